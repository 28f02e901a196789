import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs under gpurun)")
    config.addinivalue_line("markers", "slow: long CPU oracle runs (set MQ_SLOW=1)")


def pytest_collection_modifyitems(config, items):
    if os.environ.get("MQ_SLOW"):
        return
    skip = pytest.mark.skip(reason="slow oracle case; set MQ_SLOW=1")
    for it in items:
        if "slow" in it.keywords and "gpu" not in it.keywords:
            it.add_marker(skip)


def golden(name):
    path = os.path.join(GOLDEN, name)
    if not os.path.exists(path):
        pytest.skip(f"golden fixture {name} not generated")
    return np.load(path, allow_pickle=False)


def golden_names(prefix):
    return sorted(f for f in os.listdir(GOLDEN) if f.startswith(prefix) and f.endswith(".npz"))


@pytest.fixture(scope="session")
def oracle():
    from oracle import solve as orc

    orc.set_threads(os.cpu_count() or 1)
    return orc


@pytest.fixture
def tiny_fisher():
    from paper_2506_06258_b200 import FisherInstance, SparseMatrix

    u = SparseMatrix.from_dense([[0.8, 0.3], [0.2, 0.9], [0.5, 0.5]])
    return FisherInstance(u, np.array([0.4, 0.7, 0.9]))


@pytest.fixture
def small_random_fisher():
    from paper_2506_06258_b200 import GeneratorConfig, generate_fisher

    return generate_fisher(GeneratorConfig(n=12, m=6, sparsity_u=0.5, seed=3))
