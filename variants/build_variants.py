"""Build tuning variants of the fused primal kernel into variants/ (not shipped)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_06258_b200 import _build
HERE = os.path.dirname(os.path.abspath(__file__))
V = {
  "phased": dict(),
  "fused": dict(MQ_COLSUM_FUSED=1),
  "phased_triv": dict(MQ_TRIVIAL_SOLVE=1),
}
for name, d in V.items():
    flags = [f"-D{k}={v}" for k, v in d.items()]
    _build.build(force=True, extra_flags=flags, out=os.path.join(HERE, f"lib_{name}.so"))
    print(name)
