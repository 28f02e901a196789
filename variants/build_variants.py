"""Build tuning variants of the fused primal kernel into variants/ (not shipped)."""
import itertools, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_06258_b200 import _build
HERE = os.path.dirname(os.path.abspath(__file__))
V = {
  "nocolsum_g16": dict(MQ_NO_COLSUM=1, MQ_G=16),
  "nocolsum_g8": dict(MQ_NO_COLSUM=1, MQ_G=8),
  "nocolsum_g32": dict(MQ_NO_COLSUM=1, MQ_G=32),
  "g16_c6_l4": dict(MQ_G=16, MQ_NCW=6, MQ_LAG=4),
}
for name, d in V.items():
    flags = [f"-D{k}={v}" for k, v in d.items()]
    _build.build(force=True, extra_flags=flags, out=os.path.join(HERE, f"lib_{name}.so"))
    print(name)
