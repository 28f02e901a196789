"""Build tuning variants of the fused primal kernel into variants/ (not shipped)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_06258_b200 import _build
HERE = os.path.dirname(os.path.abspath(__file__))
V = {
  "base": dict(),
  "nocolsum": dict(MQ_NO_COLSUM=1),
  "gw": dict(MQ_NSW=12, MQ_NGW=4, MQ_NCW=3, MQ_STAGES=2),
  "lag8": dict(MQ_LAG=8),
  "c6s13": dict(MQ_NSW=13, MQ_NCW=6),
}
for name, d in V.items():
    flags = [f"-D{k}={v}" for k, v in d.items()]
    _build.build(force=True, extra_flags=flags, out=os.path.join(HERE, f"lib_{name}.so"))
    print(name)
