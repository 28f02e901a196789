"""Build tuning variants of the fused primal kernel into variants/ (not shipped)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_06258_b200 import _build
HERE = os.path.dirname(os.path.abspath(__file__))
V = {
  "base": dict(),
  "r0s15": dict(MQ_REG_PER=0),
  "r0s27c4": dict(MQ_REG_PER=0, MQ_NSW=27, MQ_NCW=4),
  "r0s23c8": dict(MQ_REG_PER=0, MQ_NSW=23, MQ_NCW=8),
  "r0s27_nocs": dict(MQ_REG_PER=0, MQ_NSW=27, MQ_NCW=4, MQ_NO_COLSUM=1),
  "r0s19c4": dict(MQ_REG_PER=0, MQ_NSW=19, MQ_NCW=4),
}
for name, d in V.items():
    flags = [f"-D{k}={v}" for k, v in d.items()]
    _build.build(force=True, extra_flags=flags, out=os.path.join(HERE, f"lib_{name}.so"))
    print(name)
