"""Build tuning variants of the fused primal kernel into variants/ (not shipped)."""
import itertools, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_06258_b200 import _build
HERE = os.path.dirname(os.path.abspath(__file__))
V = {
  "g16_c6_l4": dict(MQ_G=16, MQ_NCW=6, MQ_LAG=4),
  "g16_c8_l4": dict(MQ_G=16, MQ_NCW=8, MQ_LAG=4),
  "g16_c6_l2": dict(MQ_G=16, MQ_NCW=6, MQ_LAG=2),
  "g8_c6_l4": dict(MQ_G=8, MQ_NCW=6, MQ_LAG=4),
  "g32_c6_l4": dict(MQ_G=32, MQ_NCW=6, MQ_LAG=4),
  "g16_c4_l4_s12": dict(MQ_G=16, MQ_NCW=4, MQ_LAG=4, MQ_NSW=12),
}
for name, d in V.items():
    flags = [f"-D{k}={v}" for k, v in d.items()]
    _build.build(force=True, extra_flags=flags, out=os.path.join(HERE, f"lib_{name}.so"))
    print(name)
