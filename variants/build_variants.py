"""Build tuning variants of the fused primal kernel into variants/ (not shipped)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_06258_b200 import _build
HERE = os.path.dirname(os.path.abspath(__file__))
V = {
  "cta": dict(),
  "perwarp": dict(MQ_CS_PERWARP=1),
  "cta_b": dict(),
  "perwarp_b": dict(MQ_CS_PERWARP=1),
}
for name, d in V.items():
    flags = [f"-D{k}={v}" for k, v in d.items()]
    _build.build(force=True, extra_flags=flags, out=os.path.join(HERE, f"lib_{name}.so"))
    print(name)
