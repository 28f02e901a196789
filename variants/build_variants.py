"""Build tuning variants of the fused primal kernel into variants/ (not shipped).

usage: python variants/build_variants.py name=FLAG1=V,FLAG2 [name2=...]
"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_06258_b200 import _build
HERE = os.path.dirname(os.path.abspath(__file__))
for spec in sys.argv[1:]:
    name, _, rest = spec.partition("=")
    flags = [f"-D{f}" for f in rest.split(",") if f]
    _build.build(force=True, extra_flags=flags, out=os.path.join(HERE, f"lib_{name}.so"))
    print(name, flags)
