"""Build tuning variants of libldbp (same sources, different -D macros) for A/B timing on the GPU:

    python scripts/build_variants.py NAME=MACRO=V,MACRO2=V ...
    -> build/variants/NAME/libldbp.so   (run with LDBP_LIB=build/variants/NAME/libldbp.so)
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import __graft_entry__ as G  # noqa: E402

for spec in sys.argv[1:]:
    name, _, macros = spec.partition("=")
    defs = [m for m in macros.split(",") if m]
    d = os.path.join(G.BUILD, "variants", name)
    out = G.build_lib(os.path.join(d, "libldbp.so"), defs, os.path.join(d, "obj"))
    print(name, defs, "->", out)
