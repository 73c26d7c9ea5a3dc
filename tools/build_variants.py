#!/usr/bin/env python
"""Build ablation / tuning variants of librsdock.so into build/variants/ (in-tree, so they ship
to the GPU box).  bench.py picks one with RSDOCK_LIB=<path>.

    python tools/build_variants.py NAME=-DDEF1,-DDEF2 ...
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2510_26611_b200 import build_ext  # noqa: E402


def main():
    out_dir = os.path.join(ROOT, "build", "variants")
    os.makedirs(out_dir, exist_ok=True)
    for spec in sys.argv[1:]:
        name, _, defs = spec.partition("=")
        d = tuple(x[2:] if x.startswith("-D") else x for x in defs.split(",") if x)
        out = os.path.join(out_dir, f"librsdock_{name}.so")
        build_ext.build(out=out, defines=d)
        print(out)


if __name__ == "__main__":
    main()
