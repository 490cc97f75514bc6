"""Build experiment variants of libcapsim_b200.so next to it (A/B timing on the GPU box):
    python tools/build_variants.py NAME=DEF1,DEF2 NAME2=DEF3 ...
-> paper_2306_12247_b200/_lib/libcapsim_b200_NAME.so (select with CAPSIM_B200_LIB=...)."""
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2306_12247_b200.build import LIBDIR, build  # noqa: E402


def one(spec):
    name, _, defs = spec.partition("=")
    d = tuple(x for x in defs.split(",") if x)
    return build(out=LIBDIR / f"libcapsim_b200_{name}.so", defines=d)


with ThreadPoolExecutor(8) as ex:
    for p in ex.map(one, sys.argv[1:]):
        print(p)
