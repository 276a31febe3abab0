"""Build tuning variants of libcg.so (compile-time constants) for A/B timing:
    python tools/ab_build.py NAME=DEF1,DEF2 [NAME2=...]
-> paper_1503_06029_b200/lib/ab/libcg_NAME.so"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1503_06029_b200 import build_lib  # noqa: E402

for arg in sys.argv[1:]:
    name, _, defs = arg.partition("=")
    out = os.path.join(build_lib.LIBDIR, "ab", f"libcg_{name}.so")
    d = tuple(x for x in defs.split(",") if x)
    print(build_lib.build(force=True, defines=d, out=out), flush=True)
