"""Build a variant of the library with extra nvcc defines (analysis tool, not the product path).
usage: python tools/variant.py NAME [--no-ftz | --ftz-all] -DFOO=1 ...  -> tools/libcrb_NAME.so (use with CRB_LIB=...)"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2310_17274_b200 import build as B  # noqa: E402

name, defs = sys.argv[1], sys.argv[2:]
lib = os.path.join(ROOT, "tools", f"libcrb_{name}.so")
ftz = "--no-ftz" not in defs
B.compile_lib(lib, [d for d in defs if d not in ("--no-ftz", "--ftz-all")], ftz=ftz, ftz_all="--ftz-all" in defs)
print(lib)
