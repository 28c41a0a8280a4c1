"""Build a variant of the library with extra nvcc defines (analysis tool, not the product path).
usage: python tools/variant.py NAME -DFOO=1 ...  -> tools/libcrb_NAME.so (use with CRB_LIB=...)"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2310_17274_b200 import build as B  # noqa: E402

name, defs = sys.argv[1], sys.argv[2:]
lib = os.path.join(ROOT, "tools", f"libcrb_{name}.so")
cmd = [B.NVCC, *B.FLAGS, *defs, "-o", lib, B.SRC]
r = subprocess.run(cmd, capture_output=True, text=True)
if r.returncode:
    sys.exit(r.stdout + r.stderr)
for line in r.stderr.splitlines():
    if "spill" in line or "Used" in line:
        pass
print(lib)
