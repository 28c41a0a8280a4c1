"""Build libcurobo_b200.so in-tree with nvcc for sm_100a (no JIT cache: the .so travels with the
repo snapshot to the GPU box)."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
SRC = os.path.join(HERE, "csrc", "curobo_b200.cu")            # kernels (CRB_PART 0) + host side
SRC_GMEM = os.path.join(HERE, "csrc", "curobo_b200_gmem.cu")  # the <GMEM = true> (large-world) kernels
DEPS = [SRC, SRC_GMEM, os.path.join(HERE, "csrc", "crb_device.cuh"), os.path.join(ROOT, "include", "curobo_b200.h"),
        os.path.abspath(__file__)]   # the flags live here
LIB = os.path.join(HERE, "libcurobo_b200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-prec-div=false", "-prec-sqrt=false", "-Xcompiler", "-fPIC", f"-I{os.path.join(ROOT, 'include')}",
         "--expt-relaxed-constexpr"]
# flush-to-zero in both units (round 1 kept it off in the large-world unit because its tensor-core
# screen lost 9 %; that screen is gone).  One setting for every kernel: the numerics of an
# environment do not depend on which build the context picks.
FTZ = {SRC: ["-ftz=true"], SRC_GMEM: ["-ftz=true"]}


def compile_lib(out: str, defs=(), ptxas_verbose: bool = False, ftz: bool = True, ftz_all: bool = False) -> str:
    """Compile both translation units (in parallel) and link them into the shared library `out`;
    returns ptxas's report.  `defs` are extra nvcc arguments (tools/variant.py); ftz_all compiles
    the large-world unit with flush-to-zero too (A/B).  Every compiler process is waited for (or
    killed) before an error is raised, and the object files are removed in all cases."""
    objs, procs = [], []
    report = ""
    try:
        for src in (SRC, SRC_GMEM):
            obj = f"{out}.{os.path.basename(src)}.o"
            fz = (["-ftz=true"] if ftz_all else FTZ[src]) if ftz else []
            cmd = [NVCC, *FLAGS, *fz, *(["-Xptxas", "-v"] if ptxas_verbose else []), *defs, "-c", "-o", obj, src]
            procs.append(subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True))
            objs.append(obj)
        failed = None
        for p in procs:
            o, e = p.communicate()
            report += o + e
            if p.returncode != 0 and failed is None:
                failed = o + e
        if failed is not None:
            sys.stderr.write(failed)
            raise RuntimeError(f"nvcc failed building {os.path.basename(out)}")
        r = subprocess.run([NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", out, *objs],
                           capture_output=True, text=True)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError(f"nvcc failed linking {os.path.basename(out)}")
    finally:
        for p in procs:
            if p.poll() is None:
                p.kill()
                p.wait()
        for obj in objs:
            if os.path.exists(obj):
                os.remove(obj)
    return report


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(d) > t for d in DEPS)


def build(force: bool = False, verbose: bool = False) -> str:
    if force or needs_build():
        report = compile_lib(LIB, ptxas_verbose=True)
        with open(os.path.join(HERE, "csrc", "ptxas_info.txt"), "w") as f:
            f.write(report)
        if verbose:
            sys.stderr.write(report)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
