"""The C-ABI library builds for sm_100a, loads without a GPU, and exports every symbol declared in
include/curobo_b200.h; the binding refuses to work without it (no CPU fallback)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "curobo_b200.h")


def declared_symbols():
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(crb_[a-z_0-9]+)\s*\(", txt)))


@pytest.fixture(scope="module")
def lib_path():
    from paper_2310_17274_b200 import build
    return build.build()


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for s in ("crb_set_robot", "crb_set_world", "crb_evaluate_cost_grad", "crb_lbfgs_solve"):
        assert s in syms


def test_library_exports_every_declared_symbol(lib_path):
    lib = ctypes.CDLL(lib_path)
    for s in declared_symbols():
        assert hasattr(lib, s), s
    nm = subprocess.run(["nm", "-D", "--defined-only", lib_path], capture_output=True, text=True).stdout
    for s in declared_symbols():
        assert re.search(rf"\bT {s}\b", nm), s


def test_binding_lists_all_symbols(lib_path):
    from paper_2310_17274_b200 import native
    assert sorted(native.SYMBOLS) == declared_symbols()


def test_sass_is_sm100a(lib_path):
    out = subprocess.run(["cuobjdump", "--list-elf", lib_path], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["cuobjdump", "-sass", lib_path], capture_output=True, text=True).stdout
    assert "UBLKCP" in sass            # TMA bulk copy of the robot / cuboid tables
    assert "HMMA" not in sass          # no legacy tensor-core path (the path is not a contraction)


def test_create_fails_loudly_without_gpu(lib_path):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2310_17274_b200 import native
    with pytest.raises(native.CrbError):
        native.Context(0)
