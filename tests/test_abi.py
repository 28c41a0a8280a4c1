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


def test_struct_sizes_match_the_binding(lib_path):
    """crb_abi_sizes (sizeof of the five public structs in the library) against the ctypes mirrors;
    the binding also checks this at import."""
    from paper_2310_17274_b200 import native
    got = (ctypes.c_int * 5)()
    assert native._lib.crb_abi_sizes(got, 5) == 5
    assert list(got) == [ctypes.sizeof(native.crb_link), ctypes.sizeof(native.crb_robot_desc),
                         ctypes.sizeof(native.crb_cuboid), ctypes.sizeof(native.crb_cost_params),
                         ctypes.sizeof(native.crb_solver_params)]


def test_binding_lists_all_symbols(lib_path):
    from paper_2310_17274_b200 import native
    assert sorted(native.SYMBOLS) == declared_symbols()


def test_sass_is_sm100a(lib_path):
    out = subprocess.run(["cuobjdump", "--list-elf", lib_path], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["cuobjdump", "-sass", lib_path], capture_output=True, text=True).stdout
    assert "UBLKCP" in sass            # TMA bulk copy of the robot / cuboid tables
    # both builds (small-world: template argument false, large-world: true) cull the cuboids of a
    # work item with the group's AABB (warp min / max: REDUX) and a ballot, and never use the
    # round-1 tensor-core screen (removed in round 2)
    funcs = re.split(r"\n\s+Function : ", sass)
    for kern in ("solve_to_kernel", "solve_ik_kernel", "eval_to_kernel", "eval_ik_kernel"):
        body = {("ILb1E" in f.split("\n", 1)[0]): f for f in funcs if kern in f.split("\n", 1)[0]}
        assert set(body) == {False, True}, kern
        for b in (False, True):
            assert re.search(r"REDUX\.(MIN|MAX)", body[b]), (kern, b)   # group AABB over the slots
            assert "HMMA" not in body[b], (kern, b)


def test_create_fails_loudly_without_gpu(lib_path):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2310_17274_b200 import native
    with pytest.raises(native.CrbError):
        native.Context(0)
