"""Thin ctypes binding of libcurobo_b200.so (include/curobo_b200.h): argument marshalling only.

Every step of the hot path runs in the library's CUDA kernels; torch is used for device memory
and streams.  There is no CPU fallback: importing this module on a machine where the library is
missing raises immediately, and every call that returns a non-zero status raises CrbError.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Optional, Sequence

import numpy as np

from . import inputs

HERE = os.path.dirname(os.path.abspath(__file__))
# CRB_LIB: an alternative build of the same library (tools/world_stats.py); default the in-tree one
LIB_PATH = os.environ.get("CRB_LIB") or os.path.join(HERE, "libcurobo_b200.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'` "
                      "(nvcc, sm_100a).  There is no CPU fallback.")

_lib = C.CDLL(LIB_PATH)

STATUS = {0: "CRB_OK", -1: "CRB_E_ARG", -2: "CRB_E_SHAPE", -3: "CRB_E_ROBOT", -4: "CRB_E_WORLD",
          -5: "CRB_E_NOT_READY", -6: "CRB_E_LIMIT", -7: "CRB_E_CUDA", -8: "CRB_E_OOM"}


class CrbError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"{STATUS.get(code, code)}: {msg}")
        self.code = code


class crb_link(C.Structure):
    _fields_ = [("parent", C.c_int), ("type", C.c_int), ("dof", C.c_int), ("fixed", C.c_float * 12)]


F_P = C.POINTER(C.c_float)
I_P = C.POINTER(C.c_int)


class crb_robot_desc(C.Structure):
    _fields_ = [("n_links", C.c_int), ("n_dof", C.c_int), ("n_spheres", C.c_int), ("n_pairs", C.c_int),
                ("ee_link", C.c_int), ("links", C.POINTER(crb_link)),
                ("pos_lo", F_P), ("pos_hi", F_P), ("vel_max", F_P), ("acc_max", F_P), ("jerk_max", F_P),
                ("spheres", F_P), ("sphere_link", I_P), ("self_offset", F_P), ("pairs", I_P)]


class crb_cuboid(C.Structure):
    _fields_ = [("pos", C.c_float * 3), ("quat", C.c_float * 4), ("dims", C.c_float * 3), ("enabled", C.c_int)]


class crb_cost_params(C.Structure):
    _fields_ = [("a0", C.c_float), ("a1", C.c_float), ("a2", C.c_float), ("a3", C.c_float),
                ("a8", C.c_float), ("a9", C.c_float), ("w_bound", C.c_float * 4),
                ("beta_self", C.c_float), ("beta_world", C.c_float), ("eta", C.c_float),
                ("eta_bound", C.c_float), ("dt", C.c_float), ("sweep_steps", C.c_int), ("flags", C.c_uint),
                ("a4", C.c_float), ("a5", C.c_float)]


class crb_solver_params(C.Structure):
    _fields_ = [("iters", C.c_int), ("history", C.c_int), ("n_alpha", C.c_int), ("alpha", C.c_float * 8),
                ("c1", C.c_float), ("c2", C.c_float), ("ls_mode", C.c_int), ("global_seed_base", C.c_int64),
                ("particle_iters", C.c_int), ("n_particles", C.c_int), ("particle_beta", C.c_float),
                ("k_mu", C.c_float), ("k_sigma", C.c_float), ("sigma0_frac", C.c_float),
                ("rng_key", C.c_uint32), ("global_problem_base", C.c_int64), ("check_every", C.c_int),
                ("conv_rtol", C.c_float), ("cluster", C.c_int), ("trace", C.c_void_p), ("n_trace", C.c_int),
                ("trace_iter", C.c_int * 8), ("persist", C.c_int)]


_V = C.c_void_p
_lib.crb_create.argtypes = [C.c_int, C.POINTER(_V)]
_lib.crb_destroy.argtypes = [_V]
_lib.crb_last_error.argtypes = [_V]
_lib.crb_last_error.restype = C.c_char_p
_lib.crb_version.restype = C.c_char_p
_lib.crb_set_robot.argtypes = [_V, C.POINTER(crb_robot_desc)]
_lib.crb_set_world.argtypes = [_V, C.c_int, C.c_int, I_P, C.POINTER(crb_cuboid)]
_lib.crb_set_cost_params.argtypes = [_V, C.POINTER(crb_cost_params)]
_lib.crb_fk.argtypes = [_V, _V, C.c_int, _V, _V, _V]
_lib.crb_evaluate_cost_grad.argtypes = [_V, _V, C.c_int, C.c_int, _V, _V, _V, _V, _V, _V, _V]
_lib.crb_lbfgs_solve.argtypes = [_V, C.POINTER(crb_solver_params), C.c_int, C.c_int, C.c_int, _V, _V, _V, _V,
                                 _V, _V, _V, _V, _V, _V]
_lib.crb_lbfgs_solve_host.argtypes = [_V, C.POINTER(crb_solver_params), C.c_int, C.c_int, C.c_int, _V, _V, _V,
                                      _V, _V, _V, _V, _V]
_lib.crb_ls_select.argtypes = [C.c_int, C.c_int, F_P, _V, _V, _V, _V, C.c_float, C.c_float, C.c_int, _V, _V]
_lib.crb_argmin_keys.argtypes = [C.c_int, C.c_int, _V, C.c_int64, _V, _V, _V]
_lib.crb_lbfgs_direction.argtypes = [C.c_int, C.c_int, C.c_int, _V, _V, _V, _V, _V]
_lib.crb_solver_occupancy.argtypes = [_V, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int)]
_lib.crb_mask_samples.argtypes = [_V, _V, C.c_int, _V, C.c_int, C.c_float, _V, _V]
_lib.crb_steer.argtypes = [_V, C.c_int, _V, _V, _V, C.c_float, C.c_int, C.c_float, C.c_int, _V, _V, _V, _V, _V]
_lib.crb_evaluate_cost_grad_dt.argtypes = [_V, _V, C.c_int, C.c_int, _V, _V, _V, _V, _V, _V, _V, _V]
_lib.crb_lbfgs_solve_dt.argtypes = [_V, C.POINTER(crb_solver_params), C.c_int, C.c_int, C.c_int, _V, _V, _V, _V,
                                    _V, _V, _V, _V, _V, _V, _V]
_lib.crb_retime.argtypes = [_V, C.c_int, C.c_int, _V, _V, C.c_int, _V, _V, _V, _V, _V]
_lib.crb_goal_error.argtypes = [_V, C.c_int, _V, C.c_int, _V, C.c_int, _V, _V, _V]
_lib.crb_ik_scores.argtypes = [C.c_int, C.c_int, C.c_int, _V, _V, _V, _V, _V, C.c_float, C.c_float, C.c_float,
                               C.c_float, C.c_float, _V, _V]
_lib.crb_to_scores.argtypes = [C.c_int, C.c_int, C.c_int, _V, _V, _V, _V, _V, C.c_float, C.c_float, C.c_float,
                               C.c_float, C.c_float, C.c_float, _V, _V]
_lib.crb_rank_seeds.argtypes = [C.c_int, C.c_int, _V, C.c_int, _V, _V, _V]
_lib.crb_linear_seeds.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, _V, _V, C.c_int, _V, _V, _V]
_lib.crb_trajectory_states.argtypes = [C.c_int, C.c_int, C.c_int, _V, _V, C.c_int, _V, _V]
_lib.crb_gather_rows.argtypes = [C.c_int, C.c_int, C.c_int, _V, _V, C.c_int, _V, _V]
_lib.crb_interpolate.argtypes = [C.c_int, C.c_int, C.c_int, _V, _V, C.c_float, C.c_int, _V, _V, _V]
_lib.crb_particle_normals.argtypes = [C.c_uint32, C.c_uint32, C.c_int, C.c_int, C.c_int, C.c_uint32, _V, _V]
_lib.crb_launch_count.argtypes = [_V]
_lib.crb_launch_count.restype = C.c_int64


def _check_abi():
    """The ctypes mirrors must match the library's struct sizes (header drift fails loudly).  A
    CRB_LIB build older than crb_abi_sizes (tools/ab*.sh A/B runs) is not checked."""
    if os.environ.get("CRB_LIB") and not hasattr(_lib, "crb_abi_sizes"):
        return
    _lib.crb_abi_sizes.argtypes = [C.POINTER(C.c_int), C.c_int]
    _lib.crb_abi_sizes.restype = C.c_int
    got = (C.c_int * 5)()
    _lib.crb_abi_sizes(got, 5)
    mine = [C.sizeof(crb_link), C.sizeof(crb_robot_desc), C.sizeof(crb_cuboid), C.sizeof(crb_cost_params),
            C.sizeof(crb_solver_params)]
    if list(got) != mine:
        raise ImportError(f"libcurobo_b200 struct sizes {list(got)} != binding {mine}: rebuild or update native.py")


_check_abi()

SYMBOLS = ["crb_create", "crb_destroy", "crb_last_error", "crb_version", "crb_set_robot", "crb_set_world",
           "crb_set_cost_params", "crb_fk", "crb_evaluate_cost_grad", "crb_lbfgs_solve", "crb_lbfgs_solve_host",
           "crb_ls_select", "crb_argmin_keys", "crb_lbfgs_direction", "crb_launch_count", "crb_solver_occupancy",
           "crb_particle_normals", "crb_mask_samples", "crb_steer", "crb_evaluate_cost_grad_dt",
           "crb_lbfgs_solve_dt", "crb_retime", "crb_goal_error", "crb_ik_scores", "crb_to_scores",
           "crb_rank_seeds", "crb_linear_seeds", "crb_gather_rows", "crb_trajectory_states", "crb_interpolate",
           "crb_abi_sizes"]


def _ptr(t):
    """Device pointer of a torch tensor (or None)."""
    if t is None:
        return None
    assert t.is_cuda and t.is_contiguous(), "expected a contiguous CUDA tensor"
    return C.c_void_p(t.data_ptr())


def _stream():
    import torch
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def _check_free(code):
    if code != 0:
        raise CrbError(code, "(no context)")


def cost_params_struct(cp: inputs.CostParams) -> crb_cost_params:
    return crb_cost_params(cp.a0, cp.a1, cp.a2, cp.a3, cp.a8, cp.a9, (C.c_float * 4)(*cp.w_bound),
                           cp.beta_self, cp.beta_world, cp.eta, cp.eta_bound, cp.dt, int(cp.sweep_steps),
                           int(cp.flags), cp.a4, cp.a5)


def solver_params_struct(sp: inputs.SolverParams, seed_base: int = 0, problem_base: int = 0, trace=None,
                         trace_iters=()) -> crb_solver_params:
    al = list(sp.alpha) + [0.0] * (8 - len(sp.alpha))
    ti = list(trace_iters) + [-1] * (8 - len(trace_iters))
    return crb_solver_params(int(sp.iters), int(sp.history), len(sp.alpha), (C.c_float * 8)(*al), float(sp.c1),
                             float(sp.c2), int(sp.ls_mode), int(seed_base), int(sp.particle_iters),
                             int(sp.n_particles), float(sp.particle_beta), float(sp.k_mu), float(sp.k_sigma),
                             float(sp.sigma0_frac), int(sp.rng_key) & 0xFFFFFFFF, int(problem_base),
                             int(sp.check_every), float(sp.conv_rtol), int(sp.cluster),
                             None if trace is None else C.c_void_p(trace.data_ptr()), len(trace_iters),
                             (C.c_int * 8)(*ti), int(getattr(sp, "persist", -1)))


def trace_rec(N: int, m: int) -> int:
    """CRB_TRACE_REC(N, m): floats per solver trace record (include/curobo_b200.h)."""
    return 5 * N + 2 * (2 * m * N + m + 1) + 24


def parse_trace(rec, N: int, m: int) -> dict:
    """One record (numpy float array) -> named fields (header layout of crb_solver_params.trace)."""
    o = 5 * N

    def ring(off):
        S = rec[off:off + m * N].reshape(m, N); Y = rec[off + m * N:off + 2 * m * N].reshape(m, N)
        rho = rec[off + 2 * m * N:off + 2 * m * N + m]; cnt = int(rec[off + 2 * m * N + m])
        return S[:cnt], Y[:cnt], rho[:cnt], cnt
    sc = rec[-24:]
    return dict(x=rec[:N], g=rec[N:2 * N], xp=rec[2 * N:3 * N], gp=rec[3 * N:4 * N], d=rec[4 * N:5 * N],
                ring_before=ring(o), ring_after=ring(o + 2 * m * N + m + 1), g0d=sc[0], c=sc[1],
                istar=int(sc[2]), sy=sc[3], ca=sc[4:12], gda=sc[12:20], it=int(sc[20]), best=sc[21])


class Context:
    """One crb_ctx on one CUDA device."""

    def __init__(self, device: int = 0):
        h = C.c_void_p()
        code = _lib.crb_create(int(device), C.byref(h))
        if code != 0:
            raise CrbError(code, f"crb_create({device}) failed")
        self.h = h
        self.device = device
        self._keep = []

    def close(self):
        if self.h:
            _lib.crb_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _chk(self, code):
        if code != 0:
            raise CrbError(code, _lib.crb_last_error(self.h).decode())

    def solver_occupancy(self, H: int, history: int = 4, n_alpha: int = 4):
        """(CTAs resident per SM, shared-memory bytes per CTA) of the persistent solver."""
        n, b = C.c_int(), C.c_int()
        self._chk(_lib.crb_solver_occupancy(self.h, int(H), int(history), int(n_alpha), C.byref(n), C.byref(b)))
        return n.value, b.value

    @property
    def launches(self) -> int:
        return int(_lib.crb_launch_count(self.h))

    # ---- setup (host arrays) -------------------------------------------------------------
    def set_robot(self, rb: inputs.Robot):
        L = rb.n_links
        links = (crb_link * L)()
        for l in range(L):
            links[l].parent = int(rb.parent[l]); links[l].type = int(rb.jtype[l]); links[l].dof = int(rb.dof[l])
            for i in range(12):
                links[l].fixed[i] = float(rb.fixed[l][i])
        f32 = lambda a: np.ascontiguousarray(a, np.float32)
        i32 = lambda a: np.ascontiguousarray(a, np.int32)
        arrs = dict(lo=f32(rb.lo), hi=f32(rb.hi), vmax=f32(rb.vmax), amax=f32(rb.amax), jmax=f32(rb.jmax),
                    sph=f32(rb.spheres), slink=i32(rb.sphere_link), off=f32(rb.sphere_offset),
                    pairs=i32(rb.pairs.reshape(-1, 2)))
        fp = lambda a: a.ctypes.data_as(F_P)
        ip = lambda a: a.ctypes.data_as(I_P)
        desc = crb_robot_desc(L, rb.n_dof, rb.n_spheres, int(arrs["pairs"].shape[0]), int(rb.ee_link), links,
                              fp(arrs["lo"]), fp(arrs["hi"]), fp(arrs["vmax"]), fp(arrs["amax"]), fp(arrs["jmax"]),
                              fp(arrs["sph"]), ip(arrs["slink"]), fp(arrs["off"]), ip(arrs["pairs"]))
        self._chk(_lib.crb_set_robot(self.h, C.byref(desc)))
        self.robot = rb

    def set_world(self, worlds: Sequence[inputs.World]):
        n = len(worlds)
        kmax = max(1, max(w.n_boxes for w in worlds))
        arr = (crb_cuboid * (n * kmax))()
        counts = np.zeros(n, np.int32)
        for e, w in enumerate(worlds):
            counts[e] = w.n_boxes
            for k in range(w.n_boxes):
                b = arr[e * kmax + k]
                b.pos[:] = [float(x) for x in w.pos[k]]
                b.quat[:] = [float(x) for x in w.quat[k]]
                b.dims[:] = [float(x) for x in w.dims[k]]
                b.enabled = int(w.enabled[k])
        self._chk(_lib.crb_set_world(self.h, n, kmax, counts.ctypes.data_as(I_P), arr))

    def set_cost_params(self, cp: inputs.CostParams):
        s = cost_params_struct(cp)
        self._chk(_lib.crb_set_cost_params(self.h, C.byref(s)))
        self.cp = cp

    # ---- hot path (device tensors) --------------------------------------------------------
    def fk(self, q, spheres_out=None, ee_out=None):
        import torch
        B = q.shape[0]
        if spheres_out is None:
            spheres_out = torch.empty(B, self.robot.n_spheres, 4, device=q.device, dtype=torch.float32)
        if ee_out is None:
            ee_out = torch.empty(B, 7, device=q.device, dtype=torch.float32)
        self._chk(_lib.crb_fk(self.h, _ptr(q), B, _ptr(spheres_out), _ptr(ee_out), _stream()))
        return spheres_out, ee_out

    def evaluate(self, q, goal, start=None, env=None, grad=True, terms=True, dt=None):
        """q [B,H,D] (TO) or [B,D] (IK); dt [B] per-row timestep (None = the params' dt);
        returns (cost [B], grad, terms [B,5])."""
        import torch
        B = q.shape[0]
        H = 1 if q.dim() == 2 else q.shape[1]
        cost = torch.empty(B, device=q.device, dtype=torch.float32)
        g = torch.empty_like(q) if grad else None
        tc = torch.empty(B, 5, device=q.device, dtype=torch.float32) if terms else None
        self._chk(_lib.crb_evaluate_cost_grad_dt(self.h, _ptr(q), B, H, _ptr(env), _ptr(start), _ptr(goal), _ptr(dt),
                                                 _ptr(cost), _ptr(g), _ptr(tc), _stream()))
        return cost, g, tc

    def retime(self, V, start, dt=None):
        """Alg. 4 retime of V [B,H,D] (start [B or P, D]): returns (scale, dt_opt, max_jerk) [B]."""
        import torch
        B, H, _ = V.shape
        div = B // start.shape[0]
        out = [torch.empty(B, device=V.device, dtype=torch.float32) for _ in range(3)]
        self._chk(_lib.crb_retime(self.h, B, H, _ptr(V), _ptr(start), div, _ptr(dt), _ptr(out[0]), _ptr(out[1]),
                                  _ptr(out[2]), _stream()))
        return tuple(out)

    def goal_error(self, q, goal, B=None, stride=None, goal_div: int = 1):
        """Goal errors of B configurations (rows of `stride` floats from q's start, e.g. the terminal
        states of trajectories); goal [B // goal_div, 7].  Returns (pos_err, rot_err) [B]."""
        import torch
        B = goal.shape[0] * goal_div if B is None else B
        pe = torch.empty(B, device=goal.device, dtype=torch.float32)
        re = torch.empty(B, device=goal.device, dtype=torch.float32)
        stride = q.shape[-1] if stride is None else stride
        self._chk(_lib.crb_goal_error(self.h, B, _ptr(q), int(stride), _ptr(goal), int(goal_div), _ptr(pe), _ptr(re),
                                      _stream()))
        return pe, re

    def solve(self, sp: inputs.SolverParams, seeds, goal, start=None, env=None, seed_base: int = 0,
              seed_outputs: bool = False, problem_base: int = 0, dt=None, trace_iters=()):
        """seeds [P,S,H,D] (TO) or [P,S,D] (IK).  Returns dict of device tensors; with trace_iters
        (<= 8 iteration numbers) also "trace" [P,S,len(trace_iters),CRB_TRACE_REC] (parse_trace)."""
        import torch
        P, S = seeds.shape[0], seeds.shape[1]
        H = 1 if seeds.dim() == 3 else seeds.shape[2]
        D = seeds.shape[-1]
        dev = seeds.device
        out = dict(best_traj=torch.empty((P, H, D) if H > 1 else (P, D), device=dev, dtype=torch.float32),
                   best_cost=torch.empty(P, device=dev, dtype=torch.float32),
                   best_key=torch.empty(P, device=dev, dtype=torch.int64))
        if seed_outputs:
            out["seed_best_cost"] = torch.empty(P, S, device=dev, dtype=torch.float32)
            out["seed_best_traj"] = torch.empty_like(seeds)
        tr = None
        if trace_iters:
            tr = torch.zeros(P, S, len(trace_iters), trace_rec(H * D if H > 1 else D, sp.history), device=dev,
                             dtype=torch.float32)
            out["trace"] = tr
        s = solver_params_struct(sp, seed_base, problem_base, tr, tuple(trace_iters))
        self._chk(_lib.crb_lbfgs_solve_dt(self.h, C.byref(s), P, S, H, _ptr(seeds), _ptr(env), _ptr(start), _ptr(goal),
                                          _ptr(dt), _ptr(out["best_traj"]), _ptr(out["best_cost"]),
                                          _ptr(out["best_key"]), _ptr(out.get("seed_best_cost")),
                                          _ptr(out.get("seed_best_traj")), _stream()))
        return out

    def mask_samples(self, q, env=None, margin: float = 0.0, env_div: int = 1):
        """q [K,D] device fp32 (env row k // env_div) -> valid [K] uint8 (Alg. 3 mask_samples)."""
        import torch
        K = q.shape[0]
        valid = torch.empty(K, dtype=torch.uint8, device=q.device)
        self._chk(_lib.crb_mask_samples(self.h, _ptr(q), K, _ptr(env), int(env_div), float(margin), _ptr(valid),
                                        _stream()))
        return valid

    def steer(self, src, dst, dw, r: float, env: int = 0, margin: float = 0.0, n_cap: int = 256):
        """Alg. 3 parallel steering of E edges: returns dict(n [2] int32, h [E], v_new [E,D], dist [E])."""
        import torch
        E, D = src.shape
        dev = src.device
        out = dict(n=torch.empty(2, dtype=torch.int32, device=dev), h=torch.empty(E, dtype=torch.int32, device=dev),
                   v_new=torch.empty(E, D, dtype=torch.float32, device=dev),
                   dist=torch.empty(E, dtype=torch.float32, device=dev))
        self._chk(_lib.crb_steer(self.h, E, _ptr(src), _ptr(dst), _ptr(dw), float(r), int(env), float(margin),
                                 int(n_cap), _ptr(out["n"]), _ptr(out["h"]), _ptr(out["v_new"]), _ptr(out["dist"]),
                                 _stream()))
        return out

    def solve_host(self, sp: inputs.SolverParams, seeds, goal, start=None, env=None, seed_base: int = 0,
                   best_traj=None, best_cost=None, best_key=None, problem_base: int = 0):
        """Host (ideally pinned) torch CPU tensors in and out; H2D + solve + D2H + sync in the library."""
        P, S = seeds.shape[0], seeds.shape[1]
        H = 1 if seeds.dim() == 3 else seeds.shape[2]
        hp = lambda t: None if t is None else C.c_void_p(t.data_ptr())
        s = solver_params_struct(sp, seed_base, problem_base)
        self._chk(_lib.crb_lbfgs_solve_host(self.h, C.byref(s), P, S, H, hp(seeds), hp(env), hp(start), hp(goal),
                                            hp(best_traj), hp(best_cost), hp(best_key), _stream()))


# ---- test hooks -----------------------------------------------------------------------------

def ls_select(alpha, c0, g0d, ca, gda, c1=1e-4, c2=0.9, mode=2):
    import torch
    n, A = ca.shape
    out = torch.empty(n, device=ca.device, dtype=torch.int32)
    al = np.ascontiguousarray(alpha, np.float32)
    _check_free(_lib.crb_ls_select(n, A, al.ctypes.data_as(F_P), _ptr(c0), _ptr(g0d), _ptr(ca), _ptr(gda),
                                   float(c1), float(c2), int(mode), _ptr(out), _stream()))
    return out


def argmin_keys(cost, seed_base=0):
    import torch
    P, S = cost.shape
    key = torch.empty(P, device=cost.device, dtype=torch.int64)
    idx = torch.empty(P, device=cost.device, dtype=torch.int32)
    _check_free(_lib.crb_argmin_keys(P, S, _ptr(cost), int(seed_base), _ptr(key), _ptr(idx), _stream()))
    return key, idx


def lbfgs_direction(S, Y, g):
    """S, Y [B,count,n], g [B,n] device fp32 -> d [B,n] (the solver's two-loop routine)."""
    import torch
    B, n = g.shape
    count = S.shape[1]
    d = torch.empty_like(g)
    _check_free(_lib.crb_lbfgs_direction(B, n, count, _ptr(S), _ptr(Y), _ptr(g), _ptr(d), _stream()))
    return d


def ik_scores(q, q0, pos_err, rot_err, valid, pos_thr, rot_thr, w_pose, w_dist, penalty=float("inf")):
    """q [P,S,D], q0 [P,D], errors [P,S], valid [P,S] uint8 (or None) -> score [P,S]."""
    import torch
    P, S, D = q.shape
    score = torch.empty(P, S, device=q.device, dtype=torch.float32)
    _check_free(_lib.crb_ik_scores(P, S, D, _ptr(q), _ptr(q0), _ptr(pos_err), _ptr(rot_err), _ptr(valid),
                                   float(pos_thr), float(rot_thr), float(w_pose), float(w_dist), float(penalty),
                                   _ptr(score), _stream()))
    return score


def to_scores(pos_err, rot_err, max_jerk, dt_opt, valid, H, pos_thr, rot_thr, w_pose, w_jerk, w_time,
              penalty=float("inf")):
    """errors / max_jerk / dt_opt [P,S], valid [P,S,H] uint8 (or None) -> blended score [P,S]."""
    import torch
    P, S = pos_err.shape
    score = torch.empty(P, S, device=pos_err.device, dtype=torch.float32)
    _check_free(_lib.crb_to_scores(P, S, int(H), _ptr(pos_err), _ptr(rot_err), _ptr(max_jerk), _ptr(dt_opt),
                                   _ptr(valid), float(pos_thr), float(rot_thr), float(w_pose), float(w_jerk),
                                   float(w_time), float(penalty), _ptr(score), _stream()))
    return score


def rank_seeds(score, k):
    """score [P,S] -> (idx [P,k] int32, count [P] int32)."""
    import torch
    P, S = score.shape
    idx = torch.empty(P, k, device=score.device, dtype=torch.int32)
    cnt = torch.empty(P, device=score.device, dtype=torch.int32)
    _check_free(_lib.crb_rank_seeds(P, S, _ptr(score), int(k), _ptr(idx), _ptr(cnt), _stream()))
    return idx, cnt


def linear_seeds(q0, qT, H, idx=None, S=None):
    """q0 [P,D], qT [P,Sq,D], idx [P,S] (or None) -> seeds [P,S,H,D]."""
    import torch
    P, Sq, D = qT.shape
    S = idx.shape[1] if idx is not None else (S or Sq)
    seeds = torch.empty(P, S, H, D, device=qT.device, dtype=torch.float32)
    _check_free(_lib.crb_linear_seeds(P, S, int(H), D, _ptr(q0), _ptr(qT), Sq, _ptr(idx), _ptr(seeds), _stream()))
    return seeds


def trajectory_states(V, start):
    """V [B,H,D] optimisation variables, start [B or P, D] -> the states x_1..x_H [B,H,D]."""
    import torch
    B, H, D = V.shape
    x = torch.empty_like(V)
    _check_free(_lib.crb_trajectory_states(B, H, D, _ptr(V), _ptr(start), B // start.shape[0], _ptr(x), _stream()))
    return x


def gather_rows(src, idx, idx_stride=1):
    """src [P,S,...], idx [P*idx_stride] int32 -> dst [P,...] = src[p, idx[p*idx_stride]]."""
    import torch
    P, S = src.shape[0], src.shape[1]
    n = int(src[0, 0].numel())
    dst = torch.empty((P,) + tuple(src.shape[2:]), device=src.device, dtype=torch.float32)
    _check_free(_lib.crb_gather_rows(P, S, n, _ptr(src), _ptr(idx), int(idx_stride), _ptr(dst), _stream()))
    return dst


def interpolate(x, dt, dt_fine=0.025, n_max=1024):
    """B21: states x [B,H,D] at spacing dt [B] -> (points [B,n_max,D], n [B] int32 before clamping)."""
    import torch
    B, H, D = x.shape
    out = torch.empty(B, n_max, D, device=x.device, dtype=torch.float32)
    n = torch.empty(B, device=x.device, dtype=torch.int32)
    _check_free(_lib.crb_interpolate(B, H, D, _ptr(x), _ptr(dt), float(dt_fine), int(n_max), _ptr(out), _ptr(n),
                                     _stream()))
    return out, n


def particle_normals(key0, key1, n_var, n_particles, it, seed):
    """[n_particles, n_var] device fp32: the warm-up's draws as the solver makes them (B9)."""
    import torch
    out = torch.empty(n_particles, n_var, device="cuda", dtype=torch.float32)
    _check_free(_lib.crb_particle_normals(C.c_uint32(key0 & 0xFFFFFFFF), C.c_uint32(key1 & 0xFFFFFFFF), n_var,
                                          n_particles, it, C.c_uint32(seed & 0xFFFFFFFF), _ptr(out), _stream()))
    return out


def version() -> str:
    return _lib.crb_version().decode()
