"""ctypes binding of the fp64 CPU oracle (oracle.c).

TEST INFRASTRUCTURE ONLY: may be imported by tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs, nothing else.  It shares no code with the CUDA path; it
reads the same plain numpy input containers (paper_2310_17274_b200.inputs), which hold no method
arithmetic.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "oracle.c")
LIB = os.path.join(HERE, "liboracle.so")

CFLAGS = ["-O2", "-fPIC", "-shared", "-std=c11", "-ffp-contract=off", "-fno-fast-math",
          "-Wall", "-Wno-unused-function"]


def build(force: bool = False) -> str:
    """Compile oracle.c -> liboracle.so (plain gcc, fp64, no fast-math)."""
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < max(
            os.path.getmtime(SRC), os.path.getmtime(os.path.join(HERE, "oracle.h"))):
        subprocess.check_call(["gcc", *CFLAGS, "-o", LIB, SRC, "-lm", "-lpthread"])
    return LIB


D_P = C.POINTER(C.c_double)
I_P = C.POINTER(C.c_int)
F_P = C.POINTER(C.c_float)
LL_P = C.POINTER(C.c_longlong)


class _Robot(C.Structure):
    _fields_ = [("n_links", C.c_int), ("n_dof", C.c_int), ("n_spheres", C.c_int),
                ("n_pairs", C.c_int), ("ee_link", C.c_int),
                ("parent", I_P), ("jtype", I_P), ("dof", I_P), ("fixed", D_P),
                ("lo", D_P), ("hi", D_P), ("vmax", D_P), ("amax", D_P), ("jmax", D_P),
                ("sph", D_P), ("sph_link", I_P), ("sph_off", D_P), ("pairs", I_P)]


class _World(C.Structure):
    _fields_ = [("n_boxes", C.c_int), ("pos", D_P), ("quat", D_P), ("half", D_P),
                ("enabled", I_P)]


class _Params(C.Structure):
    _fields_ = [("a0", C.c_double), ("a1", C.c_double), ("a2", C.c_double), ("a3", C.c_double),
                ("a8", C.c_double), ("a9", C.c_double), ("w_bound", C.c_double * 4),
                ("beta_self", C.c_double), ("beta_world", C.c_double), ("eta", C.c_double),
                ("eta_bound", C.c_double), ("dt", C.c_double), ("sweep_steps", C.c_int),
                ("flags", C.c_int), ("a4", C.c_double), ("a5", C.c_double)]


class _Particle(C.Structure):
    _fields_ = [("iters", C.c_int), ("n", C.c_int), ("beta", C.c_double), ("k_mu", C.c_double),
                ("k_sigma", C.c_double), ("sigma0_frac", C.c_double), ("key", C.c_uint)]


class _Solver(C.Structure):
    _fields_ = [("iters", C.c_int), ("history", C.c_int), ("n_alpha", C.c_int),
                ("alpha", C.c_double * 8), ("c1", C.c_double), ("c2", C.c_double),
                ("ls_mode", C.c_int), ("pt", _Particle), ("problem_base", C.c_longlong),
                ("seed_base", C.c_longlong)]


_FUN = C.CFUNCTYPE(C.c_double, C.c_void_p, D_P, D_P)

_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(LIB)
        L.orc_set_state_margins.argtypes = [D_P]
        L.orc_cost_margin.restype = C.c_double
        L.orc_box_sdf.restype = C.c_double
        L.orc_activation.restype = C.c_double
        L.orc_bound.restype = C.c_double
        L.orc_logcosh.restype = C.c_double
        L.orc_logcosh.argtypes = [C.c_double]
        L.orc_activation.argtypes = [C.c_double, C.c_double, D_P]
        L.orc_bound.argtypes = [C.c_double, C.c_double, C.c_double, C.c_double, D_P]
        L.orc_pose_cost.restype = C.c_double
        L.orc_self_collision.restype = C.c_double
        L.orc_self_collision.argtypes = [C.POINTER(_Robot), D_P, C.c_double, D_P, I_P, D_P, LL_P]
        L.orc_sphere_world.restype = C.c_double
        L.orc_sphere_world.argtypes = [C.POINTER(_World), D_P, D_P, D_P, C.c_double, C.c_double,
                                       C.c_int, C.c_int, D_P, D_P, C.c_int, I_P, D_P, LL_P]
        L.orc_eval_traj.restype = C.c_double
        L.orc_eval_ik.restype = C.c_double
        L.orc_ls_select.restype = C.c_int
        L.orc_ls_select.argtypes = [C.c_int, D_P, C.c_double, C.c_double, D_P, D_P, C.c_double,
                                    C.c_double, C.c_int]
        L.orc_ls_select_f32.restype = C.c_int
        L.orc_ls_select_f32.argtypes = [C.c_int, F_P, C.c_float, C.c_float, F_P, F_P, C.c_float,
                                        C.c_float, C.c_int]
        L.orc_argmin_f32.restype = C.c_int
        L.orc_argmin_f32.argtypes = [C.c_int, F_P]
        L.orc_lbfgs_solve.argtypes = [_FUN, C.c_void_p, C.c_int, D_P, D_P, D_P,
                                      C.POINTER(_Solver), D_P, D_P, D_P]
        _lib = L
    return _lib


def _d(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _i(a):
    return np.ascontiguousarray(a, dtype=np.int32)


def _dp(a):
    return None if a is None else a.ctypes.data_as(D_P)


def _ip(a):
    return None if a is None else a.ctypes.data_as(I_P)


class Robot:
    """Keeps the numpy buffers alive behind the C struct."""

    def __init__(self, rb):
        self.src = rb
        self.arrs = dict(parent=_i(rb.parent), jtype=_i(rb.jtype), dof=_i(rb.dof), fixed=_d(rb.fixed),
                         lo=_d(rb.lo), hi=_d(rb.hi), vmax=_d(rb.vmax), amax=_d(rb.amax),
                         jmax=_d(rb.jmax), sph=_d(rb.spheres), sph_link=_i(rb.sphere_link),
                         sph_off=_d(rb.sphere_offset), pairs=_i(rb.pairs.reshape(-1, 2)))
        a = self.arrs
        self.s = _Robot(rb.n_links, rb.n_dof, rb.n_spheres, int(a["pairs"].shape[0]), int(rb.ee_link),
                        _ip(a["parent"]), _ip(a["jtype"]), _ip(a["dof"]), _dp(a["fixed"]),
                        _dp(a["lo"]), _dp(a["hi"]), _dp(a["vmax"]), _dp(a["amax"]), _dp(a["jmax"]),
                        _dp(a["sph"]), _ip(a["sph_link"]), _dp(a["sph_off"]), _ip(a["pairs"]))
        self.D, self.M, self.L = rb.n_dof, rb.n_spheres, rb.n_links


class World:
    def __init__(self, w):
        self.arrs = dict(pos=_d(w.pos), quat=_d(w.quat), half=_d(0.5 * np.asarray(w.dims)),
                         en=_i(w.enabled))
        a = self.arrs
        self.s = _World(int(a["pos"].shape[0]), _dp(a["pos"]), _dp(a["quat"]), _dp(a["half"]),
                        _ip(a["en"]))


def params(cp):
    return _Params(cp.a0, cp.a1, cp.a2, cp.a3, cp.a8, cp.a9, (C.c_double * 4)(*cp.w_bound),
                   cp.beta_self, cp.beta_world, cp.eta, cp.eta_bound, cp.dt, int(cp.sweep_steps),
                   int(cp.flags), cp.a4, cp.a5)


def particle(sp):
    return _Particle(int(sp.particle_iters), int(sp.n_particles), float(sp.particle_beta),
                     float(sp.k_mu), float(sp.k_sigma), float(sp.sigma0_frac), int(sp.rng_key) & 0xFFFFFFFF)


def solver(sp, problem_base=0, seed_base=0):
    al = list(sp.alpha) + [0.0] * (8 - len(sp.alpha))
    return _Solver(int(sp.iters), int(sp.history), len(sp.alpha), (C.c_double * 8)(*al),
                   float(sp.c1), float(sp.c2), int(sp.ls_mode), particle(sp), int(problem_base),
                   int(seed_base))


# ---------------------------------------------------------------------------------------------
# thin wrappers
# ---------------------------------------------------------------------------------------------

def fk(robot: Robot, q):
    q = _d(q)
    T = np.zeros((robot.L, 12)); sph = np.zeros((robot.M, 4)); ee = np.zeros(7)
    lib().orc_fk(C.byref(robot.s), _dp(q), _dp(T), _dp(sph), _dp(ee))
    return T, sph, ee


def fk_backward(robot: Robot, q, g_sph=None, g_p=None, g_q=None):
    out = np.zeros(robot.D)
    gs = None if g_sph is None else _d(g_sph)
    gp = None if g_p is None else _d(g_p)
    gq = None if g_q is None else _d(g_q)
    lib().orc_fk_backward(C.byref(robot.s), _dp(_d(q)), _dp(gs), _dp(gp), _dp(gq), _dp(out))
    return out


def box_sdf(p, pos, quat, half):
    g = np.zeros(3)
    lib().orc_box_sdf.argtypes = [D_P, D_P, D_P, D_P, D_P]
    sd = lib().orc_box_sdf(_dp(_d(p)), _dp(_d(pos)), _dp(_d(quat)), _dp(_d(half)), _dp(g))
    return sd, g


def activation(dprime, eta):
    dphi = C.c_double()
    v = lib().orc_activation(float(dprime), float(eta), C.byref(dphi))
    return v, dphi.value


def bound(x, lo, hi, eta2):
    dx = C.c_double()
    v = lib().orc_bound(float(x), float(lo), float(hi), float(eta2), C.byref(dx))
    return v, dx.value


def logcosh(x):
    return lib().orc_logcosh(float(x))


def pose_cost(cp, ee, goal):
    gp, gq = np.zeros(3), np.zeros(4)
    pr = params(cp)
    lib().orc_pose_cost.argtypes = [C.POINTER(_Params), D_P, D_P, D_P, D_P]
    c = lib().orc_pose_cost(C.byref(pr), _dp(_d(ee)), _dp(_d(goal)), _dp(gp), _dp(gq))
    return c, gp, gq


def self_collision(robot: Robot, spheres, beta):
    g = np.zeros((robot.M, 3))
    arg = C.c_int()
    margin = C.c_double(np.inf)
    c = lib().orc_self_collision(C.byref(robot.s), _dp(_d(spheres)), float(beta), _dp(g),
                                 C.byref(arg), C.byref(margin), None)
    return c, g, arg.value, margin.value


def sphere_world(world: World, c, r, eta, cprev=None, cnext=None, sweep=False, steps=4,
                 max_samples=256):
    G = np.zeros(3)
    samples = np.zeros((max_samples, 4))
    ns = C.c_int()
    margin = C.c_double(np.inf)
    cnt = np.zeros(7, np.int64)
    E = lib().orc_sphere_world(C.byref(world.s), _dp(_d(c)),
                               None if cprev is None else _dp(_d(cprev)),
                               None if cnext is None else _dp(_d(cnext)), float(r), float(eta),
                               int(sweep), int(steps), _dp(G), _dp(samples), max_samples,
                               C.byref(ns), C.byref(margin), cnt.ctypes.data_as(LL_P))
    return E, G, samples[: ns.value].copy(), margin.value, cnt


def state_map(start, V):
    V = _d(V)
    H, D = V.shape
    x = np.zeros((H + 5, D))
    lib().orc_state_map(_dp(_d(start)), _dp(V), H, D, _dp(x))
    return x


def derivs(x, H, dt):
    x = _d(x)
    D = x.shape[1]
    v, a, j = np.zeros((H, D)), np.zeros((H, D)), np.zeros((H, D))
    lib().orc_derivs.argtypes = [D_P, C.c_int, C.c_int, C.c_double, D_P, D_P, D_P]
    lib().orc_derivs(_dp(x), H, D, float(dt), _dp(v), _dp(a), _dp(j))
    return v, a, j


def cspace_cost(cp, q, goal):
    q = _d(q); goal = _d(goal)
    g = np.zeros_like(q)
    L = lib()
    L.orc_cspace_cost.restype = C.c_double
    L.orc_cspace_cost.argtypes = [C.POINTER(_Params), C.c_int, D_P, D_P, D_P]
    pr = params(cp)
    c = L.orc_cspace_cost(C.byref(pr), q.shape[0], _dp(q), _dp(goal), _dp(g))
    return c, g


def eval_traj(robot: Robot, world: World, cp, start, goal, V, state_margins=False):
    """O7 whole evaluation: (cost, grad [H][D], terms[5], margin, counters); with state_margins=True
    also (per-state margins [H], cost-discontinuity margin) appended (O10 split)."""
    V = _d(V)
    H = V.shape[0]
    sm = np.full(H, np.inf)
    if state_margins:
        lib().orc_set_state_margins(_dp(sm))
    g = np.zeros_like(V)
    terms = np.zeros(5)
    margin = C.c_double(np.inf)
    cnt = np.zeros(7, np.int64)
    pr = params(cp)
    lib().orc_eval_traj.argtypes = [C.POINTER(_Robot), C.POINTER(_World), C.POINTER(_Params),
                                    D_P, D_P, D_P, C.c_int, D_P, D_P, D_P, LL_P]
    try:
        c = lib().orc_eval_traj(C.byref(robot.s), C.byref(world.s), C.byref(pr), _dp(_d(start)),
                                _dp(_d(goal)), _dp(V), H, _dp(g), _dp(terms), C.byref(margin),
                                cnt.ctypes.data_as(LL_P))
    finally:
        if state_margins:
            lib().orc_set_state_margins(None)
    if state_margins:
        return c, g, terms, margin.value, cnt, sm, lib().orc_cost_margin()
    return c, g, terms, margin.value, cnt


def eval_ik(robot: Robot, world: World, cp, goal, q):
    g = np.zeros(robot.D)
    terms = np.zeros(5)
    margin = C.c_double(np.inf)
    cnt = np.zeros(7, np.int64)
    pr = params(cp)
    lib().orc_eval_ik.argtypes = [C.POINTER(_Robot), C.POINTER(_World), C.POINTER(_Params),
                                  D_P, D_P, D_P, D_P, D_P, LL_P]
    c = lib().orc_eval_ik(C.byref(robot.s), C.byref(world.s), C.byref(pr), _dp(_d(goal)),
                          _dp(_d(q)), _dp(g), _dp(terms), C.byref(margin), cnt.ctypes.data_as(LL_P))
    return c, g, terms, margin.value, cnt


def lbfgs_direction(S, Y, rho, g):
    """Two-loop recursion; S, Y [count][n] oldest..newest."""
    g = _d(g)
    n = g.shape[0]
    S = _d(np.asarray(S).reshape(-1, n)); Y = _d(np.asarray(Y).reshape(-1, n)); rho = _d(rho)
    d = np.zeros(n)
    lib().orc_lbfgs_direction.argtypes = [C.c_int, C.c_int, D_P, D_P, D_P, D_P, D_P]
    lib().orc_lbfgs_direction(n, S.shape[0], _dp(S), _dp(Y), _dp(rho), _dp(g), _dp(d))
    return d


def ls_select(alpha, c0, g0d, ca, gda, c1=1e-4, c2=0.9, mode=2):
    al = _d(alpha)
    return lib().orc_ls_select(len(al), _dp(al), float(c0), float(g0d), _dp(_d(ca)), _dp(_d(gda)),
                               float(c1), float(c2), int(mode))


def ls_select_f32(alpha, c0, g0d, ca, gda, c1=1e-4, c2=0.9, mode=2):
    al = np.ascontiguousarray(alpha, np.float32)
    ca = np.ascontiguousarray(ca, np.float32)
    gda = np.ascontiguousarray(gda, np.float32)
    return lib().orc_ls_select_f32(len(al), al.ctypes.data_as(F_P), np.float32(c0), np.float32(g0d),
                                   ca.ctypes.data_as(F_P), gda.ctypes.data_as(F_P), np.float32(c1),
                                   np.float32(c2), int(mode))


def argmin_f32(c):
    c = np.ascontiguousarray(c, np.float32)
    return lib().orc_argmin_f32(len(c), c.ctypes.data_as(F_P))


class _Trace(C.Structure):
    _fields_ = [("x", D_P), ("g", D_P), ("c", D_P), ("best_c", D_P), ("d", D_P), ("g0d", D_P),
                ("ca", D_P), ("gda", D_P), ("istar", I_P), ("count", I_P), ("sy", D_P),
                ("ls_margin", D_P)]


def lbfgs_solve(fun, x0, sp, lo=None, hi=None, traced=False):
    """fun(x) -> (cost, grad) in numpy fp64; returns (best_x, best_c, trace) with trace the best
    cost entering each iteration, or with traced=True a dict of the O10 per-iteration record
    (orc_solver_trace: x, g, c, best_c [iters+1], d, g0d, ca, gda, istar, count, sy, ls_margin)."""
    x0 = _d(x0)
    n = x0.shape[0]

    def cb(_ctx, xp, gp):
        x = np.ctypeslib.as_array(xp, shape=(n,)).copy()
        c, g = fun(x)
        np.ctypeslib.as_array(gp, shape=(n,))[:] = g
        return float(c)

    cfun = _FUN(cb)
    bx = np.zeros(n); bc = C.c_double()
    so = solver(sp)
    lo = None if lo is None else _d(np.broadcast_to(lo, (n,)))
    hi = None if hi is None else _d(np.broadcast_to(hi, (n,)))
    K = sp.iters
    tr = dict(x=np.zeros((K + 1, n)), g=np.zeros((K + 1, n)), c=np.zeros(K + 1), best_c=np.zeros(K + 1),
              d=np.zeros((max(K, 1), n)), g0d=np.zeros(max(K, 1)), ca=np.zeros((max(K, 1), 8)),
              gda=np.zeros((max(K, 1), 8)), istar=np.zeros(max(K, 1), np.int32),
              count=np.zeros(max(K, 1), np.int32), sy=np.zeros(max(K, 1)), ls_margin=np.zeros(max(K, 1)))
    ts = _Trace(*[tr[k].ctypes.data_as(I_P if tr[k].dtype == np.int32 else D_P) for k, _ in _Trace._fields_])
    L = lib()
    L.orc_lbfgs_solve_traced.argtypes = [_FUN, C.c_void_p, C.c_int, D_P, D_P, D_P, C.POINTER(_Solver), D_P, D_P,
                                         C.POINTER(_Trace)]
    L.orc_lbfgs_solve_traced(cfun, None, n, _dp(x0), _dp(lo), _dp(hi), C.byref(so), _dp(bx), C.byref(bc),
                             C.byref(ts))
    if not traced:
        return bx, bc.value, tr["best_c"]
    A = len(sp.alpha)
    for k in ("d", "g0d", "ca", "gda", "istar", "count", "sy", "ls_margin"):
        tr[k] = tr[k][:K]
    tr["ca"] = tr["ca"][:, :A]; tr["gda"] = tr["gda"][:, :A]
    return bx, bc.value, tr


def lbfgs_push(S, Y, rho, count, m, x, xp, g, gp):
    """O8 steps 1-2 on a ring S, Y [m][n] (oldest first), rho [m] with `count` pairs; returns
    (S, Y, rho, count, s'y) after the push (copies: the inputs are left unchanged)."""
    x = _d(x)
    n = x.shape[0]
    S = _d(np.array(S, dtype=np.float64).reshape(max(m, 1), n)).copy()
    Y = _d(np.array(Y, dtype=np.float64).reshape(max(m, 1), n)).copy()
    rho = _d(np.array(rho, dtype=np.float64).reshape(max(m, 1))).copy()
    sy = C.c_double()
    L = lib()
    L.orc_lbfgs_push.restype = C.c_int
    L.orc_lbfgs_push.argtypes = [C.c_int, C.c_int, D_P, D_P, D_P, C.c_int, D_P, D_P, D_P, D_P, D_P]
    cnt = L.orc_lbfgs_push(n, int(m), _dp(S), _dp(Y), _dp(rho), int(count), _dp(x), _dp(_d(xp)), _dp(_d(g)),
                           _dp(_d(gp)), C.byref(sy))
    return S, Y, rho, cnt, sy.value


def ls_margin(alpha, c0, g0d, ca, gda, c1=1e-4, c2=0.9, mode=2):
    al = _d(alpha)
    L = lib()
    L.orc_ls_margin.restype = C.c_double
    L.orc_ls_margin.argtypes = [C.c_int, D_P, C.c_double, C.c_double, D_P, D_P, C.c_double, C.c_double, C.c_int]
    return L.orc_ls_margin(len(al), _dp(al), float(c0), float(g0d), _dp(_d(ca)), _dp(_d(gda)), float(c1),
                           float(c2), int(mode))


def retime(robot: Robot, start, V, dt):
    """O13 Alg. 4 retime: returns (s, dt_opt, (max |v|/vmax, max sqrt(|a|/amax), max cbrt(|j|/jmax)))."""
    V = _d(V)
    H = V.shape[0]
    L = lib()
    L.orc_retime.restype = C.c_double
    L.orc_retime.argtypes = [C.POINTER(_Robot), D_P, D_P, C.c_int, C.c_double, D_P]
    r = np.zeros(3)
    s = L.orc_retime(C.byref(robot.s), _dp(_d(start)), _dp(V), H, float(dt), _dp(r))
    return s, s * dt, r


def scale_params(cp, dt, dt_ref=0.25, jerk_on=True):
    """O13 Alg. 4 weight scaling (reading B15) on an inputs.CostParams; returns a new CostParams."""
    import dataclasses
    r = dt / dt_ref
    wb = tuple(cp.w_bound)
    return dataclasses.replace(cp, dt=dt, a8=cp.a8 * r ** 4, a9=cp.a9 * r ** 6,
                               w_bound=(wb[0], wb[1] * r, wb[2] * r * r, wb[3] * r * r * r),
                               flags=cp.flags | (4 if jerk_on else 0))


def scale_params_c(cp, dt, dt_ref=0.25, jerk_on=True):
    """The same scaling done by the C oracle (orc_scale_params), returned as
    (dt, a8, a9, flags, w_bound[0..3])."""
    L = lib()
    L.orc_scale_params.argtypes = [C.POINTER(_Params), C.c_double, C.c_double, C.c_int, C.POINTER(_Params)]
    pin = params(cp); pout = _Params()
    L.orc_scale_params(C.byref(pin), float(dt), float(dt_ref), int(jerk_on), C.byref(pout))
    return (pout.dt, pout.a8, pout.a9, pout.flags) + tuple(pout.w_bound)


def goal_error(robot: Robot, q, goal):
    L = lib()
    L.orc_goal_error.argtypes = [C.POINTER(_Robot), D_P, D_P, D_P, D_P]
    pe, re = C.c_double(), C.c_double()
    L.orc_goal_error(C.byref(robot.s), _dp(_d(q)), _dp(_d(goal)), C.byref(pe), C.byref(re))
    return pe.value, re.value


def linear_seed(start, qT, H):
    start = _d(start); qT = _d(qT)
    D = start.shape[0]
    V = np.zeros((H, D))
    L = lib()
    L.orc_linear_seed.argtypes = [D_P, D_P, C.c_int, C.c_int, D_P]
    L.orc_linear_seed(_dp(start), _dp(qT), H, D, _dp(V))
    return V


def interpolate(x, dt, dt_fine=0.025, n_max=4096):
    """B21: states x [H][D] at spacing dt -> (n, points [min(n, n_max)][D]) on the grid
    k dt_fine, linear in joint space, the last point x_H."""
    x = _d(x)
    H, D = x.shape
    out = np.zeros((n_max, D))
    L = lib()
    L.orc_interpolate.restype = C.c_int
    L.orc_interpolate.argtypes = [D_P, C.c_int, C.c_int, C.c_double, C.c_double, C.c_int, D_P]
    n = L.orc_interpolate(_dp(x), H, D, float(dt), float(dt_fine), int(n_max), _dp(out))
    return n, out[:min(n, n_max)]


def ik_score(q, q0, pos_err, rot_err, w_pose, w_dist):
    q = _d(q)
    L = lib()
    L.orc_ik_score.restype = C.c_double
    L.orc_ik_score.argtypes = [C.c_int, D_P, D_P, C.c_double, C.c_double, C.c_double, C.c_double]
    return L.orc_ik_score(q.shape[0], _dp(q), _dp(_d(q0)), pos_err, rot_err, w_pose, w_dist)


def blended_score(pos_err, rot_err, max_jerk, motion_time, w_pose, w_jerk, w_time):
    L = lib()
    L.orc_blended_score.restype = C.c_double
    L.orc_blended_score.argtypes = [C.c_double] * 7
    return L.orc_blended_score(pos_err, rot_err, max_jerk, motion_time, w_pose, w_jerk, w_time)


def mask_sample(robot: Robot, world: World, q, margin=0.0):
    """O12: (valid, decision margin) of one configuration."""
    L = lib()
    L.orc_mask_sample.restype = C.c_int
    L.orc_mask_sample.argtypes = [C.POINTER(_Robot), C.POINTER(_World), D_P, C.c_double, D_P]
    mg = C.c_double()
    v = L.orc_mask_sample(C.byref(robot.s), C.byref(world.s), _dp(_d(q)), float(margin), C.byref(mg))
    return bool(v), mg.value


def steer(robot: Robot, world: World, src, dst, dw, r, margin=0.0):
    """O12 Alg. 3: returns (n, h[E], v_new[E][D], dist[E], margin[E])."""
    src = _d(src); dst = _d(dst)
    E, D = src.shape
    h = np.zeros(E, np.int32); v = np.zeros((E, D)); dist = np.zeros(E); mg = np.zeros(E)
    L = lib()
    L.orc_steer.restype = C.c_int
    L.orc_steer.argtypes = [C.POINTER(_Robot), C.POINTER(_World), C.c_int, D_P, D_P, D_P, C.c_double,
                            C.c_double, I_P, D_P, D_P, D_P]
    n = L.orc_steer(C.byref(robot.s), C.byref(world.s), E, _dp(src), _dp(dst), _dp(_d(dw)), float(r),
                    float(margin), _ip(h), _dp(v), _dp(dist), _dp(mg))
    return n, h, v, dist, mg


def margin_kind():
    """O10: the branch kind behind the last evaluation's margin (oracle.h orc_margin_kind)."""
    return int(lib().orc_margin_kind())


class cost_only_margins:
    """Context manager: while active, evaluation margins count only branches where the COST is
    discontinuous (a sweep sample in contact appearing / disappearing) -- for cost-only passes."""

    def __enter__(self):
        lib().orc_set_margin_mode(1)
        return self

    def __exit__(self, *exc):
        lib().orc_set_margin_mode(0)
        return False


def philox4x32(key, ctr):
    k = (C.c_uint * 2)(*[int(v) & 0xFFFFFFFF for v in key])
    c = (C.c_uint * 4)(*[int(v) & 0xFFFFFFFF for v in ctr])
    o = (C.c_uint * 4)()
    lib().orc_philox4x32(k, c, o)
    return [int(v) for v in o]


def normal(key0, key1, var, particle_, it, seed):
    L = lib()
    L.orc_normal.restype = C.c_double
    L.orc_normal.argtypes = [C.c_uint] * 6
    return L.orc_normal(key0 & 0xFFFFFFFF, key1 & 0xFFFFFFFF, var, particle_, it, seed & 0xFFFFFFFF)


def particle_solve(fun, x0, sp, lo, hi, problem=0, seed=0):
    """O11 warm-up. fun(x) -> cost (fp64); returns (mu, var, costs[iters][n])."""
    x0 = _d(x0)
    n = x0.shape[0]

    def cb(_ctx, xp, gp):
        x = np.ctypeslib.as_array(xp, shape=(n,)).copy()
        return float(fun(x))

    cfun = _FUN(cb)
    mu = np.zeros(n); var = np.zeros(n)
    trace = np.zeros((max(sp.particle_iters, 1), sp.n_particles))
    pp = particle(sp)
    lib().orc_particle_solve(cfun, None, n, _dp(x0), _dp(_d(np.broadcast_to(lo, (n,)))),
                             _dp(_d(np.broadcast_to(hi, (n,)))), C.byref(pp), C.c_uint(problem & 0xFFFFFFFF),
                             C.c_uint(seed & 0xFFFFFFFF), _dp(mu), _dp(var), _dp(trace))
    return mu, var, trace[:sp.particle_iters]


def _worlds_array(worlds):
    arr = (_World * len(worlds))(*[w.s for w in worlds])
    return arr


def solve_to(robot: Robot, worlds, env, cp, sp, seeds, start, goal, nthreads=1, problem_base=0,
             seed_base=0):
    seeds = _d(seeds)
    P, S, H, D = seeds.shape
    out = np.zeros_like(seeds); cost = np.zeros((P, S))
    warr = _worlds_array(worlds)
    pr, so = params(cp), solver(sp, problem_base, seed_base)
    envc = _i(env)
    lib().orc_solve_to.argtypes = [C.POINTER(_Robot), C.POINTER(_World), I_P, C.POINTER(_Params),
                                   C.POINTER(_Solver), C.c_int, C.c_int, C.c_int, D_P, D_P, D_P,
                                   C.c_int, D_P, D_P]
    lib().orc_solve_to(C.byref(robot.s), warr, _ip(envc), C.byref(pr), C.byref(so), P, S, H,
                       _dp(seeds), _dp(_d(start)), _dp(_d(goal)), int(nthreads), _dp(out), _dp(cost))
    return out, cost


def solve_ik(robot: Robot, worlds, env, cp, sp, seeds, goal, nthreads=1, problem_base=0, seed_base=0):
    seeds = _d(seeds)
    P, S, D = seeds.shape
    out = np.zeros_like(seeds); cost = np.zeros((P, S))
    warr = _worlds_array(worlds)
    pr, so = params(cp), solver(sp, problem_base, seed_base)
    envc = _i(env)
    lib().orc_solve_ik.argtypes = [C.POINTER(_Robot), C.POINTER(_World), I_P, C.POINTER(_Params),
                                   C.POINTER(_Solver), C.c_int, C.c_int, D_P, D_P, C.c_int, D_P, D_P]
    lib().orc_solve_ik(C.byref(robot.s), warr, _ip(envc), C.byref(pr), C.byref(so), P, S,
                       _dp(seeds), _dp(_d(goal)), int(nthreads), _dp(out), _dp(cost))
    return out, cost
