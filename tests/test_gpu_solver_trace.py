"""Teacher-forced solver step parity (VERDICT r1 "next" 2): the GPU solver records
its own state at chosen iterations (crb_solver_params.trace) and the fp64 oracle recomputes each
step from THAT state (Alg. 6 P:2147-2174 and Alg. 1, readings A17-A23, A35):

  * the ring push (orc_lbfgs_push: s = Theta_k - Theta_{k-1}, y = g_k - g_{k-1}, skip when
    s'y <= 1e-12, evict the oldest) from the GPU's ring before the push -> the GPU's ring after
    (count, order, S, Y, rho), wherever s'y is not within its O10 margin of 1e-12;
  * the direction d = -H g (orc_lbfgs_direction) from that ring: element-wise
    |d_i - d_i^ref| <= 1e-3 max|d^ref| and ||d - d^ref|| <= 1e-3 ||d^ref||;
  * g.d, and every candidate clip(Theta_k + alpha_a d_k, lo, hi) (a1): its fp64 cost and g_a.d
    against the GPU's (cost tolerance of the per-evaluation parity, margin-filtered);
  * i* bit-exactly through the fp32 selection mirror on the GPU's (c, g0d, c_a, g_a.d);
  * the next iterate is candidate i* (within one fp32 rounding of the fused step) and the best
    cost follows the strict update (A23).

Iterations 0, 1, 2, 5, 6, 25, 26 of a 30-iteration solve with m = 4: 25 pushes, so the ring fills
after 4 and evicts from then on.  TO (Franka, bench flags) and IK (a full and a ragged group).
"""
import numpy as np
import pytest
import torch

from paper_2310_17274_b200 import inputs, robots
from test_gpu_parity import COST_ATOL, COST_RTOL, MARGIN, T, f32, franka_trajs, make

pytestmark = pytest.mark.gpu

ITERS = (0, 1, 2, 5, 6, 25, 26)
D_TOL = 1e-3


@pytest.fixture(scope="module")
def native():
    from paper_2310_17274_b200 import native as N
    return N


def fma_candidate(x, a, d, lo, hi):
    """The GPU's candidate(): fminf(fmaxf(fmaf(alpha, d, theta), lo), hi), emulated in fp64."""
    v = np.float64(np.float32(a)) * d.astype(np.float64) + x.astype(np.float64)
    return np.clip(v, lo, hi)


class Tally:
    def __init__(self):
        self.steps = self.pushes = self.evictions = self.skips = self.excluded = self.cand = 0
        self.worst_d = self.worst_dinf = 0.0


def check_seed(native, O, recs, N, m, sp, lo, hi, evalf, tally, label, iters=ITERS):
    """recs: this seed's parsed records in `iters` order.  evalf(x) -> (c, g, margin) in fp64."""
    alpha = np.asarray(sp.alpha, np.float32)
    A = len(alpha)
    by_it = {r["it"]: r for r in recs}
    assert sorted(by_it) == sorted(iters), (label, sorted(by_it))
    for k in iters:
        r = by_it[k]
        x, g = r["x"].astype(np.float64), r["g"].astype(np.float64)
        Sb, Yb, rb_, cb = r["ring_before"]
        Sa, Ya, ra, ca_ = r["ring_after"]
        # ---- push (teacher-forced from the GPU's ring before it)
        if k == 0:
            assert cb == 0 and ca_ == 0, label
            S_ref, Y_ref, rho_ref, cnt_ref = np.zeros((0, N)), np.zeros((0, N)), np.zeros(0), 0
        else:
            pad = lambda a: np.vstack([a, np.zeros((max(m, 1) - a.shape[0], N))]).astype(np.float64)
            S_ref, Y_ref, rho_ref, cnt_ref, sy = O.lbfgs_push(pad(Sb), pad(Yb), np.r_[rb_, np.zeros(max(m, 1) - cb)], cb, m,
                                                              x, r["xp"].astype(np.float64), g,
                                                              r["gp"].astype(np.float64))
            S_ref, Y_ref, rho_ref = S_ref[:cnt_ref], Y_ref[:cnt_ref], rho_ref[:cnt_ref]
            s, y = x - r["xp"], g - r["gp"]
            scale = np.linalg.norm(s) * np.linalg.norm(y) + 1e-30
            assert abs(r["sy"] - sy) <= 1e-5 * scale + 1e-12, (label, k, r["sy"], sy)
            if abs(sy - 1e-12) < 1e-5 * scale:      # O10 skip margin: fp32 may decide either way
                tally.excluded += 1
                continue
            tally.pushes += sy > 1e-12
            tally.skips += sy <= 1e-12
            tally.evictions += (sy > 1e-12) and cb == m and m > 0
            assert ca_ == cnt_ref, (label, k, ca_, cnt_ref)
            for i in range(cnt_ref):
                np.testing.assert_allclose(Sa[i], S_ref[i], rtol=0, atol=2e-7 * (np.abs(S_ref[i]).max() + 1e-30))
                np.testing.assert_allclose(Ya[i], Y_ref[i], rtol=0, atol=2e-7 * (np.abs(Y_ref[i]).max() + 1e-30))
                assert abs(ra[i] - rho_ref[i]) <= 1e-4 * abs(rho_ref[i]), (label, k, i)
        # ---- direction from the oracle's ring (two-loop, A18/A19)
        d_ref = O.lbfgs_direction(S_ref, Y_ref, rho_ref, g)
        d = r["d"].astype(np.float64)
        e2 = np.linalg.norm(d - d_ref) / np.linalg.norm(d_ref)
        einf = np.abs(d - d_ref).max() / np.abs(d_ref).max()
        tally.worst_d = max(tally.worst_d, e2)
        tally.worst_dinf = max(tally.worst_dinf, einf)
        assert e2 <= D_TOL and einf <= D_TOL, (label, k, e2, einf)
        assert abs(r["g0d"] - g @ d) <= 1e-5 * np.linalg.norm(g) * np.linalg.norm(d) + 1e-12, (label, k)
        # ---- selection: bit-exact fp32 mirror on the GPU's own numbers
        ca, gda = r["ca"][:A], r["gda"][:A]
        assert O.ls_select_f32(alpha, r["c"], r["g0d"], ca, gda, sp.c1, sp.c2, sp.ls_mode) == r["istar"], (label, k)
        # ---- the candidates (a1) re-evaluated by the oracle
        for a in range(A):
            xa = fma_candidate(r["x"], alpha[a], r["d"], lo, hi)
            assert np.all(xa >= lo) and np.all(xa <= hi)
            c_ref, g_ref, margin = evalf(np.float32(xa).astype(np.float64))
            tally.cand += 1
            if margin < MARGIN:
                continue
            assert abs(ca[a] - c_ref) <= COST_RTOL * abs(c_ref) + COST_ATOL, (label, k, a, ca[a], c_ref)
            assert abs(gda[a] - g_ref @ d) <= 1e-3 * np.linalg.norm(g_ref) * np.linalg.norm(d) + 1e-6, (label, k, a)
        # ---- the step taken and the best update
        if k + 1 in by_it:
            nx = by_it[k + 1]
            want = np.float32(fma_candidate(r["x"], alpha[r["istar"]], r["d"], lo, hi))
            assert np.all(np.abs(nx["x"] - want) <= np.spacing(np.abs(want).astype(np.float32))), (label, k)
            assert nx["c"] == ca[r["istar"]]
            # the ring entering k+1 is the ring after k's push
            assert nx["ring_before"][3] == ca_
        bprev = r["best"]
        assert bprev <= r["c"] or not np.isfinite(r["c"])
        tally.steps += 1


def test_teacher_forced_to_steps(native, O):
    P, S, H = 2, 4, 32
    rb, starts, goals_cfg, trajs = franka_trajs(77, P * S, H)
    R = O.Robot(rb)
    world = inputs.tabletop_scene(0, 0, 20)
    W = O.World(world)
    cp = inputs.CostParams(dt=0.25)
    st = f32(starts[:P])
    gl = f32(np.array([O.fk(R, q)[2] for q in goals_cfg[:P]]))
    seeds = f32(trajs.reshape(P, S, H, 7))
    sp = inputs.SolverParams(iters=30)
    ctx = make(native, rb, [world], cp)
    out = ctx.solve(sp, T(seeds), T(gl), start=T(st), seed_outputs=True, trace_iters=ITERS)
    tr = out["trace"].cpu().numpy()
    N = H * 7
    lo, hi = np.tile(rb.lo, H), np.tile(rb.hi, H)
    tally = Tally()
    for p in range(P):
        def evalf(v, p=p):
            c, g, _, margin, _ = O.eval_traj(R, W, cp, st[p], gl[p], v.reshape(H, 7))
            return c, g.reshape(-1), margin
        for s in range(S):
            recs = [native.parse_trace(tr[p, s, j], N, sp.history) for j in range(len(ITERS))]
            check_seed(native, O, recs, N, sp.history, sp, np.float32(lo), np.float32(hi), evalf, tally, f"TO p{p} s{s}")
    print(f"TO trace: {tally.steps} steps, {tally.pushes} pushes, {tally.evictions} evictions, {tally.skips} skips, "
          f"{tally.excluded} margin-excluded, {tally.cand} candidates; worst d err 2-norm {tally.worst_d:.2e}, "
          f"inf {tally.worst_dinf:.2e}")
    assert tally.evictions >= P * S and tally.steps >= 0.9 * P * S * len(ITERS)
    # tracing does not change the solve
    ref = ctx.solve(sp, T(seeds), T(gl), start=T(st), seed_outputs=True)
    assert torch.equal(ref["seed_best_traj"], out["seed_best_traj"])
    ctx.close()


def test_teacher_forced_ik_steps(native, O):
    rb = robots.franka64()
    R = O.Robot(rb)
    world = inputs.tabletop_scene(3, 0, 20)
    W = O.World(world)
    cp = inputs.CostParams()
    P, S = 2, 40
    g = np.random.default_rng(31)
    goals = f32(np.array([O.fk(R, g.uniform(rb.lo * 0.6, rb.hi * 0.6))[2] for _ in range(P)]))
    seeds = f32(np.stack([inputs.ik_seeds(rb, p, S) for p in range(P)]))
    sp = inputs.SolverParams(iters=30)
    ctx = make(native, rb, [world], cp)
    out = ctx.solve(sp, T(seeds), T(goals), seed_outputs=True, trace_iters=ITERS)
    tr = out["trace"].cpu().numpy()
    tally = Tally()
    for p in range(P):
        def evalf(v, p=p):
            c, gg, _, margin, _ = O.eval_ik(R, W, cp, goals[p], v)
            return c, gg, margin
        for s in range(S):
            recs = [native.parse_trace(tr[p, s, j], 7, sp.history) for j in range(len(ITERS))]
            check_seed(native, O, recs, 7, sp.history, sp, np.float32(rb.lo), np.float32(rb.hi), evalf, tally,
                       f"IK p{p} s{s}")
    print(f"IK trace: {tally.steps} steps, {tally.pushes} pushes, {tally.evictions} evictions, {tally.skips} skips, "
          f"{tally.excluded} margin-excluded, {tally.cand} candidates; worst d err 2-norm {tally.worst_d:.2e}, "
          f"inf {tally.worst_dinf:.2e}")
    assert tally.evictions >= P * S and tally.steps >= 0.9 * P * S * len(ITERS)
    ref = ctx.solve(sp, T(seeds), T(goals), seed_outputs=True)
    assert torch.equal(ref["seed_best_traj"], out["seed_best_traj"])
    ctx.close()


def test_trace_argument_errors(native):
    rb = robots.franka64()
    ctx = make(native, rb, [inputs.tabletop_scene(0, 0, 5)], inputs.CostParams())
    s = native.solver_params_struct(inputs.SolverParams(iters=2), trace=torch.zeros(1, device="cuda"),
                                    trace_iters=tuple(range(8)))
    s.n_trace = 9
    import ctypes as C
    seeds = T(np.tile(rb.ready, (1, 1, 16, 1)))
    code = native._lib.crb_lbfgs_solve(ctx.h, C.byref(s), 1, 1, 16, native._ptr(seeds), None,
                                       native._ptr(T(rb.ready[None])), native._ptr(T(np.zeros((1, 7)))),
                                       None, None, None, None, None, native._stream())
    assert code == -1
    ctx.close()
