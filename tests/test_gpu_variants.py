"""GPU parity of the §8(f) f3 variants: the joint-space goal cost (Eq. cspace-cost),
gradient descent as L-BFGS with history 0 and long histories (m up to 25).
Same tolerances and margin filter as test_gpu_parity."""
import numpy as np
import pytest
import torch

from paper_2310_17274_b200 import inputs, robots
from test_gpu_parity import ref_traj, Stats, T, f32, franka_trajs, make, planar_problems

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def native():
    from paper_2310_17274_b200 import native as N
    return N


@pytest.mark.parametrize("H", [16, 8])
def test_cspace_eval_to_parity(native, O, H):
    B = 96
    rb, starts, goals_cfg, trajs = franka_trajs(500 + H, B, H)
    worlds = [inputs.tabletop_scene(5, e, 20) for e in range(2)]
    cp = inputs.CostParams(flags=inputs.CSPACE | inputs.SWEEP | inputs.SPEED, dt=0.25 if H >= 16 else 0.1)
    ctx = make(native, rb, worlds, cp)
    R = O.Robot(rb)
    Ws = [O.World(w) for w in worlds]
    env = np.arange(B, dtype=np.int32) % 2
    V, st, gl = f32(trajs), f32(starts), f32(goals_cfg)          # goal = theta_g [B][D]
    cost, grad, terms = ctx.evaluate(T(V), T(gl), start=T(st), env=T(env, torch.int32))
    cost, grad, terms = cost.cpu().numpy(), grad.cpu().numpy(), terms.cpu().numpy()
    stats = Stats()
    active = 0
    for b in range(B):
        c_ref, g_ref, t_ref, margin = ref_traj(O, R, Ws[env[b]], cp, st[b], gl[b], V[b])
        stats.check(float(cost[b]), grad[b].astype(np.float64), c_ref, g_ref, margin, f"traj {b}")
        if margin[1] >= 2e-5:
            assert terms[b, 0] == pytest.approx(t_ref[0], rel=1e-4, abs=1e-3)
        active += t_ref[0] > 0
    stats.done()
    assert active >= B // 2            # the goal term is live (seed 0 of each pair ends on the goal)
    ctx.close()


def test_cspace_eval_ik_parity(native, O):
    B = 75
    rb = robots.franka64()
    worlds = [inputs.random_world(11, e, 20, lo=-0.8, hi=0.8) for e in range(2)]
    cp = inputs.CostParams(flags=inputs.CSPACE)
    ctx = make(native, rb, worlds, cp)
    R = O.Robot(rb)
    g = np.random.default_rng(4)
    q = f32(g.uniform(rb.lo, rb.hi, (B, 7)))
    gl = f32(np.clip(q + g.normal(0, 0.05, (B, 7)), rb.lo, rb.hi))
    env = ((np.arange(B) // 32) % 2).astype(np.int32)
    cost, grad, _ = ctx.evaluate(T(q), T(gl), env=T(env, torch.int32))
    cost, grad = cost.cpu().numpy(), grad.cpu().numpy()
    stats = Stats()
    for b in range(B):
        c_ref, g_ref, _, margin, _ = O.eval_ik(R, O.World(worlds[env[b]]), cp, gl[b], q[b])
        stats.check(float(cost[b]), grad[b].astype(np.float64), c_ref, g_ref, ("ik", margin), f"ik {b}")
    stats.done()
    ctx.close()


def test_cspace_ik_solve_reaches_the_goal(native, O):
    """C-space IK to collision-free joint goals: GPU and oracle both reach theta_g."""
    rb = robots.franka64()
    R = O.Robot(rb)
    world = inputs.tabletop_scene(3, 0, 10)
    W = O.World(world)
    cp = inputs.CostParams(flags=inputs.CSPACE)
    ctx = make(native, rb, [world], cp)
    P, S = 4, 32
    goals = []
    g = np.random.default_rng(21)
    while len(goals) < P:
        q = g.uniform(rb.lo * 0.6, rb.hi * 0.6)
        c, _, t, _, _ = O.eval_ik(R, W, cp, q, q)
        if c == 0.0:                                # collision-free and inside the limits
            goals.append(q)
    goals = f32(np.array(goals))
    seeds = f32(np.stack([inputs.ik_seeds(rb, p, S) for p in range(P)]))
    sp = inputs.SolverParams(iters=60)
    out = ctx.solve(sp, T(seeds), T(goals))
    gq = out["best_traj"].cpu().numpy()
    o_q, o_c = O.solve_ik(R, [W], np.zeros(P, np.int32), cp, sp, seeds, goals, nthreads=8)
    for p in range(P):
        assert np.abs(gq[p] - goals[p]).max() < 2e-2, p
        assert np.abs(o_q[p, o_c[p].argmin()] - goals[p]).max() < 2e-2, p
    ctx.close()


def test_gradient_descent_teacher_forced(native, O):
    """history = 0 (gradient descent): the solver's recorded iterations 0-3 recomputed by
    the oracle from the GPU's own state (tests/test_gpu_solver_trace.py): d = -g element-wise,
    the candidates' costs, i* bit-exactly, the step taken."""
    from test_gpu_solver_trace import Tally, check_seed
    rb, starts, goals = planar_problems(O, 6)
    P, S, H = 6, 4, 16
    world = inputs.planar_scene()
    cp = inputs.CostParams(dt=0.25)
    ctx = make(native, rb, [world], cp)
    R, W = O.Robot(rb), O.World(world)
    seeds = f32(np.stack([inputs.to_seeds(rb, 7, p, starts[p], starts[p] + 0.6, S, H) for p in range(P)]))
    sp = inputs.SolverParams(iters=5, history=0)
    its = (0, 1, 2, 3)
    out = ctx.solve(sp, T(seeds), T(goals), start=T(starts), seed_outputs=True, trace_iters=its)
    tr = out["trace"].cpu().numpy()
    lo, hi = np.float32(np.tile(rb.lo, H)), np.float32(np.tile(rb.hi, H))
    tally = Tally()
    for p in range(P):
        def evalf(v, p=p):
            c, g, _, margin, _ = O.eval_traj(R, W, cp, starts[p], goals[p], v.reshape(H, 2))
            return c, g.reshape(-1), margin
        for s_ in range(S):
            recs = [native.parse_trace(tr[p, s_, j], H * 2, 0) for j in range(len(its))]
            for r in recs:
                np.testing.assert_array_equal(r["d"], -r["g"])     # GD: exactly -g in fp32
            check_seed(native, O, recs, H * 2, 0, sp, lo, hi, evalf, tally, f"GD p{p} s{s_}", iters=its)
    assert tally.steps >= 0.9 * P * S * len(its)
    ctx.close()


@pytest.mark.parametrize("history", [0, 25])
def test_history_variants_statistical(native, O, history):
    rb, starts, goals = planar_problems(O, 10)
    P, S, H = 10, 4, 16
    world = inputs.planar_scene()
    cp = inputs.CostParams(dt=0.25)
    ctx = make(native, rb, [world], cp)
    R, W = O.Robot(rb), O.World(world)
    seeds = f32(np.stack([inputs.to_seeds(rb, 9, p, starts[p], starts[p] + 0.4, S, H) for p in range(P)]))
    sp = inputs.SolverParams(iters=30, history=history)
    out = ctx.solve(sp, T(seeds), T(goals), start=T(starts), seed_outputs=True)
    _, o_c = O.solve_to(R, [W], np.zeros(P, np.int32), cp, sp, seeds, starts, goals, nthreads=8)
    g_best = out["best_cost"].cpu().numpy()
    assert np.median(g_best / o_c.min(1)) < 2.0
    c0, _, _ = ctx.evaluate(T(seeds.reshape(P * S, H, 2)), T(np.repeat(goals, S, 0)),
                            start=T(np.repeat(starts, S, 0)))
    assert np.all(out["seed_best_cost"].cpu().numpy().reshape(-1) <= c0.cpu().numpy() * (1 + 1e-6))
    if history == 25:
        rbf = robots.franka64()
        ctx2 = make(native, rbf, [inputs.tabletop_scene(0, 0, 20)], inputs.CostParams())
        ctas, smem = ctx2.solver_occupancy(32, 25, 4)
        assert smem > 116 * 1024 and ctas == 1          # the ring of 26 slots costs the 2nd CTA
        ctx2.close()
    ctx.close()
