"""GPU parity of the motion-generation pipeline pieces (Alg. 4 P:2049-2069,
App. B; readings B15-B18) against the oracle O13, and an end-to-end check of the
pipeline whose claims (pose error, validity of every state, limits reached after the final
retime) are re-verified with the oracle's own FK, mask and retime."""
import numpy as np
import pytest
import torch

from paper_2310_17274_b200 import inputs, robots
from test_gpu_parity import ref_traj, T, f32, make
from test_oracle_motion import _traj

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def native():
    from paper_2310_17274_b200 import native as N
    return N


def test_retime_parity(native, O):
    rb = robots.franka64()
    R = O.Robot(rb)
    ctx = make(native, rb, [inputs.tabletop_scene(0, 0, 5)], inputs.CostParams())
    B, H = 40, 32
    data = [_traj(rb, 100 + b, H, amp=0.3 + 0.05 * (b % 7)) for b in range(B)]
    st = f32(np.array([d[0] for d in data])); V = f32(np.array([d[1] for d in data]))
    dt = f32(np.linspace(0.05, 0.5, B))
    sc, dto, jm = [x.cpu().numpy() for x in ctx.retime(T(V), T(st), dt=T(dt))]
    for b in range(B):
        s, d_opt, _ = O.retime(R, st[b], V[b], dt[b])
        assert sc[b] == pytest.approx(s, rel=2e-5)
        assert dto[b] == pytest.approx(d_opt, rel=2e-5)
        _, _, j = O.derivs(O.state_map(st[b], V[b]), H, dt[b])
        assert jm[b] == pytest.approx(np.abs(j).max() / s ** 3, rel=1e-4)
    # default dt (the cost params' 0.25) and one start row per problem of 4 trajectories
    st2 = st[[0, 4]]
    sc2, _, _ = ctx.retime(T(V[:8]), T(st2))
    for b in range(8):
        assert sc2[b].item() == pytest.approx(O.retime(R, st2[b // 4], V[b], 0.25)[0], rel=2e-5)
    ctx.close()


def test_goal_error_parity(native, O):
    rb = robots.franka64()
    R = O.Robot(rb)
    ctx = make(native, rb, [inputs.tabletop_scene(0, 0, 5)], inputs.CostParams())
    g = np.random.default_rng(3)
    P, S, H = 5, 6, 16
    V = f32(g.uniform(rb.lo, rb.hi, (P, S, H, 7)))
    goals = f32(np.array([O.fk(R, g.uniform(rb.lo, rb.hi))[2] for _ in range(P)]))
    Vt = T(V)
    pe, re = ctx.goal_error(Vt.view(-1)[(H - 1) * 7:], T(goals), B=P * S, stride=H * 7, goal_div=S)
    pe, re = pe.cpu().numpy(), re.cpu().numpy()
    for b in range(P * S):
        p, s = divmod(b, S)
        rp, rr = O.goal_error(R, V[p, s, H - 1], goals[p])
        assert pe[b] == pytest.approx(rp, abs=2e-6)
        assert re[b] == pytest.approx(rr, abs=2e-6)
    ctx.close()


def test_scores_rank_seeds_gather(native, O):
    g = np.random.default_rng(9)
    P, S, D, H, k = 7, 20, 7, 8, 12
    q = f32(g.normal(size=(P, S, D))); q0 = f32(g.normal(size=(P, D)))
    pe = f32(g.uniform(0, 0.01, (P, S))); re = f32(g.uniform(0, 0.002, (P, S)))
    valid = (g.random((P, S)) < 0.7).astype(np.uint8)
    valid[3] = 0                                                   # a problem without a valid seed
    sc = native.ik_scores(T(q), T(q0), T(pe), T(re), T(valid, torch.uint8), 5e-3, 1e-3, 1.0, 0.01).cpu().numpy()
    for p in range(P):
        for s in range(S):
            ok = valid[p, s] and pe[p, s] < 5e-3 and re[p, s] < 1e-3
            ref = O.ik_score(q[p, s], q0[p], pe[p, s], re[p, s], 1.0, 0.01)
            assert (sc[p, s] == np.inf) if not ok else sc[p, s] == pytest.approx(ref, rel=1e-5)
    sc[1, 4] = sc[1, 9] = 0.5                                      # an exact tie -> lower index first
    idx, cnt = native.rank_seeds(T(sc), k)
    idx, cnt = idx.cpu().numpy(), cnt.cpu().numpy()
    for p in range(P):
        fin = [s for s in np.argsort(sc[p], kind="stable") if np.isfinite(sc[p, s])]
        assert cnt[p] == len(fin)
        if fin:
            assert list(idx[p]) == [fin[j % len(fin)] for j in range(k)]
        else:
            assert np.all(idx[p] == -1)
    # linear seeds from the ranked solutions, and gathering rows by index
    seeds = native.linear_seeds(T(q0), T(q), H, idx=T(idx, torch.int32)).cpu().numpy()
    for p in range(P):
        for s in range(k):
            j = idx[p, s]
            ref = O.linear_seed(q0[p], q[p, j] if j >= 0 else q0[p], H)
            np.testing.assert_allclose(seeds[p, s], ref, atol=2e-6)
    pick = g.integers(0, k, P).astype(np.int32); pick[2] = -1      # -1 -> a zero row
    rows = native.gather_rows(T(seeds.reshape(P, k, H * D)), T(pick, torch.int32)).cpu().numpy()
    for p in range(P):
        np.testing.assert_array_equal(rows[p], seeds[p, pick[p]].reshape(-1) if pick[p] >= 0 else 0.0)
    # blended TO score with the invalid-state penalty
    mj = f32(g.uniform(10, 500, (P, S))); dto = f32(g.uniform(0.02, 0.3, (P, S)))
    vs = (g.random((P, S, H)) < 0.97).astype(np.uint8)
    ts = native.to_scores(T(pe), T(re), T(mj), T(dto), T(vs, torch.uint8), H, 5e-3, 1e-3, 1.0, 1e-4, 1.0,
                          penalty=1e6).cpu().numpy()
    for p in range(P):
        for s in range(S):
            ok = pe[p, s] < 5e-3 and re[p, s] < 1e-3 and vs[p, s].all()
            ref = O.blended_score(pe[p, s], re[p, s], mj[p, s], (H - 1) * dto[p, s], 1.0, 1e-4, 1.0)
            assert ts[p, s] == pytest.approx(ref + (0 if ok else 1e6), rel=1e-5)


@pytest.mark.parametrize("H", [32, 16])
def test_per_problem_dt_eval_parity(native, O, H):
    """crb_evaluate_cost_grad_dt vs the oracle at the B15-scaled parameters (jerk on)."""
    from test_gpu_parity import Stats, franka_trajs
    B = 64
    rb, starts, goals_cfg, trajs = franka_trajs(700 + H, B, H, noise=0.1)
    worlds = [inputs.tabletop_scene(6, 0, 20)]
    cp = inputs.CostParams(flags=inputs.SWEEP | inputs.SPEED | inputs.JERK, dt=0.25)
    ctx = make(native, rb, worlds, cp)
    R, W = O.Robot(rb), O.World(worlds[0])
    V, st = f32(trajs), f32(starts)
    gl = f32(np.array([O.fk(R, q)[2] for q in goals_cfg]))
    dt = f32(np.geomspace(0.03, 0.6, B))
    cost, grad, terms = ctx.evaluate(T(V), T(gl), start=T(st), dt=T(dt))
    cost, grad, terms = cost.cpu().numpy(), grad.cpu().numpy(), terms.cpu().numpy()
    stats = Stats()
    for b in range(B):
        cps = O.scale_params(cp, float(dt[b]), 0.25, jerk_on=True)
        c_ref, g_ref, t_ref, margin = ref_traj(O, R, W, cps, st[b], gl[b], V[b])
        stats.check(float(cost[b]), grad[b].astype(np.float64), c_ref, g_ref, margin, f"dt {dt[b]}")
        if margin[1] >= 2e-5:
            assert terms[b, 2] == pytest.approx(t_ref[2], rel=1e-4, abs=1e-3)
    stats.done()
    ctx.close()


def test_interpolate_parity(native, O):
    """B21: the interpolation kernel against the oracle on random state sequences and
    spacings (including a spacing below dt_fine and one that truncates at n_max): the count n is
    decided exactly, points agree to fp32 rounding, rows past n repeat x_H."""
    g = np.random.default_rng(8)
    B, H, D, n_max = 9, 32, 7, 256
    x = f32(g.uniform(-2.5, 2.5, (B, H, D)))
    dt = f32(np.array([0.25, 0.1, 0.137, 0.02, 0.0253, 0.3, 0.2083, 0.05, 0.4]))
    pts, n = native.interpolate(T(x), T(dt), 0.025, n_max)
    pts, n = pts.cpu().numpy(), n.cpu().numpy()
    for b in range(B):
        # identical inputs: the kernel receives dt_fine as fp32 (the count is decided in fp64 from it)
        nr, ref = O.interpolate(x[b], float(dt[b]), float(np.float32(0.025)), n_max)
        assert n[b] == nr, (b, n[b], nr)
        m = min(nr, n_max)
        np.testing.assert_allclose(pts[b, :m], ref, rtol=0, atol=3e-6)
        if nr <= n_max:
            np.testing.assert_array_equal(pts[b, m - 1], x[b, -1])
        if m < n_max:
            np.testing.assert_array_equal(pts[b, m:], np.broadcast_to(x[b, -1], (n_max - m, D)))
    assert (n > n_max).any() and (n <= n_max).any()


def test_motion_gen_pipeline_end_to_end(native, O):
    # Trajectories diverge chaotically under fp32 reordering (north_star), so the success COUNT is a
    # statistical bound: one attempt succeeds on ~47 % of these synthetic problems (bench f2: 30-31
    # of 64), and >= 4 of 16 fails with probability < 0.5 % at that rate.  Every success is
    # re-checked against the oracle below.
    from paper_2310_17274_b200 import motion_gen, workload
    P = 16
    wl = workload.franka_to(0, list(range(P)), S=12, H=32, iters=100)
    ctx = native.Context(0)
    ctx.set_robot(wl.robot); ctx.set_world(wl.worlds); ctx.set_cost_params(wl.cost)
    mg = motion_gen.MotionGen(ctx, wl.robot, wl.cost)
    ik_seeds = T(mg.ik_seed_batch(wl.robot, range(P), 32))
    out = mg.plan(T(wl.start), T(wl.goal), T(wl.env, torch.int32), ik_seeds)
    torch.cuda.synchronize()
    R = O.Robot(wl.robot)
    succ = out["success"].cpu().numpy()
    traj = out["traj"].cpu().numpy().astype(np.float64)
    dt = out["dt"].cpu().numpy().astype(np.float64)
    assert succ.sum() >= 4, succ
    for p in np.nonzero(succ)[0]:
        W = O.World(wl.worlds[wl.env[p]])
        pe, re = O.goal_error(R, traj[p, -1], wl.goal[p])
        assert pe < 5.5e-3 and re < 0.051                           # the pose claim, re-checked
        ok = [O.mask_sample(R, W, traj[p, h]) for h in range(32)]
        assert sum(v for v, mg_ in ok if mg_ > 2e-5) == sum(1 for v, mg_ in ok if mg_ > 2e-5)
        s, _, _ = O.retime(R, wl.start[p], out["variables"][p].cpu().numpy().astype(np.float64), dt[p])   # limits at dt_f
        assert s == pytest.approx(1.0, rel=1e-3)
        # the success claim includes every state of the 0.025 s grid (B21), re-checked
        _, fine = O.interpolate(traj[p], dt[p], 0.025)
        okf = [O.mask_sample(R, W, q) for q in fine]
        assert all(v for v, mg_ in okf if mg_ > 2e-5)
    assert np.all(out["ik_count"].cpu().numpy() > 0)
    assert np.array_equal(out["success"].cpu().numpy(),
                          (out["final_score"] < float("inf")).cpu().numpy() & out["fine_valid"].cpu().numpy())
    ctx.close()


def test_motion_gen_retries_keep_successes_and_recheck(native, O):
    """plan_retry (up to three attempts with fresh linear seeds): first-attempt successes
    are kept bit for bit, the success count never drops, and every success is re-checked against
    the oracle (pose thresholds, every state valid)."""
    from paper_2310_17274_b200 import motion_gen, workload
    P = 8
    wl = workload.franka_to(0, list(range(P)), S=12, H=32, iters=100)
    ctx = native.Context(0)
    ctx.set_robot(wl.robot); ctx.set_world(wl.worlds); ctx.set_cost_params(wl.cost)
    mg = motion_gen.MotionGen(ctx, wl.robot, wl.cost)
    args = (T(wl.start), T(wl.goal), T(wl.env, torch.int32))
    one = mg.plan(*args, T(mg.ik_seed_batch(wl.robot, range(P), 32)))
    three = mg.plan_retry(*args, range(P), attempts=3)
    s1, s3 = one["success"].cpu().numpy(), three["success"].cpu().numpy()
    att = three["attempt"].cpu().numpy()
    assert s3.sum() >= s1.sum()
    assert np.all(att[s1] == 1)
    assert torch.equal(three["traj"][torch.tensor(s1)], one["traj"][torch.tensor(s1)])
    assert np.all((att >= 1) & (att <= 3))
    R = O.Robot(wl.robot)
    traj = three["traj"].cpu().numpy().astype(np.float64)
    for p in np.nonzero(s3)[0]:
        W = O.World(wl.worlds[wl.env[p]])
        pe, re = O.goal_error(R, traj[p, -1], wl.goal[p])
        assert pe < 5.5e-3 and re < 0.051
        ok = [O.mask_sample(R, W, traj[p, h]) for h in range(32)]
        assert sum(v for v, mg_ in ok if mg_ > 2e-5) == sum(1 for v, mg_ in ok if mg_ > 2e-5)
    ctx.close()
