"""GPU parity of the particle warm-up: §4.2 "Particle-Based Optimization"
(P:192-199), Alg. 5, Eqs. particle_1/2 with readings B6-B10, run inside the
persistent solver kernels before L-BFGS (crb_lbfgs_solve with particle_iters > 0).

With iters = 0 the solver returns the warm-up mean as each seed's best trajectory, so the mean
is compared directly with the fp64 oracle (orc_particle_solve) on the same seeds and the same
Philox counters.  The weights are exp(-C/beta) of fp32 vs fp64 costs: with beta of the order of
the costs they are smooth and the means agree to ~1e-4 rad; with the SPEC beta = 1 they are
one-hot, and the means agree to fp32 rounding wherever the top-2 cost gap / beta is large (the
decision is then unique: ③ "compare what is unique").  Seeds whose particles come within the
oracle's branch margin of a COST discontinuity (a sweep sample in contact appearing or
disappearing; oracle.h O10, cost-only margin mode) are excluded.
"""
import numpy as np
import pytest
import torch

from paper_2310_17274_b200 import inputs, robots
from test_gpu_parity import MARGIN, T, f32, franka_trajs, make, planar_problems

pytestmark = pytest.mark.gpu

MU_ATOL_SMOOTH = 2e-3     # rad; weights exp(-C/beta) with beta ~ C/4: dw/w ~ dC/beta ~ 1e-4
MU_ATOL_ONEHOT = 2e-5     # rad; one-hot weights: the mean is (1-k_mu) mu + k_mu theta_best in fp32


@pytest.fixture(scope="module")
def native():
    from paper_2310_17274_b200 import native as N
    return N


def test_particle_normals_match_oracle(native, O):
    """B9: identical Philox words on both sides; normals agree to fp32 rounding of Box-Muller."""
    for k0, k1, it, seed in [(0, 0, 0, 0), (1234, 7, 1, 99), (0xFFFFFFFF, 3, 2, 5)]:
        z = native.particle_normals(k0, k1, 224, 64, it, seed).cpu().numpy().astype(np.float64)
        ref = np.array([[O.normal(k0, k1, v, l, it, seed) for v in range(224)] for l in range(64)])
        np.testing.assert_allclose(z, ref, rtol=0, atol=4e-6)
        assert abs(ref.mean()) < 0.05 and abs(ref.std() - 1) < 0.05


def _oracle_means(O, R, Ws, env, cp, sp, seeds, starts, goals, lo, hi, problem_base, seed_base):
    """Per seed: (mu, min branch margin over all particle evaluations, costs[iters][n])."""
    P, S = seeds.shape[:2]
    shape = seeds.shape[2:]
    out = []
    for p in range(P):
        for s in range(S):
            mins = [np.inf]

            def f(x):
                if len(shape) == 2:
                    c, _, _, m, _ = O.eval_traj(R, Ws[env[p]], cp, starts[p], goals[p], x.reshape(shape))
                else:
                    c, _, _, m, _ = O.eval_ik(R, Ws[env[p]], cp, goals[p], x)
                mins[0] = min(mins[0], m)
                return c
            with O.cost_only_margins():     # cost-only passes: only cost jumps matter
                mu, _, costs = O.particle_solve(f, seeds[p, s].reshape(-1), sp, lo, hi,
                                                problem=problem_base + p, seed=seed_base + s)
            out.append((mu.reshape(shape), mins[0], costs))
    return out


def _to_case(O, P=3, S=4, H=16):
    rb, starts, goals_cfg, trajs = franka_trajs(321, P * S, H)
    R = O.Robot(rb)
    worlds = [inputs.tabletop_scene(4, e, 6) for e in range(2)]
    env = np.arange(P, dtype=np.int32) % 2
    st = f32(starts[:P])
    gl = f32(np.array([O.fk(R, q)[2] for q in goals_cfg[:P]]))
    seeds = f32(trajs.reshape(P, S, H, rb.n_dof))
    return rb, R, worlds, env, st, gl, seeds


@pytest.mark.parametrize("beta_mode,n_particles", [("smooth", 32), ("onehot", 32), ("smooth", 3)])
def test_particle_warmup_to_parity(native, O, beta_mode, n_particles):
    """n_particles = 3 < A = 4: the first of the A accumulation chunks is empty (and the solver
    runs sequentially: the latency mode needs a particle per CTA)."""
    P, S, H = 3, 4, 16
    rb, R, worlds, env, st, gl, seeds = _to_case(O, P, S, H)
    Ws = [O.World(w) for w in worlds]
    cp = inputs.CostParams(dt=0.25)
    c0 = [O.eval_traj(R, Ws[env[p]], cp, st[p], gl[p], seeds[p, s])[0] for p in range(P) for s in range(S)]
    beta = 0.25 * float(np.median(c0)) if beta_mode == "smooth" else 1.0
    # sigma_0 = 0.03 (hi - lo): iid per-step draws at the SPEC's 0.1 put most particles deep in
    # contact, where sweep samples cross their exit bound in nearly every evaluation
    sp = inputs.SolverParams(iters=0, particle_iters=2, n_particles=n_particles, particle_beta=beta, rng_key=77,
                             sigma0_frac=0.03)
    ctx = make(native, rb, worlds, cp)
    out = ctx.solve(sp, T(seeds), T(gl), start=T(st), env=T(env, torch.int32), seed_outputs=True,
                    seed_base=3, problem_base=5)
    mu_gpu = out["seed_best_traj"].cpu().numpy().astype(np.float64)
    lo, hi = np.tile(rb.lo, H), np.tile(rb.hi, H)
    ref = _oracle_means(O, R, Ws, env, cp, sp, seeds, st, gl, lo, hi, 5, 3)
    checked, worst = 0, 0.0
    for u, (mu, margin, costs) in enumerate(ref):
        p, s = divmod(u, S)
        if margin < MARGIN:
            continue
        if beta_mode == "onehot":
            gaps = [np.diff(np.sort(c)[:2])[0] / beta for c in costs]
            if min(gaps) < 50.0:        # weights not one-hot: the fp32/fp64 decision may differ
                continue
        err = np.abs(mu_gpu[p, s] - mu).max()
        worst = max(worst, err)
        assert err <= (MU_ATOL_SMOOTH if beta_mode == "smooth" else MU_ATOL_ONEHOT), (u, err)
        assert np.abs(mu - seeds[p, s]).max() > 1e-3, "warm-up did not move: vacuous"
        checked += 1
    assert checked >= P * S // 2, f"only {checked}/{P * S} seeds comparable"
    print(f"particle TO parity ({beta_mode}): {checked} seeds, worst |dmu| = {worst:.2e}")
    ctx.close()


def test_particle_warmup_ik_parity(native, O):
    """IK: 40 seeds = a full and a ragged 32-lane group (inactive lanes must not leak)."""
    rb = robots.franka64()
    R = O.Robot(rb)
    world = inputs.tabletop_scene(3, 0, 20)
    W = O.World(world)
    cp = inputs.CostParams()
    P, S = 2, 40
    g = np.random.default_rng(12)
    goals = f32(np.array([O.fk(R, g.uniform(rb.lo * 0.6, rb.hi * 0.6))[2] for _ in range(P)]))
    seeds = f32(np.stack([inputs.ik_seeds(rb, p, S) for p in range(P)]))
    c0 = [O.eval_ik(R, W, cp, goals[p], seeds[p, s])[0] for p in range(P) for s in range(S)]
    sp = inputs.SolverParams(iters=0, particle_iters=2, n_particles=64,
                             particle_beta=0.25 * float(np.median(c0)), rng_key=9)
    ctx = make(native, rb, [world], cp)
    out = ctx.solve(sp, T(seeds), T(goals), seed_outputs=True)
    mu_gpu = out["seed_best_traj"].cpu().numpy().astype(np.float64)
    ref = _oracle_means(O, R, [W], np.zeros(P, np.int32), cp, sp, seeds, None, goals, rb.lo, rb.hi, 0, 0)
    checked, worst = 0, 0.0
    for u, (mu, margin, _) in enumerate(ref):
        p, s = divmod(u, S)
        if margin < MARGIN:
            continue
        err = np.abs(mu_gpu[p, s] - mu).max()
        worst = max(worst, err)
        assert err <= MU_ATOL_SMOOTH, (u, err)
        checked += 1
    assert checked >= 0.8 * P * S
    print(f"particle IK parity: {checked} seeds, worst |dmu| = {worst:.2e}")
    ctx.close()


@pytest.mark.parametrize("cluster", [0, 1])
def test_particle_warmup_ik_parity_d16(native, O, cluster):
    """D = 16 makes D * 32 = 512 particle elements per 32-seed group, two per
    thread of the 256-thread CTA.  Every dof (not only the first 8) must be sampled, updated and
    given fresh sin / cos; sequential and latency-mode (cluster) kernels against the oracle."""
    from test_gpu_world_builds import capacity_robot
    rb = capacity_robot()
    D = rb.n_dof
    R = O.Robot(rb)
    world = inputs.random_world(61, 0, 24, lo=-1.2, hi=1.2, dmax=0.3)
    W = O.World(world)
    cp = inputs.CostParams()
    P, S = 1, 33
    g = np.random.default_rng(16)
    goals = f32(np.array([O.fk(R, g.uniform(-1.0, 1.0, D))[2] for _ in range(P)]))
    seeds = f32(g.uniform(-1.5, 1.5, (P, S, D)))
    c0 = [O.eval_ik(R, W, cp, goals[p], seeds[p, s])[0] for p in range(P) for s in range(S)]
    sp = inputs.SolverParams(iters=0, particle_iters=2, n_particles=16,
                             particle_beta=0.25 * float(np.median(c0)), rng_key=21, cluster=cluster)
    ctx = make(native, rb, [world], cp)
    out = ctx.solve(sp, T(seeds), T(goals), seed_outputs=True)
    mu_gpu = out["seed_best_traj"].cpu().numpy().astype(np.float64)
    ref = _oracle_means(O, R, [W], np.zeros(P, np.int32), cp, sp, seeds, None, goals, rb.lo, rb.hi, 0, 0)
    checked, worst = 0, 0.0
    for u, (mu, margin, _) in enumerate(ref):
        p, s = divmod(u, S)
        if margin < MARGIN:
            continue
        err = np.abs(mu_gpu[p, s] - mu).max()
        worst = max(worst, err)
        assert err <= MU_ATOL_SMOOTH, (u, err, np.abs(mu_gpu[p, s] - mu))
        assert np.abs(mu[8:] - seeds[p, s, 8:]).max() > 1e-3, "dofs 8..15 did not move: vacuous"
        checked += 1
    assert checked >= 0.8 * P * S
    print(f"particle IK parity D=16 (cluster={cluster}): {checked} seeds, worst |dmu| = {worst:.2e}")
    ctx.close()


def test_particle_sharding_is_bit_exact(native, O):
    """The draws are keyed by GLOBAL problem / seed indices (B9): solving a slice with
    problem_base / seed_base reproduces the full solve bit for bit (the multi-GPU seed and
    problem sharding of §8(e) relies on this)."""
    rb, starts, goals = planar_problems(O, 4)
    P, S, H = 4, 6, 16
    ctx = make(native, rb, [inputs.planar_scene()], inputs.CostParams(dt=0.25))
    seeds = f32(np.stack([inputs.to_seeds(rb, 3, p, starts[p], starts[p] + 0.5, S, H) for p in range(P)]))
    sp = inputs.SolverParams(iters=6, particle_iters=2, n_particles=16, rng_key=5)
    full = ctx.solve(sp, T(seeds), T(goals), start=T(starts), seed_outputs=True)
    a = ctx.solve(sp, T(seeds[:, :2]), T(goals), start=T(starts), seed_outputs=True)
    b = ctx.solve(sp, T(seeds[:, 2:]), T(goals), start=T(starts), seed_outputs=True, seed_base=2)
    c = ctx.solve(sp, T(seeds[1:]), T(goals[1:]), start=T(starts[1:]), seed_outputs=True, problem_base=1)
    ft, fc = full["seed_best_traj"], full["seed_best_cost"]
    assert torch.equal(torch.cat([a["seed_best_traj"], b["seed_best_traj"]], 1), ft)
    assert torch.equal(torch.cat([a["seed_best_cost"], b["seed_best_cost"]], 1), fc)
    assert torch.equal(c["seed_best_traj"], ft[1:]) and torch.equal(c["seed_best_cost"], fc[1:])
    again = ctx.solve(sp, T(seeds), T(goals), start=T(starts), seed_outputs=True)
    assert torch.equal(again["seed_best_traj"], ft)                    # deterministic
    sp2 = inputs.SolverParams(iters=6, particle_iters=2, n_particles=16, rng_key=6)
    other = ctx.solve(sp2, T(seeds), T(goals), start=T(starts), seed_outputs=True)
    assert not torch.equal(other["seed_best_traj"], ft)                # the key matters
    ctx.close()


def test_particle_ik_group_sharding_bit_exact(native, O):
    rb = robots.franka64()
    R = O.Robot(rb)
    world = inputs.tabletop_scene(3, 1, 10)
    ctx = make(native, rb, [world], inputs.CostParams())
    P, S = 2, 64
    g = np.random.default_rng(4)
    goals = f32(np.array([O.fk(R, g.uniform(rb.lo * 0.6, rb.hi * 0.6))[2] for _ in range(P)]))
    seeds = f32(np.stack([inputs.ik_seeds(rb, p, S) for p in range(P)]))
    sp = inputs.SolverParams(iters=10, particle_iters=2, n_particles=32, rng_key=1)
    full = ctx.solve(sp, T(seeds), T(goals), seed_outputs=True)
    hi = ctx.solve(sp, T(seeds[:, 32:]), T(goals), seed_outputs=True, seed_base=32)
    assert torch.equal(hi["seed_best_traj"], full["seed_best_traj"][:, 32:])
    assert torch.equal(hi["seed_best_cost"], full["seed_best_cost"][:, 32:])
    ctx.close()


def test_particle_then_lbfgs_ik_statistical_vs_oracle(native, O):
    """The paper's pipeline (2 particle iterations, then L-BFGS) on collision-free IK:
    GPU and oracle success rates agree."""
    rb = robots.franka64()
    R = O.Robot(rb)
    world = inputs.tabletop_scene(3, 0, 20)
    W = O.World(world)
    cp = inputs.CostParams()
    ctx = make(native, rb, [world], cp)
    P, S = 6, 30
    g = np.random.default_rng(11)
    goals = f32(np.array([O.fk(R, g.uniform(rb.lo * 0.6, rb.hi * 0.6))[2] for _ in range(P)]))
    seeds = f32(np.stack([inputs.ik_seeds(rb, p, S) for p in range(P)]))
    sp = inputs.SolverParams(iters=60, particle_iters=2, n_particles=64, particle_beta=1.0, rng_key=3)
    out = ctx.solve(sp, T(seeds), T(goals), seed_outputs=True)
    o_q, o_c = O.solve_ik(R, [W], np.zeros(P, np.int32), cp, sp, seeds, goals, nthreads=8)

    def pos_err(q, goal):
        return np.linalg.norm(O.fk(R, q)[2][:3] - goal[:3])
    gq = out["best_traj"].cpu().numpy().astype(np.float64)
    g_ok = sum(pos_err(gq[p], goals[p]) < 0.01 for p in range(P))
    o_ok = sum(pos_err(o_q[p, o_c[p].argmin()], goals[p]) < 0.01 for p in range(P))
    assert g_ok >= o_ok - 1, (g_ok, o_ok)
    assert np.median(out["best_cost"].cpu().numpy() / o_c.min(1)) < 2.0
    ctx.close()


def test_particle_argument_errors(native, O):
    rb, starts, goals = planar_problems(O, 1)
    ctx = make(native, rb, [inputs.planar_scene()], inputs.CostParams())
    seeds = f32(np.zeros((1, 1, 16, 2)))
    for bad in [dict(particle_iters=-1), dict(particle_iters=1, n_particles=0),
                dict(particle_iters=1, particle_beta=0.0), dict(particle_iters=1, k_mu=1.5)]:
        with pytest.raises(native.CrbError) as e:
            ctx.solve(inputs.SolverParams(iters=1, **bad), T(seeds), T(goals), start=T(starts))
        assert e.value.code == -1                   # CRB_E_ARG
    ctx.close()
