"""Pins for the whole evaluation (O7, O2-O6 composed): directional central FD, invariants, weight
linearity, the zero-cost special case.  CPU only."""
import dataclasses

import numpy as np
import pytest

from paper_2310_17274_b200 import inputs, robots


def franka_problem(seed, H, n_boxes=14, flags=0):
    rb = robots.franka64()
    g = np.random.default_rng(seed)
    start = np.clip(rb.ready + g.normal(0, 0.3, 7), rb.lo + 0.05, rb.hi - 0.05)
    tgt = np.clip(start + g.normal(0, 0.8, 7), rb.lo, rb.hi)
    h = np.arange(1, H + 1)[:, None] / H
    V = start + (tgt - start) * h + g.normal(0, 0.05, (H, 7))
    world = inputs.random_world(seed, 0, n_boxes, lo=-0.7, hi=0.7, dmin=0.05, dmax=0.35)
    goal = np.concatenate([g.uniform(-0.5, 0.5, 3) + [0.3, 0, 0.4], [1, 0, 0, 0]])
    q = g.normal(size=4); goal[3:] = q / np.linalg.norm(q)
    cp = inputs.CostParams(flags=flags, dt=0.1)
    return rb, world, cp, start, goal, V


_FD_CHECKED = []


@pytest.mark.parametrize("seed", range(20))
def test_traj_directional_fd(O, seed):
    """S:636 criterion 1 analogue: analytic gradient vs central FD on random 7-DoF problems with
    obstacles (SWEEP and SPEED off: their gradients are surrogates, pinned separately)."""
    H = 8 + seed % 5
    rb, world, cp, start, goal, V = franka_problem(seed, H)
    R, W = O.Robot(rb), O.World(world)
    c, grad, terms, margin, cnt = O.eval_traj(R, W, cp, start, goal, V)
    assert c == pytest.approx(terms.sum(), rel=1e-14)
    g = np.random.default_rng(100 + seed)
    checked = 0
    for _ in range(20):
        u = g.normal(size=V.shape)
        eps = 1e-7
        cpl = O.eval_traj(R, W, cp, start, goal, V + eps * u)
        cmi = O.eval_traj(R, W, cp, start, goal, V - eps * u)
        if min(cpl[3], cmi[3], margin) < 1e-5:      # a branch within reach of the FD step
            continue
        fd = (cpl[0] - cmi[0]) / (2 * eps)
        an = float(np.sum(grad * u))
        assert abs(fd - an) <= 1e-6 * max(1.0, abs(fd), np.abs(grad).sum())
        checked += 1
    _FD_CHECKED.append(checked)


def test_traj_fd_not_vacuous():
    assert sum(_FD_CHECKED) >= 150 and sum(c > 0 for c in _FD_CHECKED) >= 10


def test_traj_world_term_active(O):
    """The FD problems really exercise collision terms (otherwise the pin is vacuous)."""
    active = 0
    for seed in range(20):
        rb, world, cp, start, goal, V = franka_problem(seed, 10)
        _, _, terms, _, cnt = O.eval_traj(O.Robot(rb), O.World(world), cp, start, goal, V)
        active += terms[4] > 0
    assert active >= 5


_IK_CHECKED = []


@pytest.mark.parametrize("seed", range(10))
def test_ik_fd(O, seed):
    rb, world, cp, start, goal, V = franka_problem(seed, 8)
    R, W = O.Robot(rb), O.World(world)
    q = V[3]
    c, grad, terms, margin, _ = O.eval_ik(R, W, cp, goal, q)
    assert terms[2] == 0.0
    checked = 0
    for d in range(7):
        e = np.zeros(7); e[d] = 1e-7
        a, b = O.eval_ik(R, W, cp, goal, q + e), O.eval_ik(R, W, cp, goal, q - e)
        if min(a[3], b[3], margin) < 1e-5:
            continue
        fd = (a[0] - b[0]) / 2e-7
        assert abs(fd - grad[d]) <= 1e-6 * max(1.0, abs(fd), np.abs(grad).sum())
        checked += 1
    _IK_CHECKED.append(checked)


def test_ik_fd_not_vacuous():
    assert sum(_IK_CHECKED) >= 35


def test_zero_cost_case(O):
    """S:261 / S:270: goal = FK(start), constant trajectory, empty world -> C = 0, grad = 0."""
    rb = robots.franka64()
    R = O.Robot(rb)
    start = rb.ready.copy()
    _, _, ee = O.fk(R, start)
    empty = O.World(inputs.World(np.zeros((0, 3)), np.zeros((0, 4)), np.zeros((0, 3)), np.zeros(0, np.int32)))
    for flags in (0, inputs.SWEEP | inputs.SPEED | inputs.JERK):
        cp = inputs.CostParams(flags=flags)
        V = np.tile(start, (16, 1))
        c, g, terms, _, _ = O.eval_traj(R, empty, cp, start, ee, V)
        assert abs(c) < 1e-9 and np.abs(g).max() < 1e-6
        c, g, _, _, _ = O.eval_ik(R, empty, cp, ee, start)
        assert abs(c) < 1e-9 and np.abs(g).max() < 1e-6


def test_nonnegative_and_weight_linearity(O):
    """every term >= 0; doubling one weight doubles exactly that term."""
    rb, world, cp, start, goal, V = franka_problem(3, 12, flags=inputs.SWEEP | inputs.SPEED | inputs.JERK)
    R, W = O.Robot(rb), O.World(world)
    _, _, t0, _, _ = O.eval_traj(R, W, cp, start, goal, V)
    assert np.all(t0 >= 0)
    for field, idx in (("beta_world", 4), ("beta_self", 3)):
        cp2 = dataclasses.replace(cp, **{field: 2 * getattr(cp, field)})
        _, _, t2, _, _ = O.eval_traj(R, W, cp2, start, goal, V)
        assert t2[idx] == 2 * t0[idx]
        others = [i for i in range(5) if i != idx]
        np.testing.assert_array_equal(t2[others], t0[others])
    cp2 = dataclasses.replace(cp, a8=2 * cp.a8, a9=2 * cp.a9)
    _, _, t2, _, _ = O.eval_traj(R, W, cp2, start, goal, V)
    assert t2[2] == pytest.approx(2 * t0[2], rel=1e-14)


def test_dt_doubling_halves_world(O):
    """(v) S:154: with SPEED on, doubling dt halves the world term exactly (same geometry)."""
    rb, world, cp, start, goal, V = franka_problem(4, 12, flags=inputs.SWEEP | inputs.SPEED)
    R, W = O.Robot(rb), O.World(world)
    _, _, t1, _, _ = O.eval_traj(R, W, cp, start, goal, V)
    _, _, t2, _, _ = O.eval_traj(R, W, dataclasses.replace(cp, dt=2 * cp.dt), start, goal, V)
    assert t1[4] > 0
    assert t2[4] == pytest.approx(0.5 * t1[4], rel=1e-13)


def test_static_trajectory_zero_world(O):
    """(i) with SPEED on, a static trajectory has zero world cost even in collision (A13)."""
    rb, world, cp, start, goal, V = franka_problem(5, 12, flags=inputs.SWEEP | inputs.SPEED)
    V = np.tile(start, (12, 1))
    _, _, t, _, _ = O.eval_traj(O.Robot(rb), O.World(world), cp, start, goal, V)
    assert t[4] == 0.0


def test_pinned_and_aliased_get_zero_gradient(O):
    rb, world, cp, start, goal, V = franka_problem(6, 16, flags=inputs.SWEEP | inputs.SPEED | inputs.JERK)
    _, g, _, _, _ = O.eval_traj(O.Robot(rb), O.World(world), cp, start, goal, V)
    H = 16
    assert np.all(g[0:3] == 0) and np.all(g[H - 4:H - 1] == 0)
    assert np.abs(g[H - 1]).sum() > 0
