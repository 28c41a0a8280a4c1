"""Pins for the oracle's solver (O8, O9): textbook BFGS identity, known minima, hand-evaluated line
searches, the fp32 selection mirror.  CPU only."""
import dataclasses
import math

import numpy as np
import pytest

from paper_2310_17274_b200 import inputs


def dense_bfgs_direction(S, Y, g):
    """Nocedal & Wright (7.19) applied to H0 = gamma I with the same pairs, d = -H g."""
    n = g.shape[0]
    if len(S) == 0:
        return -g
    s, y = S[-1], Y[-1]
    Hm = (s @ y) / (y @ y) * np.eye(n)
    for s, y in zip(S, Y):
        rho = 1.0 / (s @ y)
        V = np.eye(n) - rho * np.outer(y, s)
        Hm = V.T @ Hm @ V + rho * np.outer(s, s)
    return -Hm @ g


def test_two_loop_matches_dense_bfgs(O):
    g = np.random.default_rng(0)
    for n in (3, 10, 40):
        for count in range(0, 9):
            A = g.normal(size=(n, n)); A = A @ A.T + n * np.eye(n)
            S = g.normal(size=(count, n)); Y = S @ A + 0.01 * g.normal(size=(count, n))
            grad = g.normal(size=n)
            rho = 1.0 / np.einsum("ij,ij->i", S, Y)
            d = O.lbfgs_direction(S, Y, rho, grad)
            ref = dense_bfgs_direction(list(S), list(Y), grad)
            np.testing.assert_allclose(d, ref, rtol=1e-10, atol=1e-12 * np.abs(ref).max())
    d = O.lbfgs_direction(np.zeros((0, 5)), np.zeros((0, 5)), np.zeros(0), np.arange(5.0))
    np.testing.assert_array_equal(d, -np.arange(5.0))                  # S:325 empty history


def test_convex_quadratic(O):
    """0.5 x'Ax - b'x, n = 10, SPD: best c within 1e-8 of -0.5 b'A^-1 b after 50 iterations."""
    g = np.random.default_rng(1)
    n = 10
    Q, _ = np.linalg.qr(g.normal(size=(n, n)))
    A = Q @ np.diag(np.linspace(1, 10, n)) @ Q.T
    b = g.normal(size=n)
    fmin = -0.5 * b @ np.linalg.solve(A, b)
    sp = inputs.SolverParams(iters=50)
    bx, bc, trace = O.lbfgs_solve(lambda x: (0.5 * x @ A @ x - b @ x, A @ x - b), np.zeros(n), sp)
    assert bc - fmin < 1e-8
    assert np.all(np.diff(trace) <= 0)                                  # best monotone


def test_rosenbrock(O):
    """S:344 / S:643: Rosenbrock from (-1.2, 1), m = 8, 200 iterations -> f < 1e-6."""
    def f(x):
        a, b = x
        return (1 - a) ** 2 + 100 * (b - a * a) ** 2, np.array([-2 * (1 - a) - 400 * a * (b - a * a), 200 * (b - a * a)])
    sp = inputs.SolverParams(iters=200, history=8)
    bx, bc, trace = O.lbfgs_solve(f, np.array([-1.2, 1.0]), sp)
    assert bc < 1e-6
    assert np.all(np.diff(trace) <= 0)


def test_line_search_hand_cases(O):
    al = [0.01, 0.3, 0.7, 1.0]
    # f = x^2 at x = 1 with the Newton direction d = -1: alpha = 1 gives c = 0 (Armijo and strong Wolfe hold)
    x, d = 1.0, -1.0
    ca = [(x + a * d) ** 2 for a in al]; gda = [2 * (x + a * d) * d for a in al]
    assert O.ls_select(al, 1.0, 2 * x * d, ca, gda) == 3
    # with d = -2 (S:334 quotes alpha = 1; by hand alpha = 1 lands at x = -1, c = 1, failing Armijo;
    # alpha = 0.7 -> x = -0.4, c = 0.16 <= 1 - 2.8e-4 and |g d| = 1.6 <= 0.9 * 4: chosen)
    d = -2.0
    ca = [(x + a * d) ** 2 for a in al]; gda = [2 * (x + a * d) * d for a in al]
    assert O.ls_select(al, 1.0, 2 * x * d, ca, gda) == 2
    # uphill direction: nothing satisfies Armijo -> index 0 (noisy step)
    d = +1.0
    ca = [(x + a * d) ** 2 for a in al]; gda = [2 * (x + a * d) * d for a in al]
    for mode in (0, 1, 2):
        assert O.ls_select(al, 1.0, 2 * x * d, ca, gda, mode=mode) == 0
        assert O.ls_select_f32(al, 1.0, 2 * x * d, ca, gda, mode=mode) == 0


def test_noisy_step_never_stalls(O):
    """S:358 / S:643: with an adversarial (always uphill) objective the solver still moves."""
    seen = []

    def f(x):
        seen.append(x.copy())
        return float(np.sum(x)), -np.ones_like(x)    # gradient lies: d = +1 is uphill
    sp = inputs.SolverParams(iters=5)
    O.lbfgs_solve(f, np.zeros(3), sp)
    for a, b in zip(seen[0::5], seen[5::5]):
        assert not np.array_equal(a, b)


def test_f32_mirror_semantics(O):
    al = np.array([0.01, 0.3, 0.7, 1.0], np.float32)
    nan, inf = float("nan"), float("inf")
    # NaN candidates are never selected; ties keep the largest satisfying index
    assert O.ls_select_f32(al, 1.0, -1.0, [0.5, nan, 0.5, nan], [0, 0, 0, 0]) == 2
    assert O.ls_select_f32(al, 1.0, -1.0, [nan] * 4, [0] * 4) == 0
    assert O.ls_select_f32(al, inf, -1.0, [1e30, 1e30, 1e30, inf], [0] * 4, mode=0) == 3
    # Armijo boundary: c_a == rhs is accepted (<=); rhs built as c0 + (c1*alpha)*g0d in fp32
    c0, g0d = np.float32(3.0), np.float32(-2.0)
    rhs = np.float32(c0 + np.float32(np.float32(np.float32(1e-4) * al[3]) * g0d))
    assert O.ls_select_f32(al, c0, g0d, [9, 9, 9, rhs], [0, 0, 0, 0]) == 3
    assert O.ls_select_f32(al, c0, g0d, [9, 9, 9, np.nextafter(rhs, np.float32(10))], [0] * 4) == 0
    # strong Wolfe uses |g_a d| <= c2 |g0d|
    assert O.ls_select_f32(al, c0, g0d, [0, 0, 0, 0], [0, 0, 1.8, 1.81], mode=2) == 2
    assert O.ls_select_f32(al, c0, g0d, [0, 0, 0, 0], [0, 0, -1.8, -1.81], mode=1) == 2
    assert O.ls_select_f32(al, c0, g0d, [0, 0, 0, 0], [0, 0, -1.81, -1.79], mode=1) == 3
    # argmin with NaN -> +inf, ties -> lowest index
    assert O.argmin_f32([3.0, nan, 1.0, 1.0]) == 2
    assert O.argmin_f32([nan, nan]) == 0
    assert O.argmin_f32([inf, 5.0]) == 1


def test_f32_mirror_matches_f64_away_from_ties(O):
    g = np.random.default_rng(3)
    al = [0.01, 0.3, 0.7, 1.0]
    agree = 0
    for _ in range(2000):
        c0 = g.uniform(0, 10); g0d = -g.uniform(0, 10)
        ca = c0 + g.normal(0, 1, 4); gda = g.normal(0, 10, 4)
        a = O.ls_select(al, c0, g0d, ca, gda); b = O.ls_select_f32(al, c0, g0d, ca, gda)
        agree += a == b
    assert agree >= 1990


def test_franka_to_solve_decreases(O):
    """The threaded rollout solve runs and improves every seed; identical for 1 and 4 threads."""
    from paper_2310_17274_b200 import robots
    rb = robots.franka64()
    R = O.Robot(rb)
    start = rb.ready.copy()
    goal_cfg = np.clip(start + np.array([0.6, 0.3, -0.4, 0.5, 0.2, -0.3, 0.4]), rb.lo, rb.hi)
    _, _, goal = O.fk(R, goal_cfg)
    world = inputs.tabletop_scene(0, 0, 8)
    seeds = inputs.to_seeds(rb, 0, 0, start, goal_cfg, 3, 12)[None]
    cp = inputs.CostParams(dt=0.25)
    sp = inputs.SolverParams(iters=6)
    W = O.World(world)
    c0 = [O.eval_traj(R, W, cp, start, goal, seeds[0, s])[0] for s in range(3)]
    out1, cost1 = O.solve_to(R, [W], [0], cp, sp, seeds, start[None], goal[None], nthreads=1)
    out4, cost4 = O.solve_to(R, [W], [0], cp, sp, seeds, start[None], goal[None], nthreads=4)
    np.testing.assert_array_equal(cost1, cost4)
    np.testing.assert_array_equal(out1, out4)
    assert np.all(cost1[0] <= np.array(c0))
