"""Pins for the §8(f) f3 variants of the path, oracle side.

* Eq. cspace-cost: C = a4 logcosh(a5 |theta_g - theta_T|^2): zero with zero gradient
  at the goal, its two asymptotes (a4 a5^2 s^2 / 2 for small s, a4 (a5 s - ln 2) for large s),
  central finite differences, and its routing through the whole rollout (directional FD of the
  trajectory cost with the flag set, the pose term replaced).
* Gradient descent = L-BFGS with history 0: on a convex quadratic it is plain GD with
  the line search, and it is slower than L-BFGS.
* Long histories (P:1950 sweeps m up to 25): the two-loop recursion still equals the dense BFGS
  inverse-Hessian recursion.
"""
import math

import numpy as np
import pytest

from paper_2310_17274_b200 import inputs, robots


def test_cspace_zero_at_goal(O):
    cp = inputs.CostParams()
    q = np.array([0.3, -0.2, 0.1, -1.5, 0.2, 1.3, 0.7])
    c, g = O.cspace_cost(cp, q, q)
    assert c == 0.0 and np.all(g == 0.0)


@pytest.mark.parametrize("scale", [1e-4, 3e-3, 0.5, 2.0])
def test_cspace_asymptotes_and_fd(O, scale):
    cp = inputs.CostParams()
    rng = np.random.default_rng(3)
    goal = rng.uniform(-1, 1, 7)
    u = rng.normal(size=7); u /= np.linalg.norm(u)
    q = goal + math.sqrt(scale) * u           # |theta_g - theta_T|^2 = scale
    c, g = O.cspace_cost(cp, q, goal)
    s, a4, a5 = scale, cp.a4, cp.a5
    if a5 * s < 1e-2:
        assert c == pytest.approx(a4 * (a5 * s) ** 2 / 2, rel=1e-3)
    if a5 * s > 20:
        assert c == pytest.approx(a4 * (a5 * s - math.log(2.0)), rel=1e-9)
    eps = 1e-7 * max(1.0, math.sqrt(scale))
    for d in range(7):
        e = np.zeros(7); e[d] = eps
        fd = (O.cspace_cost(cp, q + e, goal)[0] - O.cspace_cost(cp, q - e, goal)[0]) / (2 * eps)
        assert g[d] == pytest.approx(fd, rel=2e-5, abs=1e-6 * max(1.0, abs(c)))


def test_cspace_rollout_routes_through_terminal_state(O):
    """With CSPACE the goal term is Eq. cspace-cost at x_H; the trajectory gradient is checked by
    a directional finite difference of the whole rollout (sweep/speed off: smooth)."""
    rb = robots.franka64()
    R = O.Robot(rb)
    W = O.World(inputs.tabletop_scene(0, 0, 3))
    cp = inputs.CostParams(flags=inputs.CSPACE, dt=0.25)
    g = np.random.default_rng(8)
    H = 12
    start = rb.ready.copy()
    goal = np.clip(rb.ready + g.normal(0, 0.3, 7), rb.lo, rb.hi)
    V = np.clip(np.linspace(start, goal, H) + g.normal(0, 0.05, (H, 7)), rb.lo, rb.hi)
    c, gV, terms, _, _ = O.eval_traj(R, W, cp, start, goal, V)
    # the goal term is exactly the cspace cost at x_H = V[H-1]
    assert terms[0] == pytest.approx(O.cspace_cost(cp, V[-1], goal)[0], rel=1e-12)
    # at the goal it vanishes (the rest of the rollout is unchanged by the flag)
    V2 = V.copy(); V2[-1] = goal
    assert O.eval_traj(R, W, cp, start, goal, V2)[2][0] == 0.0
    cp_pose = inputs.CostParams(flags=0, dt=0.25)
    ee_goal = O.fk(R, goal)[2]
    assert np.allclose(O.eval_traj(R, W, cp, start, goal, V)[2][1:],
                       O.eval_traj(R, W, cp_pose, start, ee_goal, V)[2][1:], rtol=1e-12)
    for trial in range(4):
        dV = g.normal(size=V.shape)
        eps = 1e-6
        fd = (O.eval_traj(R, W, cp, start, goal, V + eps * dV)[0]
              - O.eval_traj(R, W, cp, start, goal, V - eps * dV)[0]) / (2 * eps)
        assert float((gV * dV).sum()) == pytest.approx(fd, rel=1e-5, abs=1e-4)


def test_gradient_descent_is_history_zero(O):
    """history = 0: every direction is -g (P:1948 'GD instead of L-BFGS'); on an ill-conditioned
    quadratic it converges, but more slowly than L-BFGS with m = 4."""
    A = np.diag([1.0, 10.0, 50.0])
    b = np.array([1.0, -2.0, 0.5])

    def f(x):
        return 0.5 * x @ A @ x - b @ x, A @ x - b
    xs = np.linalg.solve(A, b)
    fmin = f(xs)[0]
    gd = inputs.SolverParams(iters=60, history=0)          # the paper's alpha set
    lb = inputs.SolverParams(iters=60, history=4)
    x0 = np.array([2.0, 2.0, 2.0])
    _, c_gd, tr_gd = O.lbfgs_solve(f, x0, gd)
    _, c_lb, _ = O.lbfgs_solve(f, x0, lb)
    assert np.all(np.diff(tr_gd) <= 0)                 # best is monotone
    assert c_gd - fmin > 1e-6                          # GD has not converged
    assert c_lb - fmin < 0.1 * (c_gd - fmin)           # L-BFGS is far ahead
    # one iteration: the accepted point is x0 - alpha g0 for one of the magnitudes (d = -g)
    al = (0.001, 0.003, 0.01, 0.02)
    _, _, tr1 = O.lbfgs_solve(f, x0, inputs.SolverParams(iters=1, history=0, alpha=al))
    g0 = f(x0)[1]
    assert any(tr1[1] == pytest.approx(f(x0 - a * g0)[0], rel=1e-14) for a in al)


@pytest.mark.parametrize("count", [1, 12, 25])
def test_two_loop_long_history_equals_dense_bfgs(O, count):
    rng = np.random.default_rng(count)
    n = 30
    S = rng.normal(size=(count, n))
    M = rng.normal(size=(n, n)); Hs = M @ M.T + n * np.eye(n)
    Y = S @ Hs                                     # y = H s with H SPD: s^T y > 0
    g = rng.normal(size=n)
    rho = 1.0 / np.einsum("ij,ij->i", S, Y)
    d = O.lbfgs_direction(S, Y, rho, g)
    gamma = S[-1] @ Y[-1] / (Y[-1] @ Y[-1])
    Hk = gamma * np.eye(n)
    for i in range(count):
        r = rho[i]
        V = np.eye(n) - r * np.outer(Y[i], S[i])
        Hk = V.T @ Hk @ V + r * np.outer(S[i], S[i])
    assert np.allclose(d, -Hk @ g, rtol=1e-9, atol=1e-10)
