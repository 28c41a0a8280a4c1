"""O13 pins: the motion-generation pipeline pieces of §8(f) f2 (Alg. 4, App. B
P:2189-2190; readings B15-B18).

* retime: after scaling time by s every stencil derivative is within its limit and the binding one
  sits on it (derivatives recomputed with an independent numpy five-point stencil); dt_opt does not
  depend on the dt the trajectory was expressed at (homogeneity); a still trajectory clamps at
  s = 1e-3; the SPEC examples S:521-522 (at the limit -> s = 1; half the limit -> s = 0.5).
* weight scaling (B15): re-timing the same path from dt_ref to dt with the scaled weights leaves
  the smoothness term of the whole rollout unchanged.
* goal errors, linear seeds and the two scores: closed forms and monotonicity.
"""
import math

import numpy as np
import pytest
from scipy.spatial.transform import Rotation as Rot

from paper_2310_17274_b200 import inputs, robots


def _np_derivs(start, V, dt):
    """Independent five-point stencil over the Table 5 state map (pins x_1..x_3 = start, aliases
    x_{H-3..H+2} = x_H, pads x_{-1..0} = start)."""
    H, D = V.shape
    x = np.zeros((H + 5, D))
    x[3:3 + H] = V
    x[:6] = start                      # x_{-2..3}
    x[H - 1:] = V[-1]                  # x_{H-3..H+2}
    c = np.arange(3, 3 + H)
    v = (-x[c + 2] + 8 * x[c + 1] - 8 * x[c - 1] + x[c - 2]) / (12 * dt)
    a = (-x[c + 2] + 16 * x[c + 1] - 30 * x[c] + 16 * x[c - 1] - x[c - 2]) / (12 * dt * dt)
    j = (x[c + 2] - 2 * x[c + 1] + 2 * x[c - 1] - x[c - 2]) / (2 * dt ** 3)
    return v, a, j


def _traj(rb, seed, H=32, amp=0.8):
    g = np.random.default_rng(seed)
    start = rb.ready.copy()
    goal = np.clip(start + g.normal(0, amp, 7), rb.lo, rb.hi)
    V = np.linspace(start, goal, H) + np.sin(np.linspace(0, np.pi, H))[:, None] * g.normal(0, 0.2, 7)
    return start, np.clip(V, rb.lo, rb.hi)


@pytest.mark.parametrize("seed", range(5))
def test_retime_pushes_to_the_limits(O, seed):
    rb = robots.franka64()
    R = O.Robot(rb)
    start, V = _traj(rb, seed)
    s, dt_opt, ratios = O.retime(R, start, V, 0.25)
    v, a, j = _np_derivs(start, V, dt_opt)
    r = np.concatenate([np.abs(v) / rb.vmax, np.abs(a) / rb.amax, np.abs(j) / rb.jmax])
    assert r.max() <= 1 + 1e-9 and r.max() >= 1 - 1e-9          # within limits, one binding
    v0, a0, j0 = _np_derivs(start, V, 0.25)
    assert ratios[0] == pytest.approx(np.max(np.abs(v0) / rb.vmax), rel=1e-12)
    assert ratios[1] == pytest.approx(math.sqrt(np.max(np.abs(a0) / rb.amax)), rel=1e-12)
    assert ratios[2] == pytest.approx(np.cbrt(np.max(np.abs(j0) / rb.jmax)), rel=1e-12)
    # homogeneity: the same path expressed at another dt retimes to the same dt_opt
    for dt in (0.05, 0.5, 2.0):
        assert O.retime(R, start, V, dt)[1] == pytest.approx(dt_opt, rel=1e-12)


def test_retime_spec_examples_and_clamp(O):
    rb = robots.planar2()
    R = O.Robot(rb)
    start = np.zeros(2)
    V = np.zeros((16, 2))
    s, _, _ = O.retime(R, start, V, 0.25)
    assert s == 1e-3                                               # still trajectory: clamp
    start, V = np.zeros(2), np.linspace([0, 0], [0.3, -0.2], 16)
    s, _, _ = O.retime(R, start, V, 0.25)
    # S:521 "exactly at the limit -> s = 1": retime at dt_opt is a fixed point
    s2, dt2, _ = O.retime(R, start, V, s * 0.25)
    assert s2 == pytest.approx(1.0, rel=1e-12) and dt2 == pytest.approx(s * 0.25, rel=1e-12)
    # S:522 "half the limits -> s = 0.5, motion time halves": at dt = 2 dt_opt every ratio halves
    s3, dt3, _ = O.retime(R, start, V, 2 * s * 0.25)
    assert s3 == pytest.approx(0.5, rel=1e-12) and dt3 == pytest.approx(s * 0.25, rel=1e-12)


def test_weight_scaling_keeps_the_smoothness_term(O):
    """B15: the same path re-timed from dt_ref = 0.25 to dt with a8 (dt/dt_ref)^4 and a9
    (dt/dt_ref)^6 has exactly the same smoothness term (acceleration and jerk)."""
    rb = robots.franka64()
    R = O.Robot(rb)
    W = O.World(inputs.tabletop_scene(0, 0, 3))
    start, V = _traj(rb, 11)
    goal = O.fk(R, V[-1])[2]
    cp = inputs.CostParams(flags=inputs.JERK, dt=0.25)
    base = O.eval_traj(R, W, cp, start, goal, V)[2][2]
    for dt in (0.05, 0.1, 0.4):
        cps = O.scale_params(cp, dt)
        assert O.scale_params_c(cp, dt) == pytest.approx((dt, cps.a8, cps.a9, cps.flags) + tuple(cps.w_bound))
        assert O.eval_traj(R, W, cps, start, goal, V)[2][2] == pytest.approx(base, rel=1e-10)
    # jerk enabled by the second optimisation (Alg. 4 enable_jerk_cost)
    assert O.scale_params(inputs.CostParams(flags=0), 0.1).flags & inputs.JERK


def test_weight_scaling_keeps_large_limit_violations(O):
    """B15 for the limit terms (P:2053 'all our cost terms that relate to velocity, acceleration,
    and jerk'): beyond its band the limit cost grows with slope 1 in the derivative, which scales
    like dt^-1, dt^-2, dt^-3 for v, a, j under re-timing; with the weights scaled by r, r^2, r^3 the
    limit term of a path violating every limit by ~1e9x re-timed from 0.25 s to dt keeps its value
    up to the band offsets (relative 1e-3).  (The position-limit weight does not change.)"""
    rb = robots.franka64()
    R = O.Robot(rb)
    W = O.World(inputs.World(np.zeros((0, 3)), np.zeros((0, 4)), np.zeros((0, 3)), np.zeros(0, np.int32)))
    import dataclasses
    big = dataclasses.replace(rb, vmax=rb.vmax * 1e-9, amax=rb.amax * 1e-9, jmax=rb.jmax * 1e-9,
                              lo=rb.lo - 100.0, hi=rb.hi + 100.0)
    Rb = O.Robot(big)
    start, V = _traj(rb, 11)
    goal = O.fk(R, V[-1])[2]
    # a tiny activation band (eta_2): beyond it the limit cost is exactly |x| - limit + eta_2 / 2
    cp = inputs.CostParams(flags=inputs.JERK, dt=0.25, a8=0.0, a9=0.0, eta_bound=1e-7)
    base = O.eval_traj(Rb, W, cp, start, goal, V)[2][1]
    assert base > 1e3
    for dt in (0.05, 0.1, 0.4):
        t = O.eval_traj(Rb, W, O.scale_params(cp, dt), start, goal, V)[2][1]
        assert t == pytest.approx(base, rel=1e-3), dt
        # the unscaled weights would change it by orders of magnitude
        t0 = O.eval_traj(Rb, W, dataclasses.replace(cp, dt=dt), start, goal, V)[2][1]
        assert abs(t0 / base - 1) > 0.5
    assert O.scale_params(cp, 0.1).w_bound[0] == cp.w_bound[0]


def test_goal_error_closed_forms(O):
    rb = robots.franka64()
    R = O.Robot(rb)
    q = rb.ready
    ee = O.fk(R, q)[2]
    assert O.goal_error(R, q, ee) == pytest.approx((0.0, 0.0), abs=1e-14)
    g = ee.copy(); g[:3] += [0.01, 0.0, 0.0]
    assert O.goal_error(R, q, g)[0] == pytest.approx(0.01, rel=1e-12)
    th = 0.3
    rz = Rot.from_euler("z", th) * Rot.from_quat([ee[4], ee[5], ee[6], ee[3]])
    xq = rz.as_quat()
    g2 = np.concatenate([ee[:3], [xq[3], xq[0], xq[1], xq[2]]])
    assert O.goal_error(R, q, g2)[1] == pytest.approx(1 - math.cos(th / 2), rel=1e-9)


def test_linear_seed(O):
    start = np.array([0.1, -0.4, 1.0]); qT = np.array([1.1, 0.6, -2.0])
    V = O.linear_seed(start, qT, 9)
    assert np.array_equal(V[0], start) and np.allclose(V[-1], qT, atol=1e-15)
    assert np.allclose(np.diff(V, axis=0), (qT - start) / 8, atol=1e-15)


def test_scores(O):
    q0 = np.zeros(3)
    assert O.ik_score(np.array([3.0, 4.0, 0.0]), q0, 0.0, 0.0, 1.0, 0.01) == pytest.approx(0.05)
    assert O.ik_score(q0, q0, 0.002, 0.001, 1.0, 0.01) == pytest.approx(0.003)
    b = lambda *a: O.blended_score(*a, 1000.0, 1e-3, 1.0)
    assert b(0.001, 0.0, 100.0, 2.0) < b(0.001, 0.0, 100.0, 2.5)       # faster wins
    assert b(0.001, 0.0, 100.0, 2.0) < b(0.002, 0.0, 100.0, 2.0)
    assert b(0.001, 0.0, 100.0, 2.0) < b(0.001, 0.0, 200.0, 2.0)
    assert O.blended_score(0.001, 0.0, 100.0, 2.0, 1e4, 1e-2, 10.0) == pytest.approx(10 * b(0.001, 0.0, 100.0, 2.0))


def test_interpolation_pins(O):
    """B21: the fine grid reproduces every coarse state that falls on it, the
    end point is x_H, n = ceil((H - 1) dt / dt_fine) + 1, and a path linear in time (x_h = a + b h)
    is reproduced exactly at every fine time t (x(t) = a + b t / dt)."""
    g = np.random.default_rng(3)
    H, D = 32, 7
    a, b = g.normal(size=D), g.normal(size=D)
    x = a + b * np.arange(H)[:, None]
    for dt, dtf in ((0.25, 0.025), (0.1, 0.025), (0.137, 0.025), (0.02, 0.025)):
        n, pts = O.interpolate(x, dt, dtf)
        T = (H - 1) * dt
        assert n == math.ceil(T / dtf) + 1
        t = np.minimum(np.arange(n) * dtf, T)
        np.testing.assert_allclose(pts, a + b * (t / dt)[:, None], rtol=0, atol=1e-12)
        np.testing.assert_array_equal(pts[-1], x[-1])
    # states on the fine grid are reproduced: dt = 4 dt_fine -> every 4th point is a state
    y = g.normal(size=(H, D))
    n, pts = O.interpolate(y, 0.1, 0.025)
    np.testing.assert_allclose(pts[::4], y, rtol=0, atol=1e-12)
    # between two states the points stay on the segment (convex combination)
    mid = pts[2]
    np.testing.assert_allclose(mid, 0.5 * (y[0] + y[1]), atol=1e-12)
    # n_max truncates the output but reports the full count
    n2, p2 = O.interpolate(y, 0.1, 0.025, n_max=10)
    assert n2 == n and p2.shape == (10, D)
