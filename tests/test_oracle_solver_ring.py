"""Pins for the oracle solver's history ring, candidate clip and best update (O8, Alg. 6 lines 1-5
"Shift Buffers" P:2153-2159, Alg. 1 line 1 P:171-172, readings A20, A21, A23, A35), CPU only.

Each pin checks the oracle against what the paper and textbook L-BFGS fix, recomputed here from
the oracle's O10 per-iteration record: the ring holds the m newest curvature pairs (oldest
dropped), pairs with s'y <= 1e-12 are skipped, every candidate is clip(Theta + alpha_a d, lo, hi)
and inside the box, and the best iterate is the FIRST one reaching the minimum (strict <).
"""
import numpy as np
import pytest

from paper_2310_17274_b200 import inputs
from test_oracle_solver import dense_bfgs_direction


def _pairs(g, n, k, A):
    S = g.normal(size=(k, n))
    return S, S @ A


def test_ring_holds_m_newest_pairs(O):
    """After each of 10 pushes with s'y > 0 the ring is the min(k, m) newest pairs, oldest first."""
    g = np.random.default_rng(0)
    n, m = 6, 4
    A = g.normal(size=(n, n)); A = A @ A.T + n * np.eye(n)
    S_all, Y_all = _pairs(g, n, 10, A)
    S = np.zeros((m, n)); Y = np.zeros((m, n)); rho = np.zeros(m); cnt = 0
    x = np.zeros(n); gr = np.zeros(n)
    for k in range(10):
        xn, gn = x + S_all[k], gr + Y_all[k]
        S, Y, rho, cnt, sy = O.lbfgs_push(S, Y, rho, cnt, m, xn, x, gn, gr)
        x, gr = xn, gn
        keep = list(range(max(0, k + 1 - m), k + 1))
        assert cnt == len(keep)
        np.testing.assert_allclose(S[:cnt], S_all[keep], rtol=0, atol=1e-12)
        np.testing.assert_allclose(Y[:cnt], Y_all[keep], rtol=0, atol=1e-12)
        np.testing.assert_allclose(rho[:cnt], 1.0 / np.einsum("ij,ij->i", S_all[keep], Y_all[keep]), rtol=1e-14)
        assert sy == pytest.approx(S_all[k] @ Y_all[k], rel=1e-14)


def test_push_skips_curvature_at_or_below_threshold(O):
    """A20: a pair with s'y <= 1e-12 is skipped (ring unchanged); just above, it is kept.
    s = e0, y = t e0 makes s'y = t exactly."""
    n, m = 3, 4
    e0 = np.array([1.0, 0.0, 0.0])
    S = np.zeros((m, n)); Y = np.zeros((m, n)); rho = np.zeros(m)
    for t, kept in [(-1.0, False), (0.0, False), (1e-12, False), (np.nextafter(1e-12, 1.0), True), (0.5, True)]:
        S2, Y2, rho2, cnt, sy = O.lbfgs_push(S, Y, rho, 0, m, e0, np.zeros(n), t * e0, np.zeros(n))
        assert sy == t
        assert cnt == (1 if kept else 0), t
    # a full ring is left as it was by a skipped pair
    g = np.random.default_rng(1)
    S = g.normal(size=(m, n)); Y = S + 0.1; rho = 1.0 / np.einsum("ij,ij->i", S, Y)
    S2, Y2, rho2, cnt, _ = O.lbfgs_push(S, Y, rho, m, m, e0, np.zeros(n), -e0, np.zeros(n))
    assert cnt == m and np.array_equal(S2, S) and np.array_equal(Y2, Y) and np.array_equal(rho2, rho)
    # gradient descent (m = 0) stores nothing
    assert O.lbfgs_push(np.zeros((1, n)), np.zeros((1, n)), np.zeros(1), 0, 0, e0, np.zeros(n), e0, np.zeros(n))[3] == 0


def _wavy(n):
    """Non-convex: negative-curvature steps occur, so the s'y skip is exercised."""
    w = np.linspace(1.0, 3.0, n)

    def f(x):
        return float(np.sum(np.cos(w * x) + 0.02 * x * x)), -w * np.sin(w * x) + 0.04 * x
    return f


@pytest.mark.parametrize("m", [1, 4, 6])
def test_solver_directions_use_newest_valid_pairs(O, m):
    """Every L-BFGS direction of a solve equals -H g of the dense BFGS recursion (Nocedal & Wright
    7.19) over the m newest pairs (Theta_k - Theta_{k-1}, g_k - g_{k-1}) with s'y > 1e-12 (A20),
    recomputed from the recorded iterates; d = -g at k = 0 (A21)."""
    n, iters = 8, 30
    f = _wavy(n)
    x0 = np.random.default_rng(3).uniform(-2, 2, n)
    sp = inputs.SolverParams(iters=iters, history=m)
    _, _, tr = O.lbfgs_solve(f, x0, sp, traced=True)
    pairs, skipped, evicted = [], 0, 0
    for k in range(iters):
        if k > 0:
            s, y = tr["x"][k] - tr["x"][k - 1], tr["g"][k] - tr["g"][k - 1]
            assert tr["sy"][k] == pytest.approx(s @ y, rel=1e-12, abs=1e-300)
            if s @ y > 1e-12:
                pairs.append((s, y))
                evicted += len(pairs) > m
            else:
                skipped += 1
        else:
            assert np.isnan(tr["sy"][0])
        use = pairs[-m:]
        assert tr["count"][k] == len(use)
        ref = dense_bfgs_direction([p[0] for p in use], [p[1] for p in use], tr["g"][k])
        np.testing.assert_allclose(tr["d"][k], ref, rtol=1e-8, atol=1e-10 * np.abs(ref).max())
        assert tr["g0d"][k] == pytest.approx(tr["g"][k] @ tr["d"][k], rel=1e-12)
    assert skipped >= 1 and evicted >= 1, (skipped, evicted)   # both ring rules exercised


def test_candidates_are_clipped_steps(O):
    """Alg. 1 line 1 / A35: the A points evaluated at iteration k are exactly
    clip(Theta_k + alpha_a d_k, lo, hi), in alpha order, all inside [lo, hi]; clip is idempotent on
    them.  Tight bounds make the clip active."""
    n, iters = 6, 12
    lo, hi = -np.full(n, 0.6), np.full(n, 0.6)
    f0 = _wavy(n)
    seen = []

    def f(x):
        seen.append(x.copy())
        return f0(x)
    sp = inputs.SolverParams(iters=iters)
    x0 = np.linspace(-0.5, 0.5, n)
    _, _, tr = O.lbfgs_solve(f, x0, sp, lo=lo, hi=hi, traced=True)
    A = len(sp.alpha)
    assert len(seen) == 1 + iters * A
    clipped = 0
    for k in range(iters):
        for a in range(A):
            p = seen[1 + k * A + a]
            raw = tr["x"][k] + sp.alpha[a] * tr["d"][k]
            ref = np.minimum(np.maximum(raw, lo), hi)
            assert np.array_equal(p, ref)
            assert np.all(p >= lo) and np.all(p <= hi)
            assert np.array_equal(np.minimum(np.maximum(p, lo), hi), p)
            clipped += int(np.any(raw != ref))
        # the selected candidate becomes the next iterate (Alg. 1 line 9)
        assert np.array_equal(tr["x"][k + 1], seen[1 + k * A + tr["istar"][k]])
    assert clipped >= 5


def test_best_update_is_strict(O):
    """A23: ties keep the earlier iterate.  A flat objective with a gradient that lies makes every
    line search fail (i* = 0, the noisy step of P:165), so the solver keeps moving while every
    cost equals the first: the best point stays Theta_0."""
    n = 4

    def f(x):
        return 0.0, -np.ones_like(x)
    x0 = np.arange(n, dtype=float)
    sp = inputs.SolverParams(iters=6)
    bx, bc, tr = O.lbfgs_solve(f, x0, sp, traced=True)
    assert np.all(tr["istar"] == 0)
    assert not np.array_equal(tr["x"][-1], x0)
    assert np.array_equal(bx, x0) and bc == 0.0


def test_best_is_first_minimum_on_plateaus(O):
    """A23 with a staircase objective (equal costs on plateaus): the best point is the first
    recorded iterate with the minimal cost, and the best cost never increases."""
    n = 5

    def f(x):
        r2 = float(x @ x)
        return np.floor(4.0 * r2) / 4.0, 2.0 * x
    x0 = np.full(n, 0.9)
    sp = inputs.SolverParams(iters=15, ls_mode=0)
    bx, bc, tr = O.lbfgs_solve(f, x0, sp, traced=True)
    c = tr["c"]
    first = int(np.argmin(c))                  # argmin returns the first occurrence
    assert bc == c[first]
    assert np.array_equal(bx, tr["x"][first])
    assert np.all(np.diff(tr["best_c"]) <= 0)
    assert np.sum(c == c[first]) >= 2          # a tie actually happened after the first minimum


def test_ls_margin_hand_values(O):
    """O10 solver margin by hand: f = x^2 at x = 1, d = -1, alpha = (0.01, 0.3, 0.7, 1.0).
    Armijo rhs_a = 1 - 2e-4 alpha_a; c_a = (1 - alpha_a)^2; strong Wolfe ||g_a d| - 0.9 * 2|."""
    al = [0.01, 0.3, 0.7, 1.0]
    ca = [(1 - a) ** 2 for a in al]
    gda = [-2 * (1 - a) for a in al]
    arm = min(abs(ca[i] - (1 - 2e-4 * al[i])) for i in range(4))
    wolfe = min(abs(abs(gda[i]) - 1.8) for i in range(4))
    assert O.ls_margin(al, 1.0, -2.0, ca, gda, mode=0) == pytest.approx(arm, rel=1e-12)
    assert O.ls_margin(al, 1.0, -2.0, ca, gda, mode=2) == pytest.approx(min(arm, wolfe), rel=1e-12)
    assert O.ls_margin(al, 1.0, -2.0, ca, gda, mode=1) == pytest.approx(
        min(arm, min(abs(g + 1.8) for g in gda)), rel=1e-12)


def test_armijo_hand_boundary(O):
    """A17 Armijo, c_a <= c0 + c1 alpha_a g0d with g0d < 0, by hand at c0 = 1, g0d = -2, alpha =
    1: rhs = 1 - 2e-4.  A candidate that raises the cost by 1e-4 fails it (no uphill acceptance);
    one that lowers it by 3e-4 passes; the fp32 mirror agrees."""
    al = [0.01, 0.3, 0.7, 1.0]
    for mode in (0, 1, 2):
        gda = [0.0, 0.0, 0.0, 0.0]
        assert O.ls_select(al, 1.0, -2.0, [2, 2, 2, 1 + 1e-4], gda, mode=mode) == 0
        assert O.ls_select(al, 1.0, -2.0, [2, 2, 2, 1 - 3e-4], gda, mode=mode) == 3
        assert O.ls_select_f32(al, 1.0, -2.0, [2, 2, 2, 1 + 1e-4], gda, mode=mode) == 0
    # Wolfe (mode 1): g_a'd >= c2 g0d = -1.8 also needed
    assert O.ls_select(al, 1.0, -2.0, [2, 2, 2, 1 - 3e-4], [0, 0, 0, -1.7], mode=1) == 3
    assert O.ls_select(al, 1.0, -2.0, [2, 2, 2, 1 - 3e-4], [0, 0, 0, -1.9], mode=1) == 0
