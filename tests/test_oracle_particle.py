"""O11 pins: the particle warm-up of §4.2, Alg. 5, readings B6-B10.

The counter-based generator is pinned by the published Philox4x32-10 known-answer vectors
(Salmon et al., SC'11; the Random123 distribution's kat_vectors) and its normals by a
Kolmogorov-Smirnov test against scipy's normal CDF.  The update (Eqs. particle_1/2) is pinned by
the special cases S:352-354 names: one-hot weights with k_mu = 1 select a particle, equal costs
give uniform weights, and the warm-up converges on a 2-D quadratic with a closed-form optimum.
"""
import math

import numpy as np
import pytest
from scipy import stats

from paper_2310_17274_b200 import inputs


# Random123 kat_vectors, "philox4x32 10": counter, key -> output
KAT = [
    ((0, 0, 0, 0), (0, 0), (0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8)),
    ((0xFFFFFFFF,) * 4, (0xFFFFFFFF, 0xFFFFFFFF), (0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD)),
    ((0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344), (0xA4093822, 0x299F31D0),
     (0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1)),
]


@pytest.mark.parametrize("ctr,key,out", KAT)
def test_philox_known_answers(O, ctr, key, out):
    assert O.philox4x32(key, ctr) == list(out)


def test_normals_are_standard_normal(O):
    z = np.array([O.normal(7, 3, v, l, 0, 11) for l in range(64) for v in range(256)])
    assert abs(z.mean()) < 5 / math.sqrt(z.size)
    assert abs(z.var() - 1.0) < 5 * math.sqrt(2.0 / z.size)
    assert stats.kstest(z, "norm").pvalue > 1e-3
    # distinct streams are distinct (key word 1 = problem, counter word 3 = seed)
    assert O.normal(7, 3, 0, 0, 0, 11) != O.normal(7, 4, 0, 0, 0, 11)
    assert O.normal(7, 3, 0, 0, 0, 11) != O.normal(7, 3, 0, 0, 0, 12)


def test_normal_component_mapping(O):
    """var % 4 picks cos/sin of the two Box-Muller pairs of one Philox block (B9)."""
    w = O.philox4x32((5, 9), (1, 2, 3, 4))
    for j in range(4):
        a = (j // 2) * 2
        u1 = ((w[a] >> 8) + 1) / 2.0 ** 24
        u2 = (w[a + 1] >> 8) / 2.0 ** 24
        r = math.sqrt(-2 * math.log(u1))
        z = r * (math.sin if j & 1 else math.cos)(2 * math.pi * u2)
        assert O.normal(5, 9, 4 + j, 2, 3, 4) == pytest.approx(z, abs=1e-15)


def _sp(**kw):
    base = dict(particle_iters=1, n_particles=64, particle_beta=1.0, k_mu=0.9, k_sigma=0.5,
                sigma0_frac=0.1, rng_key=1234)
    base.update(kw)
    return inputs.SolverParams(**base)


def _particles(O, sp, mu, var, lo, hi, it, problem, seed):
    n = mu.shape[0]
    th = np.empty((sp.n_particles, n))
    for l in range(sp.n_particles):
        for v in range(n):
            z = O.normal(sp.rng_key, problem, v, l, it, seed)
            th[l, v] = min(max(mu[v] + math.sqrt(var[v]) * z, lo[v]), hi[v])
    return th


def test_iters_zero_is_identity(O):
    x0 = np.array([0.3, -0.2, 0.1])
    mu, var, _ = O.particle_solve(lambda x: float(x @ x), x0, _sp(particle_iters=0), -np.ones(3), np.ones(3))
    assert np.array_equal(mu, x0)
    assert np.allclose(var, (0.1 * 2.0) ** 2)


def test_one_hot_weights_select_the_particle(O):
    """k_mu = 1 and a dominant cost gap (beta -> 0 limit): the new mean IS the best particle."""
    n = 5
    lo, hi = -2 * np.ones(n), 2 * np.ones(n)
    x0 = np.linspace(-0.5, 0.5, n)
    target = np.full(n, 0.37)
    sp = _sp(k_mu=1.0, k_sigma=1.0, sigma0_frac=0.2)
    f = lambda x: 1e6 * float(((x - target) ** 2).sum())
    mu, var, costs = O.particle_solve(f, x0, sp, lo, hi, problem=3, seed=9)
    th = _particles(O, sp, x0, np.full(n, (0.2 * 4) ** 2), lo, hi, 0, 3, 9)
    best = int(np.argmin(((th - target) ** 2).sum(1)))
    assert np.array_equal(mu, th[best])
    assert np.allclose(var, (th[best] - x0) ** 2, rtol=0, atol=1e-15)
    assert np.allclose(costs[0], [f(t) for t in th])


def test_equal_costs_give_uniform_weights(O):
    """Zero cost variance -> w = 1/n: mean moves toward the particle average."""
    n = 4
    lo, hi = -np.ones(n), np.ones(n)
    x0 = np.array([0.1, 0.2, -0.3, 0.95])     # the last one clips often
    sp = _sp(k_mu=0.9, k_sigma=0.5)
    mu, var, _ = O.particle_solve(lambda x: 42.0, x0, sp, lo, hi, problem=1, seed=2)
    var0 = np.full(n, (0.1 * 2) ** 2)
    th = _particles(O, sp, x0, var0, lo, hi, 0, 1, 2)
    assert np.allclose(mu, 0.1 * x0 + 0.9 * th.mean(0), rtol=0, atol=1e-14)
    assert np.allclose(var, 0.5 * var0 + 0.5 * ((th - x0) ** 2).mean(0), rtol=0, atol=1e-14)


def test_non_finite_costs_get_zero_weight(O):
    n = 3
    lo, hi = -np.ones(n), np.ones(n)
    x0 = np.zeros(n)
    sp = _sp(k_mu=1.0, k_sigma=0.0)
    f = lambda x: float("nan") if x[0] > 0 else 1.0    # every particle with x0 > 0 is invalid
    mu, _, _ = O.particle_solve(f, x0, sp, lo, hi)
    th = _particles(O, sp, x0, np.full(n, 0.04), lo, hi, 0, 0, 0)
    keep = th[:, 0] <= 0
    assert 0 < keep.sum() < sp.n_particles
    assert np.allclose(mu, th[keep].mean(0), atol=1e-14)
    # all invalid: (mu, sigma) unchanged (B10)
    mu2, var2, _ = O.particle_solve(lambda x: float("inf"), x0, sp, lo, hi)
    assert np.array_equal(mu2, x0) and np.allclose(var2, 0.04)


def test_quadratic_converges(O):
    """2-D quadratic, 64 particles, 20 iterations, fixed key -> mean within 0.05 of x* (S:354)."""
    xs = np.array([0.6, -0.4])
    lo, hi = -2 * np.ones(2), 2 * np.ones(2)
    sp = _sp(particle_iters=20, sigma0_frac=0.25)
    mu, var, costs = O.particle_solve(lambda x: 10.0 * float(((x - xs) ** 2).sum()),
                                      np.array([-1.0, 1.2]), sp, lo, hi)
    assert np.linalg.norm(mu - xs) < 0.05
    assert costs.shape == (20, 64)
    assert costs[-1].min() < costs[0].min()
