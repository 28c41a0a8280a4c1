"""GPU parity of the validity mask and parallel steering (Alg. 3, P:252-268;
readings B12-B14) against the fp64 oracle O12.  Validity bits are compared exactly, except for
configurations whose oracle decision margin (distance of a limit, pair penetration or
sphere-cuboid distance to its threshold) is below 2e-5 m, where fp32 and fp64 may legitimately
disagree; the excluded fraction is asserted small.  The shared step count n is decided in fp64 on
both sides and must match exactly."""
import numpy as np
import pytest
import torch

from paper_2310_17274_b200 import inputs, robots
from test_gpu_parity import MARGIN, T, f32, make

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def native():
    from paper_2310_17274_b200 import native as N
    return N


@pytest.mark.parametrize("margin", [0.0, 0.01])
def test_mask_parity(native, O, margin):
    rb = robots.franka64()
    R = O.Robot(rb)
    worlds = [inputs.tabletop_scene(7, e, 20) for e in range(2)]
    Ws = [O.World(w) for w in worlds]
    ctx = make(native, rb, worlds, inputs.CostParams())
    K = 300                                            # 9 full groups + a ragged tail of 12
    g = np.random.default_rng(31)
    q = f32(g.uniform(rb.lo - 0.05, rb.hi + 0.05, (K, 7)))
    env = ((np.arange(K) // 32) % 2).astype(np.int32)
    valid = ctx.mask_samples(T(q), env=T(env, torch.int32), margin=margin).cpu().numpy()
    n_ex = n_valid = 0
    for k in range(K):
        v, mg = O.mask_sample(R, Ws[env[k]], q[k], margin)
        if mg < MARGIN:
            n_ex += 1
            continue
        assert bool(valid[k]) == v, (k, v)
        n_valid += v
    assert n_ex <= 0.05 * K
    assert 0.1 * K < n_valid < 0.9 * K
    ctx.close()


def test_mask_env_group_violation_is_invalid(native, O):
    rb = robots.franka64()
    ctx = make(native, rb, [inputs.tabletop_scene(7, 0, 5), inputs.tabletop_scene(7, 1, 5)], inputs.CostParams())
    q = f32(np.tile(rb.ready, (40, 1)))
    env = np.zeros(40, np.int32); env[5] = 1                        # breaks group 0's env rule
    valid = ctx.mask_samples(T(q), env=T(env, torch.int32)).cpu().numpy()
    assert valid[5] == 0 and valid[32:].all()
    ctx.close()


def test_steer_parity_franka(native, O):
    rb = robots.franka64()
    R = O.Robot(rb)
    world = inputs.tabletop_scene(9, 0, 20)
    W = O.World(world)
    ctx = make(native, rb, [world], inputs.CostParams())
    g = np.random.default_rng(5)
    src = []
    while len(src) < 40:                               # valid sources (Alg. 3 precondition)
        q = g.uniform(rb.lo, rb.hi)
        if O.mask_sample(R, W, q)[0]:
            src.append(q)
    src = f32(np.array(src))
    dst = f32(np.clip(src + g.normal(0, 0.8, src.shape), rb.lo, rb.hi))
    dw = f32(np.linspace(1.0, 0.5, 7))
    r = float(np.float32(0.05))                        # the C-ABI takes r as fp32: same input both sides
    out = ctx.steer(T(src), T(dst), T(dw), r, env=0, n_cap=512)
    n_gpu = out["n"].cpu().numpy()
    n, h, v, dist, mg = O.steer(R, W, src, dst, dw, r)
    assert n_gpu[0] == n and n_gpu[1] == n
    hg, vg, dg = out["h"].cpu().numpy(), out["v_new"].cpu().numpy(), out["dist"].cpu().numpy()
    ok = mg >= MARGIN
    assert ok.mean() >= 0.8
    assert np.array_equal(hg[ok], h[ok])
    np.testing.assert_allclose(vg[ok], v[ok], atol=2e-6)
    np.testing.assert_allclose(dg[ok], dist[ok], rtol=1e-5, atol=1e-6)
    assert 0 < (h < n).sum() < len(h)                  # both truncated and full edges occur
    ctx.close()


def test_steer_wall_and_clamp(native, O):
    rb = robots.planar2()
    R = O.Robot(rb)
    wall = inputs.World(np.array([[0.0, 1.2, 0.0]]), np.array([[1.0, 0, 0, 0]]), np.array([[0.05, 0.6, 1.0]]),
                        np.ones(1, np.int32))
    ctx = make(native, rb, [wall], inputs.CostParams())
    src = f32([[0.2, 0.0], [0.2, 0.1]])
    dst = f32([[2.8, 0.0], [0.3, 0.2]])
    dw = f32([1.0, 1.0])
    r = float(np.float32(0.02))
    out = ctx.steer(T(src), T(dst), T(dw), r, n_cap=1024)
    n, h, v, dist, _ = O.steer(R, O.World(wall), src, dst, dw, r)
    assert out["n"].cpu().tolist() == [n, n]
    assert out["h"].cpu().tolist() == h.tolist() and 0 < h[0] < n and h[1] == n
    np.testing.assert_allclose(out["v_new"].cpu().numpy(), v, atol=2e-6)
    # n_cap below n: discretised with n_cap, the unclamped n reported
    c = ctx.steer(T(src), T(dst), T(dw), r, n_cap=16)
    assert c["n"].cpu().tolist() == [16, n]
    assert 0 <= int(c["h"][0]) < 16
    ctx.close()
