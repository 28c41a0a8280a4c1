"""O12 pins: the validity mask and parallel steering of Alg. 3 (
readings B12-B14).

The mask is checked against an independent brute force: numpy over the robot's pair list and a
scipy-rotation box SDF, fed with sphere centres from the (separately pinned) FK.  Steering is
checked against the special cases S:409-412: an empty world connects fully, a wall bisecting
the segment truncates the edge strictly before the wall within one step of a dense first-
collision search, and the shared step count n is the batch maximum.
"""
import math

import numpy as np
import pytest
from scipy.spatial.transform import Rotation as Rot

from paper_2310_17274_b200 import inputs, robots


def _empty_world():
    return inputs.World(np.zeros((0, 3)), np.zeros((0, 4)), np.zeros((0, 3)), np.zeros(0, np.int32))


def _np_box_sdf(p, pos, q, half):
    r = Rot.from_quat([q[1], q[2], q[3], q[0]])
    pl = r.inv().apply(p - pos)
    qv = np.abs(pl) - half
    if qv.max() > 0:
        return np.linalg.norm(np.maximum(qv, 0))
    return qv.max()


def _brute_valid(O, R, rb, world, q, margin):
    if np.any(q < rb.lo) or np.any(q > rb.hi):
        return False
    _, sph, _ = O.fk(R, q)
    rs = rb.spheres[:, 3] + rb.sphere_offset
    for i, j in rb.pairs:
        if rs[i] <= 0 or rs[j] <= 0:
            continue
        if rs[i] + rs[j] - np.linalg.norm(sph[i, :3] - sph[j, :3]) > 0:
            return False
    for m in range(sph.shape[0]):
        r = rb.spheres[m, 3]
        if r < 0:
            continue
        for k in range(world.pos.shape[0]):
            if world.enabled[k] and _np_box_sdf(sph[m, :3], world.pos[k], world.quat[k], world.dims[k] / 2) < r + margin:
                return False
    return True


def test_mask_trivial_cases(O):
    rb = robots.franka64()
    R = O.Robot(rb)
    assert O.mask_sample(R, O.World(_empty_world()), rb.ready)[0]
    _, sph, _ = O.fk(R, rb.ready)
    box = inputs.World(sph[20:21, :3].copy(), np.array([[1.0, 0, 0, 0]]), np.array([[0.02, 0.02, 0.02]]),
                       np.ones(1, np.int32))
    assert not O.mask_sample(R, O.World(box), rb.ready)[0]                   # centre inside
    q = rb.ready.copy(); q[3] = rb.hi[3] + 1e-6
    assert not O.mask_sample(R, O.World(_empty_world()), q)[0]              # outside the limits
    # the safety margin: a box 3 cm beyond the planar arm's tip sphere is valid at margin 2 cm,
    # not at 4 cm
    pr = robots.planar2()
    PR = O.Robot(pr)
    q0 = np.zeros(2)
    _, ps, _ = O.fk(PR, q0)
    tip = int(np.argmax(ps[:, 0]))
    c = ps[tip, :3]; r = pr.spheres[tip, 3]
    box = inputs.World((c + np.array([r + 0.03 + 0.05, 0, 0]))[None], np.array([[1.0, 0, 0, 0]]),
                       np.array([[0.1, 0.1, 0.1]]), np.ones(1, np.int32))
    assert O.mask_sample(PR, O.World(box), q0, 0.02)[0]
    assert not O.mask_sample(PR, O.World(box), q0, 0.04)[0]


@pytest.mark.parametrize("margin", [0.0, 0.01])
def test_mask_equals_brute_force(O, margin):
    """S:402 in spirit: 150 Halton-like random configurations in a cluttered scene (about half
    invalid) against the independent brute force, decision by decision."""
    rb = robots.franka64()
    R = O.Robot(rb)
    world = inputs.tabletop_scene(7, 0, 20)
    W = O.World(world)
    g = np.random.default_rng(17)
    qs = g.uniform(rb.lo - 0.05, rb.hi + 0.05, (150, 7))
    n_valid = 0
    for q in qs:
        v, mg = O.mask_sample(R, W, q, margin)
        if mg < 1e-9:
            continue
        assert v == _brute_valid(O, R, rb, world, q, margin)
        n_valid += v
    assert 15 < n_valid < 135            # both outcomes are exercised


def test_steer_empty_world_connects_fully(O):
    rb = robots.franka64()
    R = O.Robot(rb)
    g = np.random.default_rng(2)
    src = np.clip(rb.ready + g.normal(0, 0.2, (3, 7)), rb.lo, rb.hi)
    dst = np.clip(src + g.normal(0, 0.5, (3, 7)), rb.lo, rb.hi)
    dw = np.linspace(1.0, 0.4, 7)
    r = 0.05
    # empty world but the self-collision term stays: use short, self-free edges
    n, h, v, dist, _ = O.steer(R, O.World(_empty_world()), src, dst, dw, r)
    gmax = np.abs(dw * (dst - src)).max()
    assert n == math.floor(gmax / r) + 1                                     # Alg. 3 line 2, batch max
    for e in range(3):
        ok = all(O.mask_sample(R, O.World(_empty_world()), src[e] + i / n * (dst[e] - src[e]))[0]
                 for i in range(n + 1))
        if ok:
            assert h[e] == n and np.allclose(v[e], dst[e], atol=1e-15)
            assert dist[e] == pytest.approx(np.linalg.norm(dw * (dst[e] - src[e])), rel=1e-14)


def test_steer_wall_truncates_before_the_wall(O):
    """Planar arm swinging through a wall: the new vertex lies strictly between the source
    and the first colliding configuration of a dense (1000-sample) search, within one step."""
    rb = robots.planar2()
    R = O.Robot(rb)
    wall = inputs.World(np.array([[0.0, 1.2, 0.0]]), np.array([[1.0, 0, 0, 0]]), np.array([[0.05, 0.6, 1.0]]),
                        np.ones(1, np.int32))
    W = O.World(wall)
    src = np.array([[0.2, 0.0]])        # link along +x, turning to +y hits the wall at x = 0
    dst = np.array([[2.8, 0.0]])
    dw = np.ones(2)
    r = 0.02
    n, h, v, dist, _ = O.steer(R, W, src, dst, dw, r)
    assert 0 < h[0] < n
    dense = [i for i in range(1001) if not O.mask_sample(R, W, src[0] + i / 1000 * (dst[0] - src[0]))[0]]
    t_hit = dense[0] / 1000
    t_new = h[0] / n
    assert t_new < t_hit <= t_new + 2.0 / n                                  # within one step
    assert dist[0] < np.linalg.norm(dst[0] - src[0])
    assert O.mask_sample(R, W, v[0])[0]


def test_steer_batch_shares_n(O):
    """A short edge batched with a long one is discretised with the long edge's n."""
    rb = robots.planar2()
    R = O.Robot(rb)
    W = O.World(_empty_world())
    src = np.array([[0.0, 0.5], [1.0, -0.5]])
    dst = np.array([[0.1, 0.6], [2.5, 0.5]])
    n, h, _, _, _ = O.steer(R, W, src, dst, np.ones(2), 0.1)
    n1, _, _, _, _ = O.steer(R, W, src[:1], dst[:1], np.ones(2), 0.1)
    assert n == math.floor(1.5 / 0.1) + 1 and n1 == math.floor(0.1 / 0.1 + 1e-12) + 1
    assert np.all(h == n)
