"""Pins for the oracle's geometry and cost primitives (O5): box SDF, activation, bound, self,
discrete / swept world, pose, stencil.  Closed forms, brute force, invariants, FD.  CPU only."""
import json
import math
import os

import numpy as np
import pytest
from scipy.spatial.transform import Rotation as Rot

from paper_2310_17274_b200 import inputs

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_values.json")))
IDQ = [1.0, 0.0, 0.0, 0.0]


def wxyz(r):
    x, y, z, w = r.as_quat()
    return np.array([w, x, y, z])


# ------------------------------------------------------------------ box SDF (A4)

def test_box_sdf_closed_form(O):
    sd, g = O.box_sdf([0, 0, 0], [0, 0, 0], IDQ, [0.5, 0.5, 0.5])
    assert sd == pytest.approx(-0.5, abs=1e-15)
    np.testing.assert_allclose(g, [1, 0, 0])            # first arg-max axis, sign(0) = +1
    sd, g = O.box_sdf([1.5, 0, 0], [0, 0, 0], IDQ, [0.5, 0.5, 0.5])
    assert sd == pytest.approx(1.0, abs=1e-15)
    np.testing.assert_allclose(g, [1, 0, 0])
    sd, g = O.box_sdf([1.5, 1.5, 0], [0, 0, 0], IDQ, [0.5, 0.5, 0.5])   # edge region
    assert sd == pytest.approx(math.sqrt(2), abs=1e-15)
    np.testing.assert_allclose(g, [math.sqrt(0.5), math.sqrt(0.5), 0], atol=1e-15)


def _surface_samples(half, n=60):
    pts = []
    u = np.linspace(-1, 1, n)
    A, B = np.meshgrid(u, u)
    for ax in range(3):
        o = [i for i in range(3) if i != ax]
        for s in (-1, 1):
            P = np.zeros((n * n, 3))
            P[:, ax] = s * half[ax]
            P[:, o[0]] = A.ravel() * half[o[0]]
            P[:, o[1]] = B.ravel() * half[o[1]]
            pts.append(P)
    return np.concatenate(pts)


def test_box_sdf_brute_force_rotated(O):
    """Rotated boxes vs dense surface sampling (within the grid step), inside sign by AABB test."""
    g = np.random.default_rng(3)
    for t in range(6):
        half = g.uniform(0.05, 0.4, 3)
        r = Rot.random(random_state=t)
        pos = g.uniform(-0.5, 0.5, 3)
        surf = _surface_samples(half)
        step = 2 * half.max() / 59
        for _ in range(30):
            p = pos + g.uniform(-0.8, 0.8, 3)
            sd, _ = O.box_sdf(p, pos, wxyz(r), half)
            pl = r.inv().apply(p - pos)
            inside = np.all(np.abs(pl) <= half)
            dist = np.min(np.linalg.norm(surf - pl[None], axis=1))
            assert abs(abs(sd) - dist) <= step
            assert (sd <= 0) == inside


def test_box_sdf_frame_invariance_and_fd(O):
    g = np.random.default_rng(4)
    for t in range(20):
        half = g.uniform(0.05, 0.4, 3)
        r = Rot.random(random_state=100 + t)
        pos = g.uniform(-0.5, 0.5, 3)
        p = pos + g.uniform(-0.6, 0.6, 3)
        sd, grad = O.box_sdf(p, pos, wxyz(r), half)
        # rigid motion of box and point, within 1e-9
        M = Rot.random(random_state=500 + t); tt = g.normal(size=3)
        sd2, grad2 = O.box_sdf(M.apply(p) + tt, M.apply(pos) + tt, wxyz(M * r), half)
        assert abs(sd - sd2) < 1e-9
        np.testing.assert_allclose(grad2, M.apply(grad), atol=1e-9)
        # gradient = central FD (away from the medial surfaces)
        fd = np.array([(O.box_sdf(p + e, pos, wxyz(r), half)[0] - O.box_sdf(p - e, pos, wxyz(r), half)[0]) / 2e-7
                       for e in np.eye(3) * 1e-7])
        if np.all(np.abs(fd - grad) < 1e-5) or True:
            pl = r.inv().apply(p - pos)
            q = np.abs(pl) - half
            srt = np.sort(q)
            if q.max() > 0 or srt[-1] - srt[-2] > 1e-4:
                np.testing.assert_allclose(grad, fd, atol=1e-6)


# ------------------------------------------------------------------ activation (Eq. smooth-distance-cases)

def test_activation_paper_values(O):
    gold = GOLD["activation_fig3"]
    eta = gold["eta"]
    # d = d' - eta (A2): d = -eta -> 0; d = 0 -> 0.015 (Fig. 3b); d = 0.1 -> 0.115
    assert O.activation(-eta + eta, eta)[0] == 0.0
    assert O.activation(gold["d"] + eta, eta)[0] == pytest.approx(gold["d_c"], abs=1e-15)
    assert O.activation(0.1 + eta, eta)[0] == pytest.approx(0.115, abs=1e-15)
    # equals the printed three-branch formula in the true-penetration variable d
    for d in np.linspace(-0.1, 0.2, 301):
        ref = d + 0.5 * eta if d > 0 else (0.5 / eta * (d + eta) ** 2 if d > -eta else 0.0)
        assert O.activation(d + eta, eta)[0] == pytest.approx(ref, abs=1e-14)


def test_activation_c1_monotone(O):
    eta = 0.025
    for b in (0.0, eta):
        for eps in (1e-7,):
            lv, ld = O.activation(b - eps, eta)
            rv, rd = O.activation(b + eps, eta)
            assert abs(rv - lv) < 1e-6 and abs(rd - ld) < 1e-5
    xs = np.linspace(-0.05, 0.1, 500)
    vals = [O.activation(x, eta)[0] for x in xs]
    assert np.all(np.diff(vals) >= 0)


# ------------------------------------------------------------------ bound (Eq. bound_cost)

def test_bound_values(O):
    e2 = GOLD["eta_bound"]["value"]
    assert O.bound(1.0, -1.0, 1.0, e2)[0] == pytest.approx(0.05, abs=1e-15)
    assert O.bound(1.2, -1.0, 1.0, e2)[0] == pytest.approx(0.25, abs=1e-15)
    assert O.bound(0.0, -1.0, 1.0, e2)[0] == 0.0
    assert O.bound(-1.2, -1.0, 1.0, e2)[0] == pytest.approx(0.25, abs=1e-15)
    for b in (-1.0, -1.0 + e2, 1.0 - e2, 1.0):
        lv, ld = O.bound(b - 1e-8, -1.0, 1.0, e2)
        rv, rd = O.bound(b + 1e-8, -1.0, 1.0, e2)
        assert abs(lv - rv) < 1e-7 and abs(ld - rd) < 1e-6
    for x in np.linspace(-1.5, 1.5, 301):
        v, d = O.bound(x, -1.0, 1.0, e2)
        fd = (O.bound(x + 1e-7, -1, 1, e2)[0] - O.bound(x - 1e-7, -1, 1, e2)[0]) / 2e-7
        assert abs(d - fd) < 1e-5


# ------------------------------------------------------------------ self-collision (Eq. self-collision)

def _two_sphere_robot(positions, radii, pairs):
    M = len(radii)
    return inputs.Robot(name="s", parent=np.array([-1], np.int32), jtype=np.array([0], np.int32),
                        dof=np.array([-1], np.int32), fixed=np.eye(3, 4).reshape(1, 12),
                        lo=-np.ones(1), hi=np.ones(1), vmax=np.ones(1), amax=np.ones(1), jmax=np.ones(1),
                        spheres=np.concatenate([positions, np.asarray(radii)[:, None]], 1),
                        sphere_link=np.zeros(M, np.int32), sphere_offset=np.zeros(M),
                        pairs=np.array(pairs, np.int32).reshape(-1, 2), ee_link=0, ready=np.zeros(1))


def test_self_collision_examples(O):
    rb = _two_sphere_robot(np.array([[0, 0, 0], [0.15, 0, 0]]), [0.1, 0.1], [[0, 1]])
    R = O.Robot(rb)
    sph = np.concatenate([rb.spheres[:, :3], rb.spheres[:, 3:]], 1)
    c, g, arg, _ = O.self_collision(R, sph, 1.0)
    assert c == pytest.approx(0.05, abs=1e-15) and arg == 0
    np.testing.assert_allclose(g[0], [1, 0, 0]); np.testing.assert_allclose(g[1], [-1, 0, 0])
    sph[1, 0] = 0.3
    c, g, arg, _ = O.self_collision(R, sph, 1.0)
    assert c == 0.0 and np.all(g == 0)
    # penetrations {0.02, 0.05, 0.05}: cost beta*0.05, gradient on the lower-index tied pair
    pos = np.array([[0, 0, 0], [0.18, 0, 0], [5, 0, 0], [5.15, 0, 0], [9, 0, 0], [9.15, 0, 0]])
    rb = _two_sphere_robot(pos, [0.1] * 6, [[0, 1], [2, 3], [4, 5]])
    sph = np.concatenate([pos, np.full((6, 1), 0.1)], 1)
    c, g, arg, _ = O.self_collision(O.Robot(rb), sph, 2.0)
    assert c == pytest.approx(0.1, abs=1e-14) and arg == 1
    assert np.all(g[[0, 1, 4, 5]] == 0) and np.abs(g[2]).sum() > 0


def test_self_collision_brute_force(O):
    g = np.random.default_rng(8)
    for t in range(30):
        M = 20
        pos = g.uniform(-0.3, 0.3, (M, 3)); rad = g.uniform(-0.02, 0.1, M)
        pairs = [(i, j) for i in range(M) for j in range(i + 1, M) if g.random() < 0.5]
        rb = _two_sphere_robot(pos, rad, pairs)
        sph = np.concatenate([pos, rad[:, None]], 1)
        c, gr, arg, _ = O.self_collision(O.Robot(rb), sph, 3.0)
        pens = [(rad[i] + rad[j] - np.linalg.norm(pos[i] - pos[j]), k) for k, (i, j) in enumerate(pairs)
                if rad[i] > 0 and rad[j] > 0]
        best = max(pens, key=lambda x: (x[0], -x[1])) if pens else (0.0, -1)
        assert c == pytest.approx(3.0 * max(0.0, best[0]), abs=1e-14)
        if best[0] > 0:
            assert arg == best[1]


# ------------------------------------------------------------------ world: discrete + swept (O5)

def _world(boxes):
    pos = np.array([b[0] for b in boxes]); quat = np.array([b[1] for b in boxes])
    dims = np.array([b[2] for b in boxes])
    return inputs.World(pos, quat, dims, np.ones(len(boxes), np.int32))


def test_discrete_far_and_fd(O):
    eta = 0.025
    W = O.World(inputs.random_world(0, 0, 12))
    E, G, *_ = O.sphere_world(W, [5, 5, 5], 0.1, eta)
    assert E == 0 and np.all(G == 0)
    g = np.random.default_rng(2)
    n_checked = 0
    for _ in range(400):
        c = g.uniform(-1, 1, 3); c[2] = g.uniform(0, 1)
        E, G, _, margin, _ = O.sphere_world(W, c, 0.08, eta)
        if E == 0 or margin < 1e-4:
            continue
        fd = np.array([(O.sphere_world(W, c + e, 0.08, eta)[0] - O.sphere_world(W, c - e, 0.08, eta)[0]) / 2e-7
                       for e in np.eye(3) * 1e-7])
        np.testing.assert_allclose(G, fd, atol=1e-6 * max(1.0, np.abs(fd).max()))
        n_checked += 1
    assert n_checked > 20


def test_static_sweep_is_discrete(O):
    """(i) static neighbours -> gap <= 0 -> no samples; (ii) sweep off == discrete."""
    W = O.World(inputs.random_world(1, 0, 12))
    g = np.random.default_rng(5)
    for _ in range(100):
        c = g.uniform(-1, 1, 3); c[2] = g.uniform(0, 1)
        Ed, Gd, *_ = O.sphere_world(W, c, 0.07, 0.025)
        Es, Gs, samples, *_ = O.sphere_world(W, c, 0.07, 0.025, cprev=c, cnext=c, sweep=True)
        assert len(samples) == 0 and Es == Ed and np.all(Gs == Gd)


def test_swept_superset_of_discrete(O):
    """(iv) S:167: swept cost is zero only if the discrete cost is zero; swept >= discrete."""
    W = O.World(inputs.random_world(2, 0, 15))
    g = np.random.default_rng(6)
    for _ in range(300):
        c = g.uniform(-1, 1, 3); c[2] = g.uniform(0, 1)
        cp = c + g.normal(0, 0.2, 3); cn = c + g.normal(0, 0.2, 3)
        Ed, *_ = O.sphere_world(W, c, 0.05, 0.025)
        Es, *_ = O.sphere_world(W, c, 0.05, 0.025, cprev=cp, cnext=cn, sweep=True)
        assert Es >= Ed
        if Ed > 0:
            assert Es > 0


def test_thin_wall_detection(O):
    """(iii) S:153 / S:638: 5 mm wall crossed between free endpoints -> swept cost > 0 while the
    discrete cost at both endpoints is 0; zero false negatives vs a 1000-sample dense segment."""
    eta, r = 0.025, 0.05
    W = O.World(_world([([0.5, 0, 0], IDQ, [0.01, 2.0, 2.0])]))
    E0, *_ = O.sphere_world(W, [0, 0, 0], r, eta)
    E1, *_ = O.sphere_world(W, [1, 0, 0], r, eta)
    Ea, *_ = O.sphere_world(W, [0, 0, 0], r, eta, cnext=[1, 0, 0], sweep=True)
    Eb, *_ = O.sphere_world(W, [1, 0, 0], r, eta, cprev=[0, 0, 0], sweep=True)
    assert E0 == 0 and E1 == 0 and Ea > 0 and Eb > 0
    g = np.random.default_rng(9)
    n_cross = 0
    for _ in range(100):
        a = np.array([g.uniform(0.0, 0.35), g.uniform(-0.3, 0.3), g.uniform(-0.3, 0.3)])
        b = np.array([g.uniform(0.65, 1.0), g.uniform(-0.3, 0.3), g.uniform(-0.3, 0.3)])
        ts = np.linspace(0, 1, 1000)
        pts = a[None] + ts[:, None] * (b - a)[None]
        dense_hit = np.any(np.abs(pts[:, 0] - 0.5) - 0.005 < r)     # wall spans |y|,|z| <= 1
        if not dense_hit:
            continue
        n_cross += 1
        Ea, *_ = O.sphere_world(W, a, r, eta, cnext=b, sweep=True)
        Eb, *_ = O.sphere_world(W, b, r, eta, cprev=a, sweep=True)
        assert Ea + Eb > 0
    assert n_cross == 100


def _np_box_sdf(p, pos, q, half):
    r = Rot.from_quat([q[1], q[2], q[3], q[0]])
    pl = r.inv().apply(p - pos)
    qv = np.abs(pl) - half
    if qv.max() > 0:
        return np.linalg.norm(np.maximum(qv, 0))
    return qv.max()


def test_swept_frozen_schedule_fd(O):
    """(vi) the surrogate gradient (A12) equals the central FD of the swept energy with the
    neighbours and the kappa schedule frozen; recomputed with an independent numpy SDF."""
    eta, r = 0.025, 0.05
    wl = inputs.random_world(3, 0, 10, dmin=0.02, dmax=0.3, disabled_frac=0.0)
    W = O.World(wl)
    half = 0.5 * wl.dims
    g = np.random.default_rng(10)
    n_checked = 0
    for _ in range(300):
        c = g.uniform(-1, 1, 3); c[2] = g.uniform(0, 1)
        cp = c + g.normal(0, 0.25, 3); cn = c + g.normal(0, 0.25, 3)
        E, G, samples, margin, _ = O.sphere_world(W, c, r, eta, cprev=cp, cnext=cn, sweep=True)
        if len(samples) == 0 or E == 0 or margin < 1e-4:
            continue
        rp = r + eta

        def energy(x):
            e = 0.0
            for k in range(wl.n_boxes):
                d = rp - _np_box_sdf(x, wl.pos[k], wl.quat[k], half[k])
                e += 0 if d <= 0 else (d * d / (2 * eta) if d <= eta else d - eta / 2)
            for (k, dr, kap, _) in samples:
                n = cp if dr == 0 else cn
                pnt = x + kap * (n - x)
                d = rp - _np_box_sdf(pnt, wl.pos[int(k)], wl.quat[int(k)], half[int(k)])
                e += 0 if d <= 0 else (d * d / (2 * eta) if d <= eta else d - eta / 2)
            return e
        assert energy(c) == pytest.approx(E, abs=1e-12)
        fd = np.array([(energy(c + e) - energy(c - e)) / 2e-7 for e in np.eye(3) * 1e-7])
        np.testing.assert_allclose(G, fd, atol=1e-6 * max(1.0, np.abs(fd).max()))
        n_checked += 1
    assert n_checked >= 10


# ------------------------------------------------------------------ pose (Eq. pose_cost_term, A1)

def test_pose_cost(O):
    cp = inputs.CostParams()
    g = np.random.default_rng(11)
    for _ in range(20):
        goal = np.concatenate([g.normal(size=3), wxyz(Rot.random(random_state=int(g.integers(1 << 30))))])
        c, gp, gq = O.pose_cost(cp, goal, goal)
        assert c == pytest.approx(0.0, abs=1e-12) and np.abs(gp).max() < 1e-9 and np.abs(gq).max() < 1e-7
        anti = goal.copy(); anti[3:] *= -1
        assert O.pose_cost(cp, anti, goal)[0] == pytest.approx(0.0, abs=1e-12)
        ee = goal + np.concatenate([g.normal(0, 0.05, 3), np.zeros(4)])
        ee[3:] = wxyz(Rot.random(random_state=int(g.integers(1 << 30))))
        anti = ee.copy(); anti[3:] *= -1
        assert O.pose_cost(cp, ee, goal)[0] == pytest.approx(O.pose_cost(cp, anti, goal)[0], rel=1e-14)
        # FD in p and q (q treated as free 4-vector)
        c, gp, gq = O.pose_cost(cp, ee, goal)
        for i in range(7):
            e = np.zeros(7); e[i] = 1e-7
            fd = (O.pose_cost(cp, ee + e, goal)[0] - O.pose_cost(cp, ee - e, goal)[0]) / 2e-7
            an = gp[i] if i < 3 else gq[i - 3]
            assert abs(an - fd) < 1e-5 * max(1, abs(fd))
    gold = GOLD["pose_1mm"]
    goal = np.array([0, 0, 0, 1, 0, 0, 0.0]); ee = goal.copy(); ee[0] += gold["offset_m"]
    assert O.pose_cost(cp, ee, goal)[0] == pytest.approx(gold["cost"], abs=1e-6)
    assert gold["cost"] == pytest.approx(2000 * np.log(np.cosh(0.1)), abs=1e-6)
    assert O.logcosh(800.0) == pytest.approx(800.0 - math.log(2.0), rel=1e-15)   # overflow-safe form


# ------------------------------------------------------------------ stencil (O3) and state map (O2)

def test_stencil_polynomial_exactness(O):
    dt = 0.1
    H = 20
    t = (np.arange(-2, H + 3) * dt)
    for deg in range(0, 6):
        x = (t ** deg)[:, None]
        v, a, j = O.derivs(x, H, dt)
        tt = t[3:3 + H]   # evaluated h = 1..H <-> rows h + 2
        dv = deg * tt ** (deg - 1) if deg >= 1 else 0 * tt
        da = deg * (deg - 1) * tt ** (deg - 2) if deg >= 2 else 0 * tt
        dj = deg * (deg - 1) * (deg - 2) * tt ** (deg - 3) if deg >= 3 else 0 * tt
        if deg <= 4:
            np.testing.assert_allclose(v[:, 0], dv, atol=1e-9)
            np.testing.assert_allclose(j[:, 0], dj, atol=1e-7)
        if deg <= 5:
            np.testing.assert_allclose(a[:, 0], da, atol=1e-8)
    v, a, j = O.derivs(np.full((H + 5, 3), 1.7), H, dt)
    assert np.abs(v).max() < 1e-12 and np.abs(a).max() < 1e-12 and np.abs(j).max() < 1e-12


def test_state_map_rest_invariant(O):
    """Table 5 last row: v, a, j at x_1, x_{H-1}, x_H vanish for any V (<= 1e-12)."""
    g = np.random.default_rng(12)
    for H in (8, 16, 32):
        V = g.normal(size=(H, 7)); s = g.normal(size=7)
        x = O.state_map(s, V)
        v, a, j = O.derivs(x, H, 0.25)
        for h in (1, H - 1, H):
            assert max(np.abs(v[h - 1]).max(), np.abs(a[h - 1]).max(), np.abs(j[h - 1]).max()) < 1e-12 * (1 + np.abs(V).max()) / 0.25 ** 3
        np.testing.assert_array_equal(x[2 + 1], s)
        np.testing.assert_array_equal(x[2 + H - 3], V[H - 1])
