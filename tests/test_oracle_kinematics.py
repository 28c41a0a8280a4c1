"""Pins for the oracle's kinematics (O4, O6): closed forms, an independent quaternion+vector
composition (scipy), central finite differences.  CPU only."""
import json
import math
import os

import numpy as np
import pytest
from scipy.spatial.transform import Rotation as Rot

from paper_2310_17274_b200 import inputs, robots

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_values.json")))


def random_chain(seed, n_links, n_spheres=6, types=None):
    """Random tree-structured chain with every Table 6 joint type."""
    g = np.random.default_rng(seed)
    parent, jtype, dof, fixed = [-1], [0], [-1], [np.eye(3, 4).reshape(12)]
    d = 0
    for l in range(1, n_links):
        parent.append(int(g.integers(0, l)) if l > 1 else 0)
        t = int(types[l % len(types)]) if types is not None else int(g.integers(0, 7))
        jtype.append(t)
        if t == 0:
            dof.append(-1)
        else:
            dof.append(d)
            d += 1
        R = Rot.random(random_state=g.integers(1 << 30)).as_matrix()
        fixed.append(np.concatenate([R, g.uniform(-0.5, 0.5, (3, 1))], axis=1).reshape(12))
    D = max(d, 1)
    sph = np.concatenate([g.uniform(-0.3, 0.3, (n_spheres, 3)), g.uniform(0.02, 0.1, (n_spheres, 1))], 1)
    slink = g.integers(0, n_links, n_spheres).astype(np.int32)
    return inputs.Robot(name="rand", parent=np.array(parent, np.int32), jtype=np.array(jtype, np.int32),
                        dof=np.array(dof, np.int32), fixed=np.array(fixed), lo=-np.ones(D) * 3,
                        hi=np.ones(D) * 3, vmax=np.ones(D), amax=np.ones(D), jmax=np.ones(D),
                        spheres=sph, sphere_link=slink, sphere_offset=np.zeros(n_spheres),
                        pairs=np.zeros((0, 2), np.int32), ee_link=n_links - 1, ready=np.zeros(D))


def reference_fk(rb, q):
    """Independent arithmetic: rigid motions as (scipy Rotation, vector), composed left to right."""
    T = []
    for l in range(rb.n_links):
        F = rb.fixed[l].reshape(3, 4)
        rF, tF = Rot.from_matrix(F[:, :3]), F[:, 3]
        if rb.parent[l] < 0:
            rP, tP = Rot.identity(), np.zeros(3)
        else:
            rP, tP = T[rb.parent[l]]
        r, t = rP * rF, tP + rP.apply(tF)
        ty = int(rb.jtype[l])
        v = q[rb.dof[l]] if rb.dof[l] >= 0 else 0.0
        if 1 <= ty <= 3:
            e = np.eye(3)[ty - 1]
            t = t + r.apply(v * e)
        elif ty >= 4:
            e = np.eye(3)[ty - 4]
            r = r * Rot.from_rotvec(v * e)
        T.append((r, t))
    sph = np.array([T[int(rb.sphere_link[m])][1] + T[int(rb.sphere_link[m])][0].apply(rb.spheres[m, :3])
                    for m in range(rb.n_spheres)])
    re, te = T[rb.ee_link]
    x, y, z, w = re.as_quat()
    qe = np.array([w, x, y, z])
    if qe[0] < 0:
        qe = -qe
    return T, sph, te, qe


def test_planar2_closed_form(O):
    R = O.Robot(robots.planar2())
    _, _, ee = O.fk(R, [0.0, 0.0])
    np.testing.assert_allclose(ee[:3], [2, 0, 0], atol=1e-14)
    np.testing.assert_allclose(ee[3:], [1, 0, 0, 0], atol=1e-14)
    _, _, ee = O.fk(R, [math.pi / 2, 0.0])
    np.testing.assert_allclose(ee[:3], [0, 2, 0], atol=1e-14)
    g = np.random.default_rng(0)
    for _ in range(50):
        q1, q2 = g.uniform(-math.pi, math.pi, 2)
        _, sph, ee = O.fk(R, [q1, q2])
        exp = [math.cos(q1) + math.cos(q1 + q2), math.sin(q1) + math.sin(q1 + q2), 0]
        np.testing.assert_allclose(ee[:3], exp, atol=1e-13)
        np.testing.assert_allclose(sph[0, :3], [0.5 * math.cos(q1), 0.5 * math.sin(q1), 0], atol=1e-14)
        half = (q1 + q2) / 2
        qexp = np.array([math.cos(half), 0, 0, math.sin(half)])
        qexp = qexp if qexp[0] >= 0 else -qexp
        np.testing.assert_allclose(ee[3:], qexp, atol=1e-12)


def test_prismatic_z_table6(O):
    """S:64 / Table 6 Prismatic Z: f_10 d_z + f_11 with identity F."""
    rb = random_chain(1, 2, types=[0, 3])
    rb.fixed[1] = np.eye(3, 4).reshape(12)
    _, _, ee = O.fk(O.Robot(rb), [0.3])
    np.testing.assert_allclose(ee[:3], [0, 0, 0.3], atol=1e-15)


@pytest.mark.parametrize("jt", [1, 2, 3, 4, 5, 6])
def test_each_joint_type_vs_rodrigues(O, jt):
    """Every Table 6 type against Rodrigues rotation / translation (A25 typo not reproduced)."""
    g = np.random.default_rng(jt)
    rb = random_chain(10 + jt, 2, types=[0, jt])
    R = O.Robot(rb)
    for _ in range(20):
        v = g.uniform(-3, 3)
        T, _, _ = O.fk(R, [v])
        F = rb.fixed[1].reshape(3, 4)
        if jt <= 3:
            J = np.eye(4); J[jt - 1, 3] = v
        else:
            k = np.eye(3)[jt - 4]
            K = np.array([[0, -k[2], k[1]], [k[2], 0, -k[0]], [-k[1], k[0], 0]])
            J = np.eye(4); J[:3, :3] = np.eye(3) + math.sin(v) * K + (1 - math.cos(v)) * K @ K
        F4 = np.eye(4); F4[:3] = F
        np.testing.assert_allclose(T[1].reshape(3, 4), (F4 @ J)[:3], atol=1e-13)


@pytest.mark.parametrize("n_links", [3, 4, 8, 12])
def test_random_chains_vs_quaternion_composition(O, n_links):
    """S:637 criterion 2 analogue: 200 random configs per chain, every joint kind, <= 1e-12."""
    for seed in range(5):
        rb = random_chain(100 * n_links + seed, n_links)
        R = O.Robot(rb)
        g = np.random.default_rng(seed)
        for _ in range(40):
            q = g.uniform(-3, 3, rb.n_dof)
            T, sph, ee = O.fk(R, q)
            Tr, sphr, te, qe = reference_fk(rb, q)
            for l in range(rb.n_links):
                np.testing.assert_allclose(T[l].reshape(3, 4)[:, :3], Tr[l][0].as_matrix(), atol=1e-12)
                np.testing.assert_allclose(T[l].reshape(3, 4)[:, 3], Tr[l][1], atol=1e-12)
            np.testing.assert_allclose(sph[:, :3], sphr, atol=1e-12)
            np.testing.assert_allclose(ee[:3], te, atol=1e-12)
            if abs(qe[0]) > 1e-6:
                np.testing.assert_allclose(ee[3:], qe, atol=1e-10)


def test_mat_to_quat_all_branches(O):
    """Shepperd branches incl. near-180-degree rotations vs scipy, canonical w >= 0."""
    import ctypes
    g = np.random.default_rng(5)
    rots = list(Rot.random(200, random_state=7)) + [Rot.from_rotvec(np.pi * 0.9999 * v / np.linalg.norm(v))
                                                     for v in g.normal(size=(50, 3))]
    for r in rots:
        R = np.ascontiguousarray(r.as_matrix().reshape(9))
        q = np.zeros(4)
        O.lib().orc_mat_to_quat(R.ctypes.data_as(O.D_P), q.ctypes.data_as(O.D_P))
        x, y, z, w = r.as_quat()
        ref = np.array([w, x, y, z])
        ref = ref if ref[0] >= 0 else -ref
        assert q[0] >= 0
        np.testing.assert_allclose(q, ref, atol=1e-12)


def test_franka_flange_golden(O):
    rb = robots.franka64()
    T, _, _ = O.fk(O.Robot(rb), np.zeros(7))
    np.testing.assert_allclose(T[8].reshape(3, 4)[:, 3], GOLD["franka_flange_q0"]["value"], atol=1e-12)


def test_franka_pairs(O):
    """S = pairs > 2 hops apart (~50 % of pairs); none penetrates at the ready pose."""
    rb = robots.franka64()
    M = rb.n_spheres
    frac = len(rb.pairs) / (M * (M - 1) / 2)
    assert 0.4 < frac < 0.65
    _, sph, _ = O.fk(O.Robot(rb), rb.ready)
    for i, j in rb.pairs:
        ri, rj = rb.spheres[i, 3], rb.spheres[j, 3]
        if ri > 0 and rj > 0:
            assert ri + rj < np.linalg.norm(sph[i, :3] - sph[j, :3])


def _fd_objective(O, R, q, Gs, gp, gq):
    _, sph, ee = O.fk(R, q)
    return float(np.sum(Gs * sph[:, :3]) + gp @ ee[:3] + gq @ ee[3:])


def test_backward_one_dof_example(O):
    """1-DoF revolute-z, sphere at (1,0,0), cotangent (0,1,0) -> 1.0."""
    rb = random_chain(3, 2, n_spheres=1, types=[0, 6])
    rb.fixed[1] = np.eye(3, 4).reshape(12)
    rb.spheres[0] = [1, 0, 0, 0.1]
    rb.sphere_link[0] = 1
    g = O.fk_backward(O.Robot(rb), [0.0], g_sph=np.array([[0.0, 1.0, 0.0]]))
    np.testing.assert_allclose(g, [1.0], atol=1e-15)


@pytest.mark.parametrize("seed", range(8))
def test_backward_vs_central_fd(O, seed):
    """O6 (Alg. 8 / Table 7 + A27) vs central FD of the pinned forward, step 1e-6."""
    rb = random_chain(1000 + seed, 7 + seed % 5, n_spheres=12)
    R = O.Robot(rb)
    g = np.random.default_rng(seed)
    for _ in range(5):
        q = g.uniform(-2.5, 2.5, rb.n_dof)
        _, _, ee = O.fk(R, q)
        if abs(ee[3]) < 0.05:
            continue   # keep away from the w = 0 canonicalisation flip
        Gs = g.normal(size=(rb.n_spheres, 3)); gp = g.normal(size=3); gq = g.normal(size=4)
        an = O.fk_backward(R, q, Gs, gp, gq)
        fd = np.zeros(rb.n_dof)
        for d in range(rb.n_dof):
            e = np.zeros(rb.n_dof); e[d] = 1e-6
            fd[d] = (_fd_objective(O, R, q + e, Gs, gp, gq) - _fd_objective(O, R, q - e, Gs, gp, gq)) / 2e-6
        np.testing.assert_allclose(an, fd, rtol=1e-7, atol=1e-7 * (1 + np.abs(fd).max()))
