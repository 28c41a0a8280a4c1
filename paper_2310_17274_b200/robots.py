"""Robot descriptions used by the synthetic workloads (data only -- no kinematics arithmetic).

* ``franka64()`` -- "Franka-Panda-shaped" 7-DoF arm, L = 14 links, M = 64 spheres.
  The fixed transforms are the public modified-DH values (a, d, alpha) of the Panda written out
  as exact 3x4 matrices F_l = RotX(alpha) TransX(a) TransZ(d) (alpha in {0, +-pi/2}, so every
  rotation entry is 0 or +-1); the joint J_l is revolute-z (Table 6).  Sphere
  counts per link follow SURVEY §8(d).1; positions are evenly spaced on hand-chosen segments.
* ``planar2()`` -- the 2-link planar arm of config 1.

The self-collision set S: every sphere pair whose links are more than two hops apart in
the kinematic tree.  SURVEY §8(d).1 also removes pairs penetrating at the ready pose; with these
sphere placements there are none (pinned by tests/test_oracle_kinematics.py::test_franka_pairs).
"""
from __future__ import annotations

import math

import numpy as np

from .inputs import Robot

S2 = math.sqrt(0.5)


def _F(R, t):
    R = np.asarray(R, dtype=np.float64)
    return np.concatenate([R, np.asarray(t, dtype=np.float64)[:, None]], axis=1).reshape(12)


_I = [[1, 0, 0], [0, 1, 0], [0, 0, 1]]
_RXm = [[1, 0, 0], [0, 0, 1], [0, -1, 0]]   # RotX(-pi/2)
_RXp = [[1, 0, 0], [0, 0, -1], [0, 1, 0]]   # RotX(+pi/2)
_RZm45 = [[S2, S2, 0], [-S2, S2, 0], [0, 0, 1]]  # RotZ(-pi/4)

# (parent, jtype, dof, F) ; F = RotX(alpha) * TransX(a) * TransZ(d) -> [RotX | (a, -sin(alpha) d, cos(alpha) d)]
_FRANKA_LINKS = [
    (-1, 0, -1, _F(_I, [0, 0, 0])),                 # 0 base
    (0, 6, 0, _F(_I, [0, 0, 0.333])),               # 1 link1: a=0, d=0.333, alpha=0
    (1, 6, 1, _F(_RXm, [0, 0, 0])),                 # 2 link2: alpha=-pi/2
    (2, 6, 2, _F(_RXp, [0, -0.316, 0])),            # 3 link3: d=0.316, alpha=+pi/2
    (3, 6, 3, _F(_RXp, [0.0825, 0, 0])),            # 4 link4: a=0.0825, alpha=+pi/2
    (4, 6, 4, _F(_RXm, [-0.0825, 0.384, 0])),       # 5 link5: a=-0.0825, d=0.384, alpha=-pi/2
    (5, 6, 5, _F(_RXp, [0, 0, 0])),                 # 6 link6: alpha=+pi/2
    (6, 6, 6, _F(_RXp, [0.088, 0, 0])),             # 7 link7: a=0.088, alpha=+pi/2
    (7, 0, -1, _F(_I, [0, 0, 0.107])),              # 8 flange
    (8, 0, -1, _F(_RZm45, [0, 0, 0])),              # 9 hand (yaw -pi/4)
    (9, 0, -1, _F(_I, [0, 0, 0.1034])),             # 10 TCP (end effector)
    (9, 0, -1, _F(_I, [0, 0.03, 0.0584])),          # 11 left finger (locked)
    (9, 0, -1, _F(_I, [0, -0.03, 0.0584])),         # 12 right finger (locked)
    (10, 0, -1, _F(_I, [0, 0, 0])),                 # 13 attached object (spheres disabled)
]

# (link, n, start, end, radius).  A child link's first sphere starts 1-1.5 cm past its joint origin,
# where the parent's last sphere sits: coincident duplicate spheres would give every pair with a
# third sphere an exact twin (ties of the self-collision arg-max, A28, at every configuration).
_FRANKA_SEGMENTS = [
    (0, 4, [0, 0, 0.06], [0, 0, 0.20], 0.08),
    (1, 6, [0, 0, -0.13], [0, 0, 0.0], 0.07),
    (2, 6, [0, -0.015, 0.0], [0, -0.18, 0.0], 0.07),
    (3, 7, [0, 0, -0.14], [0.0825, 0, 0.0], 0.065),
    (4, 7, [-0.01, 0.015, 0.0], [-0.0825, 0.12, 0.0], 0.065),
    (5, 10, [0, 0, -0.26], [0, 0, 0.0], 0.06),
    (6, 6, [0.012, 0, 0.0], [0.088, 0, 0.0], 0.06),
    (7, 5, [0, 0, 0.012], [0, 0, 0.08], 0.05),
    (9, 7, [0, -0.09, 0.04], [0, 0.09, 0.04], 0.04),
    (11, 2, [0, 0.008, 0.015], [0, 0.008, 0.04], 0.02),
    (12, 2, [0, -0.008, 0.015], [0, -0.008, 0.04], 0.02),
    (13, 2, [0, 0, 0.02], [0, 0, 0.06], -1.0),
]

# public Panda limits: pos (rad), vel (rad/s), acc 15 rad/s^2, jerk 7500.
_FRANKA_LO = [-2.8973, -1.7628, -2.8973, -3.0718, -2.8973, -0.0175, -2.8973]
_FRANKA_HI = [2.8973, 1.7628, 2.8973, -0.0698, 2.8973, 3.7525, 2.8973]
_FRANKA_VMAX = [2.175, 2.175, 2.175, 2.175, 2.61, 2.61, 2.61]
_FRANKA_READY = [0.0, -0.785, 0.0, -2.356, 0.0, 1.571, 0.785]


def _tree_hops(parent):
    L = len(parent)
    depth = [0] * L
    for l in range(L):
        depth[l] = 0 if parent[l] < 0 else depth[parent[l]] + 1

    def hops(a, b):
        n = 0
        while a != b:
            if depth[a] >= depth[b]:
                a = parent[a]
            else:
                b = parent[b]
            n += 1
        return n
    return hops


def _segment_spheres(segments):
    sph, link = [], []
    for (l, n, a, b, r) in segments:
        a, b = np.asarray(a, float), np.asarray(b, float)
        for i in range(n):
            t = i / (n - 1) if n > 1 else 0.5
            c = a + (b - a) * t
            sph.append([c[0], c[1], c[2], r])
            link.append(l)
    return np.array(sph), np.array(link, np.int32)


def franka64() -> Robot:
    parent = np.array([x[0] for x in _FRANKA_LINKS], np.int32)
    jtype = np.array([x[1] for x in _FRANKA_LINKS], np.int32)
    dof = np.array([x[2] for x in _FRANKA_LINKS], np.int32)
    fixed = np.stack([x[3] for x in _FRANKA_LINKS])
    sph, slink = _segment_spheres(_FRANKA_SEGMENTS)
    hops = _tree_hops(list(parent))
    pairs = []
    M = sph.shape[0]
    for i in range(M):
        for j in range(i + 1, M):
            if hops(int(slink[i]), int(slink[j])) > 2:
                pairs.append((i, j))
    D = 7
    return Robot(name="franka64", parent=parent, jtype=jtype, dof=dof, fixed=fixed,
                 lo=np.array(_FRANKA_LO), hi=np.array(_FRANKA_HI), vmax=np.array(_FRANKA_VMAX),
                 amax=np.full(D, 15.0), jmax=np.full(D, 7500.0), spheres=sph, sphere_link=slink,
                 sphere_offset=np.zeros(M), pairs=np.array(pairs, np.int32).reshape(-1, 2),
                 ee_link=10, ready=np.array(_FRANKA_READY))


def planar2() -> Robot:
    """Config 1: two revolute-z links of 1 m, spheres r = 0.1 at 0.5 m and 1.0 m on each link,
    S = {(sphere 0, sphere 3)}, limits +-pi, vmax 2, amax 15, jmax 500."""
    parent = np.array([-1, 0, 1, 2], np.int32)
    jtype = np.array([0, 6, 6, 0], np.int32)
    dof = np.array([-1, 0, 1, -1], np.int32)
    fixed = np.stack([_F(_I, [0, 0, 0]), _F(_I, [0, 0, 0]), _F(_I, [1, 0, 0]), _F(_I, [1, 0, 0])])
    sph = np.array([[0.5, 0, 0, 0.1], [1.0, 0, 0, 0.1], [0.5, 0, 0, 0.1], [1.0, 0, 0, 0.1]])
    slink = np.array([1, 1, 2, 2], np.int32)
    return Robot(name="planar2", parent=parent, jtype=jtype, dof=dof, fixed=fixed,
                 lo=np.full(2, -math.pi), hi=np.full(2, math.pi), vmax=np.full(2, 2.0),
                 amax=np.full(2, 15.0), jmax=np.full(2, 500.0), spheres=sph, sphere_link=slink,
                 sphere_offset=np.zeros(4), pairs=np.array([[0, 3]], np.int32), ee_link=3,
                 ready=np.zeros(2))
