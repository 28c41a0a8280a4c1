"""Pins for the whole rollout with the swept world term and the speed metric on (O5 world term,
Eq. world-collision-cost, speed P:118, readings A12-A13), CPU only.

The surrogate gradient of A12 is the exact gradient of the world cost with the sweep schedule
frozen: the neighbours w_{h-1}, w_{h+1}, every sweep sample's kappa and the speed sp are taken at
the base point and held.  These tests rebuild that frozen world cost from the oracle's pinned
pieces (state map, FK) with an independent numpy box SDF and activation, check it against the
oracle's world term at the base point, and check the oracle's whole-rollout gradient against the
central FD of  C_nonworld(V) + C_w_frozen(V)  along random directions.  A closed form with
quadratic motion fixes the speed as the CENTRAL difference ||w_{h+1} - w_{h-1}|| / (2 dt).
"""
import dataclasses

import numpy as np
import pytest
from scipy.spatial.transform import Rotation as Rot

from paper_2310_17274_b200 import inputs
from test_oracle_rollout import franka_problem

FLAGS = inputs.SWEEP | inputs.SPEED | inputs.JERK


def np_box_sdf_many(P, pos, quat, half):
    """Exact box SDF (§3.5 closest point; inside = nearest face), rows of P against rows of boxes."""
    r = Rot.from_quat(np.c_[quat[:, 1:], quat[:, :1]])
    pl = r.inv().apply(P - pos)
    q = np.abs(pl) - half
    out = np.linalg.norm(np.maximum(q, 0.0), axis=1)
    qm = q.max(axis=1)
    return np.where(qm > 0, out, qm)


def np_phi(dp, eta):
    """Eq. smooth-distance-cases in the inflated-radius form d' = r + eta - sd (A2)."""
    return np.where(dp <= 0, 0.0, np.where(dp <= eta, dp * dp / (2 * eta), dp - 0.5 * eta))


def spheres_of(O, R, start, V):
    x = O.state_map(start, V)                 # [H+5][D], x_h at row h + 2
    H = V.shape[0]
    return np.stack([O.fk(R, x[h + 2])[1] for h in range(1, H + 1)])   # [H][M][4]


class FrozenWorld:
    """The world term of one trajectory with the schedule frozen at V0 (A12)."""

    def __init__(self, O, R, rb, wl, cp, start, V0):
        W = O.World(wl)
        self.O, self.R, self.rb, self.cp, self.start = O, R, rb, cp, start
        sph = spheres_of(O, R, start, V0)
        H, M = sph.shape[:2]
        half = 0.5 * wl.dims
        en = np.flatnonzero(wl.enabled)
        self.en = en
        self.box = (wl.pos[en], wl.quat[en], half[en])
        rows = []          # (h, m, sp)
        samples = []       # (row, box k, kappa, neighbour[3])
        for h in range(H):
            for m in range(M):
                r = rb.spheres[m, 3]
                if r < 0:
                    continue
                c = sph[h, m, :3]
                cpv = sph[h - 1, m, :3] if h > 0 else None
                cnx = sph[h + 1, m, :3] if h + 1 < H else None
                a = cpv if cpv is not None else c                   # A13: missing -> w_h
                b = cnx if cnx is not None else c
                sp = np.linalg.norm(b - a) / (2 * cp.dt)            # P:118 central difference
                _, _, smp, _, _ = O.sphere_world(W, c, r, cp.eta, cprev=cpv, cnext=cnx, sweep=True,
                                                 steps=cp.sweep_steps, max_samples=4096)
                rows.append((h, m, sp))
                for (k, dr, kap, _) in smp:
                    samples.append((len(rows) - 1, int(k), kap, cpv if dr == 0 else cnx))
        self.rows = rows
        self.samples = samples

    def cost(self, V):
        sph = spheres_of(self.O, self.R, self.start, V)
        cp, rb = self.cp, self.rb
        pos, quat, half = self.box
        K = pos.shape[0]
        E = np.zeros(len(self.rows))
        if K:
            C = np.array([sph[h, m, :3] for (h, m, _) in self.rows])
            rr = np.array([rb.spheres[m, 3] + cp.eta for (_, m, _) in self.rows])
            for k in range(K):   # discrete part, every enabled box
                sd = np_box_sdf_many(C, pos[k][None], quat[k][None], half[k][None])
                E += np_phi(rr - sd, cp.eta)
            if self.samples:
                ri = np.array([s[0] for s in self.samples])
                kk = np.array([s[1] for s in self.samples])
                kap = np.array([s[2] for s in self.samples])[:, None]
                nb = np.array([s[3] for s in self.samples])
                P = C[ri] + kap * (nb - C[ri])                       # frozen kappa and neighbour
                # sample box indices are the oracle's (all boxes); map them to the enabled list
                loc = np.searchsorted(self.en, kk)
                sd = np_box_sdf_many(P, pos[loc], quat[loc], half[loc])
                np.add.at(E, ri, np_phi(rr[ri] - sd, cp.eta))
        sp = np.array([r[2] for r in self.rows])
        return cp.beta_world * float(np.sum(sp * E))


_CHECKED = []


@pytest.mark.parametrize("seed", range(8))
def test_rollout_fd_sweep_speed_frozen_schedule(O, seed):
    """SURVEY §8(c).3 'Whole rollout': directional FD with SWEEP | SPEED | JERK on and the sweep
    schedule frozen.  The oracle's world gradient is beta_2 sp G (Eq. world-collision-cost with
    the speed factor of P:121); dropping sp, or computing the speed any other way, fails here."""
    H = 10 + seed % 3
    rb, wl, cp, start, goal, V = franka_problem(seed, H, n_boxes=16, flags=FLAGS)
    R, W = O.Robot(rb), O.World(wl)
    c, grad, terms, margin, cnt = O.eval_traj(R, W, cp, start, goal, V)
    fw = FrozenWorld(O, R, rb, wl, cp, start, V)
    # the frozen world cost IS the oracle's world term at the base point
    assert fw.cost(V) == pytest.approx(terms[4], rel=1e-11, abs=1e-9)
    cp0 = dataclasses.replace(cp, beta_world=0.0)       # every other term (weight linearity pinned)
    g = np.random.default_rng(200 + seed)
    checked = 0
    for _ in range(10):
        u = g.normal(size=V.shape)
        eps = 1e-7
        cpl = O.eval_traj(R, W, cp0, start, goal, V + eps * u)
        cmi = O.eval_traj(R, W, cp0, start, goal, V - eps * u)
        if min(cpl[3], cmi[3], margin) < 1e-5:
            continue
        fd = (cpl[0] + fw.cost(V + eps * u) - cmi[0] - fw.cost(V - eps * u)) / (2 * eps)
        an = float(np.sum(grad * u))
        assert abs(fd - an) <= 1e-6 * max(1.0, abs(fd), np.abs(grad).sum()), (fd, an)
        checked += 1
    _CHECKED.append((checked, terms[4] > 0, len(fw.samples)))


def test_rollout_fd_sweep_speed_not_vacuous():
    assert sum(c for c, _, _ in _CHECKED) >= 50
    assert sum(w for _, w, _ in _CHECKED) >= 5            # world term active
    assert sum(s for _, _, s in _CHECKED) >= 100          # sweep samples taken


def _slider_robot():
    """One prismatic-x joint carrying one sphere (r = 0.05) at the joint origin: w_h = (x_h, 0, 0)."""
    I34 = np.eye(3, 4).reshape(12)
    return inputs.Robot(name="slider", parent=np.array([-1, 0], np.int32), jtype=np.array([0, 1], np.int32),
                        dof=np.array([-1, 0], np.int32), fixed=np.stack([I34, I34]), lo=np.array([-5.0]),
                        hi=np.array([5.0]), vmax=np.array([100.0]), amax=np.array([1e4]), jmax=np.array([1e7]),
                        spheres=np.array([[0.0, 0.0, 0.0, 0.05]]), sphere_link=np.array([1], np.int32),
                        sphere_offset=np.zeros(1), pairs=np.zeros((0, 2), np.int32), ee_link=1,
                        ready=np.zeros(1))


@pytest.mark.parametrize("dt", [0.1, 0.25])
def test_speed_closed_form_quadratic_motion(O, dt):
    """A13 / P:118 'velocity (calculated through finite-difference)': sp = ||w_{h+1} - w_{h-1}|| /
    (2 dt).  Quadratic motion x_h = c h^2 separates the central difference
    c ((h+1)^2 - (h-1)^2) / (2 dt) = 2 c h / dt from a one-sided one, c (2h + 1) / dt.  Only
    state h = 8 touches a thin slab 3 cm ahead of it, so with SPEED on and SWEEP off
    C_w = beta_2 * (2 c 8 / dt) * phi(r + eta - 0.03) in closed form (phi of Eq.
    smooth-distance-cases, past the quadratic zone: d' - eta/2)."""
    rb = _slider_robot()
    H, c = 16, 0.01
    xs = c * np.arange(1, H + 1) ** 2                     # x_h = c h^2
    V = xs[:, None].copy()                                # V_{h-1} = x_h for the free states
    start = np.array([xs[0]])
    wl = inputs.World(np.array([[c * 64 + 0.035, 0.0, 0.0]]), np.array([[1.0, 0, 0, 0]]),
                      np.array([[0.01, 1.0, 1.0]]), np.ones(1, np.int32))
    cp = inputs.CostParams(flags=inputs.SPEED, dt=dt, w_bound=(0.0, 0.0, 0.0, 0.0))
    R, W = O.Robot(rb), O.World(wl)
    goal = np.array([0.0, 0.0, 0.0, 1.0, 0.0, 0.0, 0.0])
    _, _, terms, _, _ = O.eval_traj(R, W, cp, start, goal, V)
    dp = 0.05 + cp.eta - 0.03                             # d' = r' - sd at x_8
    assert dp > cp.eta
    sp = (xs[8] - xs[6]) / (2 * dt)                       # states 9 and 7 (x_9 - x_7 = 2 c 8)
    assert sp == pytest.approx(2 * c * 8 / dt, rel=1e-12)
    assert terms[4] == pytest.approx(cp.beta_world * sp * (dp - 0.5 * cp.eta), rel=1e-12)
    # without SPEED the factor is 1 (P:121 d_s = s_dot d_c only with the speed metric)
    _, _, t1, _, _ = O.eval_traj(R, W, dataclasses.replace(cp, flags=0), start, goal, V)
    assert t1[4] == pytest.approx(cp.beta_world * (dp - 0.5 * cp.eta), rel=1e-12)
