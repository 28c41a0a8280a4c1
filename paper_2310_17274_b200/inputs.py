"""Seeded synthetic inputs shared by the oracle tests and the CUDA path.

This module holds data containers and counter-based random draws ONLY -- none of the method's
arithmetic (no kinematics, no signed distance, no costs).  Anything that needs the method (e.g.
the sphere centres of a start configuration, or a collision check) is passed in by the caller:
the oracle in tests/, the CUDA library in bench.py.

Workload recipe: SURVEY.md §8(d).1, restated in DESIGN.md ("Input recipe").
RNG: numpy's Philox4x64 bit generator, keyed by (run_seed, stream) with the counter's high words
set to (problem, seed) so every draw is independent of sharding and GPU count.
"""
from __future__ import annotations

import dataclasses
import math
from typing import Callable, Optional, Sequence

import numpy as np

# flags (same bit meaning in the oracle and the C-ABI; each side defines its own constants)
SWEEP, SPEED, JERK, CSPACE = 1, 2, 4, 8

STREAM_SCENE, STREAM_CONFIG, STREAM_SEED, STREAM_IK, STREAM_TEST = 1, 2, 3, 4, 5


def rng(run_seed: int, stream: int, problem: int = 0, seed: int = 0) -> np.random.Generator:
    """Counter-based generator for draw stream (run_seed, stream) at counter (problem, seed)."""
    bg = np.random.Philox(key=np.array([run_seed, stream], dtype=np.uint64),
                          counter=np.array([0, 0, seed, problem], dtype=np.uint64))
    return np.random.Generator(bg)


@dataclasses.dataclass
class Robot:
    """O1 robot description (P:2598-2605 kinematic tables)."""
    name: str
    parent: np.ndarray      # [L] int32, -1 for root, parent < own index
    jtype: np.ndarray       # [L] int32: 0 fixed, 1..3 prismatic x/y/z, 4..6 revolute x/y/z (Table 6)
    dof: np.ndarray         # [L] int32 actuated index or -1
    fixed: np.ndarray       # [L,12] float64, 3x4 row-major F_l
    lo: np.ndarray          # [D]
    hi: np.ndarray
    vmax: np.ndarray
    amax: np.ndarray
    jmax: np.ndarray
    spheres: np.ndarray     # [M,4] centre in link frame + radius (r < 0 disabled)
    sphere_link: np.ndarray  # [M] int32
    sphere_offset: np.ndarray  # [M] self-collision radius offsets
    pairs: np.ndarray       # [Pi,2] int32, i < j
    ee_link: int
    ready: np.ndarray       # [D] retract / ready configuration

    @property
    def n_links(self):
        return int(self.parent.shape[0])

    @property
    def n_dof(self):
        return int(self.lo.shape[0])

    @property
    def n_spheres(self):
        return int(self.spheres.shape[0])


@dataclasses.dataclass
class World:
    """Cuboids of one environment (§3.5).  dims are FULL extents."""
    pos: np.ndarray      # [K,3]
    quat: np.ndarray     # [K,4] (w,x,y,z)
    dims: np.ndarray     # [K,3]
    enabled: np.ndarray  # [K] int32

    @property
    def n_boxes(self):
        return int(self.pos.shape[0])


@dataclasses.dataclass
class CostParams:
    """Paper constants: P:2002 (alpha_0..3), P:2018 (alpha_8, alpha_9), P:2204 (eta = 2.5 cm,
    soft weights 5000), P:2045 (eta_2 = 0.1); sweep_steps = 4 (A11)."""
    a0: float = 2000.0
    a1: float = 350.0
    a2: float = 100.0
    a3: float = 100.0
    a8: float = 5000.0
    a9: float = 1.0
    w_bound: tuple = (5000.0, 5000.0, 5000.0, 5000.0)
    beta_self: float = 5000.0
    beta_world: float = 5000.0
    eta: float = 0.025
    eta_bound: float = 0.1
    dt: float = 0.25
    sweep_steps: int = 4
    flags: int = SWEEP | SPEED
    a4: float = 5000.0        # Eq. cspace-cost, used when flags & CSPACE
    a5: float = 50.0


@dataclasses.dataclass
class SolverParams:
    """L-BFGS history 4, alpha = {0.01, 0.3, 0.7, 1.0}, strong Wolfe with
    c1 = 1e-4, c2 = 0.9 (A17), 100 iterations."""
    iters: int = 100
    history: int = 4
    alpha: tuple = (0.01, 0.3, 0.7, 1.0)
    c1: float = 1e-4
    c2: float = 0.9
    ls_mode: int = 2
    # particle warm-up before L-BFGS (Alg. 5, Eqs. particle_1/2).  The paper runs
    # 2 iterations but gives no n / beta / k_mu / k_sigma / sigma_0: SPEC defaults
    # (S:368), non-paper values.  particle_iters = 0 disables the warm-up.
    particle_iters: int = 0
    n_particles: int = 64
    particle_beta: float = 1.0
    k_mu: float = 0.9
    k_sigma: float = 0.5
    sigma0_frac: float = 0.1
    rng_key: int = 0
    # "up to" iters in chunks of check_every iterations: a TO seed stops when
    # its best cost improved by at most conv_rtol x |best| over a chunk (reading B20); 0 = off
    check_every: int = 0
    conv_rtol: float = 0.0
    # latency mode: the line-search candidates of an iteration on the CTAs of a cluster
    # (-1 automatic for batches that fit one wave, 0 off, 1 on); bitwise identical results
    cluster: int = -1
    # IK scheduling: -1 automatic (persistent kernel over (seed group, iteration chunk) units for
    # batches of two or more waves), 0 one CTA per group, k >= 1 persistent with k chunks
    persist: int = -1


# --------------------------------------------------------------------------------------------
# scenes
# --------------------------------------------------------------------------------------------

def _uniform_quat(g: np.random.Generator) -> np.ndarray:
    """Uniform random rotation (Shoemake's subgroup algorithm), (w,x,y,z) with w >= 0."""
    u1, u2, u3 = g.random(3)
    a, b = math.sqrt(1.0 - u1), math.sqrt(u1)
    q = np.array([b * math.cos(2 * math.pi * u3), a * math.sin(2 * math.pi * u2),
                  a * math.cos(2 * math.pi * u2), b * math.sin(2 * math.pi * u3)])
    return q if q[0] >= 0 else -q


def _yaw_quat(g: np.random.Generator) -> np.ndarray:
    t = g.uniform(0.0, 2 * math.pi)
    return np.array([math.cos(t / 2), 0.0, 0.0, math.sin(t / 2)])


def _clear_of(centre, dims, keepout, eta) -> bool:
    """Conservative rejection: box bounding sphere vs keep-out spheres (no box SDF involved)."""
    if keepout is None or len(keepout) == 0:
        return True
    half_diag = 0.5 * math.sqrt(float(dims[0] ** 2 + dims[1] ** 2 + dims[2] ** 2))
    d = np.linalg.norm(keepout[:, :3] - centre[None, :], axis=1)
    return bool(np.all(d > half_diag + np.maximum(keepout[:, 3], 0.0) + eta + 1e-3))


def tabletop_scene(run_seed: int, env: int, n_boxes: int = 20, keepout: Optional[np.ndarray] = None,
                   eta: float = 0.025) -> World:
    """K = 20 'tabletop clutter': a 1.2 x 1.6 x 0.04 table with its top at z = -0.05 plus K-1
    boxes with dims U[0.05,0.30]^3, centre radius U[0.35,0.80], azimuth U[0,2pi), z U[0,0.9];
    yaw-only orientation for 70 %, uniform SO(3) for 30 %.  Boxes that touch a keep-out sphere
    (the start / goal arm, passed in by the caller) are resampled."""
    g = rng(run_seed, STREAM_SCENE, env, 0)
    pos = [np.array([0.3, 0.0, -0.07])]
    quat = [np.array([1.0, 0.0, 0.0, 0.0])]
    dims = [np.array([1.2, 1.6, 0.04])]
    while len(pos) < n_boxes:
        dm = g.uniform(0.05, 0.30, 3)
        rad, az, z = g.uniform(0.35, 0.80), g.uniform(0.0, 2 * math.pi), g.uniform(0.0, 0.9)
        c = np.array([rad * math.cos(az), rad * math.sin(az), z])
        q = _yaw_quat(g) if g.random() < 0.7 else _uniform_quat(g)
        if not _clear_of(c, dm, keepout, eta):
            continue
        pos.append(c); quat.append(q); dims.append(dm)
    return World(np.array(pos), np.array(quat), np.array(dims), np.ones(n_boxes, np.int32))


def dense_scene(run_seed: int, env: int, n_boxes: int = 1000, keepout: Optional[np.ndarray] = None,
                eta: float = 0.025) -> World:
    """K = 1000 'dense clutter': dims U[0.01,0.05]^3, centres uniform in the shell
    r in [0.25, 1.0] around (0, 0, 0.4), uniform SO(3)."""
    g = rng(run_seed, STREAM_SCENE, env, 1)
    pos, quat, dims = [], [], []
    while len(pos) < n_boxes:
        dm = g.uniform(0.01, 0.05, 3)
        v = g.normal(size=3)
        v /= np.linalg.norm(v)
        r = (g.uniform(0.25 ** 3, 1.0)) ** (1.0 / 3.0)
        c = np.array([0.0, 0.0, 0.4]) + r * v
        q = _uniform_quat(g)
        if not _clear_of(c, dm, keepout, eta):
            continue
        pos.append(c); quat.append(q); dims.append(dm)
    return World(np.array(pos), np.array(quat), np.array(dims), np.ones(n_boxes, np.int32))


def planar_scene() -> World:
    """Config 1: a 0.2 x 0.2 x 0.5 box at (1.2, 0.6, 0) and a thin
    0.02 x 0.6 x 0.5 wall at (-0.8, 0.4, 0)."""
    return World(np.array([[1.2, 0.6, 0.0], [-0.8, 0.4, 0.0]]),
                 np.array([[1.0, 0.0, 0.0, 0.0], [1.0, 0.0, 0.0, 0.0]]),
                 np.array([[0.2, 0.2, 0.5], [0.02, 0.6, 0.5]]), np.ones(2, np.int32))


def random_world(run_seed: int, env: int, n_boxes: int, lo=-1.0, hi=1.0, dmin=0.05, dmax=0.4,
                 disabled_frac=0.1) -> World:
    """Parity-test scene: boxes uniform in a cube, uniform SO(3), some disabled."""
    g = rng(run_seed, STREAM_TEST, env, 7)
    pos = g.uniform(lo, hi, (n_boxes, 3))
    pos[:, 2] = g.uniform(0.0, 1.0, n_boxes)
    quat = np.array([_uniform_quat(g) for _ in range(n_boxes)]).reshape(n_boxes, 4)
    dims = g.uniform(dmin, dmax, (n_boxes, 3))
    en = (g.random(n_boxes) >= disabled_frac).astype(np.int32)
    return World(pos, quat, dims, en)


def pad_worlds(worlds: Sequence[World]):
    """[n_env][K_max] padded arrays (disabled padding) + per-env counts."""
    kmax = max(1, max(w.n_boxes for w in worlds))
    n = len(worlds)
    pos = np.zeros((n, kmax, 3)); quat = np.zeros((n, kmax, 4)); quat[..., 0] = 1.0
    dims = np.ones((n, kmax, 3)) * 0.01
    en = np.zeros((n, kmax), np.int32)
    counts = np.zeros(n, np.int32)
    for e, w in enumerate(worlds):
        k = w.n_boxes
        counts[e] = k
        pos[e, :k], quat[e, :k], dims[e, :k], en[e, :k] = w.pos, w.quat, w.dims, w.enabled
    return pos, quat, dims, en, counts


# --------------------------------------------------------------------------------------------
# configurations and seeds
# --------------------------------------------------------------------------------------------

def uniform_configs(robot: Robot, run_seed: int, stream: int, problem: int, n: int,
                    margin: float = 0.0) -> np.ndarray:
    g = rng(run_seed, stream, problem, 11)
    lo, hi = robot.lo + margin, robot.hi - margin
    return g.uniform(lo, hi, (n, robot.n_dof))


def start_goal_configs(robot: Robot, run_seed: int, problem: int,
                       is_free: Optional[Callable[[np.ndarray], np.ndarray]] = None,
                       min_sep: float = 0.5, max_tries: int = 256):
    """Start and goal uniform in the limits with ||goal - start|| >= min_sep (§8(d).1); both
    must satisfy the caller's `is_free` predicate (self-collision check by oracle or GPU)."""
    g = rng(run_seed, STREAM_CONFIG, problem, 0)
    for _ in range(max_tries):
        s = g.uniform(robot.lo, robot.hi)
        q = g.uniform(robot.lo, robot.hi)
        if np.linalg.norm(q - s) < min_sep:
            continue
        if is_free is not None and not bool(np.all(is_free(np.stack([s, q])))):
            continue
        return s, q
    raise RuntimeError("could not draw a free start/goal pair")


def to_seeds(robot: Robot, run_seed: int, problem: int, start: np.ndarray, goal_cfg: np.ndarray,
             S: int, H: int, noise: float = 0.3) -> np.ndarray:
    """TO seeds (§8(d).1): seed 0 linear start -> goal config; seeds 1..S-1 linear to
    clip(goal + N(0, 0.3^2)) plus a sin(pi h / H) * N(0, 0.3^2) bump per DoF, clipped."""
    D = robot.n_dof
    out = np.zeros((S, H, D))
    h = np.arange(1, H + 1)[:, None] / H
    for s in range(S):
        g = rng(run_seed, STREAM_SEED, problem, s)
        if s == 0:
            tgt, bump = goal_cfg, np.zeros(D)
        else:
            tgt = np.clip(goal_cfg + g.normal(0.0, noise, D), robot.lo, robot.hi)
            bump = g.normal(0.0, noise, D)
        traj = start[None, :] + (tgt - start)[None, :] * h + np.sin(np.pi * h) * bump[None, :]
        out[s] = np.clip(traj, robot.lo, robot.hi)
    return out


def halton(index: int, base: int) -> float:
    f, r = 1.0, 0.0
    while index > 0:
        f /= base
        r += f * (index % base)
        index //= base
    return r


HALTON_BASES = (2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37)


def ik_seeds(robot: Robot, goal_index: int, S: int) -> np.ndarray:
    """IK seeds (§8(d).1): Halton sequence in the joint limits, offset by goal index."""
    D = robot.n_dof
    out = np.zeros((S, D))
    for s in range(S):
        idx = goal_index * S + s + 1
        u = np.array([halton(idx, HALTON_BASES[d]) for d in range(D)])
        out[s] = robot.lo + u * (robot.hi - robot.lo)
    return out


def random_goal_poses(run_seed: int, n: int, centre=(0.4, 0.0, 0.4), spread=0.3) -> np.ndarray:
    """Arbitrary goal poses [n,7] (p, quat wxyz) for per-evaluation parity tests."""
    g = rng(run_seed, STREAM_TEST, 0, 3)
    out = np.zeros((n, 7))
    for i in range(n):
        out[i, :3] = np.asarray(centre) + g.uniform(-spread, spread, 3)
        out[i, 3:] = _uniform_quat(g)
    return out
