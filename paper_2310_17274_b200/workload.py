"""Synthetic workloads of BASELINE.json's configs, assembled with the CUDA library.

The random draws come from `inputs` (counter-based, shard-independent); the method arithmetic the
recipe needs (FK of the start/goal arm for the keep-out spheres and the goal pose, the
self-collision check of start/goal) runs through the C-ABI (`native.Context`).  Nothing here
calls the oracle.
"""
from __future__ import annotations

import dataclasses
from typing import List, Optional

import numpy as np

from . import inputs, robots


@dataclasses.dataclass
class Workload:
    name: str
    robot: inputs.Robot
    worlds: List[inputs.World]
    env: np.ndarray          # [P] int32
    start: Optional[np.ndarray]   # [P,D] (TO) or None (IK)
    goal: np.ndarray         # [P,7]
    seeds: np.ndarray        # [P,S,H,D] (TO) or [P,S,D] (IK), float32
    cost: inputs.CostParams
    solver: inputs.SolverParams
    problem_ids: np.ndarray  # [P] global problem index

    @property
    def P(self):
        return int(self.seeds.shape[0])

    @property
    def S(self):
        return int(self.seeds.shape[1])

    @property
    def H(self):
        return 1 if self.seeds.ndim == 3 else int(self.seeds.shape[2])

    def evals_per_solve(self) -> int:
        """P*S*(A*H*iters + H): every candidate evaluation of every seed (§8(d) unit)."""
        A = len(self.solver.alpha)
        return self.P * self.S * (A * self.H * self.solver.iters + self.H)


class NativeKin:
    """FK and the self-collision check through the CUDA library (a helper context, empty world)."""

    def __init__(self, device: int, rb: inputs.Robot):
        from . import native
        self.device = device
        self.ctx = native.Context(device)
        self.ctx.set_robot(rb)
        self.ctx.set_world([inputs.World(np.zeros((0, 3)), np.zeros((0, 4)), np.zeros((0, 3)),
                                         np.zeros(0, np.int32))])
        self.ctx.set_cost_params(inputs.CostParams(flags=0))

    def fk(self, q):
        import torch
        qt = torch.tensor(np.ascontiguousarray(q, np.float32), device=f"cuda:{self.device}")
        sph, ee = self.ctx.fk(qt)
        torch.cuda.synchronize(self.device)
        return sph.cpu().numpy().astype(np.float64), ee.cpu().numpy().astype(np.float64)

    def self_free(self, q):
        import torch
        dev = f"cuda:{self.device}"
        qt = torch.tensor(np.ascontiguousarray(q, np.float32), device=dev)
        gl = torch.zeros(q.shape[0], 7, device=dev); gl[:, 3] = 1.0
        _, _, terms = self.ctx.evaluate(qt, gl, grad=False)
        torch.cuda.synchronize(self.device)
        return terms[:, 3].cpu().numpy() == 0.0

    def close(self):
        self.ctx.close()


def franka_to(device: int, problem_ids, S: int = 32, H: int = 32, n_boxes: int = 20, iters: int = 100,
              run_seed: int = 0, dense: bool = False, flags: int = inputs.SWEEP | inputs.SPEED,
              kin=None) -> Workload:
    """Configs 2 / 4 / 5: Franka TO, one scene per problem (tabletop K=20 or dense K=1000).
    `kin` supplies fk(q) -> (spheres, ee) and self_free(q) (default: the CUDA library)."""
    rb = robots.franka64()
    own = kin is None
    if own:
        kin = NativeKin(device, rb)
    worlds, starts, goals, seeds = [], [], [], []
    for p in problem_ids:
        s, qg = inputs.start_goal_configs(rb, run_seed, int(p), is_free=kin.self_free)
        sph, ee = kin.fk(np.stack([s, qg]))
        keep = sph.reshape(-1, 4)
        scene = inputs.dense_scene if dense else inputs.tabletop_scene
        worlds.append(scene(run_seed, int(p), n_boxes, keepout=keep))
        starts.append(s); goals.append(ee[1])
        seeds.append(inputs.to_seeds(rb, run_seed, int(p), s, qg, S, H))
    if own:
        kin.close()
    return Workload(name=("cfg5_franka_dense" if dense else "cfg2_franka_to"), robot=rb, worlds=worlds,
                    env=np.arange(len(problem_ids), dtype=np.int32), start=np.array(starts, np.float32),
                    goal=np.array(goals, np.float32), seeds=np.array(seeds, np.float32),
                    cost=inputs.CostParams(flags=flags, dt=0.25), solver=inputs.SolverParams(iters=iters),
                    problem_ids=np.asarray(problem_ids))


def franka_ik(device: int, problem_ids, S: int = 30, n_boxes: int = 20, iters: int = 100, run_seed: int = 0,
              kin=None) -> Workload:
    """Config 3: collision-free IK, goals = FK of configurations free in ONE shared scene (checked
    with the world term of the IK evaluation), Halton seeds offset by the goal index."""
    import torch
    from . import native
    rb = robots.franka64()
    world = inputs.tabletop_scene(run_seed, 10_000, n_boxes)
    own = kin is None
    if own:
        kin = NativeKin(device, rb)
    chk = native.Context(device)
    chk.set_robot(rb)
    chk.set_world([world])
    chk.set_cost_params(inputs.CostParams(flags=0))
    dev = f"cuda:{device}"
    qs = []
    for p in problem_ids:
        cand = inputs.uniform_configs(rb, run_seed, inputs.STREAM_IK, int(p), 64)
        gl = torch.zeros(64, 7, device=dev); gl[:, 3] = 1.0
        _, _, t = chk.evaluate(torch.tensor(cand, dtype=torch.float32, device=dev), gl, grad=False)
        t = t.cpu().numpy()
        ok = np.nonzero((t[:, 3] == 0.0) & (t[:, 4] == 0.0))[0]
        qs.append(cand[ok[0]] if len(ok) else cand[0])
    chk.close()
    _, ee = kin.fk(np.array(qs))
    if own:
        kin.close()
    seeds = np.stack([inputs.ik_seeds(rb, int(p), S) for p in problem_ids]).astype(np.float32)
    return Workload(name="cfg3_franka_ik", robot=rb, worlds=[world], env=np.zeros(len(problem_ids), np.int32),
                    start=None, goal=ee.astype(np.float32), seeds=seeds, cost=inputs.CostParams(flags=0),
                    solver=inputs.SolverParams(iters=iters), problem_ids=np.asarray(problem_ids))


def planar_to(problem_ids, S: int = 4, H: int = 16, iters: int = 25, run_seed: int = 0) -> Workload:
    """Config 1 (correctness config; goals are drawn as poses in the plane, no FK needed)."""
    rb = robots.planar2()
    g = inputs.rng(run_seed, inputs.STREAM_CONFIG, 0, 99)
    starts, goals, seeds = [], [], []
    for p in problem_ids:
        gp = inputs.rng(run_seed, inputs.STREAM_CONFIG, int(p), 0)
        s = gp.uniform(-2.5, 2.5, 2)
        r, a = gp.uniform(0.8, 1.9), gp.uniform(-np.pi, np.pi)
        goals.append([r * np.cos(a), r * np.sin(a), 0.0, 1.0, 0.0, 0.0, 0.0])
        starts.append(s)
        seeds.append(inputs.to_seeds(rb, run_seed, int(p), s, s + gp.normal(0, 0.8, 2), S, H))
    del g
    return Workload(name="cfg1_planar", robot=rb, worlds=[inputs.planar_scene()],
                    env=np.zeros(len(problem_ids), np.int32), start=np.array(starts, np.float32),
                    goal=np.array(goals, np.float32), seeds=np.array(seeds, np.float32),
                    cost=inputs.CostParams(dt=0.25), solver=inputs.SolverParams(iters=iters),
                    problem_ids=np.asarray(problem_ids))


def nominal_flops_per_eval(wl: Workload) -> float:
    """Algorithmic (nominal, data-independent) FP32 flops of one seed-timestep cost+grad eval,
    FMA = 2: the state terms, the FK chain (81 per actuated
    joint, fixed links folded), sphere transforms, the EE quaternion, every pair of S, a linear
    scan of every enabled box for every enabled sphere, the speed metric, the pose term shared by
    the H evals of a trajectory and the L-BFGS step shared by the A*H evals of an iteration.
    Data-dependent work (hits, sweep samples, backward chain terms) gets no credit."""
    rb = wl.robot
    D, M, H = rb.n_dof, rb.n_spheres, wl.H
    eff_r = rb.spheres[:, 3] + rb.sphere_offset
    pairs = sum(1 for i, j in rb.pairs if eff_r[i] > 0 and eff_r[j] > 0)
    m_en = int(np.sum(rb.spheres[:, 3] >= 0))
    K = np.mean([int(np.sum(w.enabled)) for w in wl.worlds]) if wl.worlds else 0
    n_act = int(np.sum(rb.jtype != 0))
    A, m = len(wl.solver.alpha), wl.solver.history
    N = H * D
    to = H > 1
    f = (80 if to else 10) * D + 81 * n_act + 18 * M + 40 + 9 * pairs + 26 * m_en * K
    if to and (wl.cost.flags & inputs.SPEED):
        f += 9 * m_en
    f += 80.0 / H
    f += (2 * N * (2 * m + 2) + 10 * N) / (A * H)
    return float(f)
