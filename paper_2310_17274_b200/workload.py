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


def _fk_np(ctx, q):
    import torch
    qt = torch.tensor(np.ascontiguousarray(q, np.float32), device=f"cuda:{ctx.device}")
    sph, ee = ctx.fk(qt)
    torch.cuda.synchronize(ctx.device)
    return sph.cpu().numpy().astype(np.float64), ee.cpu().numpy().astype(np.float64)


def _self_free(ctx_empty, q):
    import torch
    dev = f"cuda:{ctx_empty.device}"
    qt = torch.tensor(np.ascontiguousarray(q, np.float32), device=dev)
    gl = torch.zeros(q.shape[0], 7, device=dev); gl[:, 3] = 1.0
    _, _, terms = ctx_empty.evaluate(qt, gl, grad=False)
    torch.cuda.synchronize(ctx_empty.device)
    return terms[:, 3].cpu().numpy() == 0.0


def franka_to(device: int, problem_ids, S: int = 32, H: int = 32, n_boxes: int = 20, iters: int = 100,
              run_seed: int = 0, dense: bool = False, flags: int = inputs.SWEEP | inputs.SPEED) -> Workload:
    """Configs 2 / 4 / 5: Franka TO, one scene per problem (tabletop K=20 or dense K=1000)."""
    from . import native
    rb = robots.franka64()
    helper = native.Context(device)
    helper.set_robot(rb)
    helper.set_world([inputs.World(np.zeros((0, 3)), np.zeros((0, 4)), np.zeros((0, 3)), np.zeros(0, np.int32))])
    helper.set_cost_params(inputs.CostParams(flags=0))
    worlds, starts, goals, seeds = [], [], [], []
    for p in problem_ids:
        s, qg = inputs.start_goal_configs(rb, run_seed, int(p), is_free=lambda q: _self_free(helper, q))
        sph, ee = _fk_np(helper, np.stack([s, qg]))
        keep = sph.reshape(-1, 4)
        scene = inputs.dense_scene if dense else inputs.tabletop_scene
        worlds.append(scene(run_seed, int(p), n_boxes, keepout=keep))
        starts.append(s); goals.append(ee[1])
        seeds.append(inputs.to_seeds(rb, run_seed, int(p), s, qg, S, H))
    helper.close()
    return Workload(name=("cfg5_franka_dense" if dense else "cfg2_franka_to"), robot=rb, worlds=worlds,
                    env=np.arange(len(problem_ids), dtype=np.int32), start=np.array(starts, np.float32),
                    goal=np.array(goals, np.float32), seeds=np.array(seeds, np.float32),
                    cost=inputs.CostParams(flags=flags, dt=0.25), solver=inputs.SolverParams(iters=iters),
                    problem_ids=np.asarray(problem_ids))


def franka_ik(device: int, problem_ids, S: int = 30, n_boxes: int = 20, iters: int = 100, run_seed: int = 0) -> Workload:
    """Config 3: collision-free IK, goals = FK of free random configurations in ONE shared scene,
    Halton seeds offset by the goal index."""
    from . import native
    rb = robots.franka64()
    helper = native.Context(device)
    helper.set_robot(rb)
    world = inputs.tabletop_scene(run_seed, 10_000, n_boxes)
    helper.set_world([world])
    helper.set_cost_params(inputs.CostParams(flags=0))
    qs = []
    for p in problem_ids:
        k = 0
        while True:
            q = inputs.uniform_configs(rb, run_seed, inputs.STREAM_IK, int(p) * 64 + k, 1)[0]
            import torch
            dev = f"cuda:{device}"
            gl = torch.zeros(1, 7, device=dev); gl[:, 3] = 1.0
            _, _, t = helper.evaluate(torch.tensor(q[None], dtype=torch.float32, device=dev), gl, grad=False)
            t = t.cpu().numpy()[0]
            if t[3] == 0.0 and t[4] == 0.0:
                break
            k += 1
        qs.append(q)
    _, ee = _fk_np(helper, np.array(qs))
    helper.close()
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
