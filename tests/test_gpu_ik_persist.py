"""GPU: the persistent IK scheduling (crb_solver_params.persist) against
the one-CTA-per-group kernel.  Each seed's arithmetic does not depend on which CTA, lane or chunk
runs it, so every output is bitwise identical: flat groups (one shared environment), per-problem
groups (several environments), 1 to 5 iteration chunks (the solver state crosses global memory
between chunks), the particle warm-up in chunk 0, the solver trace, and a ragged last group."""
import dataclasses

import numpy as np
import pytest
import torch

from paper_2310_17274_b200 import inputs, workload

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda:0")
KEYS = ("seed_best_cost", "seed_best_traj", "best_cost", "best_traj", "best_key")


def T(x, dtype=torch.float32):
    return torch.tensor(np.ascontiguousarray(x), dtype=dtype, device=DEV)


@pytest.fixture(scope="module")
def native():
    from paper_2310_17274_b200 import native as N
    return N


def _ctx(native, wl, worlds=None):
    ctx = native.Context(0)
    ctx.set_robot(wl.robot)
    ctx.set_world(worlds if worlds is not None else wl.worlds)
    ctx.set_cost_params(wl.cost)
    return ctx


@pytest.mark.parametrize("particles", [0, 2])
def test_persistent_ik_bitwise_shared_env(native, particles):
    """One environment: flat 32-seed groups across problems (S = 30 leaves no lane idle except in
    the ragged last group), chunks 1..5, against persist = 0."""
    P, S = 23, 30    # 690 seeds = 21 full flat groups + 18 seeds
    wl = workload.franka_ik(0, list(range(P)), S=S, iters=17)
    sp = dataclasses.replace(wl.solver, particle_iters=particles, n_particles=16, cluster=0)
    ctx = _ctx(native, wl)
    args = (T(wl.seeds), T(wl.goal))
    kw = dict(env=T(wl.env, torch.int32), seed_outputs=True)
    ref = ctx.solve(dataclasses.replace(sp, persist=0), *args, **kw)
    assert torch.isfinite(ref["seed_best_cost"]).all()
    for chunks in (1, 2, 5):
        out = ctx.solve(dataclasses.replace(sp, persist=chunks), *args, **kw)
        for k in KEYS:
            assert torch.equal(ref[k], out[k]), (chunks, k)
    # env = NULL is the shared environment 0 as well
    out = ctx.solve(dataclasses.replace(sp, persist=3), *args, seed_outputs=True)
    for k in KEYS:
        assert torch.equal(ref[k], out[k]), ("env NULL", k)
    ctx.close()


def test_persistent_ik_bitwise_several_envs(native):
    """Several environments: per-problem groups (S = 40: a full and a ragged group per problem),
    the CTA re-stages the cuboid table when its next unit has another environment."""
    P, S = 12, 40
    wl = workload.franka_ik(0, list(range(P)), S=30, iters=13)
    rb = wl.robot
    seeds = np.stack([inputs.ik_seeds(rb, p, S) for p in range(P)]).astype(np.float32)
    worlds = [inputs.tabletop_scene(0, 10_000 + e, 20) for e in range(3)]
    env = (np.arange(P) % 3).astype(np.int32)
    ctx = _ctx(native, wl, worlds)
    sp = dataclasses.replace(wl.solver, cluster=0)
    args = (T(seeds), T(wl.goal))
    kw = dict(env=T(env, torch.int32), seed_outputs=True)
    ref = ctx.solve(dataclasses.replace(sp, persist=0), *args, **kw)
    for chunks in (1, 4):
        out = ctx.solve(dataclasses.replace(sp, persist=chunks), *args, **kw)
        for k in KEYS:
            assert torch.equal(ref[k], out[k]), (chunks, k)
    ctx.close()


def test_persistent_ik_trace_and_repeat(native):
    """The solver trace records are the same in both schedules; repeated persistent solves reuse
    the context's state buffer and flags (re-initialised per solve)."""
    P, S = 9, 30
    wl = workload.franka_ik(0, list(range(P)), S=S, iters=12)
    ctx = _ctx(native, wl)
    sp = dataclasses.replace(wl.solver, cluster=0)
    args = (T(wl.seeds), T(wl.goal))
    kw = dict(env=T(wl.env, torch.int32), seed_outputs=True, trace_iters=(0, 3, 7, 11))
    ref = ctx.solve(dataclasses.replace(sp, persist=0), *args, **kw)
    for _ in range(2):
        out = ctx.solve(dataclasses.replace(sp, persist=4), *args, **kw)
        for k in KEYS + ("trace",):
            assert torch.equal(ref[k], out[k]), k
    ctx.close()
