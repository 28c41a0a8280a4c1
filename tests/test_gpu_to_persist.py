"""GPU: the persistent chunked TO schedule (crb_solver_params.persist)
against one CTA per seed trajectory: every output bitwise identical -- several environments
(re-staged per unit), 1 to 5 iteration chunks (the seed's solver state crosses global memory
between chunks), the particle warm-up in chunk 0, the chunked convergence exit (a seed that
stopped stays stopped in later chunks), the solver trace, and H = 44 (timestep windows)."""
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


def _solve_all(native, wl, sp, variants, **extra):
    ctx = native.Context(0)
    ctx.set_robot(wl.robot)
    ctx.set_world(wl.worlds)
    ctx.set_cost_params(wl.cost)
    args = (T(wl.seeds), T(wl.goal))
    kw = dict(start=T(wl.start), env=T(wl.env, torch.int32), seed_outputs=True, **extra)
    outs = [ctx.solve(dataclasses.replace(sp, cluster=0, persist=v), *args, **kw) for v in variants]
    ctx.close()
    return outs


@pytest.mark.parametrize("particles,check_every", [(0, 0), (2, 0), (0, 4)])
def test_persistent_to_bitwise(native, particles, check_every):
    wl = workload.franka_to(0, list(range(5)), S=7, H=32, iters=17)
    sp = dataclasses.replace(wl.solver, particle_iters=particles, n_particles=8, check_every=check_every,
                             conv_rtol=0.05 if check_every else 0.0)
    outs = _solve_all(native, wl, sp, [0, 1, 2, 5])
    assert torch.isfinite(outs[0]["seed_best_cost"]).all()
    for o in outs[1:]:
        for k in KEYS:
            assert torch.equal(outs[0][k], o[k]), k


def test_persistent_to_trace_and_long_horizon(native):
    wl = workload.franka_to(0, list(range(3)), S=4, H=32, iters=12)
    sp = wl.solver
    outs = _solve_all(native, wl, sp, [0, 3], trace_iters=(0, 5, 11))
    for k in KEYS + ("trace",):
        assert torch.equal(outs[0][k], outs[1][k]), k
    wl44 = workload.franka_to(0, list(range(3)), S=4, H=44, iters=9)
    outs = _solve_all(native, wl44, wl44.solver, [0, 2])
    for k in KEYS:
        assert torch.equal(outs[0][k], outs[1][k]), ("H=44", k)


def test_persistent_degenerate(native):
    """iters = 0 and iters < chunks (the chunk count clamps to iters), a single seed, and a batch
    smaller than one wave: outputs equal one CTA per seed / group."""
    wl = workload.franka_to(0, list(range(2)), S=3, H=16, iters=5)
    for iters, chunks in ((0, 3), (2, 5), (5, 9)):
        sp = dataclasses.replace(wl.solver, iters=iters)
        outs = _solve_all(native, wl, sp, [0, chunks])
        for k in KEYS:
            assert torch.equal(outs[0][k], outs[1][k]), (iters, chunks, k)
    ik = workload.franka_ik(0, [3], S=1, iters=4)
    ctx = native.Context(0)
    ctx.set_robot(ik.robot); ctx.set_world(ik.worlds); ctx.set_cost_params(ik.cost)
    a = ctx.solve(dataclasses.replace(ik.solver, persist=0), T(ik.seeds), T(ik.goal), seed_outputs=True)
    b = ctx.solve(dataclasses.replace(ik.solver, persist=7), T(ik.seeds), T(ik.goal), seed_outputs=True)
    for k in ("seed_best_cost", "seed_best_traj", "best_cost", "best_traj"):
        assert torch.equal(a[k], b[k]), ("IK", k)
    ctx.close()


def test_persistent_large_world_build_bitwise(native):
    """The large-world (GMEM) build -- cuboid table in global memory, slow-path entries batched
    across cuboids and work items -- under the persistent schedule: every output
    bitwise equal to one CTA per seed, and, on the small environments, to the shared-memory build
    (one round per flagged cuboid).  A dense 1000-cuboid environment is in the list, so the context
    runs the GMEM kernels for every environment."""
    wl = workload.franka_to(0, list(range(6)), S=8, H=32, iters=12)
    dense = workload.franka_to(0, [0], S=8, H=32, n_boxes=1000, iters=12, dense=True)
    big = dataclasses.replace(wl, worlds=list(wl.worlds) + list(dense.worlds))
    assert max(w.n_boxes for w in big.worlds) >= 1000
    env = np.array(wl.env, np.int32)
    env[-2:] = len(big.worlds) - 1                      # two problems in the dense world
    big = dataclasses.replace(big, env=env)
    sp = wl.solver
    outs = _solve_all(native, big, sp, [0, 1, 3])
    for o in outs[1:]:
        for k in KEYS:
            assert torch.equal(outs[0][k], o[k]), ("persist", k)
    assert torch.isfinite(outs[0]["seed_best_cost"]).all()
    small = _solve_all(native, wl, sp, [0])[0]        # shared-memory build on the small worlds
    for k in ("seed_best_cost", "seed_best_traj"):    # problems 0..3 keep their small environments
        a, b = outs[0][k].reshape(6, 8, -1)[:4], small[k].reshape(6, 8, -1)[:4]
        assert torch.equal(a, b), ("builds", k)
