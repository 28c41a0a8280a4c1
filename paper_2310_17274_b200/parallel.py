"""Multi-GPU sharding of the solve; one process per GPU, torch.distributed plumbing.

* Problem sharding (configs 2/4): rank r owns a contiguous block of problems with all their seeds;
  the per-problem argmin is local and there is NO collective on the data path (weak scaling).
* Seed sharding (config 5, or one problem on n GPUs): rank r owns seeds [r*S/n, (r+1)*S/n) of every
  problem.  The exchange step is real: C1 = all_reduce(MIN) of the packed (cost bits << 32 | global
  seed) int64 keys the solve kernel emits, C2 = all_gather of the per-rank winning trajectories;
  every rank then takes the trajectory of the rank that owns the winning global seed.  Keys are
  exact integers and per-seed results are CTA-local, so the winner is bit-identical for any GPU
  count.

Both collectives run once per solve, never inside the iteration loop.
"""
from __future__ import annotations

from typing import Tuple

import torch
import torch.distributed as dist


def problem_block(P_total: int, world: int, rank: int) -> Tuple[int, int]:
    """Contiguous problem block [lo, hi) of `rank`; remainders go to the first ranks."""
    base, rem = divmod(P_total, world)
    lo = rank * base + min(rank, rem)
    return lo, lo + base + (1 if rank < rem else 0)


def seed_block(S_total: int, world: int, rank: int) -> Tuple[int, int]:
    """Seeds [lo, hi) of `rank` (requires S_total % world == 0 so ownership is arithmetic)."""
    if S_total % world != 0:
        raise ValueError(f"seed sharding needs S ({S_total}) divisible by the world size ({world})")
    s = S_total // world
    return rank * s, (rank + 1) * s


def _all_gather(t: torch.Tensor, world: int) -> torch.Tensor:
    out = torch.empty((world,) + tuple(t.shape), dtype=t.dtype, device=t.device)
    if dist.get_backend() == "nccl":
        dist.all_gather_into_tensor(out, t.contiguous())
    else:
        dist.all_gather(list(out.unbind(0)), t.contiguous())
    return out


def merge_seed_sharded(best_key: torch.Tensor, best_traj: torch.Tensor, S_total: int):
    """C1 + C2: global per-problem winner from per-rank (key, trajectory) pairs.

    best_key [P] int64 with low 32 bits = GLOBAL seed index (the solve's global_seed_base = this
    rank's first seed); best_traj [P, ...].  Returns (global_key [P], global_traj [P, ...], cost [P])."""
    world = dist.get_world_size()
    key = best_key.clone()
    dist.all_reduce(key, op=dist.ReduceOp.MIN)                    # C1
    trajs = _all_gather(best_traj, world)                          # C2
    seed = key & 0xFFFFFFFF
    owner = (seed // (S_total // world)).long()
    P = best_key.shape[0]
    out = trajs[owner, torch.arange(P, device=best_traj.device)]
    # the winner's cost straight from the key's high word (device-side bit cast, no host round
    # trip): costs are >= 0 and NaN maps to the +inf bits, so the word is < 2^31
    cost = (key >> 32).to(torch.int32).view(torch.float32)
    return key, out, cost


def max_over_ranks(x: float, device) -> float:
    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(x: float, device) -> float:
    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())
