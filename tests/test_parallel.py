"""Host-side multi-GPU logic (parallel.py) on CPU with the gloo backend, world size 2: problem /
seed blocks, and the seed-sharded exchange C1 (all_reduce MIN of packed keys) + C2 (all_gather of
winners) giving the same winner as a single-process argmin over all seeds."""
import os
import socket
import struct

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2310_17274_b200 import parallel


def _key(c, seed):
    bits = 0x7F800000 if c != c else (0 if c == 0 else struct.unpack("<I", struct.pack("<f", np.float32(c)))[0])
    return (bits << 32) | seed


def test_blocks():
    for P in (1, 7, 64, 1024):
        for w in (1, 2, 3, 8):
            spans = [parallel.problem_block(P, w, r) for r in range(w)]
            assert spans[0][0] == 0 and spans[-1][1] == P
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            assert max(h - l for l, h in spans) - min(h - l for l, h in spans) <= 1
    assert parallel.seed_block(32, 4, 3) == (24, 32)
    with pytest.raises(ValueError):
        parallel.seed_block(12, 8, 0)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, costs, trajs, S, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lo, hi = parallel.seed_block(S, world, rank)
    P = costs.shape[0]
    # what this rank's solve would emit: local argmin with keys carrying GLOBAL seed indices
    keys = torch.empty(P, dtype=torch.int64)
    best = torch.empty((P,) + trajs.shape[2:])
    for p in range(P):
        ks = [_key(float(costs[p, s]), s) for s in range(lo, hi)]
        i = int(np.argmin(ks))
        keys[p] = ks[i]
        best[p] = torch.from_numpy(trajs[p, lo + i])
    gkey, gtraj, gcost = parallel.merge_seed_sharded(keys, best, S)
    out[rank] = (gkey.numpy().copy(), gtraj.numpy().copy(), gcost.numpy().copy())
    t = parallel.max_over_ranks(float(rank + 1), torch.device("cpu"))
    assert t == world
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_seed_sharded_merge_matches_single_process(world):
    rng = np.random.default_rng(0)
    P, S = 9, 8
    costs = rng.uniform(0, 10, (P, S)).astype(np.float32)
    costs[0, 2] = costs[0, 5] = 0.01   # minimal tie across ranks -> lowest global seed (2)
    costs[1, :] = np.nan               # all NaN -> seed 0
    costs[2, 6] = np.nan
    trajs = rng.normal(size=(P, S, 4, 3)).astype(np.float32)
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), costs, trajs, S, out), nprocs=world, join=True)
    for p in range(P):
        ks = [_key(float(costs[p, s]), s) for s in range(S)]
        i = int(np.argmin(ks))
        for r in range(world):
            gkey, gtraj, gcost = out[r]
            assert gkey[p] == ks[i]
            np.testing.assert_array_equal(gtraj[p], trajs[p, i])
            if np.isfinite(costs[p, i]):
                assert gcost[p] == costs[p, i]
    assert out[0][0][0] & 0xFFFFFFFF == 2
    assert out[0][0][1] & 0xFFFFFFFF == 0
