#!/usr/bin/env python
"""Benchmark of the B200 hot path: batched per-seed L-BFGS trajectory optimisation (BASELINE.json
configs[1], Franka 7-DoF, 64 spheres, 20 cuboids, 32 seeds x 32 timesteps, 100 iterations),
P problems per GPU (weak scaling over GPUs, problem-sharded, no data-path collective).

One step = one crb_lbfgs_solve over the whole per-GPU batch: every candidate evaluation of every
seed (a1..a15 of SURVEY §8(a)).  value = seed-timestep cost+grad evals/s over all ranks, timed on
the device with CUDA events around each solve (L2 flushed between steps, outside the events),
max over ranks.  e2e = the same metric through crb_lbfgs_solve_host with pinned host buffers
(H2D of seeds/starts/goals, solve, D2H of the winners, synchronise) timed by the host clock.

--impl reference times the fp64 CPU oracle (oracle/, the correctness reference of this repo) on a
bounded sample of the same workload on the host cores.
"""
from __future__ import annotations

import argparse
import dataclasses
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "seed-timestep cost+grad evals/s"
UNIT = "evals/s"
FP32_LANES_PER_SM, SMS = 128, 148


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="native", choices=["native", "reference"])
    ap.add_argument("--problems", type=int, default=64, help="problems per GPU (32 seeds each)")
    ap.add_argument("--iters", type=int, default=100)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-extras", action="store_true", help="skip the config-3 (IK) and config-5 (dense) side metrics")
    ap.add_argument("--shard", default="problem", choices=["problem", "seed"],
                    help="problem: each rank owns its own problems (weak scaling, no collective); seed: every rank "
                         "solves its seed block of the SAME problems, then C1 all_reduce(MIN) of packed keys + C2 "
                         "all_gather of winners (strong scaling)")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def pipes_summary():
    """Issued-instruction roofline per pipe of the dominant kernel from the committed ncu capture
    (profiles/r02_pipes.json, tools/pipes_from_ncu.py; an ncu number, never re-measured here)."""
    path = os.path.join(ROOT, "profiles", "r02_pipes.json")
    try:
        return json.load(open(path))
    except Exception:
        return None


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        return json.load(open(path))
    except Exception:
        return {}


class ClockSampler:
    """SM clock + throttle reasons polled through NVML every 10 ms during the timed region (the
    recipe's clocks line; nvidia-smi -lms as a fallback when NVML is unavailable)."""
    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "sw_power_cap": 0x4}

    def __init__(self, device):
        self.device = device
        self.sm, self.mx, self.reasons = [], [], set()
        self.stop = threading.Event()
        self.th = None
        self.h = None
        try:   # NVML set up before the timed region, so polling starts at once
            import pynvml
            pynvml.nvmlInit()
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device)
        except Exception:
            self.h = None

    def _poll_nvml(self):
        import pynvml
        if self.h is None:
            raise RuntimeError("no NVML")
        h = self.h
        self.mx.append(float(pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)))
        while not self.stop.is_set():
            self.sm.append(float(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)))
            r = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
            for n, bit in self.REASONS.items():
                if r & bit:
                    self.reasons.add(n)
            time.sleep(0.01)

    def _poll_smi(self):
        fields = ["clocks.sm", "clocks.max.sm", "clocks_event_reasons.hw_slowdown",
                  "clocks_event_reasons.hw_thermal_slowdown", "clocks_event_reasons.sw_thermal_slowdown",
                  "clocks_event_reasons.sw_power_cap"]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), "--query-gpu=" + ",".join(fields),
                                 "--format=csv,noheader,nounits", "-lms", "50"],
                                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        threading.Thread(target=lambda: (self.stop.wait(), proc.terminate()), daemon=True).start()
        for ln in proc.stdout:
            parts = [p.strip() for p in ln.split(",")]
            try:
                self.sm.append(float(parts[0])); self.mx.append(float(parts[1]))
            except (ValueError, IndexError):
                continue
            for n, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    self.reasons.add(n)

    def _run(self):
        try:
            self._poll_nvml()
        except Exception:
            try:
                self._poll_smi()
            except Exception:
                pass

    def __enter__(self):
        self.th = threading.Thread(target=self._run, daemon=True)
        self.th.start()
        time.sleep(0.02)
        return self

    def __exit__(self, *a):
        self.stop.set()
        self.th.join(3)

    def summary(self):
        if not self.sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        return {"sm_mhz": statistics.median(self.sm), "sm_min_mhz": min(self.sm),
                "sm_max_mhz": max(self.mx) if self.mx else None, "reasons": sorted(self.reasons),
                "samples": len(self.sm)}


def oracle_sample_rate(wl, problem: int, iters: int, nthreads: int):
    """Time the fp64 oracle (as it stands) on problem `problem` of the workload: S seeds x iters."""
    from oracle import oracle as O
    from paper_2310_17274_b200 import inputs
    R = O.Robot(wl.robot)
    W = O.World(wl.worlds[wl.env[problem]])
    sp = inputs.SolverParams(iters=iters, history=wl.solver.history, alpha=wl.solver.alpha, c1=wl.solver.c1,
                             c2=wl.solver.c2, ls_mode=wl.solver.ls_mode)
    seeds = wl.seeds[problem:problem + 1].astype(np.float64)
    t0 = time.perf_counter()
    if wl.H > 1:
        O.solve_to(R, [W], np.zeros(1, np.int32), wl.cost, sp, seeds, wl.start[problem:problem + 1].astype(np.float64),
                   wl.goal[problem:problem + 1].astype(np.float64), nthreads=nthreads)
    else:
        O.solve_ik(R, [W], np.zeros(1, np.int32), wl.cost, sp, seeds, wl.goal[problem:problem + 1].astype(np.float64),
                   nthreads=nthreads)
    dt = time.perf_counter() - t0
    A = len(sp.alpha)
    evals = wl.S * (A * wl.H * iters + wl.H)
    return evals / dt, dt, evals


def cpu_model() -> str:
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_baseline(wl, target_s: float = 12.0, target_1t_s: float = 4.0):
    """Oracle on the host cores, bounded sample of problem 0 (about target_s seconds on all host
    threads, and about target_1t_s on one thread)."""
    nthreads = os.cpu_count() or 1
    rate1, dt1, _ = oracle_sample_rate(wl, 0, 1, nthreads)
    per_iter = dt1 / 1.0
    iters = int(max(1, min(wl.solver.iters, target_s / max(per_iter, 1e-3))))
    rate, dt, evals = oracle_sample_rate(wl, 0, iters, nthreads)
    _, d1, _ = oracle_sample_rate(wl, 0, 1, 1)
    it1 = int(max(1, min(wl.solver.iters, target_1t_s / max(d1, 1e-3))))
    r1, t1, e1 = oracle_sample_rate(wl, 0, it1, 1)
    return {"value": rate, "unit": UNIT, "cores": nthreads, "kind": "oracle",
            "sample": f"problem 0 of {wl.name}: {wl.S} seeds x {iters} L-BFGS iterations ({evals} evals, {dt:.1f} s, "
                      f"fp64 C oracle, {nthreads} threads)",
            "cpu_model": cpu_model(), "host_threads": nthreads,
            "single_thread": {"value": r1, "unit": UNIT, "cores": 1,
                              "sample": f"problem 0: {wl.S} seeds x {it1} iterations ({e1} evals, {t1:.1f} s, 1 thread)"}}


def run_reference(args):
    rank, world, local = dist_env()
    if rank != 0:
        return
    from oracle import oracle as O
    from paper_2310_17274_b200 import robots, workload

    class OracleKin:
        def __init__(self):
            self.R = O.Robot(robots.franka64())

        def fk(self, q):
            out = [O.fk(self.R, x) for x in q]
            return np.array([o[1] for o in out]), np.array([o[2] for o in out])

        def self_free(self, q):
            return np.array([O.self_collision(self.R, O.fk(self.R, x)[1], 1.0)[0] == 0.0 for x in q])

    wl = workload.franka_to(0, [0], S=32, H=32, iters=args.iters, kin=OracleKin())
    nthreads = os.cpu_count() or 1
    _, dt1, _ = oracle_sample_rate(wl, 0, 1, nthreads)
    # each step a bounded sample: ~ 150 s / (steps + warmup) of oracle work in total
    budget = 150.0 / max(1, args.steps + args.warmup)
    iters = int(max(1, min(args.iters, budget / max(dt1, 1e-3))))
    for _ in range(args.warmup):
        oracle_sample_rate(wl, 0, iters, nthreads)
    times, evals = [], 0
    for _ in range(args.steps):
        r, dt, ev = oracle_sample_rate(wl, 0, iters, nthreads)
        times.append(dt); evals += ev
    value = evals / sum(times)
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * sum(times) / len(times),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "cfg2_franka_to_batched", "sample_of_step": "problem 0 of the 64-problem step",
                       "problems_per_step": 1, "seeds": 32, "timesteps": 32, "iters_per_step": iters, "boxes": 20,
                       "spheres": 64, "dof": 7, "flags": "sweep+speed"},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": nthreads, "kind": "oracle",
                             "sample": f"1 problem x 32 seeds x {iters} iterations per step (fp64 C oracle)"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def _timed_solves(ctx, sp, seeds, goal, start, env, steps, flush, world, dev):
    import torch
    import torch.distributed as dist
    from paper_2310_17274_b200 import parallel
    ctx.solve(sp, seeds, goal, start=start, env=env)          # warm-up
    torch.cuda.synchronize()
    tot = 0.0
    for _ in range(steps):
        flush.zero_()
        if world > 1:
            dist.barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        ctx.solve(sp, seeds, goal, start=start, env=env)
        b.record()
        torch.cuda.synchronize()
        tot += a.elapsed_time(b)
    if world > 1:
        tot = parallel.max_over_ranks(tot, dev)
    return tot / steps


def motion_gen_metrics(local, rank, world, dev, steps):
    """Device-timed (CUDA events around the whole pipeline call, host launches included) motion
    generation: P = 64 problems per GPU in one batch, and P = 1 (latency)."""
    import torch
    import torch.distributed as dist
    from paper_2310_17274_b200 import motion_gen, native, parallel, workload
    res = {}
    for P in (64,):
        lo = rank * P
        wl = workload.franka_to(local, list(range(lo, lo + P)), S=12, H=32, iters=100)
        ctx = native.Context(local)
        ctx.set_robot(wl.robot); ctx.set_world(wl.worlds); ctx.set_cost_params(wl.cost)
        mg = motion_gen.MotionGen(ctx, wl.robot, wl.cost)
        args = (torch.tensor(wl.start, device=dev), torch.tensor(wl.goal, device=dev),
                torch.tensor(wl.env, device=dev), torch.tensor(mg.ik_seed_batch(wl.robot, range(lo, lo + P), 32),
                                                               device=dev))
        mg.plan(*args)
        torch.cuda.synchronize()
        tot, succ = 0.0, 0
        for _ in range(steps):
            if world > 1:
                dist.barrier()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            out = mg.plan(*args)
            b.record()
            torch.cuda.synchronize()
            tot += a.elapsed_time(b)
            succ = int(out["success"].sum().item())
        ms = tot / steps
        if world > 1:
            ms = parallel.max_over_ranks(ms, dev)
        # up to 3 attempts, failed problems re-planned with fresh seeds
        tot3, succ3 = 0.0, 0
        for _ in range(steps):
            if world > 1:
                dist.barrier()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            out = mg.plan_retry(*args[:3], range(lo, lo + P), attempts=3)
            b.record()
            torch.cuda.synchronize()
            tot3 += a.elapsed_time(b)
            succ3 = int(out["success"].sum().item())
        ms3 = tot3 / steps
        if world > 1:
            ms3 = parallel.max_over_ranks(ms3, dev)
        res[f"P{P}"] = {"problems_per_gpu": P, "ms_per_batch": ms, "problems_per_s": P * world / (ms * 1e-3),
                        "success": succ, "ik_seeds": 32, "to_seeds": 12, "timesteps": 32,
                        "iters": "IK 2p+100, TO 2p+100, refine 300",
                        "up_to_3_attempts": {"ms_per_batch": ms3, "problems_per_s": P * world / (ms3 * 1e-3),
                                             "success": succ3}}
        ctx.close()
    # single-problem latency (the paper's ~50 ms mean) over 16 different problems, each
    # planned alone (batch 1, the cluster latency mode), with its success
    n1 = 16
    lo = rank * n1
    wl = workload.franka_to(local, list(range(lo, lo + n1)), S=12, H=32, iters=100)
    ctx = native.Context(local)
    ctx.set_robot(wl.robot); ctx.set_world(wl.worlds); ctx.set_cost_params(wl.cost)
    mg = motion_gen.MotionGen(ctx, wl.robot, wl.cost)
    st_all, gl_all = torch.tensor(wl.start, device=dev), torch.tensor(wl.goal, device=dev)
    env_all = torch.tensor(wl.env, device=dev)
    iks = torch.tensor(mg.ik_seed_batch(wl.robot, range(lo, lo + n1), 32), device=dev)
    one = lambda k: (st_all[k:k + 1], gl_all[k:k + 1], env_all[k:k + 1], iks[k:k + 1])
    mg.plan(*one(0))
    torch.cuda.synchronize()
    lat, oks, lat3, ok3 = [], [], [], 0
    for k in range(n1):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        o = mg.plan(*one(k))
        b.record()
        torch.cuda.synchronize()
        lat.append(a.elapsed_time(b))
        oks.append(bool(o["success"].item()))
        a.record()
        o3 = mg.plan_retry(*one(k)[:3], [lo + k], attempts=3)
        b.record()
        torch.cuda.synchronize()
        lat3.append(a.elapsed_time(b))
        ok3 += int(o3["success"].item())
    ctx.close()
    ok = sum(oks)
    res["P1"] = {"problems": n1, "each_planned_alone": True, "median_ms": statistics.median(lat),
                 "p90_ms": float(np.quantile(lat, 0.9)), "success": ok,
                 "median_ms_successful": statistics.median([t for t, s in zip(lat, oks) if s]) if ok else None,
                 "up_to_3_attempts": {"median_ms": statistics.median(lat3), "p90_ms": float(np.quantile(lat3, 0.9)),
                                      "success": ok3}}
    return res


def side_metrics(local, rank, world, dev, flush, steps=2):
    """The other metrics of BASELINE.json on their own configs (device-timed, max over ranks):
    config 3 -- collision-free IK, 1000 goals x 30 Halton seeds, 100 iterations, one shared K = 20
    scene (IK queries/s = goals / solve time); config 5 sample -- Franka vs K = 1000 dense cuboids,
    swept + speed, 16 problems x 32 seeds x 32 timesteps x 100 iterations per GPU."""
    import torch
    from paper_2310_17274_b200 import native, workload
    out = {}
    n_ik = 1000
    lo = rank * n_ik
    wl = workload.franka_ik(local, list(range(lo, lo + n_ik)), S=30, iters=100)
    ctx = native.Context(local)
    ctx.set_robot(wl.robot); ctx.set_world(wl.worlds); ctx.set_cost_params(wl.cost)
    ms = _timed_solves(ctx, wl.solver, torch.tensor(wl.seeds, device=dev), torch.tensor(wl.goal, device=dev), None,
                       torch.tensor(wl.env, device=dev), steps, flush, world, dev)
    out["cfg3_ik"] = {"goals_per_gpu": n_ik, "seeds": 30, "iters": 100, "ms_per_solve": ms,
                      "ik_queries_per_s": n_ik * world / (ms * 1e-3),
                      "evals_per_s": wl.evals_per_solve() * world / (ms * 1e-3),
                      "ctas_per_sm": ctx.solver_occupancy(1)[0]}
    # f1: the paper's IK pipeline = 2 particle iterations, then L-BFGS
    spp = dataclasses.replace(wl.solver, particle_iters=2, n_particles=64)
    msp = _timed_solves(ctx, spp, torch.tensor(wl.seeds, device=dev), torch.tensor(wl.goal, device=dev), None,
                        torch.tensor(wl.env, device=dev), steps, flush, world, dev)
    out["cfg3_ik"]["with_particles"] = {"particle_iters": 2, "n_particles": 64, "ms_per_solve": msp,
                                        "ik_queries_per_s": n_ik * world / (msp * 1e-3),
                                        "added_ms": msp - ms}
    # single-query latency (batch size 1, "2.7ms"): the cluster latency mode runs it
    one = (torch.tensor(wl.seeds[:1], device=dev), torch.tensor(wl.goal[:1], device=dev), None,
           torch.tensor(wl.env[:1], device=dev))
    out["cfg3_ik"]["single_query_ms"] = _timed_solves(ctx, wl.solver, *one, steps, flush, 1, dev)
    out["cfg3_ik"]["single_query_ms_with_particles"] = _timed_solves(ctx, spp, *one, steps, flush, 1, dev)
    ctx.close()
    # f1 on the headline TO workload (config 2 shape): 2 x 64 cost-only particle passes per seed
    # before the same 100 L-BFGS iterations; the paper reports +2 ms for this warm-up
    n_f1 = 64
    lo = rank * n_f1
    wl = workload.franka_to(local, list(range(lo, lo + n_f1)), S=32, H=32, iters=100)
    ctx = native.Context(local)
    ctx.set_robot(wl.robot); ctx.set_world(wl.worlds); ctx.set_cost_params(wl.cost)
    args_ = (torch.tensor(wl.seeds, device=dev), torch.tensor(wl.goal, device=dev),
             torch.tensor(wl.start, device=dev), torch.tensor(wl.env, device=dev))
    ms0 = _timed_solves(ctx, wl.solver, *args_, steps, flush, world, dev)
    # config 2 single-problem latency: one problem (32 seeds x 32 timesteps x 100 iterations) per
    # call, batch 1 (the cluster latency mode), median over 8 different problems, device-timed
    lat = []
    for p in range(8):
        one = tuple(t[p:p + 1] for t in args_)
        lat.append(_timed_solves(ctx, wl.solver, *one, max(1, min(steps, 3)), flush, 1, dev))
    out["cfg2_single_problem"] = {"problems": 8, "each_solved_alone": True, "seeds": 32, "timesteps": 32,
                                  "iters": 100, "median_ms": float(np.median(lat)), "max_ms": float(max(lat)),
                                  "evals_per_s_median": wl.evals_per_solve() / n_f1 / (float(np.median(lat)) * 1e-3)}
    spp = dataclasses.replace(wl.solver, particle_iters=2, n_particles=64)
    msp = _timed_solves(ctx, spp, *args_, steps, flush, world, dev)
    sp0 = dataclasses.replace(wl.solver, iters=0, particle_iters=2, n_particles=64)
    msw = _timed_solves(ctx, sp0, *args_, steps, flush, world, dev)
    n_part = n_f1 * 32 * 2 * 64 * 32     # cost-only seed-timestep evaluations of the warm-up
    out["f1_particle_to"] = {"problems_per_gpu": n_f1, "seeds": 32, "timesteps": 32, "particle_iters": 2,
                             "n_particles": 64, "ms_lbfgs_only": ms0, "ms_particle_plus_lbfgs": msp,
                             "added_ms": msp - ms0, "ms_warmup_only": msw,
                             "warmup_cost_only_evals_per_s": n_part * world / (msw * 1e-3),
                             "to_problems_per_s_with_particles": n_f1 * world / (msp * 1e-3)}
    ctx.close()
    # config 4: batched TO, 1024 problems x 12 seeds x 32 timesteps over 8 GPUs = 128 problems per
    # GPU, each with its own K = 20 scene, 100 iterations
    n4 = 128
    lo = rank * n4
    wl = workload.franka_to(local, list(range(lo, lo + n4)), S=12, H=32, iters=100)
    ctx = native.Context(local)
    ctx.set_robot(wl.robot); ctx.set_world(wl.worlds); ctx.set_cost_params(wl.cost)
    ms = _timed_solves(ctx, wl.solver, torch.tensor(wl.seeds, device=dev), torch.tensor(wl.goal, device=dev),
                       torch.tensor(wl.start, device=dev), torch.tensor(wl.env, device=dev), steps, flush, world, dev)
    out["cfg4_batched_to"] = {"problems_per_gpu": n4, "seeds": 12, "timesteps": 32, "iters": 100,
                              "ms_per_solve": ms, "problems_per_s": n4 * world / (ms * 1e-3),
                              "evals_per_s": wl.evals_per_solve() * world / (ms * 1e-3)}
    ctx.close()
    # f2: the whole motion-generation pipeline (IK -> seeds -> TO -> retime -> TO at dt_opt ->
    # retime -> success), batched and for one problem (the paper's ~50 ms figure)
    out["f2_motion_gen"] = motion_gen_metrics(local, rank, world, dev, steps)
    # config 5 at its stated size: 256 problems x 32 seeds x 32 timesteps x 100 iterations against
    # K = 1000 dense cuboids each, swept + speed, seed-sharded over the GPUs: each
    # rank solves its 32 / N seeds of all 256 problems, then C1 + C2 pick the winners
    from paper_2310_17274_b200 import parallel
    n_dense, S5 = 256, 32
    s_lo, s_hi = parallel.seed_block(S5, world, rank)
    wl = workload.franka_to(local, list(range(n_dense)), S=S5, H=32, n_boxes=1000, iters=100, dense=True)
    ctx = native.Context(local)
    ctx.set_robot(wl.robot); ctx.set_world(wl.worlds); ctx.set_cost_params(wl.cost)
    fl = workload.nominal_flops_per_eval(wl)
    seeds5 = torch.tensor(np.ascontiguousarray(wl.seeds[:, s_lo:s_hi]), device=dev)
    g5, st5, e5 = (torch.tensor(wl.goal, device=dev), torch.tensor(wl.start, device=dev),
                   torch.tensor(wl.env, device=dev))

    def solve5(sd, base):
        o = ctx.solve(wl.solver, sd, g5, start=st5, env=e5, seed_base=base)
        if world > 1:
            parallel.merge_seed_sharded(o["best_key"], o["best_traj"], S5)
    solve5(seeds5, s_lo)
    torch.cuda.synchronize()
    tot = 0.0
    for _ in range(steps):
        flush.zero_()
        if world > 1:
            torch.distributed.barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        solve5(seeds5, s_lo)
        b.record()
        torch.cuda.synchronize()
        tot += a.elapsed_time(b)
    ms = tot / steps
    if world > 1:
        ms = parallel.max_over_ranks(ms, dev)
    evals5 = n_dense * S5 * (len(wl.solver.alpha) * 32 * 100 + 32)
    out["cfg5_dense"] = {"problems": n_dense, "seeds": S5, "seeds_per_gpu": s_hi - s_lo, "timesteps": 32,
                         "boxes": 1000, "iters": 100, "sharding": f"seed-sharded x{world} (C1 + C2 inside the timing)",
                         "ms_per_solve": ms, "evals_per_s": evals5 / (ms * 1e-3),
                         "problems_per_s": n_dense / (ms * 1e-3), "flops_per_eval": fl,
                         "nominal_tflops_per_gpu": evals5 / world / (ms * 1e-3) * fl / 1e12,
                         "ctas_per_sm": ctx.solver_occupancy(32)[0]}
    # the per-GPU share of the 8-GPU run (256 problems x 4 seeds), timed alone on this GPU
    if world == 1:
        sd8 = torch.tensor(np.ascontiguousarray(wl.seeds[:, :S5 // 8]), device=dev)
        ms8 = _timed_solves(ctx, wl.solver, sd8, g5, st5, e5, steps, flush, 1, dev)
        out["cfg5_dense"]["share_of_8_gpus"] = {"seeds_per_gpu": S5 // 8, "ms_per_solve": ms8,
                                                "evals_per_s": evals5 / 8 / (ms8 * 1e-3)}
    ctx.close()
    return out


def run_native(args):
    import torch
    import torch.distributed as dist

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device(f"cuda:{local}")
    if world > 1 or "TORCHELASTIC_RUN_ID" in os.environ:   # launched by torchrun (any world size)
        dist.init_process_group("nccl", device_id=dev)
    from paper_2310_17274_b200 import native, parallel, workload

    P = args.problems
    S_total = 32
    seed_mode = args.shard == "seed"
    if seed_mode:
        s_lo, s_hi = parallel.seed_block(S_total, world, rank)
        wl = workload.franka_to(local, list(range(P)), S=S_total, H=32, iters=args.iters)
        wl.seeds = np.ascontiguousarray(wl.seeds[:, s_lo:s_hi])
    else:
        s_lo = 0
        lo = rank * P
        wl = workload.franka_to(local, list(range(lo, lo + P)), S=S_total, H=32, iters=args.iters)
    ctx = native.Context(local)
    ctx.set_robot(wl.robot)
    ctx.set_world(wl.worlds)
    ctx.set_cost_params(wl.cost)
    seeds = torch.tensor(wl.seeds, device=dev)
    goal = torch.tensor(wl.goal, device=dev)
    start = torch.tensor(wl.start, device=dev)
    env = torch.tensor(wl.env, device=dev)
    sp = wl.solver
    ctas_per_sm, smem_per_cta = ctx.solver_occupancy(32, sp.history, len(sp.alpha))
    evals_per_step = wl.evals_per_solve()
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)   # > 126 MB L2

    p_base = 0 if seed_mode else rank * P      # global index of this rank's first problem (RNG key)

    def step():
        out = ctx.solve(sp, seeds, goal, start=start, env=env, seed_base=s_lo, problem_base=p_base)
        if seed_mode and dist.is_initialized():   # the real exchange step of seed sharding: C1 + C2
            out["best_key"], out["best_traj"], out["best_cost"] = parallel.merge_seed_sharded(
                out["best_key"], out["best_traj"], S_total)
        return out

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    stream = torch.cuda.current_stream()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    launches0 = ctx.launches
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        for k in range(args.steps):
            flush.zero_()                       # L2 flush, outside the timed events
            evs[k][0].record(stream)
            out = step()
            evs[k][1].record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    launches = ctx.launches - launches0
    step_ms = [a.elapsed_time(b) for a, b in evs]
    total_ms = sum(step_ms)
    if world > 1:
        total_ms = parallel.max_over_ranks(total_ms, dev)
    evals_all = evals_per_step * args.steps * world   # seed mode: evals_per_step counts this rank's seeds
    value = evals_all / (total_ms * 1e-3)

    # ---- roofline of the dominant kernel (solve_to_kernel; the select kernel is ~us).  The path is
    # bound by plain FP32 / ALU arithmetic ("alu"); the peak is the unit count: 148 SMs x 128 FP32
    # lanes x 2 flops x sm_max_mhz (MEASURED_PEAKS.json) = 74.4 TFLOP/s.  tools/ffma_peak.cu on
    # this pool (profiles/r02_ffma_peak.json): immediate-operand FFMA 72.4 TF (97 % of it), FADD /
    # FMUL 124.5 lanes/clk/SM; register-operand FFMA 37.4 TF with shared operands, 45.9 with
    # distinct ones (register-file bandwidth).  The round-1 denominator (64 FFMA/clk, 37.2 TF) is
    # kept as `frac_of_register_ffma_ceiling` for continuity.
    pk = peaks()
    sm_max = float(pk.get("sm_max_mhz", 1965.0))
    peak_tf = SMS * FP32_LANES_PER_SM * 2 * sm_max * 1e6 / 1e12
    flops_eval = workload.nominal_flops_per_eval(wl)
    launch_s = statistics.mean(step_ms) * 1e-3
    achieved_tf = evals_per_step * flops_eval / launch_s / 1e12
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        try:
            traffic = json.load(open(tpath)).get("solve_to_kernel_dram_bytes_per_launch")
        except Exception:
            traffic = None

    # ---- end to end through the host C-ABI call
    e2e = None
    if not args.no_e2e:
        hs = seeds.cpu().pin_memory(); hg = goal.cpu().pin_memory(); hst = start.cpu().pin_memory()
        he = env.cpu().pin_memory()
        hb = torch.empty(P, 32, 7).pin_memory(); hc = torch.empty(P).pin_memory()
        hk = torch.empty(P, dtype=torch.int64).pin_memory()

        def e2e_step():
            if not seed_mode:   # one C-ABI call: H2D, solve, D2H, synchronise
                ctx.solve_host(sp, hs, hg, start=hst, env=he, best_traj=hb, best_cost=hc, best_key=hk)
                return
            seeds.copy_(hs, non_blocking=True); goal.copy_(hg, non_blocking=True)
            start.copy_(hst, non_blocking=True); env.copy_(he, non_blocking=True)
            out = step()
            hb.copy_(out["best_traj"]); hc.copy_(out["best_cost"]); hk.copy_(out["best_key"])
            torch.cuda.synchronize()

        e2e_step()
        tt = 0.0
        for k in range(args.steps):
            flush.zero_()
            torch.cuda.synchronize()
            if world > 1:
                dist.barrier()
            t0 = time.perf_counter()
            e2e_step()
            tt += time.perf_counter() - t0
        if world > 1:
            tt = parallel.max_over_ranks(tt, dev)
        h2d = hs.numel() * 4 + hg.numel() * 4 + hst.numel() * 4 + he.numel() * 4
        d2h = hb.numel() * 4 + hc.numel() * 4 + hk.numel() * 8
        e2e = {"value": evals_all / tt, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(wl)

    extras = None
    if not args.no_extras:
        extras = {"to_problems_per_s": P * world / (total_ms / args.steps * 1e-3)}
        extras.update(side_metrics(local, rank, world, dev, flush))

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
                "scaling": "strong" if seed_mode else "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
                "config": {"workload": "cfg2_franka_to_batched", "problems_per_gpu": P,
                           "global_problems": P if seed_mode else P * world,
                           "seeds_per_gpu": int(wl.seeds.shape[1]),
                           "seeds": 32, "timesteps": 32, "dof": 7, "spheres": 64, "self_pairs": int(len(wl.robot.pairs)),
                           "boxes": 20, "iters": args.iters, "line_search": list(sp.alpha), "history": sp.history,
                           "flags": "sweep+speed", "evals_per_step_per_gpu": evals_per_step,
                           "ctas_per_sm": ctas_per_sm, "smem_bytes_per_cta": smem_per_cta,
                           "schedule": ("persistent: one wave of CTAs over (seed, 10-iteration-chunk) units"
                                        if int(wl.seeds.shape[0]) * int(wl.seeds.shape[1]) >= 2 * ctas_per_sm *
                                        torch.cuda.get_device_properties(dev).multi_processor_count
                                        else "one CTA per seed trajectory"),
                           "l2": "flushed between timed steps (256 MB write, outside the events)",
                           "parallelism": (f"seed-sharded x{world}: C1 all_reduce(MIN) of packed keys + C2 all_gather "
                                           f"of winners inside the timed step") if seed_mode else
                                          f"problem-sharded x{world}, no data-path collective"},
                "roofline": {"bound": "alu", "achieved": achieved_tf, "peak": peak_tf, "unit": "TFLOP/s",
                             "frac": achieved_tf / peak_tf, "traffic": traffic,
                             "frac_of_register_ffma_ceiling": achieved_tf / (0.5 * peak_tf),
                             "pipes": pipes_summary(),
                             "kernel": "solve_to_kernel", "flops_per_eval": flops_eval,
                             "peak_basis": f"FP32 unit count: 148 SMs x 128 lanes x 2 flops x {sm_max:.0f} MHz "
                                           "(sm_max_mhz of MEASURED_PEAKS.json); tools/ffma_peak.cu measured 72.4 TF "
                                           "immediate-operand FFMA, 37.4-45.9 TF register-operand FFMA "
                                           "(profiles/r02_ffma_peak.json); achieved = nominal algorithmic flops "
                                           "(SURVEY 8(d).2) / launch time; executed per-pipe rates in `pipes` (ncu)"},
                "cpu_baseline": cpu, "e2e": e2e, "clocks": clk.summary(), "gpu_launches": launches,
                "extras": extras}
        print(json.dumps(line), flush=True)
    ctx.close()
    if dist.is_initialized():
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_native(args)


if __name__ == "__main__":
    main()
