"""Motion-generation pipeline around the solve: the paper's Fig. 2 / §2
flow of collision-free IK -> seeds -> trajectory optimisation, with the time discretisation of
Alg. 4 and the seed selection of App. B.  Readings B15-B18 in
DESIGN.md.

Every step of the computation runs in the library's kernels (libcurobo_b200.so, through
`native`); this module only sequences the calls, allocates device memory and reshapes views:

  1. IK: L-BFGS (particle warm-up + 100 iterations) on S_ik Halton seeds per goal;
  2. goal errors + validity mask of every IK solution -> IK score -> the S_to best (B18);
  3. linear seeds start -> each selected IK solution (B17);
  4. trajectory optimisation #1 at dt = 0.25 s with the jerk term off (Alg. 4 line 1);
  5. retime every seed (Alg. 4 line 2), goal errors + state validity -> blended score -> best seed;
  6. trajectory optimisation #2 of that seed at its dt_opt with the weights re-scaled (B15) and the
     jerk term on (Alg. 4 lines 3-5);
  7. final retime (Alg. 4 line 6) and the success test: pose thresholds and every state valid;
  8. interpolation of the final trajectory to a fixed dt of 0.025 s and the validity of every
     interpolated state ("interpolate the trajectory to a fixed dt of 0.025 to validate
     success"; reading B21) -- part of the success test.

One context holds the robot, the worlds (env per problem) and the cost parameters; the jerk flag
is switched between the two optimisations by re-setting the parameters (dt stays the reference
0.25 s; the second optimisation passes its per-problem dt explicitly).
"""
from __future__ import annotations

import dataclasses

import numpy as np

from . import inputs


@dataclasses.dataclass
class MotionGenConfig:
    """Pipeline parameters.  Paper values: 30 IK seeds (P:1248, 32 here so IK rows stay in aligned
    warp groups for the mask), 12 TO seeds and 32 timesteps (Table 9 / P:2204 "Bookshelf"),
    dt_i = 0.25 s (Alg. 4 / P:2054), 2 particle iterations before L-BFGS, 100 TO
    iterations and up to 300 for the single-seed re-optimisation; the success
    thresholds are the paper's; the score weights are readings (B18)."""
    ik_seeds: int = 32
    to_seeds: int = 12
    horizon: int = 32
    dt_init: float = 0.25
    ik_iters: int = 100
    to_iters: int = 100
    refine_iters: int = 300
    refine_check: int = 25          # the re-optimisation runs "for upto 300" in 25-iteration
    refine_rtol: float = 1e-3       # chunks; stop when a chunk improves the best < 0.1 % (B20)
    particle_iters: int = 2
    pos_thr: float = 5e-3           # m: "within 5mm ... of desired position"
    rot_thr: float = 0.05           # "5% of desired ... orientation" in the A1 metric 1 - |<q_g, q>|
    w_pose: float = 1.0
    w_dist: float = 0.01
    w_jerk: float = 1e-4
    w_time: float = 1.0
    invalid_penalty: float = 1e6    # TO selection: an invalid seed still ranks after every valid one
    attempts: int = 1               # plan_retry: the paper re-attempts with new linear seeds up to 3x
                                    # before its graph planner (the planner is not built)
    dt_fine: float = 0.025          # validation grid (B21)
    interp_max: int = 1024          # fine points per trajectory (a multiple of 32: mask groups); a
                                    # longer trajectory ((H-1) dt_f > 25.6 s) counts as a failure


class MotionGen:
    def __init__(self, ctx, robot: inputs.Robot, cost: inputs.CostParams, cfg: MotionGenConfig = MotionGenConfig()):
        self.ctx, self.robot, self.cfg = ctx, robot, cfg
        self.cost_to1 = dataclasses.replace(cost, dt=cfg.dt_init, flags=cost.flags & ~inputs.JERK)
        self.cost_to2 = dataclasses.replace(cost, dt=cfg.dt_init, flags=cost.flags | inputs.JERK)
        self.sp_ik = inputs.SolverParams(iters=cfg.ik_iters, particle_iters=cfg.particle_iters)
        self.sp_to = inputs.SolverParams(iters=cfg.to_iters, particle_iters=cfg.particle_iters)
        self.sp_refine = inputs.SolverParams(iters=cfg.refine_iters, check_every=cfg.refine_check,
                                             conv_rtol=cfg.refine_rtol)

    def plan_retry(self, start, goal, env, problems, attempts=None):
        """plan() on the batch, then again on the problems that failed, with fresh IK seeds (the
        Halton sequence offset by 7919 per attempt) and particle draws (rng_key = attempt), up to
        `attempts` times in all (three attempts with linear seeds before the geometric
        planner).  Returns plan()'s dict for the whole batch (each problem's last attempt) plus
        `attempt` [P] int32 (1-based attempt of the returned result)."""
        import torch
        n = self.cfg.attempts if attempts is None else attempts
        problems = np.asarray(list(problems))
        S = self.cfg.ik_seeds
        seeds = torch.tensor(self.ik_seed_batch(self.robot, problems, S), device=start.device)
        out = self.plan(start, goal, env, seeds)
        out["attempt"] = torch.ones(start.shape[0], dtype=torch.int32, device=start.device)
        keys = ("traj", "variables", "dt", "final_score", "success", "pos_err", "rot_err", "max_jerk", "fine_valid",
                "fine_points")
        for a in range(1, n):
            fail = torch.nonzero(~out["success"]).flatten()
            if fail.numel() == 0:
                break
            fi = fail.cpu().numpy()
            seeds = torch.tensor(self.ik_seed_batch(self.robot, problems[fi] + 7919 * a, S), device=start.device)
            r = self.plan(start[fail].contiguous(), goal[fail].contiguous(), env[fail].contiguous(), seeds,
                          rng_key=a)
            for k in keys:
                out[k][fail] = r[k].view(out[k][fail].shape)
            out["attempt"][fail] = a + 1
        return out

    def plan(self, start, goal, env, ik_seeds, rng_key: int = 0):
        """start [P,D], goal [P,7] (device fp32), env [P] int32 (device), ik_seeds [P,S_ik,D]
        (device, e.g. inputs.ik_seeds).  Returns a dict of device tensors: traj [P,H,D] (the states
        x_1..x_H; `variables` holds the solver's V), dt [P],
        success [P] (bool), pos_err, rot_err [P], ik_count [P] and the intermediate results; the
        motion time is (H - 1) dt."""
        from . import native as N
        ctx, c, H = self.ctx, self.cfg, self.cfg.horizon
        P, D = start.shape
        Sik, Sto = ik_seeds.shape[1], c.to_seeds
        # 1-2: collision-free IK and the S_to best solutions
        ctx.set_cost_params(self.cost_to1)
        sp_ik = dataclasses.replace(self.sp_ik, rng_key=rng_key)
        sp_to = dataclasses.replace(self.sp_to, rng_key=rng_key)
        ik = ctx.solve(sp_ik, ik_seeds, goal, env=env, seed_outputs=True)
        q_ik = ik["seed_best_traj"]                                            # [P,Sik,D]
        pe, re = ctx.goal_error(q_ik, goal, B=P * Sik, goal_div=Sik)
        valid = ctx.mask_samples(q_ik.view(P * Sik, D), env=env, env_div=Sik)
        score = N.ik_scores(q_ik, start, pe.view(P, Sik), re.view(P, Sik), valid.view(P, Sik), c.pos_thr,
                            c.rot_thr, c.w_pose, c.w_dist)
        ik_idx, ik_count = N.rank_seeds(score, Sto)
        # 3-4: linear seeds and the first trajectory optimisation (dt_i, jerk off)
        seeds = N.linear_seeds(start, q_ik, H, idx=ik_idx)                   # [P,Sto,H,D]
        to1 = ctx.solve(sp_to, seeds, goal, start=start, env=env, seed_outputs=True)
        tr1 = to1["seed_best_traj"]                                            # [P,Sto,H,D]
        # 5: retime every seed, score it, pick the best
        _, dt1, jerk1 = ctx.retime(tr1.view(P * Sto, H, D), start)
        pe1, re1 = ctx.goal_error(tr1.view(-1)[(H - 1) * D:], goal, B=P * Sto, stride=H * D, goal_div=Sto)
        x1 = N.trajectory_states(tr1.view(P * Sto, H, D), start)             # the states x_1..x_H
        v1 = ctx.mask_samples(x1.view(P * Sto * H, D), env=env, env_div=Sto * H)
        s1 = N.to_scores(pe1.view(P, Sto), re1.view(P, Sto), jerk1.view(P, Sto), dt1.view(P, Sto),
                         v1.view(P, Sto, H), H, c.pos_thr, c.rot_thr, c.w_pose, c.w_jerk, c.w_time,
                         penalty=c.invalid_penalty)
        best1, _ = N.rank_seeds(s1, 1)
        seed2 = N.gather_rows(tr1.view(P, Sto, H * D), best1).view(P, 1, H, D)
        dt_opt = N.gather_rows(dt1.view(P, Sto, 1), best1).view(P)
        # 6: re-optimise that seed at its dt_opt, weights re-scaled (B15), jerk on
        ctx.set_cost_params(self.cost_to2)
        to2 = ctx.solve(self.sp_refine, seed2, goal, start=start, env=env, dt=dt_opt)
        tr2 = to2["best_traj"]                                                 # [P,H,D]
        # 7: final retime and success
        _, dt_f, jerk2 = ctx.retime(tr2, start, dt=dt_opt)
        pe2, re2 = ctx.goal_error(tr2.view(-1)[(H - 1) * D:], goal, B=P, stride=H * D)
        x2 = N.trajectory_states(tr2, start)
        v2 = ctx.mask_samples(x2.view(P * H, D), env=env, env_div=H)
        final = N.to_scores(pe2.view(P, 1), re2.view(P, 1), jerk2.view(P, 1), dt_f.view(P, 1), v2.view(P, 1, H), H,
                            c.pos_thr, c.rot_thr, c.w_pose, c.w_jerk, c.w_time)
        ctx.set_cost_params(self.cost_to1)
        # 8: the final trajectory on the fixed fine grid (B21), every interpolated state valid
        xi, ni = N.interpolate(x2, dt_f, c.dt_fine, c.interp_max)
        vi = ctx.mask_samples(xi.view(P * c.interp_max, D), env=env, env_div=c.interp_max)
        fine_ok = (vi.view(P, c.interp_max) != 0).all(1) & (ni <= c.interp_max)
        # success: the final blended score is finite (pose thresholds met, every state valid) and
        # every interpolated state is valid
        return dict(traj=x2, variables=tr2, dt=dt_f, final_score=final.view(P),
                    success=(final.view(P) < float("inf")) & fine_ok, fine_valid=fine_ok, fine_points=ni,
                    pos_err=pe2, rot_err=re2, max_jerk=jerk2, ik_count=ik_count, ik_q=q_ik, ik_idx=ik_idx,
                    to1_traj=tr1, to1_dt=dt1, to1_score=s1, best1=best1, dt_opt=dt_opt)

    @staticmethod
    def ik_seed_batch(robot: inputs.Robot, problems, S):
        return np.stack([inputs.ik_seeds(robot, p, S) for p in problems]).astype(np.float32)
