/*
 * curobo_b200.h -- C-ABI of libcurobo_b200.so, the B200 (sm_100a) hot path of cuRobo
 * (arXiv 2310.17274): batched seed x timestep cost+gradient evaluation driving per-seed L-BFGS
 * with the parallel noisy line search.
 *
 * Citations: P:n = line n of the paper text, with the section / equation / algorithm.
 * DESIGN.md lists every reading (A1..A37) of an ambiguous passage that these calls implement.
 *
 * Conventions for every call:
 *   - Return a crb_status; no exception or abort crosses the ABI.  crb_last_error(ctx) returns a
 *     NUL-terminated message for the last failing call on that context (owned by the context).
 *   - crb_set_* take HOST pointers, copy what they need, and return; the caller keeps ownership.
 *   - Batch inputs/outputs of crb_fk / crb_evaluate_cost_grad / crb_lbfgs_solve are DEVICE
 *     pointers (fp32 / int32 / int64, contiguous, 16-byte aligned) owned by the caller; the call is
 *     asynchronous on `stream` (a cudaStream_t, NULL = legacy default stream).
 *   - crb_lbfgs_solve_host takes HOST pointers (pinned memory recommended), performs the
 *     host->device copies, the solve and the device->host copies on `stream`, and synchronises.
 *   - A context is bound to one CUDA device and used by one host thread at a time.  Its solves
 *     share context-owned device workspaces (per-seed results when the caller passes none, the
 *     persistent schedules' state buffer and flags): solves of one context must not overlap in
 *     time on different streams (use one context per stream).
 *   - An empty batch (B == 0 or P == 0) is validated like any other and returns CRB_OK without a
 *     launch; its batch pointers may then be NULL.
 *   - Numeric types: all results are fp32 arithmetic (the paper's kernels are fp32).  The
 *     sphere-cuboid and sphere-pair terms run conservative culling (group AABBs over the slots,
 *     per-lane AABB tests, proxy-sphere bounds of rigid pair blocks) that only selects what gets
 *     the exact fp32 tests, in the paper's order: results are bitwise those of the all-pairs fp32
 *     screen.  Every kernel flushes fp32 subnormals to zero (-ftz).  Environments below 60
 *     enabled cuboids stage their cuboid tables in shared memory, larger ones read them from
 *     global memory and batch the flagged (sphere, slot, cuboid) entries of the exact path into
 *     full warp rounds; every accumulator still receives its cuboids in increasing index, so the
 *     arithmetic and the results are the same in both builds.
 *   - Non-finite inputs are not scanned: a NaN propagates into the cost, a NaN cost packs to the
 *     +inf key and never wins a selection (SURVEY §8(b) deviation).
 *   - Capacity limits (CRB_E_LIMIT): D <= 31 (D + 1 kinematic frames after folding the fixed
 *     links, 32-bit subtree masks), L <= 64 links, M <= 512 spheres and pairs <= 16384 by the
 *     packed tables, H*D <= 512, history <= 32, n_alpha <= 8, TO mode requires 8 <= H <= 64 (one
 *     timestep per lane of a warp; H > 32 runs each evaluation as 2-3 windows of 30-31 owned
 *     timesteps with a halo timestep, P:2217 uses 44), IK mode has H == 1, and the per-CTA shared memory (robot
 *     tables, M x 32 sphere positions and gradients of 16 B each, the solver state, plus one
 *     environment's cuboids below 60 cuboids) must fit in 227 KB, which in practice bounds M at
 *     about 150 (the Franka problem: M = 64, 113 KB, two CTAs per SM).  SURVEY §8(b) sketched
 *     D <= 32 and M <= 1024 (the paper's self-collision kernel limit); DESIGN.md §11.
 *     Cuboids per environment: k_max <= CRB_MAX_CUBOIDS (131071; crb_set_world returns
 *     CRB_E_SHAPE above it).
 */
#ifndef CUROBO_B200_H
#define CUROBO_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct crb_ctx crb_ctx;

typedef enum {
    CRB_OK = 0,
    CRB_E_ARG = -1,        /* NULL pointer / invalid scalar argument                         */
    CRB_E_SHAPE = -2,      /* inconsistent sizes (H, D, batch shapes)                        */
    CRB_E_ROBOT = -3,      /* robot description fails validation (see crb_set_robot)       */
    CRB_E_WORLD = -4,      /* cuboid description fails validation                           */
    CRB_E_NOT_READY = -5,  /* robot / world / cost params not set                           */
    CRB_E_LIMIT = -6,      /* capacity limit exceeded (see header comment)                  */
    CRB_E_CUDA = -7,       /* CUDA runtime error (incl. an asynchronous fault surfaced now) */
    CRB_E_OOM = -8         /* device allocation failed                                       */
} crb_status;

/* Joint types of Table 6. */
enum { CRB_FIXED = 0, CRB_PRISMATIC_X = 1, CRB_PRISMATIC_Y = 2, CRB_PRISMATIC_Z = 3,
       CRB_REVOLUTE_X = 4, CRB_REVOLUTE_Y = 5, CRB_REVOLUTE_Z = 6 };

/* Cost flags. */
enum { CRB_SWEEP = 1u,   /* continuous collision checking, §3.4 / Algs. 11-12     */
       CRB_SPEED = 2u,   /* speed metric d_s = sdot * d_c, §3.3                    */
       CRB_JERK = 4u,    /* alpha_9 jerk term of Eq. smooth_cost (off in the 1st TO) */
       CRB_CSPACE = 8u };/* goal term = Eq. cspace-cost on a joint-space goal
                            theta_g[D] instead of Eq. pose_cost_term on a pose[7]             */

/* One link of the kinematic tree (Alg. 7 kinematic data). */
typedef struct {
    int parent;          /* parent link index, < own index (topological order); -1 for the root */
    int type;            /* CRB_FIXED .. CRB_REVOLUTE_Z (Table 6)                             */
    int dof;             /* actuated joint index 0..D-1, or -1 for a fixed joint               */
    float fixed[12];     /* F_l, 3x4 row-major; full link transform = F_l * J(q) (Table 6)    */
} crb_link;

/* Robot description (O1).  Validation (CRB_E_ROBOT): parent >= own index; a fixed
 * joint with a dof or an actuated joint without one; duplicate or missing dof; pos_lo >= pos_hi;
 * non-positive vel/acc/jerk limit; sphere on an unknown link; pair with i >= j or out of range;
 * rotation block of F not orthonormal within 1e-4; ee_link out of range. */
typedef struct {
    int n_links, n_dof, n_spheres, n_pairs, ee_link;
    const crb_link *links;                                   /* [n_links]                    */
    const float *pos_lo, *pos_hi, *vel_max, *acc_max, *jerk_max;  /* [n_dof] each           */
    const float *spheres;      /* [n_spheres][4] centre in link frame + radius; r < 0 disables
                                  the sphere for world collision (Alg. 10)       */
    const int *sphere_link;    /* [n_spheres]                                                  */
    const float *self_offset;  /* [n_spheres] self-collision radius offsets (Alg. 9), or
                                  NULL for zeros; pairs with r+o <= 0 are skipped     */
    const int *pairs;          /* [n_pairs][2] self-collision set S (Eq. self-collision);
                                  the order of S breaks arg-max ties (first maximal pair)       */
} crb_robot_desc;

/* One cuboid (§3.5 oriented bounding box; Alg. 10 obb_pose/obb_bounds/obb_enable). */
typedef struct {
    float pos[3];        /* box centre, world frame                                            */
    float quat[4];       /* (w,x,y,z) box->world rotation; normalised on upload               */
    float dims[3];       /* FULL extents; Alg. 10 halves them                 */
    int enabled;         /* 0 = skipped (Alg. 10 line "obb_enable")                    */
} crb_cuboid;

/* Cost weights and switches (App. A; App. B.3). */
typedef struct {
    float a0, a1, a2, a3;      /* Eq. pose_cost_term: 2000, 350, 100, 100             */
    float a8, a9;              /* Eq. smooth_cost: 5000, 1; alpha_6 term off (A16)    */
    float w_bound[4];          /* Eq. bound_cost weights for pos/vel/acc/jerk: 5000    */
    float beta_self;           /* beta_1 of Eq. self-collision: 5000                  */
    float beta_world;          /* beta_2 of Eq. world-collision-cost: 5000            */
    float eta;                 /* activation distance, Eq. smooth-distance-cases: 0.025 */
    float eta_bound;           /* eta_2 of Eq. bound_cost: 0.1                        */
    float dt;                  /* timestep of the five-point stencil (§A.5) and speed metric   */
    int sweep_steps;           /* n_s of Alg. 12 (never given in the paper; 4, A11)            */
    unsigned flags;            /* CRB_SWEEP | CRB_SPEED | CRB_JERK | CRB_CSPACE                */
    float a4, a5;              /* Eq. cspace-cost: 5000, 50                            */
} crb_cost_params;

/* L-BFGS + parallel noisy line search (Alg. 6, Alg. 1). */
typedef struct {
    int iters;                 /* L-BFGS iterations after the initial evaluation (100) */
    int history;               /* m (4), 0..32; 0 = gradient descent d = -g  */
    int n_alpha;               /* number of magnitudes, <= 8                                    */
    float alpha[8];            /* ascending; alpha[0] is the noisy fallback    */
    float c1, c2;              /* Armijo / Wolfe constants (A17: 1e-4, 0.9)                    */
    int ls_mode;               /* 0 Armijo, 1 Armijo+Wolfe, 2 Armijo+strong Wolfe (Alg. 1)     */
    int64_t global_seed_base;  /* added to the local seed index in the packed selection key and
                                  the particle RNG counter                                       */
    /* Particle warm-up before L-BFGS (§4.2, Alg. 5, Eqs. particle_1/2;
     * DESIGN.md readings B6-B10).  The paper runs 2 iterations and gives no values for
     * the rest; the SPEC defaults are n = 64, beta = 1, k_mu = 0.9, k_sigma = 0.5,
     * sigma0_frac = 0.1.  Each iteration draws n particles theta = clip(mu + sqrt(sigma) z) with
     * z from Philox4x32-10(key = (rng_key, global problem), ctr = (var/4, particle, iteration,
     * global seed)), evaluates their cost only, and updates mu, sigma with w = softmax(-C/beta). */
    int particle_iters;        /* 0 = off; >= 0                                                  */
    int n_particles;           /* n >= 1 when particle_iters > 0                                  */
    float particle_beta;       /* beta > 0                                                        */
    float k_mu, k_sigma;       /* step sizes in [0, 1]                                            */
    float sigma0_frac;         /* initial Theta_sigma = (sigma0_frac (hi - lo))^2 per variable    */
    uint32_t rng_key;          /* Philox key word 0                                               */
    int64_t global_problem_base;   /* added to the local problem index: Philox key word 1        */
    /* "up to" an iteration count (the single-seed re-optimisation runs "for upto 300"
     * iterations) in chunks of check_every iterations (25-iteration CUDA-graph chunks):
     * after each chunk a TO seed stops when its best cost improved by at most conv_rtol x |best
     * at the chunk start| (reading B20).  check_every = 0 runs exactly `iters` (the default); IK
     * solves ignore it. */
    int check_every;           /* >= 0                                                            */
    float conv_rtol;           /* >= 0                                                            */
    /* Latency mode: the n_alpha line-search candidates of each iteration are evaluated in
     * parallel by the n_alpha CTAs of a thread-block cluster (DSMEM exchange of the candidates'
     * costs and the winner's gradient) instead of one after the other by one CTA; results are
     * bitwise identical.  -1 = automatic (the batch's CTAs x n_alpha fit in one wave of two CTAs
     * per SM; or a particle warm-up on at most 3 waves; or a better-filled last wave), 0 = off,
     * 1 = on.  TO and IK solves. */
    int cluster;
    /* Solver trace for teacher-forced parity tests (SURVEY §8(c).4 "the oracle recomputes d from
     * the GPU's (Theta, g, ring)"; O10).  trace = NULL (the default) records nothing.  Otherwise
     * a DEVICE buffer of P * S * n_trace records of CRB_TRACE_REC(N, history) floats, N = H * D
     * (TO) or D (IK); record (p * S + s) * n_trace + j is seed s of problem p at iteration
     * trace_iter[j] (0-based, ascending not required; an iteration never reached, e.g. after a
     * chunked exit, leaves its record untouched).  Tracing runs the sequential kernels (the
     * latency-mode clusters are bitwise identical, see `cluster`).  Record layout, in floats:
     *   [0, N) Theta_k entering iteration k    [N, 2N) g_k    [2N, 3N) Theta_{k-1}    [3N, 4N) g_{k-1}
     *     (Theta_{k-1}, g_{k-1} are 0 at k = 0)    [4N, 5N) the L-BFGS direction d_k
     *   ring BEFORE the push of iteration k: S [m][N], Y [m][N] (oldest first, zero rows beyond
     *     the count), rho [m], count
     *   ring AFTER the push: S [m][N], Y [m][N], rho [m], count
     *   24 scalars: g_k.d_k, c_k, i*, s'y of the offered pair (0 at k = 0), c_a [8], g_a.d [8],
     *     k, best cost after the iteration's update, 2 unused */
    float *trace;
    int n_trace;               /* 0..8                                                            */
    int trace_iter[8];
    /* Scheduling (ignored in cluster mode).  IK: -1 (default): automatic -- a
     * persistent kernel of one wave of CTAs takes (seed group, iteration chunk) work units from a
     * global counter when the batch has at least two waves of 32-seed groups (16 chunks of
     * iters / 16 iterations; the solver state of a group moves through a context-owned device
     * buffer between its chunks, so the last wave is not left to a few long CTAs); when every
     * problem uses the same environment the groups are 32 consecutive seeds of the flat P x S
     * batch (no idle lanes when S % 32 != 0).  0: one CTA per 32-seed group of a problem.  k >= 1:
     * the persistent kernel with k chunks.  TO: the same persistent kernel over (seed, iteration
     * chunk) units (one CTA per seed trajectory otherwise); automatic (10 chunks) when the seeds
     * span >= 2 waves of CTAs (e.g. 2048 seeds on 296 CTA slots); 0 off, k >= 1 k chunks.  Every seed's result is bitwise the same in all modes. */
    int persist;
} crb_solver_params;

/* Size in floats of one solver trace record (crb_solver_params.trace). */
#define CRB_TRACE_REC(N, m) (5 * (N) + 2 * (2 * (m) * (N) + (m) + 1) + 24)

crb_status crb_create(int cuda_device, crb_ctx **out);
crb_status crb_destroy(crb_ctx *ctx);
const char *crb_last_error(const crb_ctx *ctx);
const char *crb_version(void);
/* ABI self-description for bindings: writes min(n, 5) struct sizes in bytes -- crb_link,
 * crb_robot_desc, crb_cuboid, crb_cost_params, crb_solver_params -- into out (host) and returns
 * 5.  A binding compares its mirrors against these before the first call. */
int crb_abi_sizes(int *out, int n);

/* Validate, pack (spheres grouped by link, disabled self pairs dropped, float4 layout P:3014)
 * and upload the robot tables. */
crb_status crb_set_robot(crb_ctx *ctx, const crb_robot_desc *robot);

/* Upload n_env environments of cuboids: boxes[n_env * k_max], env e using its first
 * boxes_per_env[e] entries.  k_max <= CRB_MAX_CUBOIDS, else CRB_E_SHAPE (nothing uploaded).  Disabled cuboids are compacted away (Alg. 10 skips them).  Also
 * builds each cuboid's world-frame AABB (centre, half extents widened by 1e-4 m + 1e-6 |.|) for
 * the culling ahead of the exact tests.  Stream-ordered on the legacy stream: synchronises before
 * returning. */
#define CRB_MAX_CUBOIDS 131071   /* cuboids per environment (17-bit index in the slow-path entries) */
crb_status crb_set_world(crb_ctx *ctx, int n_env, int k_max, const int *boxes_per_env,
                         const crb_cuboid *boxes);

crb_status crb_set_cost_params(crb_ctx *ctx, const crb_cost_params *params);

/* Forward kinematics (Alg. 7, Table 6): q[B][D] -> spheres_out[B][M][4] (world centre, radius)
 * and ee_out[B][7] (position, quaternion (w,x,y,z) with w >= 0).  Either output may be NULL. */
crb_status crb_fk(crb_ctx *ctx, const float *q, int B, float *spheres_out, float *ee_out,
                  void *stream);

/* Batched cost and gradient (Eq. cost_motion_opt, with the App. A terms).
 *   H >= 8 (TO mode): q[B][H][D] are the optimisation variables V of B trajectories; the state
 *     map of Table 5's last row pins x_1..x_3 = start[b] and aliases x_{H-3..H-1} = x_H;
 *     cost[b] = sum over the H evaluated states of bound + smoothness + self + world terms, plus
 *     the pose term at x_H; grad[b][H][D] = dC/dV (zero on pinned / aliased variables).
 *   H == 1 (IK mode): q[B][D] configurations; pose + self + discrete world + position bound.
 *     The env index must be constant inside each aligned group of 32 rows (rows that violate it
 *     get a NaN cost).  start may be NULL.
 *   env[B] (may be NULL = all 0; device memory, so an index outside [0, n_env) is not checked
 *   on the host: such a row gets a NaN cost, never an obstacle-free one), goal[B][7] (position,
 *   quaternion w,x,y,z), or goal[B][D]
 *   (joint configuration) when the cost flags include CRB_CSPACE.
 *   term_costs[B][5] (pose, bound, smooth, self, world) may be NULL. */
crb_status crb_evaluate_cost_grad(crb_ctx *ctx, const float *q, int B, int H, const int *env,
                                  const float *start, const float *goal, float *cost,
                                  float *grad, float *term_costs, void *stream);

/* Same with a per-row timestep (Alg. 4 "run trajectory optimization with new dt", reading B15):
 * dt[B] (device, > 0; NULL = the cost params' dt).  The five-point stencil and the speed metric
 * use dt[b]; every term that relates to velocity, acceleration or jerk is rescaled relative to
 * dt_ref = the cost params' dt: alpha_8 (dt/dt_ref)^4, alpha_9 (dt/dt_ref)^6 and the
 * velocity / acceleration / jerk limit weights (dt/dt_ref)^1, ^2, ^3 (each term keeps its
 * magnitude when the same path is re-timed); the position limit weight stays.  IK rows ignore dt. */
crb_status crb_evaluate_cost_grad_dt(crb_ctx *ctx, const float *q, int B, int H, const int *env,
                                     const float *start, const float *goal, const float *dt,
                                     float *cost, float *grad, float *term_costs, void *stream);

/* Per-seed L-BFGS solve (§4.1, Alg. 6 + Alg. 1), one persistent CTA per seed trajectory (TO) or
 * per 32 seeds of one problem (IK), all `iters` iterations inside one launch.
 *   seeds[P][S][H][D] (TO, H >= 8) or [P][S][D] (IK, H == 1); env[P] (may be NULL; a problem
 *   whose env index is outside [0, n_env) evaluates to NaN costs: its best_cost is NaN and its
 *   best_key the +inf bits);
 *   start[P][D] (TO only); goal[P][7] (pose) or goal[P][D] (CRB_CSPACE).
 * Outputs (any may be NULL): best_traj[P][H][D] and best_cost[P] of the winning seed per
 * problem; best_key[P] = (float_bits(cost) << 32) | (global_seed_base + s), the packed key the
 * multi-GPU argmin reduces with MIN (NaN -> +inf bits); seed_best_cost[P][S] and
 * seed_best_traj[P][S][H][D] per seed. */
crb_status crb_lbfgs_solve(crb_ctx *ctx, const crb_solver_params *sp, int P, int S, int H,
                           const float *seeds, const int *env, const float *start,
                           const float *goal, float *best_traj, float *best_cost,
                           int64_t *best_key, float *seed_best_cost, float *seed_best_traj,
                           void *stream);

/* crb_lbfgs_solve with a per-problem timestep dt[P] (device, > 0; NULL = the cost params' dt),
 * weights rescaled as in crb_evaluate_cost_grad_dt (the second trajectory optimisation of Alg. 4). */
crb_status crb_lbfgs_solve_dt(crb_ctx *ctx, const crb_solver_params *sp, int P, int S, int H,
                              const float *seeds, const int *env, const float *start,
                              const float *goal, const float *dt, float *best_traj, float *best_cost,
                              int64_t *best_key, float *seed_best_cost, float *seed_best_traj,
                              void *stream);

/* Same as crb_lbfgs_solve with HOST buffers: copies inputs to context-owned device buffers,
 * solves, copies outputs back and synchronises `stream`.  The env indices are host data here, so
 * one outside [0, n_env) returns CRB_E_SHAPE before anything is copied. */
crb_status crb_lbfgs_solve_host(crb_ctx *ctx, const crb_solver_params *sp, int P, int S, int H,
                                const float *seeds, const int *env, const float *start,
                                const float *goal, float *best_traj, float *best_cost,
                                int64_t *best_key, void *stream);

/* ---- validity mask and parallel steering (Alg. 3) ---- */

/* mask_samples (Alg. 3 line 5, reading B12): valid[k] = 1 iff configuration q[k] is
 * inside the position limits, no self-collision pair of S penetrates, and every enabled sphere
 * keeps a distance >= r + margin (m, >= 0) to every enabled cuboid of env[k]; else 0.
 * Device pointers: q[K][D], env[K / env_div] (row k uses env[k / env_div]; may be NULL = 0; the
 * env must be constant within aligned groups of 32 rows, a row that violates it, or whose env
 * index is outside [0, n_env), is reported invalid), valid[K] (uint8).  Needs robot, world, params. */
crb_status crb_mask_samples(crb_ctx *ctx, const float *q, int K, const int *env, int env_div,
                            float margin, uint8_t *valid, void *stream);

/* Parallel steering (Alg. 3, reading B13) of E edges in environment `env`:
 *   n = floor(max_{e,d} |dw_d (dst_ed - src_ed)| / r) + 1, shared by the batch and clamped to
 *   n_cap (the grid is sized for n_cap: no host synchronisation); waypoints
 *   l_ej = src_e + (j / n)(dst_e - src_e), j = 0..n, are validated as by crb_mask_samples;
 *   h[e] = (first invalid j) - 1, or n if all are valid (-1: invalid source, v_new = src);
 *   v_new[e] = l_e,h[e]; dist[e] = |dw * (v_new[e] - src[e])|_2 (the edge weight).
 * Device pointers: src[E][D], dst[E][D], dw[D], n_out[2] (n used, n before clamping; may be
 * NULL), h[E], v_new[E][D], dist[E].  The graph bookkeeping (Alg. 2) stays with the caller. */
crb_status crb_steer(crb_ctx *ctx, int E, const float *src, const float *dst, const float *dw, float r,
                     int env, float margin, int n_cap, int *n_out, int *h, float *v_new, float *dist,
                     void *stream);

/* ---- motion-generation pipeline pieces (§2 / Fig. 2, Alg. 4, App. B P:2189-2190;
 *      SURVEY §8(f) f2; readings B15-B18).  The calls without a context are plain
 *      arithmetic on device arrays. ---- */

/* Alg. 4 retime ("find dt that pushes trajectory to robot limits"): for each of B trajectories
 * V[B][H][D] with its start row start[b / start_div][D] and timestep dt[b] (NULL = the cost
 * params' dt), the five-point-stencil v, a, j of the Table 5 state sequence give
 *   scale[b] = max(1e-3, max |v|/vmax, sqrt(|a|/amax), cbrt(|j|/jmax)),
 *   dt_opt[b] = scale[b] dt[b]  (may be NULL),  max_jerk[b] = max |j| at dt_opt (may be NULL).
 * Needs the robot (limits).  H >= 8. */
crb_status crb_retime(crb_ctx *ctx, int B, int H, const float *V, const float *start, int start_div,
                      const float *dt, float *scale, float *dt_opt, float *max_jerk, void *stream);

/* Goal errors of B configurations q (row b at q + b * q_stride, q_stride >= D floats; e.g. the
 * terminal state V[b][H-1] with q = V + (H-1) D, q_stride = H D): pos_err[b] = |p_g - p|_2,
 * rot_err[b] = 1 - |<q_g, q>| (reading A1), goal[B / goal_div][7] (row b uses goal[b / goal_div]).
 * Needs the robot. */
crb_status crb_goal_error(crb_ctx *ctx, int B, const float *q, int q_stride, const float *goal,
                          int goal_div, float *pos_err, float *rot_err, void *stream);

/* IK ranking score (App. B: "lowest weighted sum of pose error and the distance of the solution to
 * the current joint configuration"): score[p][s] = w_pose (pe + re) + w_dist |q[p][s] - q0[p]|_2,
 * plus `penalty` (e.g. +inf) unless pe < pos_thr, re < rot_thr and valid[p][s] (uint8 mask, may
 * be NULL). */
crb_status crb_ik_scores(int P, int S, int D, const float *q, const float *q0, const float *pos_err,
                         const float *rot_err, const uint8_t *valid, float pos_thr, float rot_thr,
                         float w_pose, float w_dist, float penalty, float *score, void *stream);

/* TO blended score (App. B: "a blended sum of the pose error, maximum jerk, and motion time"):
 * score[p][s] = w_pose (pe + re) + w_jerk max_jerk + w_time (H-1) dt_opt, plus `penalty` unless
 * the pose thresholds hold and all H states are valid (valid[p][s][H], uint8, may be NULL). */
crb_status crb_to_scores(int P, int S, int H, const float *pos_err, const float *rot_err,
                         const float *max_jerk, const float *dt_opt, const uint8_t *valid,
                         float pos_thr, float rot_thr, float w_pose, float w_jerk, float w_time,
                         float penalty, float *score, void *stream);

/* Per problem, the k lowest finite scores in ascending order (ties -> lower index): idx[p][j] =
 * seed index of rank j; for j >= count[p] the ranked list repeats cyclically; idx = -1 when
 * count[p] = 0 (no valid seed).  score[P][S]. */
crb_status crb_rank_seeds(int P, int S, const float *score, int k, int *idx, int *count, void *stream);

/* Linear TO seeds (reading B17): seeds[p][s][h] = q0[p] + (h/(H-1)) (qT[p][j] - q0[p]) with
 * j = idx[p][s] (idx may be NULL: j = s, then Sq >= S), qT[P][Sq][D]; j < 0 gives a still seed. */
crb_status crb_linear_seeds(int P, int S, int H, int D, const float *q0, const float *qT, int Sq,
                            const int *idx, float *seeds, void *stream);

/* The trajectory states of optimisation variables (Table 5 last row): x[b][h-1] = x_h for
 * h = 1..H with x_1..x_3 = start[b / start_div], x_{H-3..H} = V[b][H-1], else V[b][h-1] (the
 * pinned V_0..V_2 and aliased V_{H-4..H-2} are not states).  V[B][H][D] -> x[B][H][D]. */
crb_status crb_trajectory_states(int B, int H, int D, const float *V, const float *start, int start_div,
                                 float *x, void *stream);

/* Interpolation to a fine time grid ("interpolate the trajectory to a fixed dt of 0.025 to
 * validate success"; reading B21): B trajectories of states x[B][H][D] (device,
 * e.g. crb_trajectory_states) sampled at spacing dt[B] (device) -> out[B][n_max][D] (device):
 * point k is the joint-space linear interpolation at t_k = min(k dt_fine, (H-1) dt[b]) between the
 * bracketing states, for k < n_b = ceil((H-1) dt[b] / dt_fine) + 1 (the last point is x_H); rows
 * from min(n_b, n_max) on repeat x_H.  n_out[B] (device int32, may be NULL) receives n_b before
 * clamping, so a caller can detect truncation.  Errors: CRB_E_ARG (H < 2, dt_fine <= 0, n_max < 1,
 * NULL pointers), CRB_E_LIMIT (B > 65535). */
crb_status crb_interpolate(int B, int H, int D, const float *x, const float *dt, float dt_fine, int n_max,
                           float *out, int *n_out, void *stream);

/* dst[p][:] = src[p][idx[p * idx_stride]][:] for rows of n floats, src[P][S][n] (idx < 0: zeros). */
crb_status crb_gather_rows(int P, int S, int n, const float *src, const int *idx, int idx_stride,
                           float *dst, void *stream);

/* ---- test hooks: the exact device routines the solver uses, on caller data ---- */

/* Alg. 1 selection (lines 4-9) for n independent line searches, in fp32 with the fixed
 * operation order rhs = c0 + (c1 * alpha_a) * g0d (no FMA contraction): out_idx[i] = largest a
 * whose active conditions hold, else 0.  All pointers device: c0[n], g0d[n], ca[n][A],
 * gda[n][A], out_idx[n]. */
crb_status crb_ls_select(int n, int A, const float *alpha_host, const float *c0, const float *g0d,
                         const float *ca, const float *gda, float c1, float c2, int mode,
                         int *out_idx, void *stream);

/* Per-problem packed-key argmin over S seed costs (ties -> lowest seed, NaN -> +inf). Device
 * pointers: cost[P][S], out_key[P], out_idx[P]. */
crb_status crb_argmin_keys(int P, int S, const float *cost, int64_t seed_base, int64_t *out_key,
                           int *out_idx, void *stream);

/* Two-loop recursion (Alg. 6) exactly as run inside the solver: for each of B problems with n
 * variables and `count` stored pairs (oldest first), d = -H g.  Device pointers:
 * S[B][count][n], Y[B][count][n], g[B][n], d[B][n].  n <= 512, count <= 32. */
crb_status crb_lbfgs_direction(int B, int n, int count, const float *S, const float *Y,
                               const float *g, float *d, void *stream);

/* The particle warm-up's draws (Alg. 5 SAMPLE, reading B9) exactly as the solver makes them:
 * out[l][v] = theta_s for variable v of particle l in iteration `iter` of global seed `seed`,
 * key (key0, key1 = global problem).  Device pointer out[n_particles][n_var]. */
crb_status crb_particle_normals(uint32_t key0, uint32_t key1, int n_var, int n_particles, int iter,
                                uint32_t seed, float *out, void *stream);

/* Shared-memory footprint (bytes per CTA) and resident CTAs per SM of the persistent solver for
 * horizon H (1 = IK) with the current robot and world (diagnostics; needs robot, world, params). */
crb_status crb_solver_occupancy(crb_ctx *ctx, int H, int history, int n_alpha, int *ctas_per_sm,
                                int *smem_bytes);

/* Number of kernel launches this context issued since creation (bench accounting). */
int64_t crb_launch_count(const crb_ctx *ctx);

#ifdef __cplusplus
}
#endif
#endif
