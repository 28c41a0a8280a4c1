/*
 * oracle.h -- fp64 CPU oracle for the cuRobo (arXiv 2310.17274) cost+gradient / L-BFGS hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load or execute this library.  It shares no code, header, table or
 * constant with the CUDA path (paper_2310_17274_b200/csrc, include/curobo_b200.h).
 *
 * Citations: P:n = /root/reference/PAPER.md line n (section / equation / algorithm named
 * alongside); SURVEY §8(c) O1..O10 and readings A1..A37 are the paper readings this follows.
 * Everything is plain scalar fp64 C, written in the paper's order and notation.
 */
#ifndef CURobo_ORACLE_H
#define CURobo_ORACLE_H
#ifdef __cplusplus
extern "C" {
#endif

/* O1: robot.  Links in topological order (parent < own index), Table 6 joint types
 * (0 fixed, 1..3 prismatic x/y/z, 4..6 revolute x/y/z), F_l as 3x4 row-major. */
typedef struct {
    int n_links, n_dof, n_spheres, n_pairs, ee_link;
    const int *parent;       /* [L] -1 for the root                                  */
    const int *jtype;        /* [L]                                                  */
    const int *dof;          /* [L] actuated index or -1                            */
    const double *fixed;     /* [L][12]                                              */
    const double *lo, *hi, *vmax, *amax, *jmax;  /* [D]                              */
    const double *sph;       /* [M][4] centre in link frame, radius (r<0 disabled)   */
    const int *sph_link;     /* [M]                                                  */
    const double *sph_off;   /* [M] self-collision radius offsets           */
    const int *pairs;        /* [n_pairs][2] self-collision set S             */
} orc_robot;

/* §3.5 oriented bounding boxes; dims given as half extents. */
typedef struct {
    int n_boxes;
    const double *pos;       /* [K][3]                                               */
    const double *quat;      /* [K][4] (w,x,y,z), box -> world rotation              */
    const double *half;      /* [K][3]                                               */
    const int *enabled;      /* [K]                                                  */
} orc_world;

enum { ORC_SWEEP = 1, ORC_SPEED = 2, ORC_JERK = 4, ORC_CSPACE = 8 };

typedef struct {
    double a0, a1, a2, a3, a8, a9;   /* Eq. pose_cost_term, Eq. smooth_cost */
    double w_bound[4];               /* pos, vel, acc, jerk bound weights                     */
    double beta_self, beta_world;    /* beta_1 (Eq. self-collision), beta_2 (Eq. world-collision-cost) */
    double eta, eta_bound, dt;       /* eta, eta_2, timestep                        */
    int sweep_steps;                 /* n_s (A11)                                                      */
    int flags;                       /* ORC_SWEEP | ORC_SPEED | ORC_JERK | ORC_CSPACE                  */
    double a4, a5;                   /* Eq. cspace-cost: 5000, 50; goal = theta_g[D] when
                                        ORC_CSPACE is set, else the pose (p, q) [7]                  */
} orc_params;

/* O11 particle warm-up (Alg. 5; Eqs. particle_1/2 P:192-199; readings B6-B10). */
typedef struct {
    int iters;                       /* Alg. 5 N: 2 before L-BFGS; 0 = off               */
    int n;                           /* particles per iteration (SPEC default 64, no paper value) */
    double beta, k_mu, k_sigma;      /* c = -C/beta; step sizes of Eqs. particle_1/2              */
    double sigma0_frac;              /* Theta_sigma0 = (frac * (hi - lo))^2 per variable (B8)     */
    unsigned key;                    /* Philox4x32-10 key word 0 (word 1 = problem index, B9)     */
} orc_particle;

typedef struct {
    int iters, history, n_alpha;
    double alpha[8];
    double c1, c2;
    int ls_mode;                     /* 0 armijo, 1 wolfe, 2 strong wolfe (Alg. 1) */
    orc_particle pt;                 /* warm-up run before L-BFGS by orc_solve_to / orc_solve_ik  */
    long long problem_base, seed_base;   /* global indices of problem 0 / seed 0 (RNG counters) */
} orc_solver;

/* O10 instrumentation.  `margin` = the minimum distance of any quantity to a branch point where
 * the cost or its gradient is DISCONTINUOUS: the self-collision max(0, P*) switch and the top-2
 * gap of the arg-max pair, the inside-box nearest-face tie, a sweep exit |j - bound| (a sample
 * in contact appears or disappears; a free boundary sample changes nothing) and |<q_g, q>| (sign
 * switch of the orientation gradient).  Only the sweep exit makes the COST jump.  The
 * activation (Eq. smooth-distance-cases), the bound cost (Eq. bound_cost), the hit/free jump
 * switch (j += r' vs j += sd: equal at sd = r') and the gap test are C1 there and need no margin.
 * counters[] layout: */
void orc_set_margin_mode(int cost_only);   /* 1: record cost-discontinuity margins only (this thread) */
/* Which branch set the smallest margin of this thread's last orc_eval_traj / orc_eval_ik: 0 none,
 * 1 self max(0, P*) switch, 2 self top-2 gap, 3 inside-box nearest-face tie, 4 sweep exit,
 * 5 sign of <q_g, q> (diagnostics of the parity exclusions). */
int  orc_margin_kind(void);
/* Optional per-state margins of this thread's next evaluations: buf[H] (IK: buf[1]) receives, per
 * evaluated state h = 1..H at index h - 1, the smallest margin of the branches evaluated at that
 * state (their gradient discontinuities move only that state's gradient rows); NULL turns it off.
 * orc_cost_margin() is the smallest margin of a COST discontinuity (the sweep exit) of the last
 * evaluation.  Diagnostics for the parity tests (O10). */
void orc_set_state_margins(double *buf);
double orc_cost_margin(void);
enum { ORC_CNT_BOX_TESTS = 0, ORC_CNT_BOX_HITS, ORC_CNT_SWEEP_SAMPLES, ORC_CNT_SWEEP_HITS,
       ORC_CNT_PAIR_TESTS, ORC_CNT_PAIR_PEN, ORC_CNT_ACTIVE_SPHERES, ORC_CNT_N };

/* ---- individual steps (each cites its passage in oracle.c) ---- */
void   orc_quat_to_mat(const double *q, double *R);
void   orc_mat_to_quat(const double *R, double *q);
void   orc_fk(const orc_robot *rb, const double *q, double *link_T, double *spheres, double *ee);
void   orc_fk_backward(const orc_robot *rb, const double *q, const double *g_sph,
                       const double *g_p, const double *g_q, double *g_theta);
double orc_box_sdf(const double *p, const double *pos, const double *quat, const double *half,
                   double *grad);
double orc_activation(double dprime, double eta, double *dphi);
double orc_bound(double x, double lo, double hi, double eta2, double *dx);
double orc_logcosh(double x);
double orc_cspace_cost(const orc_params *pr, int D, const double *q, const double *goal, double *g);
double orc_pose_cost(const orc_params *pr, const double *ee, const double *goal, double *gp,
                     double *gq);
double orc_self_collision(const orc_robot *rb, const double *spheres, double beta, double *g,
                          int *arg_pair, double *margin, long long *counters);
double orc_sphere_world(const orc_world *w, const double *c, const double *cprev,
                        const double *cnext, double r, double eta, int sweep, int steps,
                        double *G, double *samples, int max_samples, int *n_samples,
                        double *margin, long long *counters);
void   orc_state_map(const double *start, const double *V, int H, int D, double *x);
void   orc_derivs(const double *x, int H, int D, double dt, double *v, double *a, double *j);

/* ---- whole evaluation (O7) ---- */
double orc_eval_traj(const orc_robot *rb, const orc_world *w, const orc_params *pr,
                     const double *start, const double *goal, const double *V, int H,
                     double *grad, double *terms, double *margin, long long *counters);
double orc_eval_ik(const orc_robot *rb, const orc_world *w, const orc_params *pr,
                   const double *goal, const double *q, double *grad, double *terms,
                   double *margin, long long *counters);

/* ---- solver (O8) ---- */
typedef double (*orc_fun)(void *ctx, const double *x, double *g);
void   orc_lbfgs_direction(int n, int count, const double *S, const double *Y, const double *rho,
                           const double *g, double *d);
int    orc_ls_select(int A, const double *alpha, double c0, double g0d, const double *ca,
                     const double *gda, double c1, double c2, int mode);
int    orc_ls_select_f32(int A, const float *alpha, float c0, float g0d, const float *ca,
                         const float *gda, float c1, float c2, int mode);
int    orc_argmin_f32(int n, const float *c);
/* O13: motion-generation pipeline pieces (Alg. 4 retime, weight scaling, goal errors, seeds, scores) */
double orc_retime(const orc_robot *rb, const double *start, const double *V, int H, double dt,
                  double *ratio_out);
void   orc_scale_params(const orc_params *in, double dt, double dt_ref, int jerk_on, orc_params *out);
void   orc_goal_error(const orc_robot *rb, const double *q, const double *goal, double *pos_err,
                      double *rot_err);
void   orc_linear_seed(const double *start, const double *qT, int H, int D, double *V);
/* B21: linear interpolation of states x[H][D] at spacing dt to the grid k dt_fine. */
int    orc_interpolate(const double *x, int H, int D, double dt, double dt_fine, int n_max, double *out);
double orc_ik_score(int D, const double *q, const double *q0, double pos_err, double rot_err,
                    double w_pose, double w_dist);
double orc_blended_score(double pos_err, double rot_err, double max_jerk, double motion_time,
                         double w_pose, double w_jerk, double w_time);
/* O12: validity mask and parallel steering (Alg. 3) */
int    orc_mask_sample(const orc_robot *rb, const orc_world *w, const double *q, double margin,
                       double *margin_out);
int    orc_steer(const orc_robot *rb, const orc_world *w, int E, const double *src,
                 const double *dst, const double *dw, double r, double margin, int *h,
                 double *v_new, double *dist, double *margin_out);
/* O11: counter-based generator (Philox4x32-10) and the particle warm-up */
void   orc_philox4x32(const unsigned key[2], const unsigned ctr[4], unsigned out[4]);
double orc_normal(unsigned key0, unsigned key1, unsigned var, unsigned particle, unsigned iter,
                  unsigned seed);
void   orc_particle_solve(orc_fun f, void *ctx, int n, const double *x0, const double *lo,
                          const double *hi, const orc_particle *pp, unsigned problem,
                          unsigned seed, double *mu, double *var, double *cost_trace);
void   orc_lbfgs_solve(orc_fun f, void *ctx, int n, const double *x0, const double *lo,
                       const double *hi, const orc_solver *sp, double *best_x, double *best_c,
                       double *trace);
/* O8 steps 1-2 (Alg. 6 lines 1-5): push (x - xp, g - gp) into the ring S, Y [m][n] (oldest
 * first), rho [m] of `count` pairs unless s'y <= 1e-12 (A20), dropping the oldest when full;
 * returns the new count, *sy_out = s'y. */
int    orc_lbfgs_push(int n, int m, double *S, double *Y, double *rho, int count, const double *x,
                      const double *xp, const double *g, const double *gp, double *sy_out);
/* O10 solver margin: distance of the active Armijo / (strong) Wolfe tests to their thresholds. */
double orc_ls_margin(int A, const double *alpha, double c0, double g0d, const double *ca,
                     const double *gda, double c1, double c2, int mode);
/* O10 per-iteration record of orc_lbfgs_solve_traced; every pointer may be NULL.  Row k of
 * x / g / c / best_c is the iterate entering iteration k (k = iters: the final one); rows of the
 * others are iteration k's L-BFGS step and line search (ca / gda rows have 8 slots). */
typedef struct {
    double *x, *g, *c, *best_c;          /* [iters+1][n], [iters+1][n], [iters+1], [iters+1] */
    double *d, *g0d, *ca, *gda;          /* [iters][n], [iters], [iters][8], [iters][8]        */
    int *istar, *count;                  /* [iters] selected candidate, ring size used for d  */
    double *sy, *ls_margin;              /* [iters] s'y offered at k (NaN at 0), O10 margin    */
} orc_solver_trace;
void   orc_lbfgs_solve_traced(orc_fun f, void *ctx, int n, const double *x0, const double *lo,
                              const double *hi, const orc_solver *sp, double *best_x,
                              double *best_c, orc_solver_trace *tr);
void   orc_solve_to(const orc_robot *rb, const orc_world *worlds, const int *env,
                    const orc_params *pr, const orc_solver *sp, int P, int S, int H,
                    const double *seeds, const double *start, const double *goal, int nthreads,
                    double *seed_best_traj, double *seed_best_cost);
void   orc_solve_ik(const orc_robot *rb, const orc_world *worlds, const int *env,
                    const orc_params *pr, const orc_solver *sp, int P, int S,
                    const double *seeds, const double *goal, int nthreads,
                    double *seed_best_q, double *seed_best_cost);

#ifdef __cplusplus
}
#endif
#endif
