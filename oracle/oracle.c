/*
 * oracle.c -- plain, slow, fp64 CPU oracle of the cuRobo (arXiv 2310.17274) hot path.
 *
 * TEST INFRASTRUCTURE ONLY (see oracle.h).  Never linked into, imported by, or called from the
 * product path.  No blocking, fusion or reordering beyond the paper's definitions: every function
 * follows its passage step by step in the paper's order and notation.  Compiled -O2, no fast-math,
 * -ffp-contract=off (the fp32 selection mirror depends on it).
 *
 * P:n = /root/reference/PAPER.md line n.  O1..O10 / A1..A37 = SURVEY.md §8(c) steps and readings
 * (also listed in DESIGN.md).
 */
#include "oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

#define ORC_INF (1.0 / 0.0)
#define ORC_NAN (0.0 / 0.0)

/* O10 margin kinds (diagnostics: which branch set the smallest margin of the last evaluation):
 * 1 self max(0, P*) switch, 2 self top-2 gap, 3 inside-box nearest-face tie, 4 sweep exit,
 * 5 sign of <q_g, q>. */
static _Thread_local int g_margin_kind = 0;

int orc_margin_kind(void) { return g_margin_kind; }

/* Per-state split of the margin (O10, optional; orc_set_state_margins): the margins of the
 * branches evaluated at state h (gradient discontinuities there move only the gradient rows of
 * that state) and, separately, the margins of COST discontinuities (the sweep exit). */
static _Thread_local double *g_state_margin = NULL;   /* [H] or NULL */
static _Thread_local int g_state_idx = -1;
static _Thread_local double g_cost_margin = 1.0 / 0.0;

void orc_set_state_margins(double *buf) { g_state_margin = buf; }
double orc_cost_margin(void) { return g_cost_margin; }

static void upd_margin_k(double *margin, double v, int kind) {
    if (margin && fabs(v) < *margin) { *margin = fabs(v); g_margin_kind = kind; }
    if (margin && g_state_margin && g_state_idx >= 0 && fabs(v) < g_state_margin[g_state_idx])
        g_state_margin[g_state_idx] = fabs(v);
    if (margin && kind == 4 && fabs(v) < g_cost_margin) g_cost_margin = fabs(v);
}

/* Margin kinds: upd_margin for branches where the COST jumps (a sweep sample that appears or
 * disappears while in contact), upd_margin_grad where only the gradient does (the cost is
 * continuous there).  With cost-only margins on (orc_set_margin_mode(1), per thread) the latter
 * are not recorded: what a cost-only evaluation (the particle warm-up) needs. */
static _Thread_local int g_cost_only_margins = 0;

void orc_set_margin_mode(int cost_only) { g_cost_only_margins = cost_only; }

static void upd_margin_grad(double *margin, double v, int kind) {
    if (!g_cost_only_margins) upd_margin_k(margin, v, kind);
}

/* ------------------------------------------------------------------------------------------ */
/* 4x4 homogeneous matrices, Table 6                                              */
/* ------------------------------------------------------------------------------------------ */

static void mat4_identity(double M[4][4]) {
    for (int i = 0; i < 4; ++i)
        for (int j = 0; j < 4; ++j) M[i][j] = (i == j) ? 1.0 : 0.0;
}

static void mat4_mul(double A[4][4], double B[4][4], double C[4][4]) {
    for (int i = 0; i < 4; ++i)
        for (int j = 0; j < 4; ++j) {
            double s = 0.0;
            for (int k = 0; k < 4; ++k) s += A[i][k] * B[k][j];
            C[i][j] = s;
        }
}

/* Table 6 "Joint Transformation" column.  A25: the revolute-X full-link entry
 * (3,3) typo does not arise here because we multiply F * J explicitly. */
static void joint_transform(int type, double v, double J[4][4]) {
    mat4_identity(J);
    double c = cos(v), s = sin(v);
    switch (type) {
        case 0: break;                           /* fixed                     */
        case 1: J[0][3] = v; break;              /* prismatic x: d_x          */
        case 2: J[1][3] = v; break;              /* prismatic y: d_y          */
        case 3: J[2][3] = v; break;              /* prismatic z: d_z          */
        case 4:                                  /* revolute x                */
            J[1][1] = c; J[1][2] = -s; J[2][1] = s; J[2][2] = c; break;
        case 5:                                  /* revolute y                */
            J[0][0] = c; J[0][2] = s; J[2][0] = -s; J[2][2] = c; break;
        case 6:                                  /* revolute z                */
            J[0][0] = c; J[0][1] = -s; J[1][0] = s; J[1][1] = c; break;
    }
}

/* (w,x,y,z) unit quaternion -> rotation (A31; normalised first). */
void orc_quat_to_mat(const double *q, double *R) {
    double n = sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
    double w = q[0] / n, x = q[1] / n, y = q[2] / n, z = q[3] / n;
    R[0] = 1 - 2 * (y * y + z * z); R[1] = 2 * (x * y - w * z);     R[2] = 2 * (x * z + w * y);
    R[3] = 2 * (x * y + w * z);     R[4] = 1 - 2 * (x * x + z * z); R[5] = 2 * (y * z - w * x);
    R[6] = 2 * (x * z - w * y);     R[7] = 2 * (y * z + w * x);     R[8] = 1 - 2 * (x * x + y * y);
}

/* Matrix -> quaternion (Alg. 7 mat_to_quat P:2649): Shepperd's method, branch on the
 * largest of trace / diagonal, canonical hemisphere w >= 0 (A31). */
void orc_mat_to_quat(const double *R, double *q) {
    double tr = R[0] + R[4] + R[8];
    double w, x, y, z;
    if (tr >= R[0] && tr >= R[4] && tr >= R[8]) {
        w = 0.5 * sqrt(1.0 + tr);
        x = (R[7] - R[5]) / (4 * w); y = (R[2] - R[6]) / (4 * w); z = (R[3] - R[1]) / (4 * w);
    } else if (R[0] >= R[4] && R[0] >= R[8]) {
        x = 0.5 * sqrt(1.0 + R[0] - R[4] - R[8]);
        w = (R[7] - R[5]) / (4 * x); y = (R[1] + R[3]) / (4 * x); z = (R[2] + R[6]) / (4 * x);
    } else if (R[4] >= R[8]) {
        y = 0.5 * sqrt(1.0 - R[0] + R[4] - R[8]);
        w = (R[2] - R[6]) / (4 * y); x = (R[1] + R[3]) / (4 * y); z = (R[5] + R[7]) / (4 * y);
    } else {
        z = 0.5 * sqrt(1.0 - R[0] - R[4] + R[8]);
        w = (R[3] - R[1]) / (4 * z); x = (R[2] + R[6]) / (4 * z); y = (R[5] + R[7]) / (4 * z);
    }
    if (w < 0) { w = -w; x = -x; y = -y; z = -z; }
    q[0] = w; q[1] = x; q[2] = y; q[3] = z;
}

/* O4 / Alg. 7: T_l = T_{p(l)} * F_l * J_type(x[a(l)]), T_{p(0)} = I;
 * sphere centres w_m = R_{link(m)} c_m + t_{link(m)}; EE (p, quat). */
static void fk_full(const orc_robot *rb, const double *q, double (*T)[4][4]) {
    for (int l = 0; l < rb->n_links; ++l) {
        double P[4][4], F[4][4], J[4][4], PF[4][4];
        if (rb->parent[l] < 0) mat4_identity(P);
        else memcpy(P, T[rb->parent[l]], sizeof(P));
        mat4_identity(F);
        for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 4; ++j) F[i][j] = rb->fixed[l * 12 + i * 4 + j];
        double v = (rb->dof[l] >= 0) ? q[rb->dof[l]] : 0.0;
        joint_transform(rb->jtype[l], v, J);
        mat4_mul(P, F, PF);
        mat4_mul(PF, J, T[l]);
    }
}

void orc_fk(const orc_robot *rb, const double *q, double *link_T, double *spheres, double *ee) {
    double (*T)[4][4] = malloc(sizeof(double[4][4]) * (size_t)rb->n_links);
    fk_full(rb, q, T);
    if (link_T)
        for (int l = 0; l < rb->n_links; ++l)
            for (int i = 0; i < 3; ++i)
                for (int j = 0; j < 4; ++j) link_T[l * 12 + i * 4 + j] = T[l][i][j];
    if (spheres)
        for (int m = 0; m < rb->n_spheres; ++m) {
            int l = rb->sph_link[m];
            for (int i = 0; i < 3; ++i)
                spheres[m * 4 + i] = T[l][i][0] * rb->sph[m * 4 + 0] + T[l][i][1] * rb->sph[m * 4 + 1] +
                                     T[l][i][2] * rb->sph[m * 4 + 2] + T[l][i][3];
            spheres[m * 4 + 3] = rb->sph[m * 4 + 3];
        }
    if (ee) {
        int e = rb->ee_link;
        double R[9];
        for (int i = 0; i < 3; ++i) {
            ee[i] = T[e][i][3];
            for (int j = 0; j < 3; ++j) R[i * 3 + j] = T[e][i][j];
        }
        orc_mat_to_quat(R, ee + 3);
    }
    free(T);
}

static int is_ancestor_or_self(const orc_robot *rb, int anc, int l) {
    while (l >= 0) {
        if (l == anc) return 1;
        l = rb->parent[l];
    }
    return 0;
}

/* Hamilton product a (x) b, (w,x,y,z). */
static void quat_mul(const double *a, const double *b, double *c) {
    c[0] = a[0] * b[0] - a[1] * b[1] - a[2] * b[2] - a[3] * b[3];
    c[1] = a[0] * b[1] + a[1] * b[0] + a[2] * b[3] - a[3] * b[2];
    c[2] = a[0] * b[2] - a[1] * b[3] + a[2] * b[0] + a[3] * b[1];
    c[3] = a[0] * b[3] + a[1] * b[2] - a[2] * b[1] + a[3] * b[0];
}

static void cross3(const double *a, const double *b, double *c) {
    c[0] = a[1] * b[2] - a[2] * b[1];
    c[1] = a[2] * b[0] - a[0] * b[2];
    c[2] = a[0] * b[1] - a[1] * b[0];
}

/* O6 / Alg. 8 + Table 7: for every actuated link l, sum over spheres
 * (and the EE point) whose link has l as ancestor-or-self: revolute G^T (k x (w - o)),
 * prismatic G^T k; EE quaternion: (dC/dq)^T (1/2 (0,k) (x) q) for revolute (A27). */
void orc_fk_backward(const orc_robot *rb, const double *q, const double *g_sph, const double *g_p,
                     const double *g_q, double *g_theta) {
    int L = rb->n_links;
    double (*T)[4][4] = malloc(sizeof(double[4][4]) * (size_t)L);
    fk_full(rb, q, T);
    for (int d = 0; d < rb->n_dof; ++d) g_theta[d] = 0.0;
    double ee_p[3], ee_q[4], R[9];
    int e = rb->ee_link;
    for (int i = 0; i < 3; ++i) {
        ee_p[i] = T[e][i][3];
        for (int j = 0; j < 3; ++j) R[i * 3 + j] = T[e][i][j];
    }
    orc_mat_to_quat(R, ee_q);
    for (int l = 0; l < L; ++l) {
        int a = rb->dof[l];
        if (a < 0) continue;
        int type = rb->jtype[l];
        int axis = (type >= 4) ? type - 4 : type - 1;
        double k[3] = {T[l][0][axis], T[l][1][axis], T[l][2][axis]};
        double o[3] = {T[l][0][3], T[l][1][3], T[l][2][3]};
        double acc = 0.0;
        if (g_sph) {
            for (int m = 0; m < rb->n_spheres; ++m) {
                if (!is_ancestor_or_self(rb, l, rb->sph_link[m])) continue;
                int lm = rb->sph_link[m];
                double w[3];
                for (int i = 0; i < 3; ++i)
                    w[i] = T[lm][i][0] * rb->sph[m * 4 + 0] + T[lm][i][1] * rb->sph[m * 4 + 1] +
                           T[lm][i][2] * rb->sph[m * 4 + 2] + T[lm][i][3];
                const double *G = g_sph + m * 3;
                if (type >= 4) {
                    double r[3] = {w[0] - o[0], w[1] - o[1], w[2] - o[2]}, kx[3];
                    cross3(k, r, kx);
                    acc += G[0] * kx[0] + G[1] * kx[1] + G[2] * kx[2];
                } else {
                    acc += G[0] * k[0] + G[1] * k[1] + G[2] * k[2];
                }
            }
        }
        if (is_ancestor_or_self(rb, l, e)) {
            if (g_p) {
                if (type >= 4) {
                    double r[3] = {ee_p[0] - o[0], ee_p[1] - o[1], ee_p[2] - o[2]}, kx[3];
                    cross3(k, r, kx);
                    acc += g_p[0] * kx[0] + g_p[1] * kx[1] + g_p[2] * kx[2];
                } else {
                    acc += g_p[0] * k[0] + g_p[1] * k[1] + g_p[2] * k[2];
                }
            }
            if (g_q && type >= 4) {
                double k4[4] = {0.0, k[0], k[1], k[2]}, dq[4];
                quat_mul(k4, ee_q, dq);
                for (int i = 0; i < 4; ++i) acc += g_q[i] * 0.5 * dq[i];
            }
        }
        g_theta[a] += acc;
    }
    free(T);
}

/* ------------------------------------------------------------------------------------------ */
/* World geometry: §3.5 OBB, Alg. 10, reading A4                      */
/* ------------------------------------------------------------------------------------------ */

/* Exact Euclidean box SDF from the closest point (A4): p_loc = R^T (p - t); q = |p_loc| - h;
 * outside: sd = ||max(q,0)||, grad_loc = sign(p_loc) * max(q,0) / sd; inside: sd = max_i q_i,
 * grad_loc = sign(p_loc_i*) e_i* with i* the first arg-max (x<y<z).  sign(0) := +1.
 * Returns sd, writes grad = R grad_loc (world frame) if grad != NULL. */
static double box_sdf_impl(const double *p, const double *pos, const double *quat,
                           const double *half, double *grad, double *margin) {
    double R[9];
    orc_quat_to_mat(quat, R);
    double dpw[3] = {p[0] - pos[0], p[1] - pos[1], p[2] - pos[2]};
    double pl[3], qv[3], gl[3] = {0, 0, 0};
    for (int i = 0; i < 3; ++i) pl[i] = R[0 * 3 + i] * dpw[0] + R[1 * 3 + i] * dpw[1] + R[2 * 3 + i] * dpw[2];
    for (int i = 0; i < 3; ++i) qv[i] = fabs(pl[i]) - half[i];
    double qmax = qv[0];
    int imax = 0;
    for (int i = 1; i < 3; ++i)
        if (qv[i] > qmax) { qmax = qv[i]; imax = i; }
    double sd;
    if (qmax > 0) {
        double s2 = 0;
        for (int i = 0; i < 3; ++i) {
            double mq = qv[i] > 0 ? qv[i] : 0.0;
            s2 += mq * mq;
        }
        sd = sqrt(s2);
        for (int i = 0; i < 3; ++i) {
            double mq = qv[i] > 0 ? qv[i] : 0.0;
            gl[i] = (pl[i] >= 0 ? 1.0 : -1.0) * mq / sd;
        }
    } else {
        sd = qmax;
        gl[imax] = pl[imax] >= 0 ? 1.0 : -1.0;
        if (margin) {
            /* arg-max tie margin on the inside branch */
            double second = -ORC_INF;
            for (int i = 0; i < 3; ++i)
                if (i != imax && qv[i] > second) second = qv[i];
            upd_margin_grad(margin, qmax - second, 3);
        }
    }
    if (grad)
        for (int i = 0; i < 3; ++i) grad[i] = R[i * 3 + 0] * gl[0] + R[i * 3 + 1] * gl[1] + R[i * 3 + 2] * gl[2];
    return sd;
}

double orc_box_sdf(const double *p, const double *pos, const double *quat, const double *half,
                   double *grad) {
    return box_sdf_impl(p, pos, quat, half, grad, NULL);
}

/* Eq. smooth-distance-cases in penetration-positive form (A2): with
 * d' = r' - sd (r' = r + eta) and d = d' - eta,
 * phi = 0 (d' <= 0), d'^2 / (2 eta) (0 < d' <= eta), d' - eta/2 (d' > eta). */
double orc_activation(double dprime, double eta, double *dphi) {
    if (dprime <= 0) { if (dphi) *dphi = 0.0; return 0.0; }
    if (dprime <= eta) { if (dphi) *dphi = dprime / eta; return dprime * dprime / (2.0 * eta); }
    if (dphi) *dphi = 1.0;
    return dprime - 0.5 * eta;
}

/* One box test at point p for inflated radius rp: returns phi, accumulates scale*phi'*(-grad sd). */
static double box_term(const orc_world *w, int k, const double *p, double rp, double eta,
                       double scale, double *G, double *sd_out, double *margin) {
    double g[3];
    double sd = box_sdf_impl(p, w->pos + 3 * k, w->quat + 4 * k, w->half + 3 * k, g, NULL);
    double dprime = rp - sd;
    if (sd_out) *sd_out = sd;
    if (dprime > 0) {
        if (margin) box_sdf_impl(p, w->pos + 3 * k, w->quat + 4 * k, w->half + 3 * k, NULL, margin);
        double dphi;
        double phi = orc_activation(dprime, eta, &dphi);
        for (int i = 0; i < 3; ++i) G[i] += scale * dphi * (-g[i]);
        return phi;
    }
    return 0.0;
}

/* O5 world term for one sphere (centre c, radius r >= 0) -- Alg. 10 (discrete) and §3.4 /
 * Fig. 4 / Algs. 11-12 (swept) under readings A6-A12:
 *   E = sum_k phi(r' - sd_k(c));  G = sum_k phi' (-grad sd_k(c))
 *   swept: for each box k and each existing neighbour n in {prev, next}:
 *     L = ||n - c||, gap = L - 2r' (skip if gap <= 0), bound = L/2,
 *     j = J0 = (r' - sd_k(c) > 0) ? r' : sd_k(c)   (reset per direction, A10)
 *     repeat <= n_s: if j >= bound stop; kappa = j/L; p = c + kappa (n - c); d' = r' - sd_k(p);
 *        hit: E += phi(d'), G += (1-kappa) phi'(d') (-grad sd_k(p)), j += r'   (A9, A12)
 *        else j += sd_k(p)                                                     (A8)
 * Returns E; G accumulates (without beta_2 * speed).  samples (optional) records
 * (k, dir, kappa, hit) per sweep sample. */
double orc_sphere_world(const orc_world *w, const double *c, const double *cprev,
                        const double *cnext, double r, double eta, int sweep, int steps,
                        double *G, double *samples, int max_samples, int *n_samples,
                        double *margin, long long *counters) {
    double rp = r + eta;   /* Alg. 10 line "sph.radius += eta" */
    double E = 0.0;
    if (n_samples) *n_samples = 0;
    for (int k = 0; k < w->n_boxes; ++k) {
        if (!w->enabled[k]) continue;
        double sd0;
        double phi = box_term(w, k, c, rp, eta, 1.0, G, &sd0, margin);
        E += phi;
        if (counters) { counters[ORC_CNT_BOX_TESTS]++; if (rp - sd0 > 0) counters[ORC_CNT_BOX_HITS]++; }
        if (!sweep) continue;
        for (int dir = 0; dir < 2; ++dir) {
            const double *n = (dir == 0) ? cprev : cnext;
            if (!n) continue;
            double dv[3] = {n[0] - c[0], n[1] - c[1], n[2] - c[2]};
            double L = sqrt(dv[0] * dv[0] + dv[1] * dv[1] + dv[2] * dv[2]);
            double gap = L - 2.0 * rp;
            if (gap <= 0) continue;
            double bound = 0.5 * L;
            double j = (rp - sd0 > 0) ? rp : sd0;
            for (int s = 0; s < steps; ++s) {
                if (margin && fabs(j - bound) < 1e-3) {
                    /* the sample at the exit exists on one side of j = bound only: a cost and
                     * gradient jump iff it is in contact (a free sample adds nothing and ends
                     * the sweep either way) */
                    double kb = j / L;
                    double pb[3] = {c[0] + kb * dv[0], c[1] + kb * dv[1], c[2] + kb * dv[2]};
                    double sdb = box_sdf_impl(pb, w->pos + 3 * k, w->quat + 4 * k, w->half + 3 * k, NULL, NULL);
                    if (rp - sdb > -1e-6) upd_margin_k(margin, j - bound, 4);
                }
                if (j >= bound) break;
                double kappa = j / L;
                double p[3] = {c[0] + kappa * dv[0], c[1] + kappa * dv[1], c[2] + kappa * dv[2]};
                double sdp;
                double phis = box_term(w, k, p, rp, eta, 1.0 - kappa, G, &sdp, margin);
                int hit = (rp - sdp > 0);
                if (counters) { counters[ORC_CNT_SWEEP_SAMPLES]++; if (hit) counters[ORC_CNT_SWEEP_HITS]++; }
                if (samples && n_samples && *n_samples < max_samples) {
                    double *sm = samples + 4 * (*n_samples);
                    sm[0] = k; sm[1] = dir; sm[2] = kappa; sm[3] = hit;
                    (*n_samples)++;
                }
                if (hit) { E += phis; j += rp; }
                else j += sdp;
            }
        }
    }
    return E;
}

/* ------------------------------------------------------------------------------------------ */
/* Self-collision: Eq. self-collision, Alg. 9, readings A28-A30        */
/* ------------------------------------------------------------------------------------------ */
double orc_self_collision(const orc_robot *rb, const double *spheres, double beta, double *g,
                          int *arg_pair, double *margin, long long *counters) {
    double best = -ORC_INF, second = -ORC_INF;
    int ibest = -1;
    for (int p = 0; p < rb->n_pairs; ++p) {
        int i = rb->pairs[2 * p], j = rb->pairs[2 * p + 1];
        double ri = rb->sph[i * 4 + 3] + (rb->sph_off ? rb->sph_off[i] : 0.0);
        double rj = rb->sph[j * 4 + 3] + (rb->sph_off ? rb->sph_off[j] : 0.0);
        if (ri <= 0.0 || rj <= 0.0) continue;            /* Alg. 9 "continue" */
        double dx = spheres[i * 4] - spheres[j * 4], dy = spheres[i * 4 + 1] - spheres[j * 4 + 1],
               dz = spheres[i * 4 + 2] - spheres[j * 4 + 2];
        double P = ri + rj - sqrt(dx * dx + dy * dy + dz * dz);
        if (counters) { counters[ORC_CNT_PAIR_TESTS]++; if (P > 0) counters[ORC_CNT_PAIR_PEN]++; }
        if (P > best) { second = best; best = P; ibest = p; }   /* first maximal pair (A28) */
        else if (P > second) second = P;
    }
    if (arg_pair) *arg_pair = -1;
    if (ibest < 0) return 0.0;
    upd_margin_grad(margin, best, 1);
    if (best <= 0) return 0.0;
    if (margin && second > -ORC_INF) upd_margin_grad(margin, best - second, 2);
    if (arg_pair) *arg_pair = ibest;
    int i = rb->pairs[2 * ibest], j = rb->pairs[2 * ibest + 1];
    double u[3] = {spheres[i * 4] - spheres[j * 4], spheres[i * 4 + 1] - spheres[j * 4 + 1],
                   spheres[i * 4 + 2] - spheres[j * 4 + 2]};
    double nu = sqrt(u[0] * u[0] + u[1] * u[1] + u[2] * u[2]);
    if (nu < 1e-12) { u[0] = 1; u[1] = 0; u[2] = 0; }
    else for (int t = 0; t < 3; ++t) u[t] /= nu;
    if (g)
        for (int t = 0; t < 3; ++t) {
            g[i * 3 + t] += -beta * u[t];
            g[j * 3 + t] += beta * u[t];
        }
    return beta * best;
}

/* ------------------------------------------------------------------------------------------ */
/* Bound, smoothness, pose (Appendix A)                                            */
/* ------------------------------------------------------------------------------------------ */

/* Eq. bound_cost, the five branches in the paper's order. */
double orc_bound(double x, double lo, double hi, double eta2, double *dx) {
    if (x < lo) { if (dx) *dx = -1.0; return lo - x + 0.5 * eta2; }
    if (lo + eta2 > x && x >= lo) {
        if (dx) *dx = -(lo - x + eta2) / eta2;
        return 0.5 / eta2 * (lo - x + eta2) * (lo - x + eta2);
    }
    if (x > hi) { if (dx) *dx = 1.0; return x - hi + 0.5 * eta2; }
    if (hi - eta2 < x && x <= hi) {
        if (dx) *dx = (x - hi + eta2) / eta2;
        return 0.5 / eta2 * (x - hi + eta2) * (x - hi + eta2);
    }
    if (dx) *dx = 0.0;
    return 0.0;
}

/* log cosh in the overflow-safe form |x| + log1p(exp(-2|x|)) - log 2. */
double orc_logcosh(double x) {
    double ax = fabs(x);
    return ax + log1p(exp(-2.0 * ax)) - log(2.0);
}

/* Eq. cspace-cost, the goal cost "for tasks that require reaching a joint
 * configuration": C = a4 logcosh(a5 ||theta_g - theta_T||_2^2);
 * dC/dtheta_T = a4 a5 tanh(a5 ||.||^2) * 2 (theta_T - theta_g). */
double orc_cspace_cost(const orc_params *pr, int D, const double *q, const double *goal, double *g) {
    double s = 0.0;
    for (int d = 0; d < D; ++d) s += (goal[d] - q[d]) * (goal[d] - q[d]);
    double C = pr->a4 * orc_logcosh(pr->a5 * s);
    if (g)
        for (int d = 0; d < D; ++d) g[d] = pr->a4 * pr->a5 * tanh(pr->a5 * s) * 2.0 * (q[d] - goal[d]);
    return C;
}

/* Eq. pose_cost_term with reading A1: e_r = 1 - |<q_g, q>|. */
double orc_pose_cost(const orc_params *pr, const double *ee, const double *goal, double *gp,
                     double *gq) {
    double ep[3] = {goal[0] - ee[0], goal[1] - ee[1], goal[2] - ee[2]};
    double n = sqrt(ep[0] * ep[0] + ep[1] * ep[1] + ep[2] * ep[2]);
    double d = goal[3] * ee[3] + goal[4] * ee[4] + goal[5] * ee[5] + goal[6] * ee[6];
    double er = 1.0 - fabs(d);
    double C = pr->a0 * orc_logcosh(pr->a2 * n) + pr->a1 * orc_logcosh(pr->a3 * er);
    if (gp) {
        /* dC/dp = -a0 a2 tanh(a2 n)/n e_p, limit -a0 a2^2 e_p as n -> 0 */
        double f = (n > 1e-12) ? tanh(pr->a2 * n) / n : pr->a2;
        for (int i = 0; i < 3; ++i) gp[i] = -pr->a0 * pr->a2 * f * ep[i];
    }
    if (gq) {
        double sg = (d >= 0) ? 1.0 : -1.0;
        double f = -pr->a1 * pr->a3 * tanh(pr->a3 * er) * sg;
        for (int i = 0; i < 4; ++i) gq[i] = f * goal[3 + i];
    }
    return C;
}

/* O2 state map (A14, Table 5 last row P:2097): x has H+5 rows, row i <-> h = i-2. */
void orc_state_map(const double *start, const double *V, int H, int D, double *x) {
#define XR(h) (x + ((h) + 2) * D)
    for (int h = 1; h <= H; ++h) memcpy(XR(h), V + (h - 1) * D, sizeof(double) * D);
    for (int h = 1; h <= 3; ++h) memcpy(XR(h), start, sizeof(double) * D);          /* pin   */
    for (int h = H - 3; h <= H - 1; ++h) memcpy(XR(h), XR(H), sizeof(double) * D);  /* alias */
    for (int h = -2; h <= 0; ++h) memcpy(XR(h), start, sizeof(double) * D);         /* pads  */
    for (int h = H + 1; h <= H + 2; ++h) memcpy(XR(h), XR(H), sizeof(double) * D);
#undef XR
}

/* O3 five-point stencil (§A.5; reading A15), at h = 1..H; outputs [H][D]. */
void orc_derivs(const double *x, int H, int D, double dt, double *v, double *a, double *j) {
#define X(h, d) x[((h) + 2) * D + (d)]
    for (int h = 1; h <= H; ++h)
        for (int d = 0; d < D; ++d) {
            double xm2 = X(h - 2, d), xm1 = X(h - 1, d), x0 = X(h, d), xp1 = X(h + 1, d), xp2 = X(h + 2, d);
            v[(h - 1) * D + d] = (-xp2 + 8 * xp1 - 8 * xm1 + xm2) / (12 * dt);
            a[(h - 1) * D + d] = (-xp2 + 16 * xp1 - 30 * x0 + 16 * xm1 - xm2) / (12 * dt * dt);
            j[(h - 1) * D + d] = (xp2 - 2 * xp1 + 2 * xm1 - xm2) / (2 * dt * dt * dt);
        }
#undef X
}

/* ------------------------------------------------------------------------------------------ */
/* O7: whole evaluation                                                                        */
/* ------------------------------------------------------------------------------------------ */

/* Per-configuration bound cost; returns cost, writes dC/dx into gx (may be NULL).
 * kind: 0 pos, 1 vel, 2 acc, 3 jerk. */
static double bound_vec(const orc_robot *rb, const orc_params *pr, int kind, const double *x,
                        double *gx, double *margin) {
    double c = 0.0;
    for (int d = 0; d < rb->n_dof; ++d) {
        double lo, hi;
        switch (kind) {
            case 0: lo = rb->lo[d]; hi = rb->hi[d]; break;
            case 1: lo = -rb->vmax[d]; hi = rb->vmax[d]; break;
            case 2: lo = -rb->amax[d]; hi = rb->amax[d]; break;
            default: lo = -rb->jmax[d]; hi = rb->jmax[d]; break;
        }
        double dx;
        c += pr->w_bound[kind] * orc_bound(x[d], lo, hi, pr->eta_bound, &dx);
        if (gx) gx[d] = pr->w_bound[kind] * dx;
    }
    return c;
}

double orc_eval_traj(const orc_robot *rb, const orc_world *w, const orc_params *pr,
                     const double *start, const double *goal, const double *V, int H,
                     double *grad, double *terms, double *margin, long long *counters) {
    int D = rb->n_dof, M = rb->n_spheres;
    g_margin_kind = 0;
    g_cost_margin = 1.0 / 0.0;
    if (g_state_margin)
        for (int h = 0; h < H; ++h) g_state_margin[h] = 1.0 / 0.0;
    double *x = calloc((size_t)(H + 5) * D, sizeof(double));
    double *v = calloc((size_t)H * D, sizeof(double)), *a = calloc((size_t)H * D, sizeof(double)),
           *jk = calloc((size_t)H * D, sizeof(double));
    double *gxf = calloc((size_t)(H + 5) * D, sizeof(double));      /* dC/dx_h, h = -2..H+2 */
    double *gv = calloc((size_t)H * D, sizeof(double)), *ga = calloc((size_t)H * D, sizeof(double)),
           *gj = calloc((size_t)H * D, sizeof(double));
    double *sph = calloc((size_t)(H + 1) * M * 4, sizeof(double));  /* w[h][m], h = 1..H */
    double *gs = calloc((size_t)(H + 1) * M * 3, sizeof(double));
    double *tmp = calloc((size_t)D, sizeof(double));
    double ee[7], tm[5] = {0, 0, 0, 0, 0};

    orc_state_map(start, V, H, D, x);                                /* O2 */
    orc_derivs(x, H, D, pr->dt, v, a, jk);                           /* O3 */
#define XR(h) (x + ((h) + 2) * D)
#define GX(h) (gxf + ((h) + 2) * D)
    for (int h = 1; h <= H; ++h) {
        /* bound (Eq. bound_cost) on pos/vel/acc/jerk and smoothness (Eq. smooth_cost, A16) */
        tm[1] += bound_vec(rb, pr, 0, XR(h), tmp, margin);
        for (int d = 0; d < D; ++d) GX(h)[d] += tmp[d];
        tm[1] += bound_vec(rb, pr, 1, v + (h - 1) * D, gv + (h - 1) * D, margin);
        tm[1] += bound_vec(rb, pr, 2, a + (h - 1) * D, ga + (h - 1) * D, margin);
        tm[1] += bound_vec(rb, pr, 3, jk + (h - 1) * D, gj + (h - 1) * D, margin);
        for (int d = 0; d < D; ++d) {
            double ad = a[(h - 1) * D + d], jd = jk[(h - 1) * D + d];
            tm[2] += pr->a8 * ad * ad;
            ga[(h - 1) * D + d] += 2 * pr->a8 * ad;
            if (pr->flags & ORC_JERK) {
                tm[2] += pr->a9 * jd * jd;
                gj[(h - 1) * D + d] += 2 * pr->a9 * jd;
            }
        }
        /* FK (O4) */
        orc_fk(rb, XR(h), NULL, sph + h * M * 4, (h == H) ? ee : NULL);
        /* self-collision (O5) */
        g_state_idx = h - 1;
        tm[3] += orc_self_collision(rb, sph + h * M * 4, pr->beta_self, gs + h * M * 3, NULL,
                                    margin, counters);
    }
    /* world: discrete + swept + speed (O5, Eq. world-collision-cost) */
    int sweep = (pr->flags & ORC_SWEEP) != 0;
    for (int h = 1; h <= H; ++h)
        for (int m = 0; m < M; ++m) {
            double r = rb->sph[m * 4 + 3];
            if (r < 0) continue;
            const double *c = sph + (h * M + m) * 4;
            g_state_idx = h - 1;
            const double *cp = (h > 1) ? sph + ((h - 1) * M + m) * 4 : NULL;
            const double *cn = (h < H) ? sph + ((h + 1) * M + m) * 4 : NULL;
            double sp = 1.0;
            if (pr->flags & ORC_SPEED) {                                 /* A13 */
                const double *pa = cp ? cp : c, *pb = cn ? cn : c;
                double dx = pb[0] - pa[0], dy = pb[1] - pa[1], dz = pb[2] - pa[2];
                sp = sqrt(dx * dx + dy * dy + dz * dz) / (2.0 * pr->dt);
            }
            double G[3] = {0, 0, 0};
            double E = orc_sphere_world(w, c, sweep ? cp : NULL, sweep ? cn : NULL, r, pr->eta, sweep,
                                        pr->sweep_steps, G, NULL, 0, NULL, margin, counters);
            if (counters && E > 0) counters[ORC_CNT_ACTIVE_SPHERES]++;
            tm[4] += pr->beta_world * sp * E;
            for (int i = 0; i < 3; ++i) gs[(h * M + m) * 3 + i] += pr->beta_world * sp * G[i];
        }
    /* goal term at x_H: Eq. pose_cost_term, or Eq. cspace-cost (goal = theta_g[D]) */
    double gp[3], gq[4];
    int cspace = (pr->flags & ORC_CSPACE) != 0;
    if (cspace) {
        tm[0] = orc_cspace_cost(pr, D, XR(H), goal, tmp);
        for (int d = 0; d < D; ++d) GX(H)[d] += tmp[d];
    } else {
        tm[0] = orc_pose_cost(pr, ee, goal, gp, gq);
        g_state_idx = H - 1;
        if (margin) upd_margin_grad(margin, goal[3] * ee[3] + goal[4] * ee[4] + goal[5] * ee[5] + goal[6] * ee[6], 5);
    }
    g_state_idx = -1;
    /* backward (O6) per evaluated configuration */
    for (int h = 1; h <= H; ++h) {
        int pose = (h == H) && !cspace;
        orc_fk_backward(rb, XR(h), gs + h * M * 3, pose ? gp : NULL, pose ? gq : NULL, tmp);
        for (int d = 0; d < D; ++d) GX(h)[d] += tmp[d];
    }
    /* transposed stencil: chain rule through O3 */
    for (int h = 1; h <= H; ++h)
        for (int d = 0; d < D; ++d) {
            double gvd = gv[(h - 1) * D + d], gad = ga[(h - 1) * D + d], gjd = gj[(h - 1) * D + d];
            double cv[5] = {1.0 / (12 * pr->dt), -8.0 / (12 * pr->dt), 0.0, 8.0 / (12 * pr->dt), -1.0 / (12 * pr->dt)};
            double dt2 = pr->dt * pr->dt, dt3 = dt2 * pr->dt;
            double ca[5] = {-1.0 / (12 * dt2), 16.0 / (12 * dt2), -30.0 / (12 * dt2), 16.0 / (12 * dt2), -1.0 / (12 * dt2)};
            double cj[5] = {-1.0 / (2 * dt3), 2.0 / (2 * dt3), 0.0, -2.0 / (2 * dt3), 1.0 / (2 * dt3)};
            for (int o = -2; o <= 2; ++o) GX(h + o)[d] += cv[o + 2] * gvd + ca[o + 2] * gad + cj[o + 2] * gjd;
        }
    /* transposed state map (O2 gradient routing) */
    if (grad) {
        memset(grad, 0, sizeof(double) * (size_t)H * D);
        for (int h = 4; h <= H - 4; ++h)
            for (int d = 0; d < D; ++d) grad[(h - 1) * D + d] = GX(h)[d];
        for (int d = 0; d < D; ++d) {
            double s = GX(H)[d] + GX(H - 1)[d] + GX(H - 2)[d] + GX(H - 3)[d] + GX(H + 1)[d] + GX(H + 2)[d];
            grad[(H - 1) * D + d] = s;
        }
    }
#undef XR
#undef GX
    if (terms) memcpy(terms, tm, sizeof(tm));
    double C = tm[0] + tm[1] + tm[2] + tm[3] + tm[4];
    free(x); free(v); free(a); free(jk); free(gxf); free(gv); free(ga); free(gj);
    free(sph); free(gs); free(tmp);
    return C;
}

/* IK mode (A34): pose + self + discrete world (speed 1) + position bound. */
double orc_eval_ik(const orc_robot *rb, const orc_world *w, const orc_params *pr,
                   const double *goal, const double *q, double *grad, double *terms,
                   double *margin, long long *counters) {
    int D = rb->n_dof, M = rb->n_spheres;
    g_margin_kind = 0;
    g_cost_margin = 1.0 / 0.0;
    if (g_state_margin) g_state_margin[0] = 1.0 / 0.0;
    g_state_idx = 0;
    double *sph = calloc((size_t)M * 4, sizeof(double)), *gs = calloc((size_t)M * 3, sizeof(double));
    double *gb = calloc((size_t)D, sizeof(double));
    double ee[7], tm[5] = {0, 0, 0, 0, 0};
    orc_fk(rb, q, NULL, sph, ee);
    tm[1] = bound_vec(rb, pr, 0, q, gb, margin);
    tm[3] = orc_self_collision(rb, sph, pr->beta_self, gs, NULL, margin, counters);
    for (int m = 0; m < M; ++m) {
        double r = rb->sph[m * 4 + 3];
        if (r < 0) continue;
        double G[3] = {0, 0, 0};
        double E = orc_sphere_world(w, sph + m * 4, NULL, NULL, r, pr->eta, 0, 0, G, NULL, 0, NULL,
                                    margin, counters);
        if (counters && E > 0) counters[ORC_CNT_ACTIVE_SPHERES]++;
        tm[4] += pr->beta_world * E;
        for (int i = 0; i < 3; ++i) gs[m * 3 + i] += pr->beta_world * G[i];
    }
    double gp[3], gq[4];
    int cspace = (pr->flags & ORC_CSPACE) != 0;
    double *gc = calloc(D, sizeof(double));
    if (cspace) {
        tm[0] = orc_cspace_cost(pr, D, q, goal, gc);          /* Eq. cspace-cost */
    } else {
        tm[0] = orc_pose_cost(pr, ee, goal, gp, gq);
        if (margin) upd_margin_grad(margin, goal[3] * ee[3] + goal[4] * ee[4] + goal[5] * ee[5] + goal[6] * ee[6], 5);
    }
    g_state_idx = -1;
    if (grad) {
        orc_fk_backward(rb, q, gs, cspace ? NULL : gp, cspace ? NULL : gq, grad);
        for (int d = 0; d < D; ++d) grad[d] += gb[d] + gc[d];
    }
    free(gc);
    if (terms) memcpy(terms, tm, sizeof(tm));
    free(sph); free(gs); free(gb);
    return tm[0] + tm[1] + tm[2] + tm[3] + tm[4];
}

/* ------------------------------------------------------------------------------------------ */
/* O8: L-BFGS (Alg. 6) + parallel noisy line search (Alg. 1)           */
/* ------------------------------------------------------------------------------------------ */

static double dot(int n, const double *a, const double *b) {
    double s = 0.0;
    for (int i = 0; i < n; ++i) s += a[i] * b[i];
    return s;
}

/* Two-loop recursion (Nocedal & Wright, Alg. 6) over `count` stored pairs, index 0
 * oldest .. count-1 newest; H0 = gamma I, gamma = s^T y / y^T y of the newest pair (A19), 1 if
 * empty; d = -r (A18). */
void orc_lbfgs_direction(int n, int count, const double *S, const double *Y, const double *rho,
                         const double *g, double *d) {
    double *q = malloc(sizeof(double) * (size_t)n);
    double alpha[64];
    memcpy(q, g, sizeof(double) * (size_t)n);
    for (int i = count - 1; i >= 0; --i) {
        alpha[i] = rho[i] * dot(n, S + (size_t)i * n, q);
        for (int t = 0; t < n; ++t) q[t] -= alpha[i] * Y[(size_t)i * n + t];
    }
    double gamma = 1.0;
    if (count > 0) {
        const double *s = S + (size_t)(count - 1) * n, *y = Y + (size_t)(count - 1) * n;
        gamma = dot(n, s, y) / dot(n, y, y);
    }
    for (int t = 0; t < n; ++t) q[t] *= gamma;       /* r = H0 q */
    for (int i = 0; i < count; ++i) {
        double beta = rho[i] * dot(n, Y + (size_t)i * n, q);
        for (int t = 0; t < n; ++t) q[t] += (alpha[i] - beta) * S[(size_t)i * n + t];
    }
    for (int t = 0; t < n; ++t) d[t] = -q[t];
    free(q);
}

/* Alg. 1 lines 4-9 in fp64 (A17, A22): Armijo c_a <= c0 + c1 alpha_a g0d; Wolfe g_a^T d >= c2 g0d;
 * strong |g_a^T d| <= c2 |g0d|; largest index with all conditions true, else 0. */
int orc_ls_select(int A, const double *alpha, double c0, double g0d, const double *ca,
                  const double *gda, double c1, double c2, int mode) {
    int best = 0;
    for (int a = 0; a < A; ++a) {
        int ok = ca[a] <= c0 + (c1 * alpha[a]) * g0d;
        if (mode == 1) ok = ok && (gda[a] >= c2 * g0d);
        if (mode == 2) ok = ok && (fabs(gda[a]) <= c2 * fabs(g0d));
        if (ok) best = a;
    }
    return best;
}

/* fp32 mirror of the pure selection function: fixed operation order, no FMA
 * contraction (-ffp-contract=off), NaN compares false. */
int orc_ls_select_f32(int A, const float *alpha, float c0, float g0d, const float *ca,
                      const float *gda, float c1, float c2, int mode) {
    int best = 0;
    for (int a = 0; a < A; ++a) {
        volatile float t1 = c1 * alpha[a];
        volatile float t2 = t1 * g0d;
        volatile float rhs = c0 + t2;
        int ok = ca[a] <= rhs;
        if (mode == 1) { volatile float w = c2 * g0d; ok = ok && (gda[a] >= w); }
        if (mode == 2) { volatile float w = c2 * fabsf(g0d); ok = ok && (fabsf(gda[a]) <= w); }
        if (ok) best = a;
    }
    return best;
}

/* O9 selection: argmin with ties to the lowest index, NaN treated as +inf. */
int orc_argmin_f32(int n, const float *c) {
    int best = 0;
    float bv = (c[0] != c[0]) ? (float)ORC_INF : c[0];
    for (int i = 1; i < n; ++i) {
        float v = (c[i] != c[i]) ? (float)ORC_INF : c[i];
        if (v < bv) { bv = v; best = i; }
    }
    return best;
}

/* ------------------------------------------------------------------------------------------ */
/* O13 motion-generation pipeline pieces (§2 / Fig. 2, Alg. 4, App. B; */
/* readings B15-B18)                                                                           */
/* ------------------------------------------------------------------------------------------ */

/* Alg. 4 retime ("find dt that pushes trajectory to robot limits (velocity, acceleration or
 * jerk)"), reading B15 after SPEC S:515: with v, a, j the five-point-stencil derivatives (O3) of
 * the state sequence (O2 state map of V with `start`) at dt, over h = 1..H and every joint,
 *   s = max(1e-3, max(|v|/vmax, sqrt(|a|/amax), cbrt(|j|/jmax)));  dt_opt = s dt.
 * Time scaling by s divides v, a, j by s, s^2, s^3, so at dt_opt every derivative is within its
 * limit and the binding one sits on it.  ratio_out[3] (may be NULL) = the three maxima at dt. */
double orc_retime(const orc_robot *rb, const double *start, const double *V, int H, double dt,
                  double *ratio_out) {
    int D = rb->n_dof;
    double *x = malloc(sizeof(double) * (H + 5) * D), *v = malloc(sizeof(double) * H * D),
           *a = malloc(sizeof(double) * H * D), *j = malloc(sizeof(double) * H * D);
    orc_state_map(start, V, H, D, x);
    orc_derivs(x, H, D, dt, v, a, j);
    double rv = 0.0, ra = 0.0, rj = 0.0;
    for (int h = 0; h < H; ++h)
        for (int d = 0; d < D; ++d) {
            double qv = fabs(v[h * D + d]) / rb->vmax[d];
            double qa = sqrt(fabs(a[h * D + d]) / rb->amax[d]);
            double qj = cbrt(fabs(j[h * D + d]) / rb->jmax[d]);
            if (qv > rv) rv = qv;
            if (qa > ra) ra = qa;
            if (qj > rj) rj = qj;
        }
    double sc = rv;
    if (ra > sc) sc = ra;
    if (rj > sc) sc = rj;
    if (sc < 1e-3) sc = 1e-3;
    if (ratio_out) { ratio_out[0] = rv; ratio_out[1] = ra; ratio_out[2] = rj; }
    free(x); free(v); free(a); free(j);
    return sc;
}

/* Alg. 4 "scale_traj_opt(dt_opt)" + "enable_jerk_cost()", reading B15: the smoothness weights are
 * rescaled so that the terms keep their magnitude when the same path is re-timed from dt_ref to
 * dt (a ~ dt^-2, j ~ dt^-3): a8 (dt/dt_ref)^4, a9 (dt/dt_ref)^6; the limit (bound) weights are
 * physical constraints and stay. */
void orc_scale_params(const orc_params *in, double dt, double dt_ref, int jerk_on, orc_params *out) {
    *out = *in;
    double r = dt / dt_ref;
    out->dt = dt;
    /* P:2053 "scale all our cost terms that relate to velocity, acceleration, and jerk": each term
     * keeps its magnitude when the same path is re-timed from dt_ref to dt (reading B15): the
     * squared acceleration / jerk by r^4 / r^6, the velocity / acceleration / jerk limit terms
     * (slope 1 in the derivative beyond the band) by r, r^2, r^3; the position limit term stays. */
    out->a8 = in->a8 * r * r * r * r;
    out->a9 = in->a9 * r * r * r * r * r * r;
    out->w_bound[1] = in->w_bound[1] * r;
    out->w_bound[2] = in->w_bound[2] * r * r;
    out->w_bound[3] = in->w_bound[3] * r * r * r;
    if (jerk_on) out->flags |= ORC_JERK;
}

/* Goal errors of a configuration (App. B P:2190 "pose error"): position |p_g - p|_2 and
 * orientation 1 - |<q_g, q>| (reading A1). */
void orc_goal_error(const orc_robot *rb, const double *q, const double *goal, double *pos_err,
                    double *rot_err) {
    int L = rb->n_links, M = rb->n_spheres;
    double *T = malloc(sizeof(double) * 12 * L), *sph = malloc(sizeof(double) * 4 * M), ee[7];
    orc_fk(rb, q, T, sph, ee);
    double dx = goal[0] - ee[0], dy = goal[1] - ee[1], dz = goal[2] - ee[2];
    *pos_err = sqrt(dx * dx + dy * dy + dz * dz);
    *rot_err = 1.0 - fabs(goal[3] * ee[3] + goal[4] * ee[4] + goal[5] * ee[5] + goal[6] * ee[6]);
    free(T); free(sph);
}

/* Linear TO seed ("linear interpolation from the start configuration to the solved terminal
 * configuration"), reading B17: V_h = start + (h / (H-1)) (q_T - start), h = 0..H-1. */
void orc_linear_seed(const double *start, const double *qT, int H, int D, double *V) {
    for (int h = 0; h < H; ++h)
        for (int d = 0; d < D; ++d) V[h * D + d] = start[d] + ((double)h / (H - 1)) * (qT[d] - start[d]);
}

/* Interpolation of a solved trajectory to a fine time grid ("interpolate the trajectory
 * to a fixed dt of 0.025 to validate success"; reading B21): the states x_1..x_H sit at
 * t = 0, dt, .., (H-1) dt; the fine grid t_k = min(k dt_fine, T), k = 0..n-1 with T = (H-1) dt and
 * n = ceil(T / dt_fine) + 1 (so the last point is x_H), decided in fp64; linear in joint space
 * between the bracketing states: i = min(floor(t_k / dt), H - 2), f = t_k / dt - i,
 * x(t_k) = (1 - f) x_i + f x_{i+1}.  Writes min(n, n_max) points of out [n_max][D]; returns n. */
int orc_interpolate(const double *x, int H, int D, double dt, double dt_fine, int n_max, double *out) {
    const double T = (H - 1) * dt;
    const int n = (int)ceil(T / dt_fine) + 1;
    for (int k = 0; k < n && k < n_max; ++k) {
        double t = k * dt_fine;
        double u = (t >= T) ? (double)(H - 1) : t / dt;        /* the last point is x_H exactly */
        int i = (int)floor(u);
        if (i > H - 2) i = H - 2;
        double f = u - i;
        for (int d = 0; d < D; ++d) out[k * D + d] = (1.0 - f) * x[i * D + d] + f * x[(i + 1) * D + d];
    }
    return n;
}

/* Scores (App. B, reading B18).  IK: "a lowest weighted sum of pose error and the
 * distance of the solution to the current joint configuration":
 *   w_pose (pos_err + rot_err) + w_dist |q - q_0|_2.
 * TO: "a blended sum of the pose error, maximum jerk, and motion time":
 *   w_pose (pos_err + rot_err) + w_jerk max|j| + w_time (H - 1) dt  (after retiming). */
double orc_ik_score(int D, const double *q, const double *q0, double pos_err, double rot_err,
                    double w_pose, double w_dist) {
    double s2 = 0.0;
    for (int d = 0; d < D; ++d) s2 += (q[d] - q0[d]) * (q[d] - q0[d]);
    return w_pose * (pos_err + rot_err) + w_dist * sqrt(s2);
}

double orc_blended_score(double pos_err, double rot_err, double max_jerk, double motion_time,
                         double w_pose, double w_jerk, double w_time) {
    return w_pose * (pos_err + rot_err) + w_jerk * max_jerk + w_time * motion_time;
}

/* ------------------------------------------------------------------------------------------ */
/* O12 validity mask and parallel steering (Alg. 3; readings B12-B14) */
/* ------------------------------------------------------------------------------------------ */

/* mask_samples (Alg. 3 line 5, "check for validity"), reading B12: a configuration is valid iff
 * every joint is inside its position limits, no self-collision pair of S penetrates
 * ((r_i+o_i) + (r_j+o_j) - |w_i - w_j| <= 0, pairs with r+o <= 0 skipped as in Alg. 9), and every
 * enabled sphere (r >= 0) keeps sd_k(c) >= r + margin to every enabled cuboid (strict
 * non-penetration with a safety margin).  margin_out (may be NULL) = the smallest distance of a
 * decision quantity to its threshold (for fp32-vs-fp64 parity filtering). */
int orc_mask_sample(const orc_robot *rb, const orc_world *w, const double *q, double margin,
                    double *margin_out) {
    int D = rb->n_dof, M = rb->n_spheres, L = rb->n_links;
    int valid = 1;
    double mg = ORC_INF;
    for (int d = 0; d < D; ++d) {
        double a = q[d] - rb->lo[d], b = rb->hi[d] - q[d];
        if (a < 0 || b < 0) valid = 0;
        if (fabs(a) < mg) mg = fabs(a);
        if (fabs(b) < mg) mg = fabs(b);
    }
    double *T = malloc(sizeof(double) * 12 * L), *sph = malloc(sizeof(double) * 4 * M), ee[7];
    orc_fk(rb, q, T, sph, ee);
    for (int p = 0; p < rb->n_pairs; ++p) {
        int i = rb->pairs[2 * p], j = rb->pairs[2 * p + 1];
        double ri = rb->sph[i * 4 + 3] + (rb->sph_off ? rb->sph_off[i] : 0.0);
        double rj = rb->sph[j * 4 + 3] + (rb->sph_off ? rb->sph_off[j] : 0.0);
        if (ri <= 0.0 || rj <= 0.0) continue;
        double dx = sph[i * 4] - sph[j * 4], dy = sph[i * 4 + 1] - sph[j * 4 + 1],
               dz = sph[i * 4 + 2] - sph[j * 4 + 2];
        double P = ri + rj - sqrt(dx * dx + dy * dy + dz * dz);
        if (P > 0) valid = 0;
        if (fabs(P) < mg) mg = fabs(P);
    }
    for (int m = 0; m < M; ++m) {
        double r = rb->sph[m * 4 + 3];
        if (r < 0) continue;
        for (int k = 0; k < w->n_boxes; ++k) {
            if (!w->enabled[k]) continue;
            double sd = orc_box_sdf(sph + m * 4, w->pos + 3 * k, w->quat + 4 * k, w->half + 3 * k, NULL);
            if (sd < r + margin) valid = 0;
            if (fabs(sd - (r + margin)) < mg) mg = fabs(sd - (r + margin));
        }
    }
    free(T); free(sph);
    if (margin_out) *margin_out = mg;
    return valid;
}

/* Alg. 3 (Parallel Steering) under reading B13, for E edges (src_e, dst_e):
 *   g_e = d_w * (dst_e - src_e)                       (distvec, per-joint weighted)
 *   n = floor(max_{e,j} |g_ej| / r) + 1               (line 2, ONE n shared by the batch)
 *   l_ei = src_e + (i / n) (dst_e - src_e), i = 0..n  (lines 3-4)
 *   mask = validity of every l_ei                     (line 5)
 *   h_e = (first invalid i) - 1, or n if none          (lines 6-7)
 *   v_new_e = l_e,h_e; dist_e = |d_w * (v_new_e - src_e)|_2   (lines 8-9)
 * h_e = -1 (source invalid, outside Alg. 3's precondition) gives v_new = src and dist 0.
 * Returns n; margin_out[E] (may be NULL) = the smallest decision margin over each edge's
 * waypoints up to and including its first invalid one. */
int orc_steer(const orc_robot *rb, const orc_world *w, int E, const double *src, const double *dst,
              const double *dw, double r, double margin, int *h, double *v_new, double *dist,
              double *margin_out) {
    int D = rb->n_dof;
    double gmax = 0.0;
    for (int e = 0; e < E; ++e)
        for (int d = 0; d < D; ++d) {
            double gv = fabs(dw[d] * (dst[e * D + d] - src[e * D + d]));
            if (gv > gmax) gmax = gv;
        }
    int n = (int)floor(gmax / r) + 1;
    double *l = malloc(sizeof(double) * D);
    for (int e = 0; e < E; ++e) {
        int first = -1;
        double me = ORC_INF;
        for (int i = 0; i <= n; ++i) {
            for (int d = 0; d < D; ++d)
                l[d] = src[e * D + d] + ((double)i / n) * (dst[e * D + d] - src[e * D + d]);
            double mi;
            int ok = orc_mask_sample(rb, w, l, margin, &mi);
            if (mi < me) me = mi;
            if (!ok) { first = i; break; }
        }
        int he = first < 0 ? n : first - 1;
        h[e] = he;
        double s2 = 0.0;
        for (int d = 0; d < D; ++d) {
            double v = he < 0 ? src[e * D + d]
                              : src[e * D + d] + ((double)he / n) * (dst[e * D + d] - src[e * D + d]);
            v_new[e * D + d] = v;
            double gd = dw[d] * (v - src[e * D + d]);
            s2 += gd * gd;
        }
        dist[e] = sqrt(s2);
        if (margin_out) margin_out[e] = me;
    }
    free(l);
    return n;
}

/* ------------------------------------------------------------------------------------------ */
/* O11 particle-based warm-up (§4.2 "Particle-Based Optimization"; Alg. 5,          */
/* P:2130-2144; two iterations before L-BFGS)                                          */
/* ------------------------------------------------------------------------------------------ */

/* Counter-based generator for the particle draws (reading B9).  Philox4x32-10 as published by
 * Salmon et al. (SC'11): 10 rounds of two 32x32->64 multiplies with M0 = 0xD2511F53,
 * M1 = 0xCD9E8D57, the key bumped by the Weyl constants W0 = 0x9E3779B9, W1 = 0xBB67AE85 after
 * every round.  Pinned by the published known-answer vectors (tests/test_oracle_particle.py). */
void orc_philox4x32(const unsigned key[2], const unsigned ctr[4], unsigned out[4]) {
    unsigned k0 = key[0], k1 = key[1];
    unsigned x0 = ctr[0], x1 = ctr[1], x2 = ctr[2], x3 = ctr[3];
    for (int r = 0; r < 10; ++r) {
        unsigned long long p0 = (unsigned long long)0xD2511F53u * x0;
        unsigned long long p1 = (unsigned long long)0xCD9E8D57u * x2;
        unsigned hi0 = (unsigned)(p0 >> 32), lo0 = (unsigned)p0;
        unsigned hi1 = (unsigned)(p1 >> 32), lo1 = (unsigned)p1;
        unsigned y0 = hi1 ^ x1 ^ k0, y1 = lo1, y2 = hi0 ^ x3 ^ k1, y3 = lo0;
        x0 = y0; x1 = y1; x2 = y2; x3 = y3;
        k0 += 0x9E3779B9u; k1 += 0xBB67AE85u;
    }
    out[0] = x0; out[1] = x1; out[2] = x2; out[3] = x3;
}

/* theta_s ~ N(0, 1) for variable `var` of particle `particle` in iteration `iter` of a seed
 * (B9): Philox(key = (key0, key1), ctr = (var / 4, particle, iter, seed)) gives 4 words; words
 * (0,1) and (2,3) are two Box-Muller pairs with 24-bit uniforms u1 = (w_a >> 8 + 1) 2^-24 in
 * (0, 1], u2 = (w_b >> 8) 2^-24 in [0, 1): z = sqrt(-2 ln u1) (cos | sin)(2 pi u2); variable
 * var takes output var % 4 (cos for even, sin for odd). */
double orc_normal(unsigned key0, unsigned key1, unsigned var, unsigned particle, unsigned iter,
                  unsigned seed) {
    unsigned key[2] = {key0, key1}, ctr[4] = {var >> 2, particle, iter, seed}, w[4];
    orc_philox4x32(key, ctr, w);
    int j = (int)(var & 3u), a = (j >> 1) * 2;
    double u1 = ((double)(w[a] >> 8) + 1.0) / 16777216.0;
    double u2 = (double)(w[a + 1] >> 8) / 16777216.0;
    double r = sqrt(-2.0 * log(u1));
    const double two_pi = 6.283185307179586476925286766559;
    return (j & 1) ? r * sin(two_pi * u2) : r * cos(two_pi * u2);
}

/* Alg. 5: mu <- Theta_init, sigma <- sigma_0; for each iteration: Theta_l <- SAMPLE(mu, sigma)
 * (theta_l = mu + sqrt(Theta_sigma) * theta_s, clipped to the box constraints, B7);
 * c_l <- C(Theta_l) (cost only); UPDATE: c = -C/beta, w = e^{c_i} / sum e^{c_i} (the max is
 * subtracted first: the same ratio), Eq. particle_1 mu = (1-k_mu) mu + k_mu sum_i w_i theta_i,
 * Eq. particle_2 as read in B6: sigma = (1-k_sigma) sigma + k_sigma sum_i w_i (theta_i - mu_prev)^2
 * (diagonal covariance).  A non-finite cost gets weight 0; if every weight is 0 the iteration
 * leaves (mu, sigma) unchanged (B10).  cost_trace[it * n + l] = c_l (may be NULL). */
void orc_particle_solve(orc_fun f, void *ctx, int n, const double *x0, const double *lo,
                        const double *hi, const orc_particle *pp, unsigned problem,
                        unsigned seed, double *mu, double *var, double *cost_trace) {
    int L = pp->n;
    double *theta = malloc(sizeof(double) * (size_t)L * n);
    double *C = malloc(sizeof(double) * L), *w = malloc(sizeof(double) * L);
    for (int v = 0; v < n; ++v) {
        double s0 = pp->sigma0_frac * (hi[v] - lo[v]);
        mu[v] = x0[v];
        var[v] = s0 * s0;
    }
    for (int it = 0; it < pp->iters; ++it) {
        /* SAMPLE */
        for (int l = 0; l < L; ++l)
            for (int v = 0; v < n; ++v) {
                double z = orc_normal(pp->key, problem, (unsigned)v, (unsigned)l, (unsigned)it, seed);
                double x = mu[v] + sqrt(var[v]) * z;
                if (x < lo[v]) x = lo[v];
                if (x > hi[v]) x = hi[v];
                theta[(size_t)l * n + v] = x;
            }
        /* C(Theta_l), cost only */
        for (int l = 0; l < L; ++l) {
            C[l] = f(ctx, theta + (size_t)l * n, NULL);
            if (cost_trace) cost_trace[(size_t)it * L + l] = C[l];
        }
        /* UPDATE: exponential utility */
        double cmax = -ORC_INF;
        for (int l = 0; l < L; ++l) {
            double cl = -C[l] / pp->beta;
            if (isfinite(C[l]) && cl > cmax) cmax = cl;
        }
        if (!(cmax > -ORC_INF)) continue;            /* B10: no finite particle */
        double Z = 0.0;
        for (int l = 0; l < L; ++l) {
            w[l] = isfinite(C[l]) ? exp(-C[l] / pp->beta - cmax) : 0.0;
            Z += w[l];
        }
        for (int l = 0; l < L; ++l) w[l] /= Z;
        for (int v = 0; v < n; ++v) {
            double m1 = 0.0, m2 = 0.0;
            for (int l = 0; l < L; ++l) {
                double x = theta[(size_t)l * n + v];
                m1 += w[l] * x;                                   /* w * theta (Eq. particle_1) */
                m2 += w[l] * (x - mu[v]) * (x - mu[v]);   /* B6: mu[v] is still Theta_mu-1 here */
            }
            mu[v] = (1.0 - pp->k_mu) * mu[v] + pp->k_mu * m1;
            var[v] = (1.0 - pp->k_sigma) * var[v] + pp->k_sigma * m2;
        }
    }
    free(theta); free(C); free(w);
}

/* O8 steps 1-2, Alg. 6 lines 1-5 ("Shift Buffers"): the pair of the last move,
 * s = x - xp, y = g - gp, joins the history ring S, Y [m][n] (oldest first), rho [m] holding
 * `count` pairs, unless s'y <= 1e-12 (A20, the pair is skipped); a full ring drops its oldest
 * pair first.  Returns the new count; *sy_out = s'y (O10: |s'y - 1e-12| is the skip margin).
 * m = 0 is gradient descent: nothing is ever stored. */
int orc_lbfgs_push(int n, int m, double *S, double *Y, double *rho, int count, const double *x,
                   const double *xp, const double *g, const double *gp, double *sy_out) {
    double *s = malloc(sizeof(double) * (size_t)n), *y = malloc(sizeof(double) * (size_t)n);
    for (int t = 0; t < n; ++t) { s[t] = x[t] - xp[t]; y[t] = g[t] - gp[t]; }
    double sy = dot(n, s, y);
    if (sy_out) *sy_out = sy;
    if (m > 0 && sy > 1e-12) {                    /* A20 */
        if (count == m) {                         /* shift buffers: drop the oldest pair */
            memmove(S, S + n, sizeof(double) * (size_t)(m - 1) * n);
            memmove(Y, Y + n, sizeof(double) * (size_t)(m - 1) * n);
            memmove(rho, rho + 1, sizeof(double) * (m - 1));
            count = m - 1;
        }
        memcpy(S + (size_t)count * n, s, sizeof(double) * n);
        memcpy(Y + (size_t)count * n, y, sizeof(double) * n);
        rho[count] = 1.0 / sy;
        count++;
    }
    free(s); free(y);
    return count;
}

/* O10 solver margin of one line search (Alg. 1 lines 4-9): the smallest distance of an active
 * condition to its decision point, over the A candidates: |c_a - (c0 + c1 alpha_a g0d)| (Armijo),
 * |g_a'd - c2 g0d| (Wolfe, mode 1), ||g_a'd| - c2 |g0d|| (strong Wolfe, mode 2). */
double orc_ls_margin(int A, const double *alpha, double c0, double g0d, const double *ca,
                     const double *gda, double c1, double c2, int mode) {
    double mg = ORC_INF;
    for (int a = 0; a < A; ++a) {
        mg = fmin(mg, fabs(ca[a] - (c0 + (c1 * alpha[a]) * g0d)));
        if (mode == 1) mg = fmin(mg, fabs(gda[a] - c2 * g0d));
        if (mode == 2) mg = fmin(mg, fabs(fabs(gda[a]) - c2 * fabs(g0d)));
    }
    return mg;
}

/* O8 per-seed solver in fp64: evaluate at x0, then `iters` iterations of
 * L-BFGS step -> clipped candidates -> batched evaluation -> selection -> best update.
 * tr (may be NULL; every member may be NULL) records each iteration (O10 instrumentation). */
void orc_lbfgs_solve_traced(orc_fun f, void *ctx, int n, const double *x0, const double *lo,
                            const double *hi, const orc_solver *sp, double *best_x, double *best_c,
                            orc_solver_trace *tr) {
    int m = sp->history, A = sp->n_alpha;
    double *x = malloc(sizeof(double) * n), *g = malloc(sizeof(double) * n);
    double *xp = malloc(sizeof(double) * n), *gpv = malloc(sizeof(double) * n);
    double *d = malloc(sizeof(double) * n);
    size_t mm = m > 0 ? (size_t)m : 1;
    double *S = malloc(sizeof(double) * mm * n), *Y = malloc(sizeof(double) * mm * n);
    double *rho = malloc(sizeof(double) * mm);
    double *xa = malloc(sizeof(double) * (size_t)A * n), *ga = malloc(sizeof(double) * (size_t)A * n);
    double ca[8], gda[8];
    int count = 0;
    memcpy(x, x0, sizeof(double) * n);
    double c = f(ctx, x, g);
    double bc = c;
    memcpy(best_x, x, sizeof(double) * n);
    for (int it = 0; it <= sp->iters; ++it) {
        if (tr) {                                     /* the iterate entering iteration it */
            if (tr->x) memcpy(tr->x + (size_t)it * n, x, sizeof(double) * n);
            if (tr->g) memcpy(tr->g + (size_t)it * n, g, sizeof(double) * n);
            if (tr->c) tr->c[it] = c;
            if (tr->best_c) tr->best_c[it] = bc;
        }
        if (it == sp->iters) break;
        double sy = ORC_NAN;
        if (it > 0) count = orc_lbfgs_push(n, m, S, Y, rho, count, x, xp, g, gpv, &sy);   /* A21: none at 0 */
        memcpy(xp, x, sizeof(double) * n);
        memcpy(gpv, g, sizeof(double) * n);
        orc_lbfgs_direction(n, count, S, Y, rho, g, d);
        double g0d = dot(n, g, d);
        for (int a = 0; a < A; ++a) {
            double *xc = xa + (size_t)a * n;
            for (int t = 0; t < n; ++t) {                 /* clip (A35) */
                double v = x[t] + sp->alpha[a] * d[t];
                if (lo && v < lo[t]) v = lo[t];
                if (hi && v > hi[t]) v = hi[t];
                xc[t] = v;
            }
            ca[a] = f(ctx, xc, ga + (size_t)a * n);
            gda[a] = dot(n, ga + (size_t)a * n, d);
        }
        int i = orc_ls_select(A, sp->alpha, c, g0d, ca, gda, sp->c1, sp->c2, sp->ls_mode);
        if (tr) {
            if (tr->d) memcpy(tr->d + (size_t)it * n, d, sizeof(double) * n);
            if (tr->g0d) tr->g0d[it] = g0d;
            for (int a = 0; a < A; ++a) {
                if (tr->ca) tr->ca[it * 8 + a] = ca[a];
                if (tr->gda) tr->gda[it * 8 + a] = gda[a];
            }
            if (tr->istar) tr->istar[it] = i;
            if (tr->count) tr->count[it] = count;
            if (tr->sy) tr->sy[it] = sy;
            if (tr->ls_margin)
                tr->ls_margin[it] = orc_ls_margin(A, sp->alpha, c, g0d, ca, gda, sp->c1, sp->c2, sp->ls_mode);
        }
        memcpy(x, xa + (size_t)i * n, sizeof(double) * n);
        memcpy(g, ga + (size_t)i * n, sizeof(double) * n);
        c = ca[i];
        if (c < bc) { bc = c; memcpy(best_x, x, sizeof(double) * n); }   /* A23 strict < */
    }
    *best_c = bc;
    free(x); free(g); free(xp); free(gpv); free(d); free(S); free(Y); free(rho); free(xa); free(ga);
}

void orc_lbfgs_solve(orc_fun f, void *ctx, int n, const double *x0, const double *lo,
                     const double *hi, const orc_solver *sp, double *best_x, double *best_c,
                     double *trace) {
    orc_solver_trace tr;
    memset(&tr, 0, sizeof(tr));
    tr.best_c = trace;                                /* best cost after each iteration */
    orc_lbfgs_solve_traced(f, ctx, n, x0, lo, hi, sp, best_x, best_c, trace ? &tr : NULL);
}

/* ---- rollout objectives and threaded multi-seed solves (timing harness for cpu_baseline) ---- */
typedef struct {
    const orc_robot *rb; const orc_world *w; const orc_params *pr;
    const double *start, *goal; int H;
} traj_ctx;

static double traj_fun(void *vctx, const double *x, double *g) {
    traj_ctx *c = vctx;
    return orc_eval_traj(c->rb, c->w, c->pr, c->start, c->goal, x, c->H, g, NULL, NULL, NULL);
}

static double ik_fun(void *vctx, const double *x, double *g) {
    traj_ctx *c = vctx;
    return orc_eval_ik(c->rb, c->w, c->pr, c->goal, x, g, NULL, NULL, NULL);
}

typedef struct {
    const orc_robot *rb; const orc_world *worlds; const int *env; const orc_params *pr;
    const orc_solver *sp; int P, S, H, ik; const double *seeds, *start, *goal;
    double *out_x, *out_c; int tid, nthreads;
} solve_job;

static void *solve_worker(void *arg) {
    solve_job *jb = arg;
    int D = jb->rb->n_dof, N = jb->ik ? D : jb->H * D;
    double *lo = malloc(sizeof(double) * N), *hi = malloc(sizeof(double) * N);
    for (int t = 0; t < N; ++t) { lo[t] = jb->rb->lo[t % D]; hi[t] = jb->rb->hi[t % D]; }
    for (int u = jb->tid; u < jb->P * jb->S; u += jb->nthreads) {
        int p = u / jb->S;
        traj_ctx ctx = {jb->rb, jb->worlds + (jb->env ? jb->env[p] : 0), jb->pr,
                        jb->start ? jb->start + (size_t)p * D : NULL, jb->goal + (size_t)p * 7, jb->H};
        const double *x0 = jb->seeds + (size_t)u * N;
        double *mu = NULL, *var = NULL;
        if (jb->sp->pt.iters > 0) {                   /* O11 warm-up, then L-BFGS from its mean */
            mu = malloc(sizeof(double) * N); var = malloc(sizeof(double) * N);
            orc_particle_solve(jb->ik ? ik_fun : traj_fun, &ctx, N, x0, lo, hi, &jb->sp->pt,
                               (unsigned)(jb->sp->problem_base + p),
                               (unsigned)(jb->sp->seed_base + (u - p * jb->S)), mu, var, NULL);
            x0 = mu;
        }
        orc_lbfgs_solve(jb->ik ? ik_fun : traj_fun, &ctx, N, x0, lo, hi, jb->sp,
                        jb->out_x + (size_t)u * N, jb->out_c + u, NULL);
        free(mu); free(var);
    }
    free(lo); free(hi);
    return NULL;
}

static void solve_threads(solve_job base, int nthreads) {
    if (nthreads < 1) nthreads = 1;
    pthread_t th[256];
    solve_job jobs[256];
    if (nthreads > 256) nthreads = 256;
    for (int t = 0; t < nthreads; ++t) {
        jobs[t] = base; jobs[t].tid = t; jobs[t].nthreads = nthreads;
        pthread_create(&th[t], NULL, solve_worker, &jobs[t]);
    }
    for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
}

void orc_solve_to(const orc_robot *rb, const orc_world *worlds, const int *env,
                  const orc_params *pr, const orc_solver *sp, int P, int S, int H,
                  const double *seeds, const double *start, const double *goal, int nthreads,
                  double *seed_best_traj, double *seed_best_cost) {
    solve_job b = {rb, worlds, env, pr, sp, P, S, H, 0, seeds, start, goal, seed_best_traj,
                   seed_best_cost, 0, 1};
    solve_threads(b, nthreads);
}

void orc_solve_ik(const orc_robot *rb, const orc_world *worlds, const int *env,
                  const orc_params *pr, const orc_solver *sp, int P, int S,
                  const double *seeds, const double *goal, int nthreads,
                  double *seed_best_q, double *seed_best_cost) {
    solve_job b = {rb, worlds, env, pr, sp, P, S, 1, 1, seeds, NULL, goal, seed_best_q,
                   seed_best_cost, 0, 1};
    solve_threads(b, nthreads);
}
