// crb_device.cuh -- sm_100a device code of the fused cost+gradient evaluation (one CTA, 32
// configurations per pass) shared by the evaluate, FK and persistent-solver kernels.
//
// Mapping: a CTA of NT = 512 threads (16 warps); the 32 lanes of every
// warp are the 32 configuration slots of the pass (TO: the H timesteps of one candidate
// trajectory; IK: 32 seeds of one problem).  Warps split the kinematic-chain rows (FK), the
// spheres (world collision), the pair list (self-collision) and the (dof, config) elements; all
// cross-warp combination goes through shared memory in a fixed order, so every result is
// bitwise deterministic.  The robot tables and this environment's cuboids are staged into shared
// memory once per CTA with TMA bulk copies (cp.async.bulk + mbarrier).
//
// P:n = line n of the paper; A* = readings listed in DESIGN.md.
#pragma once
#include <cstdint>

namespace crb {

constexpr int NT = 512;          // threads per CTA
constexpr int NW = NT / 32;      // warps per CTA
constexpr int NC = 32;           // configuration slots per pass (= lanes)
constexpr unsigned FULL = 0xffffffffu;

enum : unsigned { F_SWEEP = 1u, F_SPEED = 2u, F_JERK = 4u };
enum { MODE_TO = 0, MODE_IK = 1 };

// Packed robot tables (built by the host in crb_set_robot).  Offsets are in 4-byte words from
// the start of the blob; every section starts on a 16-byte boundary.
struct RobotPack {
    int L, D, M, P, ee;
    int o_links;    // L x 16 words: F[12] (3x4 row-major), parent, type, dof, pad
    int o_sph;      // M float4 (centre in link frame, radius), spheres grouped by link
    int o_sphlink;  // M ints
    int o_sbeg;     // L+1 ints: spheres of link l are [sbeg[l], sbeg[l+1])
    int o_pairs;    // P x 2 words: (i | j << 16), float bits of r_i+o_i+r_j+o_j
    int o_lim;      // 5 x D floats: lo, hi, vmax, amax, jmax
    int o_doflink;  // D ints: link carrying dof d
    int o_perm;     // M ints: packed sphere index -> caller's sphere index
    int words;      // total (multiple of 4)
};

// Shared-memory layout (offsets in 4-byte words from the dynamic smem base).
struct Layout {
    int robot, boxes, mbar;
    int q_cfg, xs, lt, sw, sg, ls, sbest, sidx, wpart, cbb, csm, gxd, gva, pose_ft, pose_c,
        goal, cfg_cost, cfg_terms, gV, red, st;
    int solver;      // start of the solver region
    int total;       // words
    int XS;          // row length of xs (H + 5)
};

struct KParams {
    RobotPack rp;
    Layout lay;
    const float4 *robot;     // packed robot blob (global)
    const float4 *boxes;     // [n_env][kmax][4] float4: (R col i, -col_i . t) x3, (h, 0)
    const int *box_count;    // [n_env] enabled (compacted) boxes
    int kmax, n_env;
    // cost parameters (App. A)
    float a0, a1, a2, a3, a8, a9, wb[4], beta_self, beta_world, eta, eta_bound, dt;
    int sweep_steps;
    unsigned flags;
    // solver parameters (Alg. 6, Alg. 1)
    int iters, m, A, ls_mode;
    float alpha[8], c1, c2;
    long long seed_base;
    // problem
    int mode, H, S, P, B;
    const float *q_in;
    const int *env;
    const float *start, *goal;
    float *cost_out, *grad_out, *terms_out, *spheres_out, *ee_out;
    float *seed_best_cost, *seed_best_traj;
};

// ------------------------------------------------------------------------------------------
// small helpers
// ------------------------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ float warp_sum(float v) {
    // xor butterfly: every lane ends with the same bits (fp addition is commutative)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
    return v;
}

// Deterministic CTA-wide sum of one value per thread (fixed order over warps).
__device__ __forceinline__ float block_sum(float v, float *red) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    v = warp_sum(v);
    if (lane == 0) red[warp] = v;
    __syncthreads();
    float s = 0.f;
#pragma unroll
    for (int w = 0; w < NW; ++w) s += red[w];
    __syncthreads();
    return s;
}

// TMA bulk copy global -> shared, completion on an mbarrier (SASS: UBLKCP / SYNCS).
__device__ __forceinline__ void mbar_init(uint64_t *bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, unsigned phase) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
        "r"(phase)
        : "memory");
}

// Stage the robot tables and environment `env`'s cuboids into shared memory (one TMA bulk copy
// each, P:3014 float4 layout).  Must be called by all threads; ends with the data visible.
__device__ __forceinline__ int stage_tables(const KParams &kp, float *smem, int env) {
    uint64_t *bar = reinterpret_cast<uint64_t *>(smem + kp.lay.mbar);
    int K = (env >= 0 && env < kp.n_env) ? kp.box_count[env] : 0;
    if (threadIdx.x == 0) {
        mbar_init(bar, 1);
        uint32_t rbytes = (uint32_t)kp.rp.words * 4u;
        uint32_t bbytes = (uint32_t)K * 64u;
        mbar_expect_tx(bar, rbytes + bbytes);
        bulk_g2s(smem + kp.lay.robot, kp.robot, rbytes, bar);
        if (K > 0) bulk_g2s(smem + kp.lay.boxes, kp.boxes + (size_t)env * kp.kmax * 4, bbytes, bar);
    }
    __syncthreads();
    mbar_wait(bar, 0);
    return K;
}

// ------------------------------------------------------------------------------------------
// scalar pieces of the method
// ------------------------------------------------------------------------------------------

// Eq. smooth-distance-cases in penetration-positive form d' = r' - sd (A2).
__device__ __forceinline__ float activation(float dp, float eta, float &dphi) {
    if (dp <= 0.f) { dphi = 0.f; return 0.f; }
    if (dp <= eta) { dphi = dp / eta; return dp * dp / (2.f * eta); }
    dphi = 1.f;
    return dp - 0.5f * eta;
}

// Eq. bound_cost, the five branches in the paper's order.
__device__ __forceinline__ float bound_cost(float x, float lo, float hi, float e2, float &dx) {
    if (x < lo) { dx = -1.f; return lo - x + 0.5f * e2; }
    if (lo + e2 > x && x >= lo) { float t = lo - x + e2; dx = -t / e2; return 0.5f / e2 * t * t; }
    if (x > hi) { dx = 1.f; return x - hi + 0.5f * e2; }
    if (hi - e2 < x && x <= hi) { float t = x - hi + e2; dx = t / e2; return 0.5f / e2 * t * t; }
    dx = 0.f;
    return 0.f;
}

// log cosh accurate in fp32 for all x: log1p(2 sinh^2(x/2)) for |x| < 5, else the
// overflow-safe |x| + log1p(exp(-2|x|)) - log 2.
__device__ __forceinline__ float logcoshf(float x) {
    float ax = fabsf(x);
    if (ax < 5.f) {
        float s = sinhf(0.5f * ax);
        return log1pf(2.f * s * s);
    }
    return ax + log1pf(expf(-2.f * ax)) - 0.69314718055994531f;
}

// Signed distance of a point to one cuboid stored as 4 float4 (R columns with -col.t, half
// extents): exact Euclidean box SDF (A4).  Returns sd; `out` = outside flag; writes the local
// gradient on request.
struct BoxView {
    float4 c0, c1, c2, h;
};

__device__ __forceinline__ BoxView load_box(const float *boxes, int k) {
    const float4 *b = reinterpret_cast<const float4 *>(boxes) + 4 * k;
    return BoxView{b[0], b[1], b[2], b[3]};
}

__device__ __forceinline__ void box_local(const BoxView &b, float px, float py, float pz, float &lx,
                                          float &ly, float &lz) {
    lx = fmaf(b.c0.x, px, fmaf(b.c0.y, py, fmaf(b.c0.z, pz, b.c0.w)));
    ly = fmaf(b.c1.x, px, fmaf(b.c1.y, py, fmaf(b.c1.z, pz, b.c1.w)));
    lz = fmaf(b.c2.x, px, fmaf(b.c2.y, py, fmaf(b.c2.z, pz, b.c2.w)));
}

// Full SDF + world-frame gradient at a point (used on hits and sweep samples).
__device__ __forceinline__ float box_sdf_grad(const BoxView &b, float px, float py, float pz, float &gx,
                                              float &gy, float &gz) {
    float lx, ly, lz;
    box_local(b, px, py, pz, lx, ly, lz);
    float qx = fabsf(lx) - b.h.x, qy = fabsf(ly) - b.h.y, qz = fabsf(lz) - b.h.z;
    float qm = fmaxf(qx, fmaxf(qy, qz));
    float glx = 0.f, gly = 0.f, glz = 0.f, sd;
    if (qm > 0.f) {
        float mx = fmaxf(qx, 0.f), my = fmaxf(qy, 0.f), mz = fmaxf(qz, 0.f);
        sd = sqrtf(mx * mx + my * my + mz * mz);
        float inv = 1.f / sd;
        glx = copysignf(mx * inv, lx >= 0.f ? 1.f : -1.f);
        gly = copysignf(my * inv, ly >= 0.f ? 1.f : -1.f);
        glz = copysignf(mz * inv, lz >= 0.f ? 1.f : -1.f);
    } else {
        sd = qm;  // first arg-max in x, y, z order; sign(0) = +1
        if (qx >= qy && qx >= qz) glx = lx >= 0.f ? 1.f : -1.f;
        else if (qy >= qz) gly = ly >= 0.f ? 1.f : -1.f;
        else glz = lz >= 0.f ? 1.f : -1.f;
    }
    // grad sd (world) = R grad_loc = sum_i grad_loc_i * col_i
    gx = glx * b.c0.x + gly * b.c1.x + glz * b.c2.x;
    gy = glx * b.c0.y + gly * b.c1.y + glz * b.c2.y;
    gz = glx * b.c0.z + gly * b.c1.z + glz * b.c2.z;
    return sd;
}

// Alg. 1 lines 4-9 in fp32 with a fixed operation order and no FMA contraction (the same
// function runs in the solver and in the crb_ls_select test hook).
__device__ __forceinline__ int ls_select(int A, const float *alpha, float c0, float g0d, const float *ca,
                                         const float *gda, float c1, float c2, int mode) {
    int best = 0;
    for (int a = 0; a < A; ++a) {
        float rhs = __fadd_rn(c0, __fmul_rn(__fmul_rn(c1, alpha[a]), g0d));
        bool ok = ca[a] <= rhs;
        if (mode == 1) ok = ok && (gda[a] >= __fmul_rn(c2, g0d));
        if (mode == 2) ok = ok && (fabsf(gda[a]) <= __fmul_rn(c2, fabsf(g0d)));
        if (ok) best = a;
    }
    return best;
}

// Packed selection key (O9, north star): (float bits of c << 32) | seed; NaN -> +inf bits.
__device__ __forceinline__ unsigned long long pack_key(float c, long long seed) {
    unsigned bits;
    if (c != c) bits = 0x7f800000u;
    else if (c == 0.f) bits = 0u;
    else bits = __float_as_uint(c);
    return ((unsigned long long)bits << 32) | (unsigned long long)(unsigned)(seed & 0xffffffffll);
}

// Candidate of the line search (Alg. 1 line 1, A35): clip(theta + alpha d, lo, hi).  One
// function everywhere so the recomputed winner is bitwise the evaluated candidate.
__device__ __forceinline__ float candidate(float th, float alpha, float d, float lo, float hi) {
    return fminf(fmaxf(__fmaf_rn(alpha, d, th), lo), hi);
}

// ------------------------------------------------------------------------------------------
// the fused evaluation pass over 32 configuration slots
// ------------------------------------------------------------------------------------------
struct Smem {
    const int *iw;          // robot blob as ints
    const float *fw;        // robot blob as floats
    const float *boxes;
    float *q_cfg, *xs, *lt, *sw, *sg, *ls, *sbest, *wpart, *cbb, *csm, *gxd, *gva, *pose_ft, *pose_c,
        *goal, *cfg_cost, *cfg_terms, *gV, *red, *st;
    int *sidx;
};

__device__ __forceinline__ Smem make_smem(const KParams &kp, float *smem) {
    const Layout &L = kp.lay;
    Smem s;
    s.iw = reinterpret_cast<const int *>(smem + L.robot);
    s.fw = smem + L.robot;
    s.boxes = smem + L.boxes;
    s.q_cfg = smem + L.q_cfg; s.xs = smem + L.xs; s.lt = smem + L.lt; s.sw = smem + L.sw;
    s.sg = smem + L.sg; s.ls = smem + L.ls; s.sbest = smem + L.sbest;
    s.sidx = reinterpret_cast<int *>(smem + L.sidx);
    s.wpart = smem + L.wpart; s.cbb = smem + L.cbb; s.csm = smem + L.csm; s.gxd = smem + L.gxd;
    s.gva = smem + L.gva; s.pose_ft = smem + L.pose_ft; s.pose_c = smem + L.pose_c;
    s.goal = smem + L.goal; s.cfg_cost = smem + L.cfg_cost; s.cfg_terms = smem + L.cfg_terms;
    s.gV = smem + L.gV; s.red = smem + L.red; s.st = smem + L.st;
    return s;
}

// Forward kinematics of the 32 slots (Alg. 7 / Table 6): warps 0..2 each own one row of the
// 3x4 link transforms (the paper's "parallel threads per matrix"), lane = slot.  Writes
// lt[l][12][32]; then every warp places its spheres: sw[m][3][32] = R_link c_m + t_link.
__device__ __forceinline__ void fk_phase(const KParams &kp, const Smem &s) {
    const RobotPack &rp = kp.rp;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (warp < 3) {
        const int r = warp;
        float4 cur = make_float4(0.f, 0.f, 0.f, 0.f);
        for (int l = 0; l < rp.L; ++l) {
            const float *F = s.fw + rp.o_links + 16 * l;
            const int parent = s.iw[rp.o_links + 16 * l + 12];
            const int type = s.iw[rp.o_links + 16 * l + 13];
            const int dof = s.iw[rp.o_links + 16 * l + 14];
            float4 pr;
            if (parent < 0) pr = make_float4(r == 0, r == 1, r == 2, 0.f);
            else if (parent == l - 1) pr = cur;
            else {
                const float *src = s.lt + (parent * 12 + r * 4) * NC + lane;
                pr = make_float4(src[0], src[NC], src[2 * NC], src[3 * NC]);
            }
            // local transform M = F * J(v): Table 6 "Full Link Transformation" column (A25 fixed)
            float m00 = F[0], m01 = F[1], m02 = F[2], m03 = F[3];
            float m10 = F[4], m11 = F[5], m12 = F[6], m13 = F[7];
            float m20 = F[8], m21 = F[9], m22 = F[10], m23 = F[11];
            if (type != 0) {
                const float v = s.q_cfg[dof * NC + lane];
                if (type <= 3) {           // prismatic: col3 += v * col_axis
                    if (type == 1) { m03 = fmaf(m00, v, m03); m13 = fmaf(m10, v, m13); m23 = fmaf(m20, v, m23); }
                    else if (type == 2) { m03 = fmaf(m01, v, m03); m13 = fmaf(m11, v, m13); m23 = fmaf(m21, v, m23); }
                    else { m03 = fmaf(m02, v, m03); m13 = fmaf(m12, v, m13); m23 = fmaf(m22, v, m23); }
                } else {
                    float sn, cs;
                    sincosf(v, &sn, &cs);
                    if (type == 4) {        // revolute x: col1' = c f1 + s f2, col2' = -s f1 + c f2
                        float a0 = m01, a1 = m11, a2 = m21;
                        m01 = cs * a0 + sn * m02; m11 = cs * a1 + sn * m12; m21 = cs * a2 + sn * m22;
                        m02 = -sn * a0 + cs * m02; m12 = -sn * a1 + cs * m12; m22 = -sn * a2 + cs * m22;
                    } else if (type == 5) { // revolute y: col0' = c f0 - s f2, col2' = s f0 + c f2
                        float a0 = m00, a1 = m10, a2 = m20;
                        m00 = cs * a0 - sn * m02; m10 = cs * a1 - sn * m12; m20 = cs * a2 - sn * m22;
                        m02 = sn * a0 + cs * m02; m12 = sn * a1 + cs * m12; m22 = sn * a2 + cs * m22;
                    } else {                // revolute z: col0' = c f0 + s f1, col1' = -s f0 + c f1
                        float a0 = m00, a1 = m10, a2 = m20;
                        m00 = cs * a0 + sn * m01; m10 = cs * a1 + sn * m11; m20 = cs * a2 + sn * m21;
                        m01 = -sn * a0 + cs * m01; m11 = -sn * a1 + cs * m11; m21 = -sn * a2 + cs * m21;
                    }
                }
            }
            float4 nr;
            nr.x = pr.x * m00 + pr.y * m10 + pr.z * m20;
            nr.y = pr.x * m01 + pr.y * m11 + pr.z * m21;
            nr.z = pr.x * m02 + pr.y * m12 + pr.z * m22;
            nr.w = pr.x * m03 + pr.y * m13 + pr.z * m23 + pr.w;
            float *dst = s.lt + (l * 12 + r * 4) * NC + lane;
            dst[0] = nr.x; dst[NC] = nr.y; dst[2 * NC] = nr.z; dst[3 * NC] = nr.w;
            cur = nr;
        }
    }
    __syncthreads();
    const float4 *sph = reinterpret_cast<const float4 *>(s.fw + rp.o_sph);
    for (int m = warp; m < rp.M; m += NW) {
        const int l = s.iw[rp.o_sphlink + m];
        const float4 c = sph[m];
        const float *T = s.lt + l * 12 * NC + lane;
        float wx = T[0] * c.x + T[NC] * c.y + T[2 * NC] * c.z + T[3 * NC];
        float wy = T[4 * NC] * c.x + T[5 * NC] * c.y + T[6 * NC] * c.z + T[7 * NC];
        float wz = T[8 * NC] * c.x + T[9 * NC] * c.y + T[10 * NC] * c.z + T[11 * NC];
        float *dst = s.sw + m * 3 * NC + lane;
        dst[0] = wx; dst[NC] = wy; dst[2 * NC] = wz;
    }
    __syncthreads();
}

// Matrix -> quaternion (Shepperd), canonical w >= 0 (A31).
__device__ __forceinline__ void mat_to_quat(float r00, float r01, float r02, float r10, float r11, float r12,
                                            float r20, float r21, float r22, float q[4]) {
    float tr = r00 + r11 + r22;
    float w, x, y, z;
    if (tr >= r00 && tr >= r11 && tr >= r22) {
        w = 0.5f * sqrtf(1.f + tr); float k = 0.25f / w;
        x = (r21 - r12) * k; y = (r02 - r20) * k; z = (r10 - r01) * k;
    } else if (r00 >= r11 && r00 >= r22) {
        x = 0.5f * sqrtf(1.f + r00 - r11 - r22); float k = 0.25f / x;
        w = (r21 - r12) * k; y = (r01 + r10) * k; z = (r02 + r20) * k;
    } else if (r11 >= r22) {
        y = 0.5f * sqrtf(1.f - r00 + r11 - r22); float k = 0.25f / y;
        w = (r02 - r20) * k; x = (r01 + r10) * k; z = (r12 + r21) * k;
    } else {
        z = 0.5f * sqrtf(1.f - r00 - r11 + r22); float k = 0.25f / z;
        w = (r10 - r01) * k; x = (r02 + r20) * k; y = (r12 + r21) * k;
    }
    if (w < 0.f) { w = -w; x = -x; y = -y; z = -z; }
    q[0] = w; q[1] = x; q[2] = y; q[3] = z;
}

// World term of one sphere at one slot (Alg. 10 discrete + §3.4 / Algs. 11-12 swept under
// readings A6-A12; O5 in DESIGN.md).  Accumulates E and dE/dc (before beta_2 * speed).
__device__ __forceinline__ float sphere_world(const float *boxes, int K, float cx, float cy, float cz, float rp,
                                              float eta, bool doB, float bx, float by, float bz, float LB,
                                              bool doF, float fx, float fy, float fz, float LF, int steps,
                                              float &Gx, float &Gy, float &Gz) {
    float E = 0.f;
    const float boundB = 0.5f * LB, boundF = 0.5f * LF;
    float maxb = 0.f;
    if (doB) maxb = boundB;
    if (doF) maxb = fmaxf(maxb, boundF);
    const float rp2 = rp * rp, maxb2 = maxb * maxb;
    for (int k = 0; k < K; ++k) {
        const BoxView b = load_box(boxes, k);
        float lx, ly, lz;
        box_local(b, cx, cy, cz, lx, ly, lz);
        const float qx = fabsf(lx) - b.h.x, qy = fabsf(ly) - b.h.y, qz = fabsf(lz) - b.h.z;
        const float qm = fmaxf(qx, fmaxf(qy, qz));
        const float mx = fmaxf(qx, 0.f), my = fmaxf(qy, 0.f), mz = fmaxf(qz, 0.f);
        const float s2 = mx * mx + my * my + mz * mz;
        const bool hit = (qm <= 0.f) || (s2 < rp2);
        const bool sweep = (doB || doF) && (hit || s2 < maxb2);
        if (!hit && !sweep) continue;
        float sd0 = 0.f;
        if (hit) {
            float gx, gy, gz;
            sd0 = box_sdf_grad(b, cx, cy, cz, gx, gy, gz);
            float dphi;
            const float phi = activation(rp - sd0, eta, dphi);
            E += phi;
            Gx -= dphi * gx; Gy -= dphi * gy; Gz -= dphi * gz;
        } else {
            sd0 = sqrtf(s2);
        }
        if (!sweep) continue;
        const float J0 = (rp - sd0 > 0.f) ? rp : sd0;
#pragma unroll
        for (int dir = 0; dir < 2; ++dir) {
            const bool on = dir == 0 ? doB : doF;
            if (!on) continue;
            const float L = dir == 0 ? LB : LF, bound = dir == 0 ? boundB : boundF;
            const float vx = dir == 0 ? bx : fx, vy = dir == 0 ? by : fy, vz = dir == 0 ? bz : fz;
            float j = J0;
            for (int st = 0; st < steps; ++st) {
                if (j >= bound) break;
                const float kap = j / L;
                const float px = fmaf(kap, vx, cx), py = fmaf(kap, vy, cy), pz = fmaf(kap, vz, cz);
                float gx, gy, gz;
                const float sd = box_sdf_grad(b, px, py, pz, gx, gy, gz);
                const float dp = rp - sd;
                if (dp > 0.f) {
                    float dphi;
                    E += activation(dp, eta, dphi);
                    const float w = (1.f - kap) * dphi;
                    Gx -= w * gx; Gy -= w * gy; Gz -= w * gz;
                    j += rp;
                } else {
                    j += sd;
                }
            }
        }
    }
    return E;
}

// One evaluation pass over the 32 slots.  Inputs already in shared memory:
//   TO: s.gV is NOT an input; the candidate V[H][D] is in `thA`, start in s.st, goal in s.goal.
//   IK: configurations in s.q_cfg[D][32], goals in s.goal[7][32].
// Outputs: s.cfg_cost[32], s.cfg_terms[5][32]; TO: s.gV[H][D] = dC/dV; IK: s.gV[D][32].
// n_act = number of valid slots (TO: H, IK: active seeds).
template <int MODE>
__device__ void eval_pass(const KParams &kp, const Smem &s, const float *thA, int K, int n_act) {
    const RobotPack &rp = kp.rp;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int D = rp.D, H = kp.H, XS = kp.lay.XS;
    const float *lim = s.fw + rp.o_lim;

    // ---- a2: state map (O2, Table 5 last row) into xs[D][H+5] and the slot configurations
    if (MODE == MODE_TO) {
        for (int idx = tid; idx < D * XS; idx += NT) {
            const int d = idx / XS, i = idx - d * XS, h = i - 2;
            float v;
            if (h <= 3) v = s.st[d];
            else if (h >= H - 3) v = thA[(H - 1) * D + d];
            else v = thA[(h - 1) * D + d];
            s.xs[idx] = v;
        }
        for (int idx = tid; idx < D * NC; idx += NT) {
            const int d = idx / NC, c = idx - d * NC;
            const int h = c + 1 <= H ? c + 1 : H;
            float v;
            if (h <= 3) v = s.st[d];
            else if (h >= H - 3) v = thA[(H - 1) * D + d];
            else v = thA[(h - 1) * D + d];
            s.q_cfg[idx] = v;
        }
        __syncthreads();
    }

    // ---- a3: forward kinematics
    fk_phase(kp, s);

    // ---- a4: self-collision (Eq. self-collision, Alg. 9): warp w scans pairs w, w+NW, ...;
    // lane = slot; first maximal pair per warp (strict >), merged in pair order below (A28).
    {
        float best = 0.f;
        int bidx = -1;
        const uint2 *pairs = reinterpret_cast<const uint2 *>(s.iw + rp.o_pairs);
        for (int p = warp; p < rp.P; p += NW) {
            const uint2 pr = pairs[p];
            const int i = pr.x & 0xffff, j = pr.x >> 16;
            const float R = __uint_as_float(pr.y);
            const float *wi = s.sw + i * 3 * NC + lane, *wj = s.sw + j * 3 * NC + lane;
            const float dx = wi[0] - wj[0], dy = wi[NC] - wj[NC], dz = wi[2 * NC] - wj[2 * NC];
            const float d2 = dx * dx + dy * dy + dz * dz;
            if (d2 < R * R) {
                const float pen = R - sqrtf(d2);
                if (pen > best) { best = pen; bidx = p; }
            }
        }
        s.sbest[warp * NC + lane] = best;
        s.sidx[warp * NC + lane] = bidx;
    }

    // ---- a5/a6: world collision, discrete + swept + speed (Eq. world-collision-cost)
    {
        float wsum = 0.f;
        const bool to = MODE == MODE_TO;
        const bool sweepf = to && (kp.flags & F_SWEEP);
        const bool speedf = to && (kp.flags & F_SPEED);
        const float4 *sph = reinterpret_cast<const float4 *>(s.fw + rp.o_sph);
        const bool hasp = to && lane > 0 && lane < H;
        const bool hasn = to && lane + 1 < H;
        for (int m = warp; m < rp.M; m += NW) {
            float *g = s.sg + m * 3 * NC + lane;
            const float r = sph[m].w;
            float Gx = 0.f, Gy = 0.f, Gz = 0.f;
            float Ew = 0.f;
            if (r >= 0.f) {   // r < 0 disables the sphere (Alg. 10)
                const float *w = s.sw + m * 3 * NC + lane;
                const float cx = w[0], cy = w[NC], cz = w[2 * NC];
                float px = cx, py = cy, pz = cz, nx = cx, ny = cy, nz = cz;
                if (hasp) { px = w[-1]; py = w[NC - 1]; pz = w[2 * NC - 1]; }
                if (hasn) { nx = w[1]; ny = w[NC + 1]; nz = w[2 * NC + 1]; }
                float sp = 1.f;
                if (speedf) {   // A13: central difference, missing neighbour -> w_h
                    const float ddx = nx - px, ddy = ny - py, ddz = nz - pz;
                    sp = sqrtf(ddx * ddx + ddy * ddy + ddz * ddz) / (2.f * kp.dt);
                }
                if (sp != 0.f) {
                    const float rpr = r + kp.eta;   // Alg. 10 "sph.radius += eta"
                    const float bx = px - cx, by = py - cy, bz = pz - cz;
                    const float fx = nx - cx, fy = ny - cy, fz = nz - cz;
                    const float LB = sqrtf(bx * bx + by * by + bz * bz);
                    const float LF = sqrtf(fx * fx + fy * fy + fz * fz);
                    const bool doB = sweepf && hasp && (LB - 2.f * rpr > 0.f);   // A6
                    const bool doF = sweepf && hasn && (LF - 2.f * rpr > 0.f);
                    const float E = sphere_world(s.boxes, K, cx, cy, cz, rpr, kp.eta, doB, bx, by, bz, LB, doF,
                                                 fx, fy, fz, LF, kp.sweep_steps, Gx, Gy, Gz);
                    const float sc = kp.beta_world * sp;
                    Ew = sc * E;
                    Gx *= sc; Gy *= sc; Gz *= sc;
                }
            }
            g[0] = Gx; g[NC] = Gy; g[2 * NC] = Gz;
            wsum += Ew;
        }
        s.wpart[warp * NC + lane] = wsum;
    }

    // ---- a8: bound (Eq. bound_cost) on pos/vel/acc/jerk and smoothness (Eq. smooth_cost)
    for (int idx = tid; idx < D * NC; idx += NT) {
        const int d = idx / NC, c = idx - d * NC;
        float cb = 0.f, cs = 0.f, gx = 0.f, gv = 0.f, ga = 0.f, gj = 0.f;
        if (c < n_act) {
            const float lo = lim[d], hi = lim[D + d];
            float dd;
            if (MODE == MODE_TO) {
                const float *x = s.xs + d * XS + c + 3;   // x_h with h = c + 1
                const float xm2 = x[-2], xm1 = x[-1], x0 = x[0], xp1 = x[1], xp2 = x[2];
                const float dt = kp.dt, dt2 = dt * dt, dt3 = dt2 * dt;
                // O3 five-point stencil (§A.5, A15)
                const float v = (-xp2 + 8.f * xp1 - 8.f * xm1 + xm2) / (12.f * dt);
                const float a = (-xp2 + 16.f * xp1 - 30.f * x0 + 16.f * xm1 - xm2) / (12.f * dt2);
                const float j = (xp2 - 2.f * xp1 + 2.f * xm1 - xm2) / (2.f * dt3);
                const float vm = lim[2 * D + d], am = lim[3 * D + d], jm = lim[4 * D + d];
                cb += kp.wb[0] * bound_cost(x0, lo, hi, kp.eta_bound, dd); gx = kp.wb[0] * dd;
                cb += kp.wb[1] * bound_cost(v, -vm, vm, kp.eta_bound, dd); gv = kp.wb[1] * dd;
                cb += kp.wb[2] * bound_cost(a, -am, am, kp.eta_bound, dd); ga = kp.wb[2] * dd;
                cb += kp.wb[3] * bound_cost(j, -jm, jm, kp.eta_bound, dd); gj = kp.wb[3] * dd;
                cs = kp.a8 * a * a;
                ga += 2.f * kp.a8 * a;
                if (kp.flags & F_JERK) { cs += kp.a9 * j * j; gj += 2.f * kp.a9 * j; }
            } else {
                const float x0 = s.q_cfg[d * NC + c];
                cb = kp.wb[0] * bound_cost(x0, lo, hi, kp.eta_bound, dd);
                gx = kp.wb[0] * dd;
            }
        }
        s.cbb[idx] = cb; s.csm[idx] = cs; s.gxd[idx] = gx;
        if (MODE == MODE_TO) { s.gva[idx] = gv; s.gva[D * NC + idx] = ga; s.gva[2 * D * NC + idx] = gj; }
    }

    // ---- a7: pose cost (Eq. pose_cost_term, A1) at the terminal slot (TO) / every slot (IK)
    if (warp == NW - 1) {
        const int c = lane;
        const bool on = (MODE == MODE_TO) ? (c == H - 1) : (c < n_act);
        float ft[6] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f}, C = 0.f;
        if (on) {
            const float *T = s.lt + rp.ee * 12 * NC + c;
            const float px = T[3 * NC], py = T[7 * NC], pz = T[11 * NC];
            float q[4];
            mat_to_quat(T[0], T[NC], T[2 * NC], T[4 * NC], T[5 * NC], T[6 * NC], T[8 * NC], T[9 * NC],
                        T[10 * NC], q);
            const float *G = s.goal;   // [7][32]
            const float ex = G[0 * NC + c] - px, ey = G[1 * NC + c] - py, ez = G[2 * NC + c] - pz;
            const float n = sqrtf(ex * ex + ey * ey + ez * ez);
            const float gw = G[3 * NC + c], gxq = G[4 * NC + c], gyq = G[5 * NC + c], gzq = G[6 * NC + c];
            const float dq = gw * q[0] + gxq * q[1] + gyq * q[2] + gzq * q[3];
            const float er = 1.f - fabsf(dq);
            C = kp.a0 * logcoshf(kp.a2 * n) + kp.a1 * logcoshf(kp.a3 * er);
            const float f = (n > 1e-12f) ? tanhf(kp.a2 * n) / n : kp.a2;
            const float kpo = -kp.a0 * kp.a2 * f;
            const float gpx = kpo * ex, gpy = kpo * ey, gpz = kpo * ez;
            const float kq = -kp.a1 * kp.a3 * tanhf(kp.a3 * er) * (dq >= 0.f ? 1.f : -1.f);
            const float gqw = kq * gw, gqx = kq * gxq, gqy = kq * gyq, gqz = kq * gzq;
            // torque of the quaternion gradient: tau = 1/2 (w g_v - g_w v + v x g_v)  (A27)
            const float tx = 0.5f * (q[0] * gqx - gqw * q[1] + (q[2] * gqz - q[3] * gqy));
            const float ty = 0.5f * (q[0] * gqy - gqw * q[2] + (q[3] * gqx - q[1] * gqz));
            const float tz = 0.5f * (q[0] * gqz - gqw * q[3] + (q[1] * gqy - q[2] * gqx));
            ft[0] = gpx; ft[1] = gpy; ft[2] = gpz;
            ft[3] = py * gpz - pz * gpy + tx;
            ft[4] = pz * gpx - px * gpz + ty;
            ft[5] = px * gpy - py * gpx + tz;
        }
#pragma unroll
        for (int k = 0; k < 6; ++k) s.pose_ft[k * NC + c] = ft[k];
        s.pose_c[c] = C;
    }
    __syncthreads();

    // ---- a10 (per slot): merge self-collision, apply its gradient, per-slot costs
    if (warp == 0) {
        const int c = lane;
        float bp = 0.f;
        int bi = -1;
        for (int w = 0; w < NW; ++w) {
            const float p = s.sbest[w * NC + c];
            const int i = s.sidx[w * NC + c];
            if (i >= 0 && (p > bp || (p == bp && i < bi))) { bp = p; bi = i; }
        }
        float cself = 0.f;
        if (bi >= 0 && bp > 0.f) {
            const uint2 pr = reinterpret_cast<const uint2 *>(s.iw + rp.o_pairs)[bi];
            const int i = pr.x & 0xffff, j = pr.x >> 16;
            const float *wi = s.sw + i * 3 * NC + c, *wj = s.sw + j * 3 * NC + c;
            float ux = wi[0] - wj[0], uy = wi[NC] - wj[NC], uz = wi[2 * NC] - wj[2 * NC];
            const float nu = sqrtf(ux * ux + uy * uy + uz * uz);
            if (nu < 1e-12f) { ux = 1.f; uy = 0.f; uz = 0.f; }
            else { ux /= nu; uy /= nu; uz /= nu; }
            const float b = kp.beta_self;
            float *gi = s.sg + i * 3 * NC + c, *gj = s.sg + j * 3 * NC + c;
            gi[0] -= b * ux; gi[NC] -= b * uy; gi[2 * NC] -= b * uz;
            gj[0] += b * ux; gj[NC] += b * uy; gj[2 * NC] += b * uz;
            cself = b * bp;
        }
        float cw = 0.f;
        for (int w = 0; w < NW; ++w) cw += s.wpart[w * NC + c];
        float cb = 0.f, cs = 0.f;
        for (int d = 0; d < D; ++d) { cb += s.cbb[d * NC + c]; cs += s.csm[d * NC + c]; }
        const bool valid = c < n_act;
        const float cp = s.pose_c[c];
        const float t0 = valid ? cp : 0.f, t1 = valid ? cb : 0.f, t2 = valid ? cs : 0.f,
                    t3 = valid ? cself : 0.f, t4 = valid ? cw : 0.f;
        s.cfg_terms[0 * NC + c] = t0; s.cfg_terms[1 * NC + c] = t1; s.cfg_terms[2 * NC + c] = t2;
        s.cfg_terms[3 * NC + c] = t3; s.cfg_terms[4 * NC + c] = t4;
        s.cfg_cost[c] = (((t0 + t1) + t2) + t3) + t4;
    }
    __syncthreads();

    // ---- a9: backward to joint space (Alg. 8 / Table 7 as subtree sums):
    // per link: F_l = sum G_m, T_l = sum w_m x G_m over its spheres (+ the pose pseudo-sphere)
    for (int idx = tid; idx < rp.L * NC; idx += NT) {
        const int l = idx / NC, c = idx - l * NC;
        float F0 = 0.f, F1 = 0.f, F2 = 0.f, T0 = 0.f, T1 = 0.f, T2 = 0.f;
        const int b = s.iw[rp.o_sbeg + l], e = s.iw[rp.o_sbeg + l + 1];
        for (int m = b; m < e; ++m) {
            const float *g = s.sg + m * 3 * NC + c, *w = s.sw + m * 3 * NC + c;
            const float gx = g[0], gy = g[NC], gz = g[2 * NC];
            const float wx = w[0], wy = w[NC], wz = w[2 * NC];
            F0 += gx; F1 += gy; F2 += gz;
            T0 += wy * gz - wz * gy; T1 += wz * gx - wx * gz; T2 += wx * gy - wy * gx;
        }
        if (l == rp.ee) {
            F0 += s.pose_ft[0 * NC + c]; F1 += s.pose_ft[1 * NC + c]; F2 += s.pose_ft[2 * NC + c];
            T0 += s.pose_ft[3 * NC + c]; T1 += s.pose_ft[4 * NC + c]; T2 += s.pose_ft[5 * NC + c];
        }
        float *o = s.ls + l * 6 * NC + c;
        o[0] = F0; o[NC] = F1; o[2 * NC] = F2; o[3 * NC] = T0; o[4 * NC] = T1; o[5 * NC] = T2;
    }
    __syncthreads();
    // subtree accumulation, child -> parent in reverse topological order; warp k owns component k
    if (warp < 6) {
        const int k = warp;
        for (int l = rp.L - 1; l >= 1; --l) {
            const int p = s.iw[rp.o_links + 16 * l + 12];
            if (p >= 0) s.ls[(p * 6 + k) * NC + lane] += s.ls[(l * 6 + k) * NC + lane];
        }
    }
    __syncthreads();
    // joint gradient: revolute k . (T_l - o_l x F_l), prismatic k . F_l (Table 7), + bound_pos
    float *gq = s.sbest;   // reuse [D][32] (self scratch is dead now)
    for (int idx = tid; idx < D * NC; idx += NT) {
        const int d = idx / NC, c = idx - d * NC;
        const int l = s.iw[rp.o_doflink + d];
        const int type = s.iw[rp.o_links + 16 * l + 13];
        const int ax = type >= 4 ? type - 4 : type - 1;
        const float *T = s.lt + l * 12 * NC + c;
        const float kx = T[ax * NC], ky = T[(4 + ax) * NC], kz = T[(8 + ax) * NC];
        const float *S6 = s.ls + l * 6 * NC + c;
        const float F0 = S6[0], F1 = S6[NC], F2 = S6[2 * NC];
        float g;
        if (type >= 4) {
            const float ox = T[3 * NC], oy = T[7 * NC], oz = T[11 * NC];
            const float t0 = S6[3 * NC] - (oy * F2 - oz * F1);
            const float t1 = S6[4 * NC] - (oz * F0 - ox * F2);
            const float t2 = S6[5 * NC] - (ox * F1 - oy * F0);
            g = kx * t0 + ky * t1 + kz * t2;
        } else {
            g = kx * F0 + ky * F1 + kz * F2;
        }
        gq[idx] = (c < n_act) ? g + s.gxd[idx] : 0.f;
    }
    __syncthreads();

    // ---- transposed stencil + transposed state map (O2/O3 gradient routing) -> dC/dV
    if (MODE == MODE_TO) {
        const float dt = kp.dt, dt2 = dt * dt, dt3 = dt2 * dt;
        const float cv[5] = {1.f / (12.f * dt), -8.f / (12.f * dt), 0.f, 8.f / (12.f * dt), -1.f / (12.f * dt)};
        const float ca[5] = {-1.f / (12.f * dt2), 16.f / (12.f * dt2), -30.f / (12.f * dt2), 16.f / (12.f * dt2),
                             -1.f / (12.f * dt2)};
        const float cj[5] = {-1.f / (2.f * dt3), 2.f / (2.f * dt3), 0.f, -2.f / (2.f * dt3), 1.f / (2.f * dt3)};
        for (int idx = tid; idx < D * NC; idx += NT) {
            const int d = idx / NC, h = idx - d * NC;   // V_h <-> x_{h+1}
            if (h >= H) continue;
            const int hx = h + 1;
            int xlo, xhi;
            if (hx >= 4 && hx <= H - 4) { xlo = hx; xhi = hx; }
            else if (hx == H) { xlo = H - 3; xhi = H + 2; }
            else { s.gV[h * D + d] = 0.f; continue; }
            float acc = 0.f;
            for (int xi = xlo; xi <= xhi; ++xi) {
                float gx = (xi >= 1 && xi <= H) ? gq[d * NC + xi - 1] : 0.f;
                const int h0 = xi - 2 > 1 ? xi - 2 : 1, h1 = xi + 2 < H ? xi + 2 : H;
                for (int hp = h0; hp <= h1; ++hp) {
                    const int o = xi - hp + 2;
                    const int e = d * NC + hp - 1;
                    gx += cv[o] * s.gva[e] + ca[o] * s.gva[D * NC + e] + cj[o] * s.gva[2 * D * NC + e];
                }
                acc += gx;
            }
            s.gV[h * D + d] = acc;
        }
    } else {
        for (int idx = tid; idx < D * NC; idx += NT) s.gV[idx] = gq[idx];
    }
    __syncthreads();
}

}  // namespace crb
