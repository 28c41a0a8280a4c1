// curobo_b200.cu -- kernels and host side of the C-ABI declared in include/curobo_b200.h.
//
// Kernels (all sm_100a, NT = 256 threads, 2 CTAs per SM by shared-memory footprint):
//   solve_to_kernel   per-seed L-BFGS for trajectory optimisation: one CTA = one seed trajectory,
//                     all iterations in one launch (replaces the paper's ~20 kernels x 25-iteration
//                     CUDA graph); PERSIST: one wave taking (seed, iteration chunk)
//                     units; LONG: H > 32 in timestep windows
//   solve_ik_kernel   same for collision-free IK: one CTA = 32 seeds (PERSIST: chunked units)
//   solve_*_cluster_kernel   latency mode: the line-search candidates on a thread-block cluster
//   eval_to_kernel / eval_ik_kernel   one-shot batched cost+gradient (crb_evaluate_cost_grad)
//   fk_kernel         forward kinematics only (crb_fk)
//   select_kernel     per-problem packed-key argmin over seeds (O9)
//   + the motion-generation, mask / steering and test-hook kernels
//
// Two translation units, compiled in parallel with the same flags (build.py): this file
// (CRB_PART 0: the <GMEM = false> kernels that stage the cuboid table in shared memory, every
// non-template kernel and the host side) and curobo_b200_gmem.cu, which includes it with
// CRB_PART 1 and instantiates only the <GMEM = true> kernels (environments of >= CRB_GMEM_MIN_K
// cuboids: the cuboid table is read from global memory through L1 / L2 so two CTAs fit per SM).
// crb_gmem_kernel() hands those kernels to the host side.
#ifndef CRB_PART
#define CRB_PART 0
#endif
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <array>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <limits>
#include <string>
#include <vector>

#include "curobo_b200.h"
#include "crb_device.cuh"

#ifndef CRB_SELF_CULL
#define CRB_SELF_CULL 1   // frame-pair culling of the self-collision blocks (0: every block screened)
#endif
#ifndef CRB_SELF_LEN
#define CRB_SELF_LEN 16   // partners per self-collision work item (<= 511)
#endif

using namespace crb;

namespace {

constexpr int SMEM_MAX = 232448;   // 227 KB opt-in per CTA

// Two-loop recursion (Alg. 6; A18/A19) over the ring `order` (oldest first); each
// thread owns elements t and t + NT (N <= 2 NT); every dot product a deterministic block sum.
__device__ void two_loop_block(int N, int Np, int count, const int *order, const float *Sb, const float *Yb,
                               const float *rho, const float *syv, const float *yyv, const float *g, float *d,
                               float *red, int &ph) {
    const int t0 = threadIdx.x, t1 = threadIdx.x + NT;
    float al[32];
    float q0 = t0 < N ? g[t0] : 0.f, q1 = t1 < N ? g[t1] : 0.f;
#pragma unroll 1
    for (int i = count - 1; i >= 0; --i) {
        const float *S = Sb + order[i] * Np, *Y = Yb + order[i] * Np;
        const float part = (t0 < N ? S[t0] * q0 : 0.f) + (t1 < N ? S[t1] * q1 : 0.f);
        const float a = rho[order[i]] * block_sum(part, red, ph);
        al[i] = a;
        if (t0 < N) q0 -= a * Y[t0];
        if (t1 < N) q1 -= a * Y[t1];
    }
    float gamma = 1.f;
    if (count > 0) {
        const int sl = order[count - 1];
        gamma = syv[sl] / yyv[sl];
    }
    float r0 = gamma * q0, r1 = gamma * q1;
#pragma unroll 1
    for (int i = 0; i < count; ++i) {
        const float *S = Sb + order[i] * Np, *Y = Yb + order[i] * Np;
        const float part = (t0 < N ? Y[t0] * r0 : 0.f) + (t1 < N ? Y[t1] * r1 : 0.f);
        const float b = rho[order[i]] * block_sum(part, red, ph);
        if (t0 < N) r0 += (al[i] - b) * S[t0];
        if (t1 < N) r1 += (al[i] - b) * S[t1];
    }
    if (t0 < N) d[t0] = -r0;
    if (t1 < N) d[t1] = -r1;
}

// L-BFGS step of a TO seed by the whole CTA (Alg. 6): push (s, y, rho) of the last
// move unless s^T y <= 1e-12 (A20), then the two-loop recursion d = -H g; returns g^T d.  One
// definition for the sequential and the cluster solver (identical arithmetic).
__device__ __forceinline__ float lbfgs_step_to(int it, int N, int Np, int m, const float *th, const float *g, float *thp,
                                               float *gp, float *dd, float *Sb, float *Yb, float *rho, float *syv,
                                               float *yyv, int *order, int *ring, float *red, int &ph, float (&d_e)[2],
                                               float &sy_out) {
    const int t = threadIdx.x;
    sy_out = 0.f;
    // ---- a13: L-BFGS buffers (Alg. 6 lines 1-5): push (s, y, rho) unless s^T y <= 1e-12 (A20)
    if (it > 0) {
        const int fs = ring[1];
        float sy_p = 0.f, yy_p = 0.f;
#pragma unroll
        for (int e = 0; e < 2; ++e) {
            const int i = t + e * NT;
            if (i < N) {
                const float sv = th[i] - thp[i], yv = g[i] - gp[i];
                Sb[fs * Np + i] = sv; Yb[fs * Np + i] = yv;
                sy_p += sv * yv; yy_p += yv * yv;
            }
        }
        const float sy = block_sum(sy_p, red, ph);
        const float yy = block_sum(yy_p, red, ph);
        sy_out = sy;
        if (m > 0 && sy > 1e-12f && t == 0) {   // m = 0: gradient descent
            rho[fs] = 1.f / sy; syv[fs] = sy; yyv[fs] = yy;
            const int cnt = ring[0];
            if (cnt < m) { order[cnt] = fs; ring[0] = cnt + 1; ring[1] = cnt + 1; }
            else {
                const int ev = order[0];
                for (int i = 0; i < m - 1; ++i) order[i] = order[i + 1];
                order[m - 1] = fs;
                ring[1] = ev;
            }
        }
        __syncthreads();
    }
#pragma unroll
    for (int e = 0; e < 2; ++e) {
        const int i = t + e * NT;
        if (i < N) { thp[i] = th[i]; gp[i] = g[i]; }
    }
    // ---- two-loop recursion -> d = -H g
    two_loop_block(N, Np, ring[0], order, Sb, Yb, rho, syv, yyv, g, dd, red, ph);
    float gd_p = 0.f;
#pragma unroll
    for (int e = 0; e < 2; ++e) {
        const int i = t + e * NT;
        d_e[e] = i < N ? dd[i] : 0.f;
        if (i < N) gd_p += g[i] * d_e[e];
    }
    return block_sum(gd_p, red, ph);   // also publishes dd to every thread
}

// ------------------------------------------------------------------------------------------
// solver trace for the teacher-forced parity tests (crb_solver_params.trace; record layout in
// the header).  Out of line, behind one uniform branch: the hot loop keeps its code size.
// ------------------------------------------------------------------------------------------
__device__ __forceinline__ int trace_slot(const KParams &kp, int it) {
    if (kp.trace == nullptr) return -1;
    for (int j = 0; j < kp.n_trace; ++j)
        if (kp.trace_iter[j] == it) return j;
    return -1;
}

__device__ __forceinline__ float *trace_rec(const KParams &kp, size_t seed_unit, int j, int N) {
    return kp.trace + (seed_unit * (size_t)kp.n_trace + (size_t)j) * (size_t)CRB_TRACE_REC(N, kp.m);
}

// TO: the ring (slots via order[], oldest first) as S [m][N], Y [m][N], rho [m], count; every
// element is read by the thread that wrote it in the push (e = t, t + NT)
__device__ __forceinline__ void trace_to_ring(float *dst, int N, int Np, int m, const float *Sb, const float *Yb,
                                              const float *rho, const int *order, int cnt) {
    for (int i = 0; i < m; ++i)
        for (int e = threadIdx.x; e < N; e += NT) {
            dst[i * N + e] = i < cnt ? Sb[order[i] * Np + e] : 0.f;
            dst[(m + i) * N + e] = i < cnt ? Yb[order[i] * Np + e] : 0.f;
        }
    for (int i = threadIdx.x; i < m; i += NT) dst[2 * m * N + i] = i < cnt ? rho[order[i]] : 0.f;
    if (threadIdx.x == 0) dst[2 * m * N + m] = (float)cnt;
}

// One TO trace phase (all threads; few scalar arguments, the solver arrays are re-derived from
// the shared-memory layout of solve_to_kernel): 0 = entering iteration `it` (before the push),
// 1 = after the L-BFGS step, 2 = after the selection (thread 0 only writes).
static __device__ __noinline__ void trace_to(const KParams &kp, int phase, int unit, int it, int tj, float c, float g0d,
                                             float sy, int istar, float cbest) {
    extern __shared__ __align__(16) float smem[];
    const int D = kp.rp.D, N = kp.H * D, Np = (N + 3) & ~3, m = kp.m, A = kp.A;
    float *th = smem + kp.lay.solver, *g = th + Np, *dd = g + Np, *thp = dd + Np, *gp = thp + Np, *best = gp + Np,
          *thA = best + Np, *cg = thA + Np, *Sb = cg + A * Np, *Yb = Sb + (m + 1) * Np, *rho = Yb + (m + 1) * Np,
          *syv = rho + 40, *yyv = syv + 40;
    const int *order = reinterpret_cast<const int *>(yyv + 40);
    const float *scal = yyv + 80;
    const int *ring = reinterpret_cast<const int *>(scal + 24);
    float *rec = trace_rec(kp, (size_t)unit, tj, N), *sc = rec + CRB_TRACE_REC(N, m) - 24;
    if (phase == 0) {
        for (int e = threadIdx.x; e < N; e += NT) {
            rec[e] = th[e]; rec[N + e] = g[e];
            rec[2 * N + e] = it > 0 ? thp[e] : 0.f; rec[3 * N + e] = it > 0 ? gp[e] : 0.f;
        }
        trace_to_ring(rec + 5 * N, N, Np, m, Sb, Yb, rho, order, ring[0]);
        if (threadIdx.x == 0) { sc[1] = c; sc[20] = (float)it; }
    } else if (phase == 1) {
        for (int e = threadIdx.x; e < N; e += NT) rec[4 * N + e] = dd[e];
        trace_to_ring(rec + 5 * N + 2 * m * N + m + 1, N, Np, m, Sb, Yb, rho, order, ring[0]);
        if (threadIdx.x == 0) { sc[0] = g0d; sc[3] = sy; }
    } else if (threadIdx.x == 0) {
        sc[2] = (float)istar;
        for (int a = 0; a < 8; ++a) { sc[4 + a] = a < A ? scal[a] : 0.f; sc[12 + a] = a < A ? scal[8 + a] : 0.f; }
        sc[21] = cbest;
    }
}

// One IK trace phase for seed `lane` of the CTA's group (warp 0, per lane; arrays re-derived from
// the shared-memory layout of solve_ik_kernel; cnt = the lane's ring count).
static __device__ __noinline__ void trace_ik(const KParams &kp, int phase, size_t seed_unit, int it, int tj, int cnt,
                                             float c, float g0d, float sy, int istar, float cbest) {
    extern __shared__ __align__(16) float smem[];
    const int D = kp.rp.D, m = kp.m, A = kp.A, DC = D * NC, lane = threadIdx.x & 31;
    float *th = smem + kp.lay.solver, *g = th + DC, *dd = g + DC, *thp = dd + DC, *gp = thp + DC, *best = gp + DC,
          *Sb = best + DC, *Yb = Sb + (m + 1) * DC, *rho = Yb + (m + 1) * DC, *syv = rho + (m + 1) * NC,
          *yyv = syv + (m + 1) * NC, *cg = yyv + (m + 1) * NC, *cc = cg + A * DC, *cgd = cc + A * NC;
    const int *order = reinterpret_cast<const int *>(cgd + A * NC);
    float *rec = trace_rec(kp, seed_unit, tj, D), *sc = rec + CRB_TRACE_REC(D, m) - 24;
    if (phase == 2) {
        sc[2] = (float)istar;
        for (int a = 0; a < 8; ++a) { sc[4 + a] = a < A ? cc[a * NC + lane] : 0.f; sc[12 + a] = a < A ? cgd[a * NC + lane] : 0.f; }
        sc[21] = cbest;
        return;
    }
    float *dst = rec + 5 * D + (phase == 1 ? 2 * m * D + m + 1 : 0);
    for (int i = 0; i < m; ++i) {
        const int sl = i < cnt ? order[i * NC + lane] : 0;
        for (int d = 0; d < D; ++d) {
            dst[i * D + d] = i < cnt ? Sb[sl * DC + d * NC + lane] : 0.f;
            dst[(m + i) * D + d] = i < cnt ? Yb[sl * DC + d * NC + lane] : 0.f;
        }
        dst[2 * m * D + i] = i < cnt ? rho[sl * NC + lane] : 0.f;
    }
    dst[2 * m * D + m] = (float)cnt;
    if (phase == 0) {
        for (int d = 0; d < D; ++d) {
            const int e = d * NC + lane;
            rec[d] = th[e]; rec[D + d] = g[e];
            rec[2 * D + d] = it > 0 ? thp[e] : 0.f; rec[3 * D + d] = it > 0 ? gp[e] : 0.f;
        }
        sc[1] = c; sc[20] = (float)it;
    } else {
        for (int d = 0; d < D; ++d) rec[4 * D + d] = dd[d * NC + lane];
        sc[0] = g0d; sc[3] = sy;
    }
}

// ------------------------------------------------------------------------------------------
// persistent TO solver: one CTA per (problem, seed)
// ------------------------------------------------------------------------------------------
template <bool GMEM, bool LONG, bool PERSIST>
__global__ void __launch_bounds__(NT, 2) solve_to_kernel(const __grid_constant__ KParams kp) {
    extern __shared__ __align__(16) float smem[];
    const Smem s = make_smem(kp, smem);
    const int D = kp.rp.D, H = kp.H, N = H * D, Np = (N + 3) & ~3, m = kp.m, A = kp.A;
    const int t = threadIdx.x;
    float *base = smem + kp.lay.solver;
    float *th = base, *g = th + Np, *dd = g + Np, *thp = dd + Np, *gp = thp + Np, *best = gp + Np,
          *thA = best + Np, *cg = thA + Np, *Sb = cg + A * Np, *Yb = Sb + (m + 1) * Np,
          *rho = Yb + (m + 1) * Np, *syv = rho + 40, *yyv = syv + 40;   // m + 1 <= 33 slots each
    int *order = reinterpret_cast<int *>(yyv + 40);
    float *scal = yyv + 80;           // [0..7] c_a, [8..15] gd_a, [17] i*
    int *ring = reinterpret_cast<int *>(scal + 24);   // [0] count, [1] free slot
    const float *lim = s.fw + kp.rp.o_lim;
    int ph = 0;
    // Work units: one seed trajectory per CTA and all iterations, or
    // (kp.ik_chunks = C > 0, persistent launch of one wave) units (seed, iteration chunk) in
    // chunk-major order from a global counter, the solver state crossing global memory between a
    // seed's chunks as in the persistent IK kernel.  Every seed's arithmetic is the same (bitwise).
    const int C = PERSIST ? kp.ik_chunks : 1;
    const int NU = kp.P * kp.S;
    // saved per seed: th, g, dd, thp, gp, best (6 Np) | Sb .. order (2 (m + 1) Np + 160) | ring,
    // c, cbest, chunk_best, done
    const int SWA = 6 * Np, SWB = 2 * (m + 1) * Np + 160, SWT = SWA + SWB + 8;
    int *bcast = reinterpret_cast<int *>(smem + kp.lay.mbar) + 3;
    // the persistent kernel keeps its unit bookkeeping in shared memory (the staged environment in
    // mbar[2], K in s.scal[6], the unit in mbar[3]) so the pass loop does not carry it in registers
    int *envs = reinterpret_cast<int *>(smem + kp.lay.mbar) + 2, *Ks = reinterpret_cast<int *>(s.scal + 6);
    int *PHs = Ks + 1;   // the pass loop's end (PERSIST), -1 after the chunked convergence exit
    int K = 0;
    int unit = blockIdx.x;
    if (PERSIST) {
        if (t == 0) { *bcast = atomicAdd(kp.ik_flags, 1); *envs = -0x7fffffff; }
        __syncthreads();
        unit = *bcast;
    }
    while (unit < NU * C) {
    const int ch = PERSIST ? unit / NU : 0, u = unit - ch * NU;
    const int p = u / kp.S;
    {
        const int env = kp.env ? kp.env[p] : 0;
        if (!PERSIST) K = stage_tables(kp, smem, env);
        else {
            const int staged = *envs;
            if (staged == -0x7fffffff) K = stage_tables(kp, smem, env);
            else if (env != staged) K = restage_world(kp, smem, env);
            else K = *Ks;
            if (t == 0) *Ks = K;
        }
    }
    if (t < D) s.st[t] = kp.start[p * D + t];
    if (t < kp.cp.gw * NC) s.goal[t] = kp.goal[p * kp.cp.gw + t / NC];
    stage_dt(kp, s, p);
    const float *seed = kp.q_in + (size_t)u * N;
    float lo_e[2], hi_e[2];
#pragma unroll
    for (int e = 0; e < 2; ++e) {
        const int i = t + e * NT;
        lo_e[e] = i < N ? lim[i % D] : 0.f;
        hi_e[e] = i < N ? lim[D + i % D] : 0.f;
        if (ch == 0 && i < N) { th[i] = seed[i]; thA[i] = seed[i]; }
    }
    // One loop over evaluation passes with a single eval_pass call site: first the particle
    // warm-up (f1: pn_iters x pn cost-only passes, Alg. 5), then pass 0 evaluates Theta_0 (O8
    // initialise) and every iteration is an L-BFGS step followed by A candidate passes.
    // During the warm-up th holds mu, g holds Theta_sigma, dd / thp the UPDATE sums S1 / S2.
    float c = 0.f, cbest = 0.f, g0d = 0.f, chunk_best = 0.f;
    int done = 0;
    float d_e[2] = {0.f, 0.f};
    const int npart = kp.pn_iters * kp.pn;
    const int it_lo = (int)((long long)ch * kp.iters / C), it_hi = (int)((long long)(ch + 1) * kp.iters / C);
    const int pass_lo = ch == 0 ? 0 : npart + 1 + it_lo * A, pass_hi = npart + 1 + it_hi * A;
    if (ch == 0) {
        if (t == 0) { ring[0] = 0; ring[1] = 0; }
        __syncthreads();
    } else {   // (u, ch - 1) has saved the seed's state
        if (t == 0) {
            int *flag = kp.ik_flags + 2 + u;
            int v;
            for (;;) {
                asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(flag) : "memory");
                if (v >= ch) break;
                __nanosleep(256);
            }
        }
        __syncthreads();
        const float *src = kp.ik_state + (size_t)u * SWT;
        for (int i = t; i < SWA; i += NT) base[i] = __ldcg(src + i);
        for (int i = t; i < SWB; i += NT) Sb[i] = __ldcg(src + SWA + i);
        const float *sc = src + SWA + SWB;
        if (t < 2) ring[t] = __float_as_int(__ldcg(sc + t));
        c = __ldcg(sc + 2); cbest = __ldcg(sc + 3); chunk_best = __ldcg(sc + 4); done = __float_as_int(__ldcg(sc + 5));
        __syncthreads();
    }
    if (PERSIST) {
        __syncthreads();   // every thread has read PHs of the previous unit
        if (t == 0) *PHs = done ? -1 : pass_hi;
        __syncthreads();
    }
    // the seed of this unit (PERSIST: re-derived from the broadcast unit where needed, so the pass
    // loop does not carry it)
    auto seed_u = [&]() { if (PERSIST) { const int un = *bcast; return un - (un / NU) * NU; } return u; };
    ParticleAcc pacc;
    pacc.reset();
    float tm = -INFINITY, tZ = 0.f;   // merged particle chunks of the current warm-up iteration
    if (ch == 0 && npart > 0) {
#pragma unroll
        for (int e = 0; e < 2; ++e) {
            const int i = t + e * NT;
            if (i < N) { const float s0 = kp.s0_frac * (hi_e[e] - lo_e[e]); g[i] = s0 * s0; }   // B8
        }
    }
    for (int pass = pass_lo; PERSIST ? pass < *PHs : pass < (done ? pass_lo : pass_hi); ++pass) {
        const bool part = pass < npart;
        const int pit = part ? pass / kp.pn : 0, pl = pass - pit * kp.pn;
        const int lpass = pass - npart;
        const int a = part ? -2 : (lpass == 0 ? -1 : (lpass - 1) % A);
        if (part) {
            // ---- f1 SAMPLE (Alg. 5): theta_l = clip(mu + sqrt(Theta_sigma) theta_s) (B7)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int i = t + e * NT;
                if (i < N) {
                    const int su = seed_u(), sp_ = su / kp.S;
                    const float z = particle_normal(kp.rng_key, (unsigned)(kp.prob_base + sp_), (unsigned)i, (unsigned)pl,
                                                    (unsigned)pit, (unsigned)(kp.seed_base + (su - sp_ * kp.S)));
                    thA[i] = fminf(fmaxf(fmaf(sqrtf(g[i]), z, th[i]), lo_e[e]), hi_e[e]);
                }
            }
            __syncthreads();
        }
        if (a == 0) {
            const int it = (lpass - 1) / A;
            const int tj = trace_slot(kp, it);
            if (tj >= 0) trace_to(kp, 0, seed_u(), it, tj, c, 0.f, 0.f, 0, 0.f);
            float sy;
            g0d = lbfgs_step_to(it, N, Np, m, th, g, thp, gp, dd, Sb, Yb, rho, syv, yyv, order, ring, s.red, ph, d_e, sy);
            if (tj >= 0) trace_to(kp, 1, seed_u(), it, tj, c, g0d, sy, 0, 0.f);
        }
        // ---- a1: candidate a = clip(theta + alpha_a d) (pass 0: theta_0 is already in thA)
        if (a >= 0) {
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int i = t + e * NT;
                if (i < N) thA[i] = candidate(th[i], kp.alpha[a], dd[i], lo_e[e], hi_e[e]);   // d from dd (the step's output)
            }
            __syncthreads();
        }
        // ---- a2..a10: one evaluation pass (cost only for particles)
        eval_pass<MODE_TO, GMEM, LONG>(kp, smem, thA, PERSIST ? *Ks : K, H, a >= 0 ? dd : nullptr, !part);
        if (part) {
            // ---- f1 UPDATE, streamed over the particles of a chunk (Eqs. particle_1/2, B6), the
            // chunks merged in order (chunk_merge; totals in cg, unused during the warm-up)
            const int nch = A >= 2 ? A : 1, ch = particle_chunk(pl, kp.pn, nch);
            const int clo = ch * kp.pn / nch, chi = (ch + 1) * kp.pn / nch;
            float *S1t = cg, *S2t = cg + Np;
            float r;
            const float w = pacc.add(s.scal[0], kp.p_inv_beta, r);
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int i = t + e * NT;
                if (i < N) {
                    const float x = thA[i], dx = x - th[i];
                    dd[i] = (pl == clo ? 0.f : dd[i] * r) + w * x;
                    thp[i] = (pl == clo ? 0.f : thp[i] * r) + w * dx * dx;
                }
            }
            if (pl == chi - 1 && nch > 1) {
                if (clo == 0) { tm = -INFINITY; tZ = 0.f; }   // the iteration's first (non-empty) chunk
                float ft, fc;
                chunk_merge(tm, tZ, pacc.m, pacc.Z, ft, fc);
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const int i = t + e * NT;
                    if (i < N) {
                        S1t[i] = (clo == 0 ? 0.f : S1t[i]) * ft + dd[i] * fc;
                        S2t[i] = (clo == 0 ? 0.f : S2t[i]) * ft + thp[i] * fc;
                    }
                }
                pacc.reset();
            }
            if (pl == kp.pn - 1) {
                const float Zs = nch > 1 ? tZ : pacc.Z;
                const float *S1 = nch > 1 ? S1t : dd, *S2 = nch > 1 ? S2t : thp;
                const bool upd = Zs > 0.f;
                const float iz = upd ? 1.f / Zs : 0.f;
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const int i = t + e * NT;
                    if (i < N) {
                        if (upd) {
                            th[i] = (1.f - kp.k_mu) * th[i] + kp.k_mu * (S1[i] * iz);
                            g[i] = (1.f - kp.k_sigma) * g[i] + kp.k_sigma * (S2[i] * iz);
                        }
                        if (pass == npart - 1) thA[i] = th[i];   // Theta_0 of L-BFGS = mu
                    }
                }
                pacc.reset();
                __syncthreads();
            }
            continue;
        }
        if (a < 0) {
            c = s.scal[0];
            cbest = c;
            chunk_best = c;
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int i = t + e * NT;
                if (i < N) { g[i] = s.gV[i]; best[i] = th[i]; }
            }
            continue;
        }
#pragma unroll
        for (int e = 0; e < 2; ++e) {
            const int i = t + e * NT;
            if (i < N) cg[a * Np + i] = s.gV[i];
        }
        if (t == 0) { scal[a] = s.scal[0]; scal[8 + a] = pass_gdot(s); }
        if (a == A - 1) {
            __syncthreads();
            // ---- a11: selection (Alg. 1 lines 4-9), fp32 mirror, then take candidate i*
            const int istar = ls_select(A, kp.alpha, c, g0d, scal, scal + 8, kp.c1, kp.c2, kp.ls_mode);
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int i = t + e * NT;
                if (i < N) {
                    th[i] = candidate(th[i], kp.alpha[istar], dd[i], lo_e[e], hi_e[e]);
                    g[i] = cg[istar * Np + i];
                }
            }
            c = scal[istar];
            // ---- a12: best update, strict < (A23)
            if (c < cbest) {
                cbest = c;
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const int i = t + e * NT;
                    if (i < N) best[i] = th[i];
                }
            }
            if (kp.trace) {
                const int tj = trace_slot(kp, (lpass - 1) / A);
                if (tj >= 0) trace_to(kp, 2, seed_u(), 0, tj, c, 0.f, 0.f, istar, cbest);
            }
            // ---- a14: "up to" iters in chunks (B20): every thread holds the same cbest, so the
            // exit is CTA-uniform
            if (kp.check_every > 0) {
                const int it = (lpass - 1) / A + 1;   // iterations done
                if (it % kp.check_every == 0) {
                    if (!(cbest < chunk_best - kp.conv_rtol * fabsf(chunk_best))) {   // (CTA-uniform)
                        done = 1;
                        if (PERSIST && t == 0) *PHs = -1;   // read after the barrier below
                        break;
                    }
                    chunk_best = cbest;
                }
            }
        }
    }
    __syncthreads();
    {   // (PERSIST: the unit re-derived from shared memory, not carried through the pass loop)
    const int un = PERSIST ? *bcast : unit;
    const int ch = PERSIST ? un / NU : 0, u = un - ch * NU;
    const int done_ = PERSIST ? (*PHs == -1 ? 1 : 0) : done;
    if (ch == C - 1) {
        if (t == 0) kp.seed_best_cost[u] = cbest;
#pragma unroll
        for (int e = 0; e < 2; ++e) {
            const int i = t + e * NT;
            if (i < N) kp.seed_best_traj[(size_t)u * N + i] = best[i];
        }
    } else {   // save the seed's state for (u, ch + 1), then publish the chunk
        float *dst = kp.ik_state + (size_t)u * SWT;
        for (int i = t; i < SWA; i += NT) __stcg(dst + i, base[i]);
        for (int i = t; i < SWB; i += NT) __stcg(dst + SWA + i, Sb[i]);
        if (t == 0) {
            float *sc = dst + SWA + SWB;
            __stcg(sc, __int_as_float(ring[0])); __stcg(sc + 1, __int_as_float(ring[1]));
            __stcg(sc + 2, c); __stcg(sc + 3, cbest); __stcg(sc + 4, chunk_best); __stcg(sc + 5, __int_as_float(done_));
        }
        __syncthreads();
        if (t == 0) {
            __threadfence();
            int *flag = kp.ik_flags + 2 + u;
            const int v = ch + 1;
            asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(flag), "r"(v) : "memory");
        }
    }
    }
    if (!PERSIST) break;
    if (t == 0) *bcast = atomicAdd(kp.ik_flags, 1);
    __syncthreads();
    unit = *bcast;
    __syncthreads();   // every thread has read the unit before thread 0 may overwrite it
    }
}

// ------------------------------------------------------------------------------------------
// persistent IK solver: one CTA per (problem, group of 32 seeds); lane = seed
// ------------------------------------------------------------------------------------------
// latency mode of the TO solver (small batches): the A line-search candidates of an iteration are
// evaluated by the A CTAs of a thread-block cluster, one candidate each, instead of one after the
// other by one CTA.  Every CTA of the cluster holds the whole solver state and runs the identical
// L-BFGS step; after the candidate passes each reads the A costs / directional derivatives and the
// winner's gradient from the owners' shared memory (DSMEM), so every step is bitwise the
// sequential kernel's.  The particle warm-up and pass 0 run redundantly in every CTA.
// ------------------------------------------------------------------------------------------
template <bool GMEM, bool LONG>
__global__ void __launch_bounds__(NT, 2) solve_to_cluster_kernel(const __grid_constant__ KParams kp) {
    extern __shared__ __align__(16) float smem[];
    namespace cg = cooperative_groups;
    cg::cluster_group cluster = cg::this_cluster();
    const int A = kp.A;
    const int rank = (int)cluster.block_rank();
    const int unit = blockIdx.x / A;
    const int p = unit / kp.S;
    const int env = kp.env ? kp.env[p] : 0;
    const int K = stage_tables(kp, smem, env);
    const Smem s = make_smem(kp, smem);
    const int D = kp.rp.D, H = kp.H, N = H * D, Np = (N + 3) & ~3, m = kp.m;
    const int t = threadIdx.x;
    float *base = smem + kp.lay.solver;
    float *th = base, *g = th + Np, *dd = g + Np, *thp = dd + Np, *gp = thp + Np, *best = gp + Np,
          *thA = best + Np, *cg_ = thA + Np, *Sb = cg_ + A * Np, *Yb = Sb + (m + 1) * Np,
          *rho = Yb + (m + 1) * Np, *syv = rho + 40, *yyv = syv + 40;
    int *order = reinterpret_cast<int *>(yyv + 40);
    float *scal = yyv + 80;           // [0] this CTA's candidate cost, [8] its g . d
    int *ring = reinterpret_cast<int *>(scal + 24);
    const float *lim = s.fw + kp.rp.o_lim;
    int ph = 0;

    if (t < D) s.st[t] = kp.start[p * D + t];
    if (t < kp.cp.gw * NC) s.goal[t] = kp.goal[p * kp.cp.gw + t / NC];
    stage_dt(kp, s, p);
    const float *seed = kp.q_in + (size_t)unit * N;
    // (the joint limits are read from the staged tables where used, and the direction from dd:
    // no per-thread copies live across the evaluation passes)
#pragma unroll
    for (int e = 0; e < 2; ++e) {
        const int i = t + e * NT;
        if (i < N) { th[i] = seed[i]; thA[i] = seed[i]; }
    }
    if (t == 0) { ring[0] = 0; ring[1] = 0; }
    __syncthreads();

    float c = 0.f, cbest = 0.f, g0d = 0.f, chunk_best = 0.f;
    float d_e[2] = {0.f, 0.f};
    // particle warm-up: this CTA evaluates chunk `rank` of every iteration's particles (the
    // sequential kernel's chunks), the chunks are merged in order through DSMEM
    const int clo = rank * kp.pn / A, chi = (rank + 1) * kp.pn / A, csz = chi - clo;   // csz >= 1 (host)
    const int npart = kp.pn_iters * csz;
    const int npass = npart + 1 + kp.iters;   // warm-up, pass 0, then one candidate pass per iteration
    float tm = -INFINITY, tZ = 0.f;
    const unsigned pk1 = (unsigned)(kp.prob_base + p), psd = (unsigned)(kp.seed_base + (unit - p * kp.S));
    ParticleAcc pacc;
    pacc.reset();
    if (npart > 0) {
#pragma unroll
        for (int e = 0; e < 2; ++e) {
            const int i = t + e * NT;
            if (i < N) { const float s0 = kp.s0_frac * (lim[D + i % D] - lim[i % D]); g[i] = s0 * s0; }   // B8
        }
    }
    for (int pass = 0; pass < npass; ++pass) {
        const bool part = pass < npart;
        const int pit = part ? pass / csz : 0, pl = part ? clo + (pass - pit * csz) : 0;
        const int lpass = pass - npart;        // 0: Theta_0, it + 1: iteration it
        if (part) {
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int i = t + e * NT;
                if (i < N) {
                    const float z = particle_normal(kp.rng_key, pk1, (unsigned)i, (unsigned)pl, (unsigned)pit, psd);
                    thA[i] = fminf(fmaxf(fmaf(sqrtf(g[i]), z, th[i]), lim[i % D]), lim[D + i % D]);
                }
            }
            __syncthreads();
        }
        if (lpass > 0) {
            const int it = lpass - 1;
            // ---- a13 (identical in every CTA of the cluster)
            float sy;
            g0d = lbfgs_step_to(it, N, Np, m, th, g, thp, gp, dd, Sb, Yb, rho, syv, yyv, order, ring, s.red, ph, d_e, sy);
            // ---- a1: this CTA's candidate
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int i = t + e * NT;
                if (i < N) thA[i] = candidate(th[i], kp.alpha[rank], dd[i], lim[i % D], lim[D + i % D]);   // d from dd
            }
            __syncthreads();
        }
        eval_pass<MODE_TO, GMEM, LONG>(kp, smem, thA, K, H, lpass > 0 ? dd : nullptr, !part);
        if (part) {
            float r;
            const float w = pacc.add(s.scal[0], kp.p_inv_beta, r);
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int i = t + e * NT;
                if (i < N) {
                    const float x = thA[i], dx = x - th[i];
                    dd[i] = (pl == clo ? 0.f : dd[i] * r) + w * x;
                    thp[i] = (pl == clo ? 0.f : thp[i] * r) + w * dx * dx;
                }
            }
            if (pl == chi - 1) {
                // publish this chunk, merge all chunks in order (identical in every CTA)
                if (t == 0) { scal[0] = pacc.m; scal[1] = pacc.Z; }
                cluster.sync();
                float *S1t = cg_, *S2t = cg_ + Np;
                tm = -INFINITY; tZ = 0.f;
                for (int c = 0; c < A; ++c) {
                    const float *pc = cluster.map_shared_rank(scal, c);
                    const float *pd = cluster.map_shared_rank(dd, c), *pq = cluster.map_shared_rank(thp, c);
                    float ft, fc;
                    chunk_merge(tm, tZ, pc[0], pc[1], ft, fc);
#pragma unroll
                    for (int e = 0; e < 2; ++e) {
                        const int i = t + e * NT;
                        if (i < N) {
                            S1t[i] = (c == 0 ? 0.f : S1t[i]) * ft + pd[i] * fc;
                            S2t[i] = (c == 0 ? 0.f : S2t[i]) * ft + pq[i] * fc;
                        }
                    }
                }
                cluster.sync();                // peers have read this chunk before it is overwritten
                const bool upd = tZ > 0.f;
                const float iz = upd ? 1.f / tZ : 0.f;
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const int i = t + e * NT;
                    if (i < N) {
                        if (upd) {
                            th[i] = (1.f - kp.k_mu) * th[i] + kp.k_mu * (S1t[i] * iz);
                            g[i] = (1.f - kp.k_sigma) * g[i] + kp.k_sigma * (S2t[i] * iz);
                        }
                        if (pass == npart - 1) thA[i] = th[i];
                    }
                }
                pacc.reset();
                __syncthreads();
            }
            continue;
        }
        if (lpass == 0) {
            c = s.scal[0];
            cbest = c;
            chunk_best = c;
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int i = t + e * NT;
                if (i < N) { g[i] = s.gV[i]; best[i] = th[i]; }
            }
            continue;
        }
        // ---- publish this candidate, then a11 over all of them (DSMEM)
        if (t == 0) { scal[0] = s.scal[0]; scal[8] = pass_gdot(s); }
        cluster.sync();
        float ca[8], gda[8];
        for (int a = 0; a < A; ++a) {
            const float *ps = cluster.map_shared_rank(scal, a);
            ca[a] = ps[0];
            gda[a] = ps[8];
        }
        const int istar = ls_select(A, kp.alpha, c, g0d, ca, gda, kp.c1, kp.c2, kp.ls_mode);
        const float *gsrc = cluster.map_shared_rank(s.gV, istar);
#pragma unroll
        for (int e = 0; e < 2; ++e) {
            const int i = t + e * NT;
            if (i < N) {
                th[i] = candidate(th[i], kp.alpha[istar], dd[i], lim[i % D], lim[D + i % D]);
                g[i] = gsrc[i];
            }
        }
        c = ca[istar];
        if (c < cbest) {                       // a12 (A23)
            cbest = c;
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int i = t + e * NT;
                if (i < N) best[i] = th[i];
            }
        }
        cluster.sync();                        // peers have read this CTA's candidate before it is overwritten
        if (kp.check_every > 0 && lpass % kp.check_every == 0) {   // a14 chunk exit (B20), cluster-uniform
            if (!(cbest < chunk_best - kp.conv_rtol * fabsf(chunk_best))) break;
            chunk_best = cbest;
        }
    }
    __syncthreads();
    if (rank == 0) {
        if (t == 0) kp.seed_best_cost[unit] = cbest;
#pragma unroll
        for (int e = 0; e < 2; ++e) {
            const int i = t + e * NT;
            if (i < N) kp.seed_best_traj[(size_t)unit * N + i] = best[i];
        }
    }
}

// One seed's L-BFGS step of the IK solver (Alg. 6 ring push and two-loop recursion, A18-A20) on
// the lane that owns the seed (warp 0 of the CTA).  The per-dof vectors of the recursion live in
// registers (DM >= D, loops unrolled and predicated) so its dependent dot-product / update chains
// run without local memory; alpha_i of the first loop goes to `alv` [m][32] (shared scratch, dead
// between passes).  Returns g.d; sy = s'y of the pushed pair (trace).
template <int DM>
__device__ __forceinline__ float ik_step_lane(int D, int m, int DC, int lane, int it, int &cnt, int &fs, float &sy,
                                              const float *th, const float *g, float *dd, float *thp, float *gp,
                                              float *Sb, float *Yb, float *rho, float *syv, float *yyv, int *order,
                                              float *alv) {
    sy = 0.f;
    if (it > 0) {   // ---- ring push (per seed, A20)
        float yy = 0.f;
#pragma unroll
        for (int d = 0; d < DM; ++d)
            if (d < D) {
                const int e = d * NC + lane;
                const float sv = th[e] - thp[e], yv = g[e] - gp[e];
                Sb[fs * DC + e] = sv; Yb[fs * DC + e] = yv;
                sy += sv * yv; yy += yv * yv;
            }
        if (m > 0 && sy > 1e-12f) {
            rho[fs * NC + lane] = 1.f / sy; syv[fs * NC + lane] = sy; yyv[fs * NC + lane] = yy;
            if (cnt < m) { order[cnt * NC + lane] = fs; ++cnt; fs = cnt; }
            else {
                const int ev = order[lane];
                for (int i = 0; i < m - 1; ++i) order[i * NC + lane] = order[(i + 1) * NC + lane];
                order[(m - 1) * NC + lane] = fs;
                fs = ev;
            }
        }
    }
    float q[DM];
#pragma unroll
    for (int d = 0; d < DM; ++d) {
        q[d] = 0.f;
        if (d < D) {
            const int e = d * NC + lane;
            const float gv = g[e];
            thp[e] = th[e]; gp[e] = gv; q[d] = gv;
        }
    }
    // ---- two-loop recursion per seed (Alg. 6)
    for (int i = cnt - 1; i >= 0; --i) {
        const int sl = order[i * NC + lane];
        const float *S = Sb + sl * DC + lane, *Y = Yb + sl * DC + lane;
        float ai = 0.f;
#pragma unroll
        for (int d = 0; d < DM; ++d)
            if (d < D) ai += S[d * NC] * q[d];
        ai *= rho[sl * NC + lane];
        alv[i * NC + lane] = ai;
#pragma unroll
        for (int d = 0; d < DM; ++d)
            if (d < D) q[d] -= ai * Y[d * NC];
    }
    float gamma = 1.f;
    if (cnt > 0) { const int sl = order[(cnt - 1) * NC + lane]; gamma = syv[sl * NC + lane] / yyv[sl * NC + lane]; }
#pragma unroll
    for (int d = 0; d < DM; ++d) q[d] *= gamma;
    for (int i = 0; i < cnt; ++i) {
        const int sl = order[i * NC + lane];
        const float *S = Sb + sl * DC + lane, *Y = Yb + sl * DC + lane;
        float bi = 0.f;
#pragma unroll
        for (int d = 0; d < DM; ++d)
            if (d < D) bi += Y[d * NC] * q[d];
        bi *= rho[sl * NC + lane];
        const float k = alv[i * NC + lane] - bi;
#pragma unroll
        for (int d = 0; d < DM; ++d)
            if (d < D) q[d] += k * S[d * NC];
    }
    float g0d = 0.f;
#pragma unroll
    for (int d = 0; d < DM; ++d)
        if (d < D) { dd[d * NC + lane] = -q[d]; g0d += g[d * NC + lane] * (-q[d]); }
    return g0d;
}

// the register bucket of the IK step for D (<= 8, <= 16, <= 32), warp-uniform
__device__ __forceinline__ float ik_step(int D, int m, int DC, int lane, int it, int &cnt, int &fs, float &sy,
                                         const float *th, const float *g, float *dd, float *thp, float *gp, float *Sb,
                                         float *Yb, float *rho, float *syv, float *yyv, int *order, float *alv) {
    if (D <= 8)
        return ik_step_lane<8>(D, m, DC, lane, it, cnt, fs, sy, th, g, dd, thp, gp, Sb, Yb, rho, syv, yyv, order, alv);
    if (D <= 16)
        return ik_step_lane<16>(D, m, DC, lane, it, cnt, fs, sy, th, g, dd, thp, gp, Sb, Yb, rho, syv, yyv, order, alv);
    return ik_step_lane<32>(D, m, DC, lane, it, cnt, fs, sy, th, g, dd, thp, gp, Sb, Yb, rho, syv, yyv, order, alv);
}

// The per-candidate bookkeeping of the IK solver on the seed's lane (warp 0) after a pass: the
// candidate's cost, gradient and g.d; after the last candidate the line-search selection (Alg. 1
// lines 4-9, ls_select in fp32), the accepted point and the best update (strict <, A23).  Per-dof
// loops unrolled over DM >= D so the loads issue back to back.  istar = the selected candidate.
template <int DM>
__device__ __forceinline__ void ik_post_pass(const KParams &kp, const Smem &s, int a, int D, int lane, float *th,
                                             float *g, const float *dd, float *best, float *cg, float *cc,
                                             float *cgd, const float *lim, float &c, float &cbest, float g0d,
                                             int &istar) {
    const int DC = D * NC, A = kp.A;
    cc[a * NC + lane] = s.cfg_cost[lane];
    float gd = 0.f;
#pragma unroll
    for (int d = 0; d < DM; ++d)
        if (d < D) {
            const float v = s.gV[d * NC + lane];
            cg[a * DC + d * NC + lane] = v;
            gd += v * dd[d * NC + lane];
        }
    cgd[a * NC + lane] = gd;
    if (a != A - 1) return;
    const int i = ls_select(A, kp.alpha, c, g0d, cc + lane, cgd + lane, kp.c1, kp.c2, kp.ls_mode, NC);
    const float al = kp.alpha[i];
    float nt[DM];
#pragma unroll
    for (int d = 0; d < DM; ++d) {
        nt[d] = 0.f;
        if (d < D) {
            const int e = d * NC + lane;
            nt[d] = candidate(th[e], al, dd[e], lim[d], lim[D + d]);
            th[e] = nt[d];
            g[e] = cg[i * DC + e];
        }
    }
    c = cc[i * NC + lane];
    if (c < cbest) {
        cbest = c;
#pragma unroll
        for (int d = 0; d < DM; ++d)
            if (d < D) best[d * NC + lane] = nt[d];
    }
    istar = i;
}

// ------------------------------------------------------------------------------------------
template <bool GMEM, bool PERSIST>
__global__ void __launch_bounds__(NT, 2) solve_ik_kernel(const __grid_constant__ KParams kp) {
    extern __shared__ __align__(16) float smem[];
    const Smem s = make_smem(kp, smem);
    const int D = kp.rp.D, m = kp.m, A = kp.A;
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const int DC = D * NC;
    const int G = (kp.S + NC - 1) / NC;
    // Work units.  Sequential kernel: one 32-seed group of one problem
    // per CTA, all iterations.  Persistent kernel (PERSIST): the grid holds one wave of CTAs that
    // take units u = c * NG + g (chunk-major) from a global counter; unit (g, c) runs iterations
    // [c iters / C, (c + 1) iters / C) of seed group g, restoring the solver state that (g, c - 1)
    // saved to global memory (it waits on its completion flag; the chunk-major order makes the
    // wait rare).  With one environment for every problem (ik_flags[1], set by a device check)
    // the groups are flat: 32 consecutive seeds of the P x S batch, so no lane idles when S is
    // not a multiple of 32.  Each seed's arithmetic is the same in every mapping (bitwise).
    const bool flat = PERSIST && kp.ik_flags[1] != 0;
    const long long PS = (long long)kp.P * kp.S;
    const int NG = flat ? (int)((PS + NC - 1) / NC) : kp.P * G;
    const int C = PERSIST ? kp.ik_chunks : 1;
    const int SW = (6 + 2 * (m + 1)) * DC + 3 * (m + 1) * NC;   // saved solver words: th .. yyv
    const int SWT = SW + (m + 5) * NC;                            // + ring order, 4 per-lane scalars
    float *base = smem + kp.lay.solver;
    float *th = base, *g = th + DC, *dd = g + DC, *thp = dd + DC, *gp = thp + DC, *best = gp + DC,
          *Sb = best + DC, *Yb = Sb + (m + 1) * DC, *rho = Yb + (m + 1) * DC, *syv = rho + (m + 1) * NC,
          *yyv = syv + (m + 1) * NC, *cg = yyv + (m + 1) * NC, *cc = cg + A * DC, *cgd = cc + A * NC;
    int *order = reinterpret_cast<int *>(cgd + A * NC);   // [m][32]
    const float *lim = s.fw + kp.rp.o_lim;
    int *bcast = reinterpret_cast<int *>(smem + kp.lay.mbar) + 3;
    int staged = -0x7fffffff, K = 0;
    int unit = blockIdx.x;
    if (PERSIST) {
        if (t == 0) *bcast = atomicAdd(kp.ik_flags, 1);
        __syncthreads();
        unit = *bcast;
    }
    while (unit < NG * C) {
        const int ch = unit / NG, gi = unit - ch * NG;
        // this lane's seed: flat index fsd = p * S + sd
        long long fsd;
        int n_act;
        if (flat) {
            fsd = (long long)gi * NC + lane;
            n_act = (int)min((long long)NC, PS - (long long)gi * NC);
        } else {
            const int pg = gi / G, grp = gi - pg * G;
            fsd = (long long)pg * kp.S + grp * NC + lane;
            n_act = min(NC, kp.S - grp * NC);
        }
        const bool active = lane < n_act;
        const int p = (int)(min(fsd, PS - 1) / kp.S), sd = (int)(min(fsd, PS - 1) - (long long)p * kp.S);
        {   // the unit's environment (flat: one for all problems)
            const int p0 = flat ? 0 : gi / G;
            const int env = kp.env ? kp.env[p0] : 0;
            if (staged == -0x7fffffff) K = stage_tables(kp, smem, env);
            else if (env != staged) K = restage_world(kp, smem, env);
            staged = env;
        }
        const int npart = kp.pn_iters * kp.pn;
        const int it_lo = (int)((long long)ch * kp.iters / C), it_hi = (int)((long long)(ch + 1) * kp.iters / C);
        const int pass_lo = ch == 0 ? 0 : npart + 1 + it_lo * A, pass_hi = npart + 1 + it_hi * A;
        if (t < kp.cp.gw * NC) s.goal[t] = kp.goal[(size_t)p * kp.cp.gw + t / NC];   // t & 31 == lane of thread t
        float c = 0.f, cbest = 0.f, g0d = 0.f;
        int cnt = 0, fs = 0;
        if (ch == 0) {
            if (warp == 0)
                for (int d = 0; d < D; ++d) {
                    const float v = active ? kp.q_in[(size_t)fsd * D + d] : lim[d];
                    th[d * NC + lane] = v;
                    s.q_cfg[d * NC + lane] = v;
                }
            __syncthreads();
            prep_sincos(s, kp.rp);
        } else {
            if (t == 0) {   // (g, c - 1) has saved its state
                int *flag = kp.ik_flags + 2 + gi;
                int v;
                for (;;) {
                    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(flag) : "memory");
                    if (v >= ch) break;
                    __nanosleep(256);
                }
            }
            __syncthreads();
            const float *src = kp.ik_state + (size_t)gi * SWT;
            for (int i = t; i < SW; i += NT) base[i] = __ldcg(src + i);
            for (int i = t; i < (m + 1) * NC; i += NT) order[i] = __float_as_int(__ldcg(src + SW + i));
            if (warp == 0) {
                const float *sc = src + SW + (m + 1) * NC;   // per-lane scalars
                c = __ldcg(sc + lane); cbest = __ldcg(sc + NC + lane);
                cnt = __float_as_int(__ldcg(sc + 2 * NC + lane)); fs = __float_as_int(__ldcg(sc + 3 * NC + lane));
            }
            __syncthreads();
        }
        // single eval_pass call site: the particle warm-up (f1, cost only: thread t < D*32 owns
        // element t with mu in th, Theta_sigma in g, the UPDATE sums in dd / thp), then pass 0 =
        // Theta_0 and (L-BFGS step, A candidates) per iteration
        const unsigned pk1 = (unsigned)(kp.prob_base + p);
        const unsigned psd = (unsigned)(kp.seed_base + sd);
        ParticleAcc pacc;
        pacc.reset();
        float tm = -INFINITY, tZ = 0.f;   // merged particle chunks of the current warm-up iteration
        if (ch == 0 && npart > 0)
            for (int idx = t; idx < DC; idx += NT) {   // D * 32 elements: D > 8 needs more than one per thread
                const int d = idx / NC;
                const float s0 = kp.s0_frac * (lim[D + d] - lim[d]);   // B8
                g[idx] = s0 * s0;
            }
        for (int pass = pass_lo; pass < pass_hi; ++pass) {
            const bool part = pass < npart;
            const int pit = part ? pass / kp.pn : 0, pl = pass - pit * kp.pn;
            const int lpass = pass - npart;
            const int a = part ? -2 : (lpass == 0 ? -1 : (lpass - 1) % A);
            if (part)
                for (int idx = t; idx < DC; idx += NT) {
                    // ---- f1 SAMPLE (Alg. 5) for every seed of the group: variable d of seed idx & 31
                    // (idx & 31 == t & 31: psd is this thread's seed for all its elements)
                    const int d = idx / NC;
                    const float z = particle_normal(kp.rng_key, pk1, (unsigned)d, (unsigned)pl, (unsigned)pit, psd);
                    const float v = fminf(fmaxf(fmaf(sqrtf(g[idx]), z, th[idx]), lim[d]), lim[D + d]);
                    s.q_cfg[idx] = v;
                    joint_csq(s, kp.rp, idx, v);
                }
            if (a == 0 && warp == 0) {
                const int it = (lpass - 1) / A;
                const int tj = active ? trace_slot(kp, it) : -1;
                if (tj >= 0) trace_ik(kp, 0, (size_t)fsd, it, tj, cnt, c, 0.f, 0.f, 0, 0.f);
                float sy;
                g0d = ik_step(D, m, DC, lane, it, cnt, fs, sy, th, g, dd, thp, gp, Sb, Yb, rho, syv, yyv, order, s.ls);
                if (tj >= 0) trace_ik(kp, 1, (size_t)fsd, it, tj, cnt, c, g0d, sy, 0, 0.f);
            }
            if (a >= 0) {
                if (a == 0) __syncthreads();   // the L-BFGS step (warp 0) wrote the directions
                for (int idx = t; idx < DC; idx += NT) {   // all threads: candidate + its sin / cos
                    const int d = idx / NC;
                    const float v = candidate(th[idx], kp.alpha[a], dd[idx], lim[d], lim[D + d]);
                    s.q_cfg[idx] = v;
                    joint_csq(s, kp.rp, idx, v);
                }
            }
            eval_pass<MODE_IK, GMEM>(kp, smem, nullptr, K, n_act, nullptr, !part);
            if (part) {
                // ---- f1 UPDATE, streamed over the particles of a chunk (Eqs. particle_1/2, B6), per
                // seed; the chunks merged in order (chunk_merge; totals in cg, unused during the warm-up)
                const int nch = A >= 2 ? A : 1, pch = particle_chunk(pl, kp.pn, nch);
                const int clo = pch * kp.pn / nch, chi = (pch + 1) * kp.pn / nch;
                float *S1t = cg, *S2t = cg + DC;
                float r;
                const float w = pacc.add(s.cfg_cost[t & 31], kp.p_inv_beta, r);
                for (int idx = t; idx < DC; idx += NT) {   // w, r: seed idx & 31 == t & 31
                    const float x = s.q_cfg[idx], dx = x - th[idx];
                    dd[idx] = (pl == clo ? 0.f : dd[idx] * r) + w * x;
                    thp[idx] = (pl == clo ? 0.f : thp[idx] * r) + w * dx * dx;
                }
                if (pl == chi - 1 && nch > 1) {
                    if (clo == 0) { tm = -INFINITY; tZ = 0.f; }   // the iteration's first (non-empty) chunk
                    float ft, fc;
                    chunk_merge(tm, tZ, pacc.m, pacc.Z, ft, fc);
                    for (int idx = t; idx < DC; idx += NT) {
                        S1t[idx] = (clo == 0 ? 0.f : S1t[idx]) * ft + dd[idx] * fc;
                        S2t[idx] = (clo == 0 ? 0.f : S2t[idx]) * ft + thp[idx] * fc;
                    }
                    pacc.reset();
                }
                if (pl == kp.pn - 1) {
                    const float Zs = nch > 1 ? tZ : pacc.Z;
                    const float *S1 = nch > 1 ? S1t : dd, *S2 = nch > 1 ? S2t : thp;
                    for (int idx = t; idx < DC; idx += NT) {
                        if (Zs > 0.f) {
                            const float iz = 1.f / Zs;
                            th[idx] = (1.f - kp.k_mu) * th[idx] + kp.k_mu * (S1[idx] * iz);
                            g[idx] = (1.f - kp.k_sigma) * g[idx] + kp.k_sigma * (S2[idx] * iz);
                        }
                        if (pass == npart - 1) {   // Theta_0 of L-BFGS = mu
                            const float v = th[idx];
                            s.q_cfg[idx] = v;
                            joint_csq(s, kp.rp, idx, v);
                        }
                    }
                    pacc.reset();
                }
                continue;
            }
            if (warp != 0) continue;
            if (a < 0) {
                c = s.cfg_cost[lane];
                cbest = c;
                for (int d = 0; d < D; ++d) { g[d * NC + lane] = s.gV[d * NC + lane]; best[d * NC + lane] = th[d * NC + lane]; }
                continue;
            }
            int i = 0;
            if (D <= 8) ik_post_pass<8>(kp, s, a, D, lane, th, g, dd, best, cg, cc, cgd, lim, c, cbest, g0d, i);
            else if (D <= 16) ik_post_pass<16>(kp, s, a, D, lane, th, g, dd, best, cg, cc, cgd, lim, c, cbest, g0d, i);
            else ik_post_pass<32>(kp, s, a, D, lane, th, g, dd, best, cg, cc, cgd, lim, c, cbest, g0d, i);
            if (a == A - 1) {
                if (kp.trace && active) {
                    const int tj = trace_slot(kp, (lpass - 1) / A);
                    if (tj >= 0) trace_ik(kp, 2, (size_t)fsd, 0, tj, cnt, c, 0.f, 0.f, i, cbest);
                }
            }
        }
        __syncthreads();
        if (ch == C - 1) {
            if (warp == 0 && active) {
                kp.seed_best_cost[fsd] = cbest;
                for (int d = 0; d < D; ++d) kp.seed_best_traj[(size_t)fsd * D + d] = best[d * NC + lane];
            }
        } else {   // save the state for (g, c + 1), then publish the chunk
            float *dst = kp.ik_state + (size_t)gi * SWT;
            for (int i = t; i < SW; i += NT) __stcg(dst + i, base[i]);
            for (int i = t; i < (m + 1) * NC; i += NT) __stcg(dst + SW + i, __int_as_float(order[i]));
            if (warp == 0) {
                float *sc = dst + SW + (m + 1) * NC;
                __stcg(sc + lane, c); __stcg(sc + NC + lane, cbest);
                __stcg(sc + 2 * NC + lane, __int_as_float(cnt)); __stcg(sc + 3 * NC + lane, __int_as_float(fs));
            }
            __syncthreads();
            if (t == 0) {
                __threadfence();
                int *flag = kp.ik_flags + 2 + gi;
                const int v = ch + 1;
                asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(flag), "r"(v) : "memory");
            }
        }
        if (!PERSIST) break;
        if (t == 0) *bcast = atomicAdd(kp.ik_flags, 1);
        __syncthreads();
        unit = *bcast;
        __syncthreads();   // every thread has read the unit before thread 0 may overwrite it
    }
}

// latency mode of the IK solver: the A candidates of an iteration on the A CTAs of a cluster (as
// solve_to_cluster_kernel; per-seed selection on warp 0 from the peers' costs and gradients)
template <bool GMEM>
__global__ void __launch_bounds__(NT, 2) solve_ik_cluster_kernel(const __grid_constant__ KParams kp) {
    extern __shared__ __align__(16) float smem[];
    cooperative_groups::cluster_group cluster = cooperative_groups::this_cluster();
    const int rank = (int)cluster.block_rank();
    const int G = (kp.S + NC - 1) / NC;
    const int cid = blockIdx.x / kp.A;   // cluster = one 32-seed group, A CTAs
    const int p = cid / G, grp = cid - p * G;
    const int env = kp.env ? kp.env[p] : 0;
    const int K = stage_tables(kp, smem, env);
    const Smem s = make_smem(kp, smem);
    const int D = kp.rp.D, m = kp.m, A = kp.A;
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const int n_act = min(NC, kp.S - grp * NC);
    const int DC = D * NC;
    float *base = smem + kp.lay.solver;
    float *th = base, *g = th + DC, *dd = g + DC, *thp = dd + DC, *gp = thp + DC, *best = gp + DC,
          *Sb = best + DC, *Yb = Sb + (m + 1) * DC, *rho = Yb + (m + 1) * DC, *syv = rho + (m + 1) * NC,
          *yyv = syv + (m + 1) * NC, *cg = yyv + (m + 1) * NC, *cc = cg + A * DC, *cgd = cc + A * NC;
    int *order = reinterpret_cast<int *>(cgd + A * NC);   // [m][32]
    const float *lim = s.fw + kp.rp.o_lim;
    const int sd = grp * NC + lane;
    const bool active = lane < n_act;

    if (t < kp.cp.gw * NC) s.goal[t] = kp.goal[p * kp.cp.gw + t / NC];
    if (warp == 0)
        for (int d = 0; d < D; ++d) {
            const float v = active ? kp.q_in[((size_t)p * kp.S + sd) * D + d] : lim[d];
            th[d * NC + lane] = v;
            s.q_cfg[d * NC + lane] = v;
        }
    __syncthreads();
    prep_sincos(s, kp.rp);
    // single eval_pass call site: the particle warm-up (f1, cost only: thread t < D*32 owns
    // element t with mu in th, Theta_sigma in g, the UPDATE sums in dd / thp), then pass 0 =
    // Theta_0 and (L-BFGS step, A candidates) per iteration
    float c = 0.f, cbest = 0.f, g0d = 0.f;
    int cnt = 0, fs = 0;
    // particle warm-up: this CTA evaluates chunk `rank` of every iteration's particles
    const int clo = rank * kp.pn / A, chi = (rank + 1) * kp.pn / A, csz = chi - clo;   // csz >= 1 (host)
    const int npart = kp.pn_iters * csz;
    const int npass = npart + 1 + kp.iters;   // one candidate pass per iteration (this CTA's rank)
    float tm = -INFINITY, tZ = 0.f;
    const unsigned pk1 = (unsigned)(kp.prob_base + p);
    const unsigned psd = (unsigned)(kp.seed_base + grp * NC + (t & 31));
    ParticleAcc pacc;
    pacc.reset();
    if (npart > 0)
        for (int idx = t; idx < DC; idx += NT) {   // D * 32 elements: D > 8 needs more than one per thread
            const int d = idx / NC;
            const float s0 = kp.s0_frac * (lim[D + d] - lim[d]);   // B8
            g[idx] = s0 * s0;
        }
    for (int pass = 0; pass < npass; ++pass) {
        const bool part = pass < npart;
        const int pit = part ? pass / csz : 0, pl = part ? clo + (pass - pit * csz) : 0;
        const int lpass = pass - npart;
        const int a = part ? -2 : (lpass == 0 ? -1 : rank);
        if (part)
            for (int idx = t; idx < DC; idx += NT) {
                // ---- f1 SAMPLE (Alg. 5) for every seed of the group: variable d of seed idx & 31
                // (idx & 31 == t & 31: psd is this thread's seed for all its elements)
                const int d = idx / NC;
                const float z = particle_normal(kp.rng_key, pk1, (unsigned)d, (unsigned)pl, (unsigned)pit, psd);
                const float v = fminf(fmaxf(fmaf(sqrtf(g[idx]), z, th[idx]), lim[d]), lim[D + d]);
                s.q_cfg[idx] = v;
                joint_csq(s, kp.rp, idx, v);
            }
        if (a >= 0 && warp == 0) {
            const int it = lpass - 1;
            float sy;
            g0d = ik_step(D, m, DC, lane, it, cnt, fs, sy, th, g, dd, thp, gp, Sb, Yb, rho, syv, yyv, order, s.ls);
        }
        if (a >= 0) {
            __syncthreads();               // the L-BFGS step (warp 0) wrote the directions
            for (int idx = t; idx < DC; idx += NT) {   // all threads: candidate + its sin / cos
                const int d = idx / NC;
                const float v = candidate(th[idx], kp.alpha[a], dd[idx], lim[d], lim[D + d]);
                s.q_cfg[idx] = v;
                joint_csq(s, kp.rp, idx, v);
            }
        }
        eval_pass<MODE_IK, GMEM>(kp, smem, nullptr, K, n_act, nullptr, !part);
        if (part) {
            // ---- f1 UPDATE over this CTA's chunk, then all chunks merged in order (DSMEM)
            float r;
            const float w = pacc.add(s.cfg_cost[t & 31], kp.p_inv_beta, r);
            for (int idx = t; idx < DC; idx += NT) {   // w, r: seed idx & 31 == t & 31
                const float x = s.q_cfg[idx], dx = x - th[idx];
                dd[idx] = (pl == clo ? 0.f : dd[idx] * r) + w * x;
                thp[idx] = (pl == clo ? 0.f : thp[idx] * r) + w * dx * dx;
            }
            if (pl == chi - 1) {
                if (t < NC) { cc[t] = pacc.m; cgd[t] = pacc.Z; }   // this chunk's per-seed (m, Z)
                cluster.sync();
                float *S1t = cg, *S2t = cg + DC;
                tm = -INFINITY; tZ = 0.f;
                for (int c = 0; c < A; ++c) {
                    const float mc = cluster.map_shared_rank(cc, c)[t & 31], Zc = cluster.map_shared_rank(cgd, c)[t & 31];
                    float ft, fc;
                    chunk_merge(tm, tZ, mc, Zc, ft, fc);
                    const float *pd = cluster.map_shared_rank(dd, c), *pq = cluster.map_shared_rank(thp, c);
                    for (int idx = t; idx < DC; idx += NT) {
                        S1t[idx] = (c == 0 ? 0.f : S1t[idx]) * ft + pd[idx] * fc;
                        S2t[idx] = (c == 0 ? 0.f : S2t[idx]) * ft + pq[idx] * fc;
                    }
                }
                cluster.sync();                // peers have read this chunk before it is overwritten
                pacc.m = tm; pacc.Z = tZ;      // the merged totals feed the update below
                for (int idx = t; idx < DC; idx += NT) { dd[idx] = S1t[idx]; thp[idx] = S2t[idx]; }
            }
            if (pl == chi - 1) {
                for (int idx = t; idx < DC; idx += NT) {
                    if (pacc.Z > 0.f) {
                        const float iz = 1.f / pacc.Z;
                        th[idx] = (1.f - kp.k_mu) * th[idx] + kp.k_mu * (dd[idx] * iz);
                        g[idx] = (1.f - kp.k_sigma) * g[idx] + kp.k_sigma * (thp[idx] * iz);
                    }
                    if (pass == npart - 1) {   // Theta_0 of L-BFGS = mu
                        const float v = th[idx];
                        s.q_cfg[idx] = v;
                        joint_csq(s, kp.rp, idx, v);
                    }
                }
                pacc.reset();
            }
            continue;
        }
        if (a < 0) {
            if (warp != 0) continue;
            c = s.cfg_cost[lane];
            cbest = c;
            for (int d = 0; d < D; ++d) { g[d * NC + lane] = s.gV[d * NC + lane]; best[d * NC + lane] = th[d * NC + lane]; }
            continue;
        }
        // ---- publish this CTA's candidate (per seed), then a11 over all of them (DSMEM)
        if (warp == 0) {
            float gd = 0.f;
            for (int d = 0; d < D; ++d) gd += s.gV[d * NC + lane] * dd[d * NC + lane];
            cc[lane] = s.cfg_cost[lane];
            cgd[lane] = gd;
        }
        cluster.sync();
        if (warp == 0) {
            float ca[8], gda[8];
            for (int k = 0; k < A; ++k) {
                ca[k] = cluster.map_shared_rank(cc, k)[lane];
                gda[k] = cluster.map_shared_rank(cgd, k)[lane];
            }
            const int i = ls_select(A, kp.alpha, c, g0d, ca, gda, kp.c1, kp.c2, kp.ls_mode);
            const float *gsrc = cluster.map_shared_rank(s.gV, i);
            for (int d = 0; d < D; ++d) {
                const int e = d * NC + lane;
                th[e] = candidate(th[e], kp.alpha[i], dd[e], lim[d], lim[D + d]);
                g[e] = gsrc[e];
            }
            c = ca[i];
            if (c < cbest) {
                cbest = c;
                for (int d = 0; d < D; ++d) best[d * NC + lane] = th[d * NC + lane];
            }
        }
        cluster.sync();                        // peers have read this CTA's candidate
    }
    __syncthreads();
    if (rank == 0 && warp == 0 && active) {
        const size_t u = (size_t)p * kp.S + sd;
        kp.seed_best_cost[u] = cbest;
        for (int d = 0; d < D; ++d) kp.seed_best_traj[u * D + d] = best[d * NC + lane];
    }
}

// ------------------------------------------------------------------------------------------
// one-shot evaluation, FK, selection
// ------------------------------------------------------------------------------------------
template <bool GMEM, bool LONG>
__global__ void __launch_bounds__(NT, 2) eval_to_kernel(const __grid_constant__ KParams kp) {
    extern __shared__ __align__(16) float smem[];
    const int b = blockIdx.x;
    const int env = kp.env ? kp.env[b] : 0;
    const int K = stage_tables(kp, smem, env);
    const Smem s = make_smem(kp, smem);
    const int D = kp.rp.D, H = kp.H, N = H * D, t = threadIdx.x;
    float *thA = smem + kp.lay.solver;
    if (t < D) s.st[t] = kp.start[(size_t)b * D + t];
    if (t < kp.cp.gw * NC) s.goal[t] = kp.goal[(size_t)b * kp.cp.gw + t / NC];
    stage_dt(kp, s, b);
    for (int i = t; i < N; i += NT) thA[i] = kp.q_in[(size_t)b * N + i];
    __syncthreads();
    eval_pass<MODE_TO, GMEM, LONG>(kp, smem, thA, K, H, nullptr);
    if (t < 32) {
        float tr[5];
        for (int k = 0; k < 5; ++k) tr[k] = warp_sum(s.cfg_terms[k * NC + t]);
        if (t == 0) {
            kp.cost_out[b] = s.scal[0];
            if (kp.terms_out)
                for (int k = 0; k < 5; ++k) kp.terms_out[(size_t)b * 5 + k] = tr[k];
        }
    }
    if (kp.grad_out)
        for (int i = t; i < N; i += NT) kp.grad_out[(size_t)b * N + i] = s.gV[i];
}

template <bool GMEM>
__global__ void __launch_bounds__(NT, 2) eval_ik_kernel(const __grid_constant__ KParams kp) {
    extern __shared__ __align__(16) float smem[];
    const int b0 = blockIdx.x * NC;
    const int n_act = min(NC, kp.B - b0);
    const int env0 = kp.env ? kp.env[b0] : 0;
    const int K = stage_tables(kp, smem, env0);
    const Smem s = make_smem(kp, smem);
    const int D = kp.rp.D, t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const float *lim = s.fw + kp.rp.o_lim;
    if (warp == 0) {
        const bool act = lane < n_act;
        for (int d = 0; d < D; ++d) s.q_cfg[d * NC + lane] = act ? kp.q_in[(size_t)(b0 + lane) * D + d] : lim[d];
        const int gw = kp.cp.gw;
        for (int k = 0; k < gw; ++k)
            s.goal[k * NC + lane] = act ? kp.goal[(size_t)(b0 + lane) * gw + k] : (k == 3 && gw == 7 ? 1.f : 0.f);
    }
    __syncthreads();
    prep_sincos(s, kp.rp);
    eval_pass<MODE_IK, GMEM>(kp, smem, nullptr, K, n_act, nullptr);
    if (warp == 0 && lane < n_act) {
        const int b = b0 + lane;
        const bool ok = !kp.env || kp.env[b] == env0;
        kp.cost_out[b] = ok ? s.cfg_cost[lane] : __int_as_float(0x7fc00000);
        if (kp.terms_out)
            for (int k = 0; k < 5; ++k) kp.terms_out[(size_t)b * 5 + k] = s.cfg_terms[k * NC + lane];
        if (kp.grad_out)
            for (int d = 0; d < D; ++d) kp.grad_out[(size_t)b * D + d] = s.gV[d * NC + lane];
    }
}

#if CRB_PART == 0   // the non-template kernels: only in the main translation unit
// Persistent IK scheduling set-up (solve_ik_kernel<., true>): flags[0] = unit counter (0),
// flags[1] = 1 iff every problem uses the same environment (env = NULL counts as env 0), flags[2..]
// = completed chunks per seed group (0).
__global__ void ik_persist_init_kernel(const int *env, int P, int NG, int *flags) {
    __shared__ int diff;
    if (threadIdx.x == 0) diff = 0;
    __syncthreads();
    if (env)
        for (int p = threadIdx.x; p < P; p += blockDim.x)
            if (env[p] != env[0]) diff = 1;
    for (int i = threadIdx.x; i < NG; i += blockDim.x) flags[2 + i] = 0;
    __syncthreads();
    if (threadIdx.x == 0) { flags[0] = 0; flags[1] = diff ? 0 : 1; }
}

__global__ void __launch_bounds__(NT, 2) fk_kernel(const __grid_constant__ KParams kp) {
    extern __shared__ __align__(16) float smem[];
    const int b0 = blockIdx.x * NC;
    const int n_act = min(NC, kp.B - b0);
    stage_tables(kp, smem, -1);
    const Smem s = make_smem(kp, smem);
    const RobotPack &rp = kp.rp;
    const int D = rp.D, t = threadIdx.x, lane = t & 31, warp = t >> 5;
    if (warp == 0)
        for (int d = 0; d < D; ++d) s.q_cfg[d * NC + lane] = lane < n_act ? kp.q_in[(size_t)(b0 + lane) * kp.q_stride + d] : 0.f;
    __syncthreads();
    prep_sincos(s, kp.rp);
    __syncthreads();
    fk_phase(kp.rp, s);
    const float4 *sph = reinterpret_cast<const float4 *>(s.fw + rp.o_sph);
    if (kp.spheres_out)
        for (int m = warp; m < rp.M; m += NW) {
            if (lane >= n_act) continue;
            const int um = s.iw[rp.o_perm + m];
            float *o = kp.spheres_out + ((size_t)(b0 + lane) * rp.M + um) * 4;
            const float4 w = s.sw[m * NC + lane];
            o[0] = w.x; o[1] = w.y; o[2] = w.z; o[3] = sph[m].w;
        }
    if ((kp.ee_out || kp.pos_err_out) && warp == 0 && lane < n_act) {
        const float *E = ee_frame(s, D) + lane;   // R (9, row-major) then p (3)
        float q[4];
        mat_to_quat(E[0], E[NC], E[2 * NC], E[3 * NC], E[4 * NC], E[5 * NC], E[6 * NC], E[7 * NC], E[8 * NC], q);
        if (kp.ee_out) {
            float *o = kp.ee_out + (size_t)(b0 + lane) * 7;
            o[0] = E[9 * NC]; o[1] = E[10 * NC]; o[2] = E[11 * NC];
            o[3] = q[0]; o[4] = q[1]; o[5] = q[2]; o[6] = q[3];
        }
        if (kp.pos_err_out) {   // goal errors (App. B "pose error"): |p_g - p|, 1 - |<q_g, q>| (A1)
            const float *G = kp.goal + (size_t)((b0 + lane) / kp.goal_div) * 7;
            const float ex = G[0] - E[9 * NC], ey = G[1] - E[10 * NC], ez = G[2] - E[11 * NC];
            kp.pos_err_out[b0 + lane] = sqrtf(ex * ex + ey * ey + ez * ez);
            kp.rot_err_out[b0 + lane] = 1.f - fabsf(G[3] * q[0] + G[4] * q[1] + G[5] * q[2] + G[6] * q[3]);
        }
    }
}

// O9: per problem, the seed with the smallest packed key (cost bits, global seed index).
// ------------------------------------------------------------------------------------------
// validity mask and parallel steering (Alg. 3; readings B12-B14)
// ------------------------------------------------------------------------------------------
// One CTA per 32 configurations (lane = configuration): FK, then limits (warp 0), self pairs
// (pair blocks by warp) and sphere-cuboid distances (spheres by warp) each set a bit of the slot's
// flag; valid = no bit.  The cuboid screen's s2 is the exact squared outside distance, so
// sd < r + margin  <=>  s2 < (r + margin)^2 for r + margin > 0 (inside: s2 = 0).
__global__ void __launch_bounds__(NT, 2) mask_kernel(const __grid_constant__ KParams kp) {
    extern __shared__ __align__(16) float smem[];
    const RobotPack &rp = kp.rp;
    const int D = rp.D, t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const bool edges = kp.e_src != nullptr;
    const int n = edges ? kp.e_n[0] : 0;
    const int total = edges ? kp.E * (n + 1) : kp.B;
    const int b0 = blockIdx.x * NC;
    if (b0 >= total) return;                          // grid sized for n_cap >= n
    const int n_act = min(NC, total - b0);
    const int env = edges ? kp.e_env : (kp.env ? kp.env[b0 / kp.env_div] : 0);
    const int K = stage_tables(kp, smem, env);
    const Smem s = make_smem(kp, smem);
    const float *lim = s.fw + rp.o_lim;
    int *flag = reinterpret_cast<int *>(s.cfg_cost);  // [32] per-slot invalid bits (unused otherwise here)
    if (warp == 0) {
        flag[lane] = 0;
        const int i = b0 + lane;
        for (int d = 0; d < D; ++d) {
            float v = lim[d];
            if (lane < n_act) {
                if (edges) {                          // l_ej = src_e + (j / n)(dst_e - src_e)
                    const int e = i / (n + 1), j = i - e * (n + 1);
                    const float a = kp.e_src[(size_t)e * D + d], b = kp.e_dst[(size_t)e * D + d];
                    v = fmaf((float)j / (float)n, b - a, a);
                } else {
                    v = kp.q_in[(size_t)i * D + d];
                }
            }
            s.q_cfg[d * NC + lane] = v;
        }
        if (!edges && kp.env && lane < n_act && kp.env[(b0 + lane) / kp.env_div] != env) flag[lane] = 8;   // env group rule
    }
    __syncthreads();
    prep_sincos(s, kp.rp);
    __syncthreads();
    fk_phase(rp, s);
    int bad = (env < 0 || env >= kp.n_env) ? 16 : 0;  // env index outside [0, n_env): invalid
    if (warp == 0)                                    // position limits
        for (int d = 0; d < D; ++d) {
            const float v = s.q_cfg[d * NC + lane];
            if (v < lim[d] || v > lim[D + d]) bad |= 1;
        }
    {                                                 // self pairs (every pair of S with r + o > 0)
        const uint4 *blk = reinterpret_cast<const uint4 *>(s.iw + rp.o_blocks);
        const float *rself = s.fw + rp.o_rself;
        for (int bi = warp; bi < rp.NB; bi += NW) {
            const uint4 B = blk[bi];
            const int ia = B.x & 0x1ff, na = ((B.x >> 9) & 3) + 1, jb = (B.x >> 11) & 0x1ff, len = (B.x >> 20) & 0x1ff;
            for (int u = 0; u < na; ++u) {
                const float4 wi = s.sw[(ia + u) * NC + lane];
                const float ri = rself[ia + u];
                for (int v = 0; v < len; ++v) {
                    const float4 wj = s.sw[(jb + v) * NC + lane];
                    const float R = ri + rself[jb + v];
                    const float dx = wi.x - wj.x, dy = wi.y - wj.y, dz = wi.z - wj.z;
                    if (dx * dx + dy * dy + dz * dz < R * R) bad |= 2;
                }
            }
        }
    }
    {                                                 // world: sd_k(c) >= r + margin for all k
        const float4 *sph = reinterpret_cast<const float4 *>(s.fw + rp.o_sph);
        for (int m = warp; m < rp.M; m += NW) {
            const float r = sph[m].w;
            if (r < 0.f) continue;                    // disabled sphere
            const float4 c = s.sw[m * NC + lane];
            const float thr = r + kp.margin, thr2 = thr * thr;
            for (int k = 0; k < K; ++k) {
                const BoxView b = load_box(s.boxes, k);
                const float s2 = box_screen(c.x, c.y, c.z, b);
                bool hit;
                if (thr > 0.f) hit = s2 < thr2;
                else {                                // degenerate r + margin = 0: strictly inside
                    float gx, gy, gz;
                    hit = s2 == 0.f && box_sdf_grad(b, c.x, c.y, c.z, gx, gy, gz) < thr;
                }
                if (hit) bad |= 4;
            }
        }
    }
    if (bad) atomicOr(&flag[lane], bad);
    __syncthreads();
    if (warp == 0 && lane < n_act) kp.mask_out[b0 + lane] = flag[lane] == 0 ? 1 : 0;
}

// Alg. 3 line 2: n = floor(max_{e,d} |dw_d (dst - src)| / r) + 1, in fp64 from the fp32 inputs
// (the integer is decided exactly as the oracle decides it), clamped to n_cap; out[0] = n used,
// out[1] = n before clamping.
__global__ void steer_n_kernel(int E, int D, const float *src, const float *dst, const float *dw, float r, int n_cap,
                               int *out) {
    __shared__ double red[NT];
    double gm = 0.0;
    for (int i = threadIdx.x; i < E * D; i += blockDim.x) {
        const int d = i % D;
        const double g = fabs((double)dw[d] * ((double)dst[i] - (double)src[i]));
        gm = fmax(gm, g);
    }
    red[threadIdx.x] = gm;
    __syncthreads();
    for (int o = blockDim.x / 2; o > 0; o >>= 1) {
        if (threadIdx.x < o) red[threadIdx.x] = fmax(red[threadIdx.x], red[threadIdx.x + o]);
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        const double q = floor(red[0] / (double)r) + 1.0;
        const int n = q > 2.0e9 ? 2000000000 : (int)q;
        out[0] = min(n, n_cap);
        out[1] = n;
    }
}

// Alg. 3 lines 6-9, one warp per edge: h = first invalid - 1 (n if none), v_new = l_h,
// dist = |dw (v_new - src)|_2; h = -1 (invalid source) gives v_new = src, dist = 0.
__global__ void steer_scan_kernel(int E, int D, const float *src, const float *dst, const float *dw, const int *n_dev,
                                  const unsigned char *mask, int *h_out, float *v_out, float *dist_out) {
    const int e = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
    if (e >= E) return;
    const int n = n_dev[0];
    int first = -1;
    for (int j0 = 0; j0 <= n && first < 0; j0 += 32) {
        const int j = j0 + lane;
        const bool inval = j <= n && !mask[(size_t)e * (n + 1) + j];
        const unsigned bal = __ballot_sync(0xffffffffu, inval);
        if (bal) first = j0 + __ffs(bal) - 1;
    }
    const int h = first < 0 ? n : first - 1;
    float s2 = 0.f;
    for (int d = lane; d < D; d += 32) {
        const float a = src[(size_t)e * D + d], b = dst[(size_t)e * D + d];
        const float v = h < 0 ? a : fmaf((float)h / (float)n, b - a, a);
        v_out[(size_t)e * D + d] = v;
        const float g = dw[d] * (v - a);
        s2 += g * g;
    }
    for (int o = 16; o > 0; o >>= 1) s2 += __shfl_xor_sync(0xffffffffu, s2, o);
    if (lane == 0) { h_out[e] = h; dist_out[e] = sqrtf(s2); }
}

// ------------------------------------------------------------------------------------------
// motion-generation pipeline pieces (§8(f) f2; Alg. 4, App. B; readings B15-B18)
// ------------------------------------------------------------------------------------------
// Alg. 4 retime, one warp per trajectory: the five-point-stencil v, a, j of the state sequence
// (O2 map of V with the start) at dt[b]; s = max(1e-3, max |v|/vmax, sqrt(|a|/amax),
// cbrt(|j|/jmax)); dt_opt = s dt; max_jerk = max |j| / s^3 (the jerk at dt_opt).
__global__ void retime_kernel(int B, int H, int D, const float *V, const float *start, int start_div, const float *dt,
                              float dt_default, const float *lim, float *s_out, float *dt_out, float *jerk_out) {
    const int b = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
    if (b >= B) return;
    const float *Vb = V + (size_t)b * H * D, *st = start + (size_t)(b / start_div) * D;
    const float h_dt = dt ? dt[b] : dt_default;
    const float i12 = 1.f / (12.f * h_dt), i12b = 1.f / (12.f * h_dt * h_dt), i2c = 1.f / (2.f * h_dt * h_dt * h_dt);
    float rv = 0.f, ra = 0.f, rj = 0.f, jm = 0.f;
    for (int e = lane; e < H * D; e += 32) {
        const int h = e / D + 1, d = e - (h - 1) * D;     // state x_h, h = 1..H
        float x[5];
#pragma unroll
        for (int o = 0; o < 5; ++o) {
            const int k = h - 2 + o;                        // Table 5 map: pin / alias / V
            x[o] = k <= 3 ? st[d] : (k >= H - 3 ? Vb[(H - 1) * D + d] : Vb[(k - 1) * D + d]);
        }
        const float v = (-x[4] + 8.f * x[3] - 8.f * x[1] + x[0]) * i12;
        const float a = (-x[4] + 16.f * x[3] - 30.f * x[2] + 16.f * x[1] - x[0]) * i12b;
        const float j = (x[4] - 2.f * x[3] + 2.f * x[1] - x[0]) * i2c;
        rv = fmaxf(rv, fabsf(v) / lim[2 * D + d]);
        ra = fmaxf(ra, sqrtf(fabsf(a) / lim[3 * D + d]));
        rj = fmaxf(rj, cbrtf(fabsf(j) / lim[4 * D + d]));
        jm = fmaxf(jm, fabsf(j));
    }
    for (int o = 16; o > 0; o >>= 1) {
        rv = fmaxf(rv, __shfl_xor_sync(0xffffffffu, rv, o));
        ra = fmaxf(ra, __shfl_xor_sync(0xffffffffu, ra, o));
        rj = fmaxf(rj, __shfl_xor_sync(0xffffffffu, rj, o));
        jm = fmaxf(jm, __shfl_xor_sync(0xffffffffu, jm, o));
    }
    if (lane == 0) {
        const float sc = fmaxf(fmaxf(fmaxf(rv, ra), rj), 1e-3f);
        s_out[b] = sc;
        if (dt_out) dt_out[b] = sc * h_dt;
        if (jerk_out) jerk_out[b] = jm / (sc * sc * sc);
    }
}

// App. B scores (reading B18); +inf marks an invalid seed.  IK: w_pose (pe + re) + w_dist |q - q0|
// for seeds inside the pose thresholds whose configuration is valid (mask).  TO: the blended
// w_pose (pe + re) + w_jerk max|j| + w_time (H-1) dt_opt for seeds inside the pose thresholds whose
// H states are all valid.
__global__ void ik_scores_kernel(int P, int S, int D, const float *q, const float *q0, const float *pe, const float *re,
                                 const unsigned char *valid, float pos_thr, float rot_thr, float w_pose, float w_dist,
                                 float penalty, float *score) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= P * S) return;
    const int p = i / S;
    float d2 = 0.f;
    for (int d = 0; d < D; ++d) {
        const float e = q[(size_t)i * D + d] - q0[(size_t)p * D + d];
        d2 = fmaf(e, e, d2);
    }
    const bool ok = (!valid || valid[i]) && pe[i] < pos_thr && re[i] < rot_thr;
    score[i] = w_pose * (pe[i] + re[i]) + w_dist * sqrtf(d2) + (ok ? 0.f : penalty);
}

__global__ void to_scores_kernel(int P, int S, int H, const float *pe, const float *re, const float *max_jerk,
                                 const float *dt_opt, const unsigned char *valid, float pos_thr, float rot_thr,
                                 float w_pose, float w_jerk, float w_time, float penalty, float *score) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= P * S) return;
    bool ok = pe[i] < pos_thr && re[i] < rot_thr;
    if (valid)
        for (int h = 0; h < H && ok; ++h) ok = valid[(size_t)i * H + h] != 0;
    score[i] = w_pose * (pe[i] + re[i]) + w_jerk * max_jerk[i] + w_time * (float)(H - 1) * dt_opt[i] + (ok ? 0.f : penalty);
}

// Per problem: the k lowest finite scores in ascending order (ties -> lower seed index), one warp
// per problem; idx[p][j] for j >= count repeats the ranked list cyclically (-1 if count = 0).
__global__ void rank_kernel(int P, int S, const float *score, int k, int *idx, int *count) {
    const int p = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
    if (p >= P) return;
    const float *sc = score + (size_t)p * S;
    int cnt = 0;
    for (int s0 = 0; s0 < S; s0 += 32) {
        const int sidx = s0 + lane;
        const bool fin = sidx < S && sc[sidx] < INFINITY;
        cnt += __popc(__ballot_sync(0xffffffffu, fin));
    }
    for (int s0 = 0; s0 < S; s0 += 32) {
        const int si = s0 + lane;
        if (si < S) {
            const float v = sc[si];
            if (v < INFINITY) {
                int r = 0;                                     // rank = #(finite entries before it)
                for (int t = 0; t < S; ++t) {
                    const float w = sc[t];
                    r += (w < v) || (w == v && t < si);
                }
                for (int j = r; j < k; j += cnt) idx[(size_t)p * k + j] = si;
            }
        }
    }
    if (cnt == 0)
        for (int j = lane; j < k; j += 32) idx[(size_t)p * k + j] = -1;
    if (lane == 0) count[p] = cnt;
}

// Linear TO seeds (reading B17): V_h = q0 + (h / (H-1)) (qT - q0) from the ranked terminal
// configurations qT[p][idx[p][s]] (idx may be NULL = s; idx < 0 -> the start, a still seed).
__global__ void linear_seeds_kernel(int P, int S, int H, int D, const float *q0, const float *qT, int Sq, const int *idx,
                                    float *seeds) {
    const size_t n = (size_t)P * S * H * D;
    for (size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (size_t)gridDim.x * blockDim.x) {
        const int d = (int)(e % D), h = (int)((e / D) % H), s = (int)((e / ((size_t)D * H)) % S), p = (int)(e / ((size_t)D * H * S));
        const int j = idx ? idx[(size_t)p * S + s] : s;
        const float a = q0[(size_t)p * D + d];
        const float b = j >= 0 ? qT[((size_t)p * Sq + j) * D + d] : a;
        seeds[e] = a + ((float)h / (float)(H - 1)) * (b - a);
    }
}

// The trajectory states x_1..x_H of optimisation variables V (Table 5 last row, O2): x_h = start for
// h <= 3, x_h = V_{H-1} for h >= H-3, else V_{h-1} (V_0..V_2 and V_{H-4..H-2} are not states).
__global__ void states_kernel(int B, int H, int D, const float *V, const float *start, int start_div, float *x) {
    const size_t n = (size_t)B * H * D;
    for (size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (size_t)gridDim.x * blockDim.x) {
        const int d = (int)(e % D), h = (int)((e / D) % H) + 1, b = (int)(e / ((size_t)D * H));
        const float *Vb = V + (size_t)b * H * D;
        x[e] = h <= 3 ? start[(size_t)(b / start_div) * D + d] : (h >= H - 3 ? Vb[(H - 1) * D + d] : Vb[(h - 1) * D + d]);
    }
}

// Interpolation to a fine time grid (reading B21): trajectory b's states x[b][H][D] at
// spacing dt[b] -> out[b][k][D] at t_k = min(k dt_fine, T), T = (H-1) dt[b], k < n_b = ceil(T /
// dt_fine) + 1 (the count and the bracketing index decided in fp64 from the fp32 inputs, as the
// oracle decides them); rows k >= min(n_b, n_max) repeat x_H (neutral for a validity mask).
__global__ void interp_kernel(int B, int H, int D, const float *x, const float *dt, float dt_fine, int n_max,
                              float *out, int *n_out) {
    const int b = blockIdx.y;
    if (b >= B) return;
    const double dtb = (double)dt[b], T = (H - 1) * dtb;
    const int n = (int)ceil(T / (double)dt_fine) + 1;
    if (blockIdx.x == 0 && threadIdx.x == 0 && n_out) n_out[b] = n;
    const float *xb = x + (size_t)b * H * D;
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < n_max * D; e += gridDim.x * blockDim.x) {
        const int k = e / D, d = e - k * D;
        float v;
        if (k >= n - 1) {
            v = xb[(H - 1) * D + d];
        } else {
            const double u = (k * (double)dt_fine) / dtb;
            int i = (int)floor(u);
            if (i > H - 2) i = H - 2;
            const float f = (float)(u - i);
            v = fmaf(f, xb[(i + 1) * D + d] - xb[i * D + d], xb[i * D + d]);
        }
        out[((size_t)b * n_max + k) * D + d] = v;
    }
}

// dst[p][:] = src[p][idx[p]][:] (rows of n floats; idx < 0 -> zeros)
__global__ void gather_kernel(int P, int S, int n, const float *src, const int *idx, int idx_stride, float *dst) {
    const size_t tot = (size_t)P * n;
    for (size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x; e < tot; e += (size_t)gridDim.x * blockDim.x) {
        const int p = (int)(e / n), c = (int)(e % n);
        const int j = idx[(size_t)p * idx_stride];
        dst[e] = j >= 0 ? src[((size_t)p * S + j) * n + c] : 0.f;
    }
}

__global__ void select_kernel(int P, int S, int N, const float *seed_cost, const float *seed_traj,
                              long long seed_base, float *best_traj, float *best_cost, long long *best_key) {
    const int p = blockIdx.x;
    __shared__ int sbest;
    if (threadIdx.x == 0) {
        unsigned long long k = ~0ull;
        int bi = 0;
        for (int s = 0; s < S; ++s) {
            const unsigned long long ks = pack_key(seed_cost[(size_t)p * S + s], seed_base + s);
            if (ks < k) { k = ks; bi = s; }
        }
        sbest = bi;
        if (best_cost) best_cost[p] = seed_cost[(size_t)p * S + bi];
        if (best_key) best_key[p] = (long long)k;
    }
    __syncthreads();
    if (best_traj)
        for (int i = threadIdx.x; i < N; i += blockDim.x)
            best_traj[(size_t)p * N + i] = seed_traj[((size_t)p * S + sbest) * N + i];
}

struct LsParams {
    float alpha[8];
};

__global__ void ls_select_kernel(int n, int A, LsParams ap, const float *c0, const float *g0d, const float *ca,
                                 const float *gda, float c1, float c2, int mode, int *out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    float a8[8], b8[8];
    for (int a = 0; a < A; ++a) { a8[a] = ca[(size_t)i * A + a]; b8[a] = gda[(size_t)i * A + a]; }
    out[i] = ls_select(A, ap.alpha, c0[i], g0d[i], a8, b8, c1, c2, mode);
}

__global__ void argmin_keys_kernel(int P, int S, const float *cost, long long base, long long *out_key, int *out_idx) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= P) return;
    unsigned long long k = ~0ull;
    int bi = 0;
    for (int s = 0; s < S; ++s) {
        const unsigned long long ks = pack_key(cost[(size_t)p * S + s], base + s);
        if (ks < k) { k = ks; bi = s; }
    }
    if (out_key) out_key[p] = (long long)k;
    if (out_idx) out_idx[p] = bi;
}

__global__ void particle_normals_kernel(unsigned k0, unsigned k1, int n_var, int n, int it, unsigned seed,
                                        float *out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n * n_var) return;
    const int l = i / n_var, v = i - l * n_var;
    out[i] = particle_normal(k0, k1, (unsigned)v, (unsigned)l, (unsigned)it, seed);
}

__global__ void __launch_bounds__(NT, 2) lbfgs_direction_kernel(int n, int count, const float *S, const float *Y,
                                                                const float *g, float *d) {
    extern __shared__ __align__(16) float smem[];
    const int b = blockIdx.x, t = threadIdx.x, Np = (n + 3) & ~3;
    float *Sb = smem, *Yb = Sb + count * Np, *gg = Yb + count * Np, *dd = gg + Np, *rho = dd + Np,
          *syv = rho + 32, *yyv = syv + 32, *red = yyv + 32;   // count <= 32
    int *order = reinterpret_cast<int *>(red + 3 * NW);
    int ph = 0;
    for (int i = 0; i < count; ++i)
        for (int e = t; e < n; e += NT) {
            Sb[i * Np + e] = S[((size_t)b * count + i) * n + e];
            Yb[i * Np + e] = Y[((size_t)b * count + i) * n + e];
        }
    for (int e = t; e < n; e += NT) gg[e] = g[(size_t)b * n + e];
    if (t < count) order[t] = t;
    __syncthreads();
    for (int i = 0; i < count; ++i) {   // same reductions as the solver's push
        float sy_p = 0.f, yy_p = 0.f;
        for (int e = t; e < n; e += NT) { sy_p += Sb[i * Np + e] * Yb[i * Np + e]; yy_p += Yb[i * Np + e] * Yb[i * Np + e]; }
        const float sy = block_sum(sy_p, red, ph);
        const float yy = block_sum(yy_p, red, ph);
        if (t == 0) { rho[i] = 1.f / sy; syv[i] = sy; yyv[i] = yy; }
    }
    __syncthreads();
    two_loop_block(n, Np, count, order, Sb, Yb, rho, syv, yyv, gg, dd, red, ph);
    for (int e = t; e < n; e += NT) d[(size_t)b * n + e] = dd[e];
}

#endif  // CRB_PART == 0

}  // namespace

// the <GMEM = true> kernels, instantiated in CRB_PART 1
enum { KW_EVAL_TO, KW_EVAL_IK, KW_SOLVE_TO, KW_SOLVE_IK, KW_SOLVE_TO_CLUSTER, KW_SOLVE_IK_CLUSTER, KW_SOLVE_IK_PERSIST,
       KW_EVAL_TO_LONG, KW_SOLVE_TO_LONG, KW_SOLVE_TO_CLUSTER_LONG, KW_SOLVE_TO_PERSIST, KW_SOLVE_TO_LONG_PERSIST };
const void *crb_gmem_kernel(int k);

#if CRB_STATS
static int stats_copy(unsigned long long *out, int reset) {   // this translation unit's counters
    if (cudaDeviceSynchronize() != cudaSuccess) return -1;
    if (cudaMemcpyFromSymbol(out, ::g_crb_stats, sizeof(unsigned long long) * 32) != cudaSuccess) return -1;
    if (reset) {
        unsigned long long z[32] = {};
        cudaMemcpyToSymbol(::g_crb_stats, z, sizeof(z));
    }
    return 0;
}
int crb_gmem_stats(unsigned long long *out, int reset);
#endif

#if CRB_PART == 1
#if CRB_STATS
int crb_gmem_stats(unsigned long long *out, int reset) { return stats_copy(out, reset); }
#endif
const void *crb_gmem_kernel(int k) {
    switch (k) {
    case KW_EVAL_TO: return (const void *)eval_to_kernel<true, false>;
    case KW_EVAL_TO_LONG: return (const void *)eval_to_kernel<true, true>;
    case KW_EVAL_IK: return (const void *)eval_ik_kernel<true>;
    case KW_SOLVE_TO: return (const void *)solve_to_kernel<true, false, false>;
    case KW_SOLVE_TO_LONG: return (const void *)solve_to_kernel<true, true, false>;
    case KW_SOLVE_TO_PERSIST: return (const void *)solve_to_kernel<true, false, true>;
    case KW_SOLVE_TO_LONG_PERSIST: return (const void *)solve_to_kernel<true, true, true>;
    case KW_SOLVE_IK: return (const void *)solve_ik_kernel<true, false>;
    case KW_SOLVE_IK_PERSIST: return (const void *)solve_ik_kernel<true, true>;
    case KW_SOLVE_TO_CLUSTER: return (const void *)solve_to_cluster_kernel<true, false>;
    case KW_SOLVE_TO_CLUSTER_LONG: return (const void *)solve_to_cluster_kernel<true, true>;
    case KW_SOLVE_IK_CLUSTER: return (const void *)solve_ik_cluster_kernel<true>;
    }
    return nullptr;
}
#else
// ==========================================================================================
// host side
// ==========================================================================================
struct crb_ctx {
    int device = 0;
    std::string err;
    int64_t launches = 0;
    // robot
    bool robot_ok = false;
    RobotPack rp{};
    float4 *d_robot = nullptr;
    std::vector<float> lo, hi;
    // world
    bool world_ok = false;
    float4 *d_boxes = nullptr;
    float4 *d_boxes_ab = nullptr;         // world-frame AABB (centre, half extents) per cuboid (culling)
    int *d_box_count = nullptr;
    int n_env = 0, kmax = 0, kmax_enabled = 0;
    int sm_count = 148;
    // params
    bool params_ok = false;
    crb_cost_params cp{};
    // workspaces (grow on demand)
    float *ws_cost = nullptr, *ws_traj = nullptr;
    size_t cap_cost = 0, cap_traj = 0;
    unsigned char *ws_mask = nullptr;     // steering waypoint validity [E][n_cap + 1]
    size_t cap_mask = 0;
    int *ws_n = nullptr;                  // steering step count (used, unclamped)
    size_t cap_n = 0;
    float *ws_ik_state = nullptr;         // persistent IK: solver state per seed group
    size_t cap_ik_state = 0;
    int *ws_ik_flags = nullptr;           // persistent IK: unit counter, flat flag, chunk flags
    size_t cap_ik_flags = 0;
    // host-API buffers
    float *h_seeds = nullptr, *h_start = nullptr, *h_goal = nullptr, *h_best = nullptr, *h_bcost = nullptr;
    int *h_env = nullptr;
    int64_t *h_key = nullptr;
    size_t cap_h_seeds = 0, cap_h_start = 0, cap_h_goal = 0, cap_h_best = 0, cap_h_bcost = 0, cap_h_env = 0,
           cap_h_key = 0;
};

namespace {

crb_status fail(crb_ctx *ctx, crb_status st, const std::string &msg) {
    if (ctx) ctx->err = msg;
    return st;
}

crb_status cuda_check(crb_ctx *ctx, cudaError_t e, const char *what) {
    if (e == cudaSuccess) return CRB_OK;
    return fail(ctx, e == cudaErrorMemoryAllocation ? CRB_E_OOM : CRB_E_CUDA,
                std::string(what) + ": " + cudaGetErrorString(e));
}

crb_status enter(crb_ctx *ctx) {
    if (!ctx) return CRB_E_ARG;
    cudaError_t e = cudaSetDevice(ctx->device);
    if (e != cudaSuccess) return cuda_check(ctx, e, "cudaSetDevice");
    e = cudaGetLastError();   // surfaces an asynchronous fault of an earlier launch
    if (e != cudaSuccess) return cuda_check(ctx, e, "earlier asynchronous error");
    return CRB_OK;
}

template <typename T>
crb_status grow(crb_ctx *ctx, T **p, size_t *cap, size_t n) {
    if (n <= *cap) return CRB_OK;
    if (*p) cudaFree(*p);
    *p = nullptr;
    *cap = 0;
    cudaError_t e = cudaMalloc(p, std::max<size_t>(n, 1) * sizeof(T));
    if (e != cudaSuccess) return cuda_check(ctx, e, "cudaMalloc workspace");
    *cap = n;
    return CRB_OK;
}

int r4(int w) { return (w + 3) & ~3; }

// Shared-memory layout for one kernel configuration; returns total bytes.
size_t make_layout(const RobotPack &rp, int kmax, int mode, int H, int m, int A, bool solver, Layout &L) {
    const int D = rp.D;
    int w = 0;
    auto take = [&](int words) { int o = w; w += r4(words); return o; };
    L.robot = take(rp.words);
    L.boxes = take(kmax * 16);
    L.mbar = take(4);
    L.XS = mode == MODE_TO ? H + 5 : 0;
    L.q_cfg = take(D * NC);
    L.xs = take(D * L.XS);
    L.ltg = take(std::max(rp.L * 12, rp.M * 4) * NC);     // link transforms, then sphere gradients + E
    L.frames = take((D * 6 + 12) * NC);
    L.swl = take(std::max(std::max(rp.M * 4, rp.L * 6), std::max(2 * D, m)) * NC);   // joint sin/cos (before the chain),
    L.scs = L.swl;                                                      // then sphere centres (+hb), then link sums
    L.sbest = take(NW * NC);
    L.srank = take(NW * NC);
    L.sij = take(NW * NC);
    L.cbb = take(D * NC);
    L.csm = take(D * NC);
    L.gxd = take(D * NC);
    L.HS = mode == MODE_TO ? ((std::max(H, 1) + NC - 1) / NC) * NC : NC;   // slot stride (timestep windows)
    L.gq = take(D * L.HS);
    L.gva = take(mode == MODE_TO ? 3 * D * L.HS : 4);
    L.pose_ft = take(6 * NC);
    L.tdp = take(12);
    L.goal = take(std::max(7, D) * NC);   // pose [7][32] or joint-space goal [D][32] (CRB_CSPACE)
    L.cfg_cost = take(NC);
    L.cfg_terms = take(5 * NC);
    L.gV = take(std::max(H * D, D * NC));
    L.red = take(3 * NW);
    L.st = take(std::max(D, 16));   // start state (TO), D <= 31
    L.scal = take(8);
    L.wq = take(2 * ((rp.M + 3) / 4) + NW);   // world work-queue order + last-pass cost per group + per-warp current group
    L.solver = w;
    const int N = H * D, Np = r4(N), DC = D * NC;
    if (mode == MODE_TO) {
        if (solver) w += 7 * Np + A * Np + 2 * (m + 1) * Np + 192;   // + rho/syv/yyv/order/scal/ring tail
        else w += Np + 8;
    } else if (solver) {
        w += 6 * DC + 2 * (m + 1) * DC + 3 * (m + 1) * NC + A * DC + 2 * A * NC + (m + 1) * NC;
    }
    L.total = r4(w);
    return (size_t)L.total * 4;
}

KParams base_params(const crb_ctx *ctx) {
    KParams kp;
    memset(&kp, 0, sizeof(kp));
    kp.rp = ctx->rp;
    kp.robot = ctx->d_robot;
    kp.boxes = ctx->d_boxes;
    kp.boxes_ab = ctx->d_boxes_ab;
    kp.box_count = ctx->d_box_count;
    kp.kmax = ctx->kmax;
    kp.n_env = ctx->n_env;
    const crb_cost_params &c = ctx->cp;
    CostP &k = kp.cp;
    k.a0 = c.a0; k.a1 = c.a1; k.a2 = c.a2; k.a3 = c.a3; k.a8 = c.a8; k.a9 = c.a9;
    for (int i = 0; i < 4; ++i) k.wb[i] = c.w_bound[i];
    k.beta_self = c.beta_self; k.beta_world = c.beta_world; k.eta = c.eta; k.eta_bound = c.eta_bound;
    k.dt = c.dt; k.sweep_steps = c.sweep_steps; k.flags = c.flags;
    k.a4 = c.a4; k.a5 = c.a5;
    k.gw = (c.flags & CRB_CSPACE) ? ctx->rp.D : 7;
    k.inv_eta = 1.0f / c.eta;
    k.inv_eta_bound = 1.0f / c.eta_bound;
    k.inv_2dt = 1.0f / (2.0f * c.dt);
    k.inv_12dt = (float)(1.0 / (12.0 * c.dt));
    k.inv_12dt2 = (float)(1.0 / (12.0 * (double)c.dt * c.dt));
    k.inv_2dt3 = (float)(1.0 / (2.0 * (double)c.dt * c.dt * c.dt));
    return kp;
}

crb_status ready(crb_ctx *ctx, bool need_world) {
    if (!ctx->robot_ok) return fail(ctx, CRB_E_NOT_READY, "robot not set (crb_set_robot)");
    if (need_world && !ctx->world_ok) return fail(ctx, CRB_E_NOT_READY, "world not set (crb_set_world)");
    if (need_world && !ctx->params_ok) return fail(ctx, CRB_E_NOT_READY, "cost params not set");
    return CRB_OK;
}

// The solver / evaluation kernels come in two builds: <GMEM = true> (cuboid table read from global
// memory) when some environment holds >= CRB_GMEM_MIN_K enabled cuboids, else the table is staged
// in shared memory.  The world arithmetic is the same.
bool use_gmem_world(const crb_ctx *ctx) { return ctx->kmax_enabled >= CRB_GMEM_MIN_K; }

crb_status launch_fn(crb_ctx *ctx, const void *fn, int grid, size_t smem, cudaStream_t st, const KParams &kp,
                     const char *nm) {
    if (grid <= 0) return CRB_OK;
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return cuda_check(ctx, e, nm);
    void *args[] = {(void *)&kp};
    e = cudaLaunchKernel(fn, dim3(grid), dim3(NT), args, smem, st);
    ctx->launches++;
    if (e != cudaSuccess) return cuda_check(ctx, e, nm);
    return cuda_check(ctx, cudaGetLastError(), nm);
}

template <typename Kern>
crb_status launch(crb_ctx *ctx, Kern k, int grid, size_t smem, cudaStream_t st, const KParams &kp, const char *nm) {
    if (grid <= 0) return CRB_OK;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return cuda_check(ctx, e, nm);
    k<<<grid, NT, smem, st>>>(kp);
    ctx->launches++;
    return cuda_check(ctx, cudaGetLastError(), nm);
}

}  // namespace

extern "C" {

const char *crb_version(void) { return "curobo_b200 0.2 (sm_100a)"; }

int crb_abi_sizes(int *out, int n) {
    const int v[5] = {(int)sizeof(crb_link), (int)sizeof(crb_robot_desc), (int)sizeof(crb_cuboid),
                      (int)sizeof(crb_cost_params), (int)sizeof(crb_solver_params)};
    for (int i = 0; i < 5 && i < n && out; ++i) out[i] = v[i];
    return 5;
}

crb_status crb_create(int cuda_device, crb_ctx **out) {
    if (!out) return CRB_E_ARG;
    *out = nullptr;
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || cuda_device < 0 || cuda_device >= n) return CRB_E_CUDA;
    crb_ctx *c = new crb_ctx();
    c->device = cuda_device;
    if (cudaSetDevice(cuda_device) != cudaSuccess) { delete c; return CRB_E_CUDA; }
    cudaDeviceGetAttribute(&c->sm_count, cudaDevAttrMultiProcessorCount, cuda_device);
    *out = c;
    return CRB_OK;
}

crb_status crb_destroy(crb_ctx *ctx) {
    if (!ctx) return CRB_E_ARG;
    cudaSetDevice(ctx->device);
    cudaFree(ctx->d_robot); cudaFree(ctx->d_boxes); cudaFree(ctx->d_box_count);
    cudaFree(ctx->d_boxes_ab);
    cudaFree(ctx->ws_cost); cudaFree(ctx->ws_traj); cudaFree(ctx->ws_mask); cudaFree(ctx->ws_n);
    cudaFree(ctx->ws_ik_state); cudaFree(ctx->ws_ik_flags);
    cudaFree(ctx->h_seeds); cudaFree(ctx->h_start); cudaFree(ctx->h_goal); cudaFree(ctx->h_best);
    cudaFree(ctx->h_bcost); cudaFree(ctx->h_env); cudaFree(ctx->h_key);
    delete ctx;
    return CRB_OK;
}

const char *crb_last_error(const crb_ctx *ctx) { return ctx ? ctx->err.c_str() : "null context"; }

int64_t crb_launch_count(const crb_ctx *ctx) { return ctx ? ctx->launches : 0; }

crb_status crb_set_robot(crb_ctx *ctx, const crb_robot_desc *r) {
    crb_status st = enter(ctx);
    if (st != CRB_OK) return st;
    if (!r || !r->links || !r->pos_lo || !r->pos_hi || !r->vel_max || !r->acc_max || !r->jerk_max ||
        (r->n_spheres > 0 && (!r->spheres || !r->sphere_link)) || (r->n_pairs > 0 && !r->pairs))
        return fail(ctx, CRB_E_ARG, "null pointer in robot description");
    const int L = r->n_links, D = r->n_dof, M = r->n_spheres, P = r->n_pairs;
    if (L < 1 || L > 64 || D < 1 || D > 31 || M < 0 || M > 512 || P < 0 || P > 16383)
        return fail(ctx, CRB_E_LIMIT, "robot size outside limits (L<=64, D<=31, M<=512, pairs<=16384)");
    if (r->ee_link < 0 || r->ee_link >= L) return fail(ctx, CRB_E_ROBOT, "ee_link out of range");
    std::vector<int> doflink(D, -1);
    for (int l = 0; l < L; ++l) {
        const crb_link &k = r->links[l];
        if (k.parent >= l || (l > 0 && k.parent < 0 && false)) return fail(ctx, CRB_E_ROBOT, "parent >= own index (unsorted chain or cycle)");
        if (k.parent < -1) return fail(ctx, CRB_E_ROBOT, "invalid parent");
        if (k.type < 0 || k.type > 6) return fail(ctx, CRB_E_ROBOT, "unknown joint type");
        if (k.type == 0 && k.dof != -1) return fail(ctx, CRB_E_ROBOT, "fixed joint carries a dof");
        if (k.type != 0) {
            if (k.dof < 0 || k.dof >= D) return fail(ctx, CRB_E_ROBOT, "actuated joint without a valid dof");
            if (doflink[k.dof] != -1) return fail(ctx, CRB_E_ROBOT, "duplicate dof");
            doflink[k.dof] = l;
        }
        for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j) {
                double dot = 0;
                for (int q = 0; q < 3; ++q) dot += (double)k.fixed[q * 4 + i] * k.fixed[q * 4 + j];
                if (std::fabs(dot - (i == j ? 1.0 : 0.0)) > 1e-4)
                    return fail(ctx, CRB_E_ROBOT, "rotation block of a fixed transform is not orthonormal");
            }
    }
    for (int d = 0; d < D; ++d) {
        if (doflink[d] < 0) return fail(ctx, CRB_E_ROBOT, "dof without a joint");
        if (!(r->pos_lo[d] < r->pos_hi[d])) return fail(ctx, CRB_E_ROBOT, "pos_lo >= pos_hi");
        if (!(r->vel_max[d] > 0) || !(r->acc_max[d] > 0) || !(r->jerk_max[d] > 0))
            return fail(ctx, CRB_E_ROBOT, "non-positive vel/acc/jerk limit");
    }
    for (int m = 0; m < M; ++m)
        if (r->sphere_link[m] < 0 || r->sphere_link[m] >= L) return fail(ctx, CRB_E_ROBOT, "sphere on an unknown link");
    for (int p = 0; p < P; ++p) {
        const int i = r->pairs[2 * p], j = r->pairs[2 * p + 1];
        if (i < 0 || j >= M || i >= j) return fail(ctx, CRB_E_ROBOT, "self-collision pair with i >= j or out of range");
    }
    // ---- kinematic folding (exact algebra, fp64 on the host): every fixed link l is rigidly
    // attached to its nearest actuated ancestor b(l), T_l = T_b(l) * C_l with C_l the product of the
    // fixed transforms on the path (Table 6: full link = F * J, J = I for fixed joints).  The
    // device chain then runs over frame 0 (the root, identity) and the D actuated links only;
    // spheres and the end effector are re-expressed in their frame.
    typedef std::array<double, 12> M34;
    auto compose = [](const M34 &A, const M34 &B) {   // [A|a] * [B|b] (3x4 homogeneous)
        M34 C{};
        for (int i = 0; i < 3; ++i) {
            for (int j = 0; j < 4; ++j) {
                double v = 0.0;
                for (int k = 0; k < 3; ++k) v += A[i * 4 + k] * B[k * 4 + j];
                C[i * 4 + j] = v + (j == 3 ? A[i * 4 + 3] : 0.0);
            }
        }
        return C;
    };
    std::vector<int> bl(L), frame_of(L, -1);
    std::vector<M34> Cl(L);
    for (int l = 0; l < L; ++l) {
        M34 F;
        for (int i = 0; i < 12; ++i) F[i] = r->links[l].fixed[i];
        const int p = r->links[l].parent;
        if (p < 0) { bl[l] = -1; Cl[l] = F; }
        else if (r->links[p].type != 0) { bl[l] = p; Cl[l] = F; }
        else { bl[l] = bl[p]; Cl[l] = compose(Cl[p], F); }
    }
    const int NF = D + 1;
    std::vector<int> fparent(NF, -1), ftype(NF, 0), fdof(NF, -1);
    std::vector<M34> fC(NF);
    fC[0] = M34{1, 0, 0, 0, 0, 1, 0, 0, 0, 0, 1, 0};
    for (int l = 0, f = 1; l < L; ++l)
        if (r->links[l].type != 0) {
            frame_of[l] = f;
            fparent[f] = bl[l] < 0 ? 0 : frame_of[bl[l]];
            ftype[f] = r->links[l].type; fdof[f] = r->links[l].dof; fC[f] = Cl[l];
            ++f;
        }
    auto frame_and_offset = [&](int l, M34 &off) {   // frame carrying link l, offset of l in it
        if (r->links[l].type != 0) { off = M34{1, 0, 0, 0, 0, 1, 0, 0, 0, 0, 1, 0}; return frame_of[l]; }
        off = Cl[l];
        return bl[l] < 0 ? 0 : frame_of[bl[l]];
    };
    std::vector<int> sframe(M);
    std::vector<std::array<double, 3>> scen(M);
    for (int m = 0; m < M; ++m) {
        M34 off;
        sframe[m] = frame_and_offset(r->sphere_link[m], off);
        for (int i = 0; i < 3; ++i)
            scen[m][i] = off[i * 4 + 0] * r->spheres[4 * m + 0] + off[i * 4 + 1] * r->spheres[4 * m + 1] +
                         off[i * 4 + 2] * r->spheres[4 * m + 2] + off[i * 4 + 3];
    }
    M34 eeoff;
    const int fee = frame_and_offset(r->ee_link, eeoff);
    // Joint-axis normalisation: frame f is re-expressed as T'_f = T_f P_f, P_f the cyclic axis
    // permutation taking z to the joint's axis (R_a(q) = P R_z(q) P^T, Trans(q e_a) = P Trans(q e_z)
    // P^T), so every device joint is a z-axis joint: F'_f = P_parent^T F_f P_f, spheres and the EE
    // offset of frame f pre-multiplied by P_f^T.  World poses are unchanged; the joint axis of the
    // backward is column z of R'_f (= column a of R_f).  Entries are permuted, not rounded.
    {
        auto P_of = [&](int f) {   // columns (P e_x, P e_y, P e_z) as a row-major 3x3
            std::array<double, 9> P{1, 0, 0, 0, 1, 0, 0, 0, 1};
            if (f == 0) return P;
            const int a = (ftype[f] - 1) % 3;
            if (a == 0) P = {0, 0, 1, 1, 0, 0, 0, 1, 0};        // z -> x (e_x -> e_y, e_y -> e_z)
            else if (a == 1) P = {0, 1, 0, 0, 0, 1, 1, 0, 0};   // z -> y (e_x -> e_z, e_y -> e_x)
            return P;
        };
        auto xform = [&](const std::array<double, 9> &Pl, const M34 &A, const std::array<double, 9> &Pr) {
            M34 B;   // [Pl^T R Pr | Pl^T t]
            for (int i = 0; i < 3; ++i) {
                for (int j = 0; j < 3; ++j) {
                    double v = 0.0;
                    for (int k = 0; k < 3; ++k)
                        for (int q = 0; q < 3; ++q) v += Pl[k * 3 + i] * A[k * 4 + q] * Pr[q * 3 + j];
                    B[i * 4 + j] = v;
                }
                double t = 0.0;
                for (int k = 0; k < 3; ++k) t += Pl[k * 3 + i] * A[k * 4 + 3];
                B[i * 4 + 3] = t;
            }
            return B;
        };
        const std::array<double, 9> I3{1, 0, 0, 0, 1, 0, 0, 0, 1};
        std::vector<std::array<double, 9>> Pf(NF);
        for (int f = 0; f < NF; ++f) Pf[f] = P_of(f);
        for (int f = 1; f < NF; ++f) fC[f] = xform(Pf[fparent[f]], fC[f], Pf[f]);
        for (int m = 0; m < M; ++m) {
            const auto &Pm = Pf[sframe[m]];
            std::array<double, 3> c{};
            for (int i = 0; i < 3; ++i)
                for (int k = 0; k < 3; ++k) c[i] += Pm[k * 3 + i] * scen[m][k];
            scen[m] = c;
        }
        eeoff = xform(Pf[fee], eeoff, I3);
        for (int f = 1; f < NF; ++f) ftype[f] = ftype[f] <= 3 ? 3 : 6;
    }
    // ---- pack: spheres grouped by frame (stable), pairs remapped, disabled pairs dropped
    std::vector<int> ord(M);
    for (int m = 0; m < M; ++m) ord[m] = m;
    std::stable_sort(ord.begin(), ord.end(), [&](int a, int b) { return sframe[a] < sframe[b]; });
    std::vector<int> inv(M);
    for (int k = 0; k < M; ++k) inv[ord[k]] = k;
    RobotPack rp{};
    rp.L = NF; rp.D = D; rp.M = M; rp.ee = fee;
    int w = 0;
    rp.o_links = w; w += 16 * NF;
    rp.o_eeoff = w; w += 12 + 4;
    rp.o_sph = w; w += 4 * M;
    rp.o_sphlink = w; w += r4(M);
    rp.o_sbeg = w; w += r4(NF + 1);
    // self pairs (Eq. self-collision): drop r+o <= 0 (Alg. 9 "continue", P:2778 -- exact),
    // remap to packed sphere indices a < b, then cover S with rectangular blocks
    // {ia..ia+na-1} x {jb..jb+len-1} (na <= 4): consecutive first spheres with identical partner runs
    // share a block.  Blocks are balanced over the NW warps (LPT); the rank of every pair in S is
    // kept so arg-max ties resolve to the first maximal pair in S order (A28).
    std::vector<float> rself(M);
    for (int k = 0; k < M; ++k) {
        const int m = ord[k];
        rself[k] = (float)((double)r->spheres[4 * m + 3] + (r->self_offset ? r->self_offset[m] : 0.0));
    }
    std::vector<int> rank_of((size_t)M * M, -1);
    int npairs = 0;
    for (int p = 0; p < P; ++p) {
        const int i = r->pairs[2 * p], j = r->pairs[2 * p + 1];
        const double ri = (double)r->spheres[4 * i + 3] + (r->self_offset ? r->self_offset[i] : 0.0);
        const double rj = (double)r->spheres[4 * j + 3] + (r->self_offset ? r->self_offset[j] : 0.0);
        if (ri <= 0.0 || rj <= 0.0) continue;
        const int a = std::min(inv[i], inv[j]), b = std::max(inv[i], inv[j]);
        if (rank_of[(size_t)a * M + b] < 0) ++npairs;
        rank_of[(size_t)a * M + b] = rank_of[(size_t)a * M + b] < 0 ? p : std::min(rank_of[(size_t)a * M + b], p);
    }
    // packed sphere k -> its frame (spheres are sorted by frame)
    std::vector<int> pf(M);
    for (int k = 0; k < M; ++k) pf[k] = sframe[ord[k]];
    auto runs_of = [&](int a) {
        // partner runs of first sphere a; with CRB_SELF_CULL a run is also cut where the partner
        // frame changes, so every block below lies within one frame pair
        std::vector<std::pair<int, int>> rr;
        for (int b = a + 1; b < M;) {
            if (rank_of[(size_t)a * M + b] < 0) { ++b; continue; }
            int e = b;
            while (e < M && rank_of[(size_t)a * M + e] >= 0 && (!CRB_SELF_CULL || pf[e] == pf[b])) ++e;
            rr.push_back({b, e});
            b = e;
        }
        return rr;
    };
    // Block culling (crb_device.cuh): per block a proxy sphere on each
    // side (the one minimising the side's bound) and T^2, T = max_i (|c_i - c_pa| + r_i) +
    // max_j (|c_j - c_pb| + r_j) + 2 mm in frame coordinates (both sides rigid: one frame each).
    auto proxy = [&](int b0, int n, int &pbest) {
        double best = 1e300;
        for (int c = b0; c < b0 + n; ++c) {
            double mx = 0.0;
            for (int k = b0; k < b0 + n; ++k) {
                double d2 = 0.0;
                for (int i = 0; i < 3; ++i) d2 += (scen[ord[k]][i] - scen[ord[c]][i]) * (scen[ord[k]][i] - scen[ord[c]][i]);
                mx = std::max(mx, std::sqrt(d2) + (double)rself[k]);
            }
            if (mx < best) { best = mx; pbest = c; }
        }
        return best;
    };
    auto cull_of = [&](int ia, int na, int jb, int len, uint32_t &z, uint32_t &wv) {
        z = 0xffffffffu; wv = 0u;
        bool one = true;
        for (int k = ia; k < ia + na; ++k) one = one && pf[k] == pf[ia];
        for (int k = jb; k < jb + len; ++k) one = one && pf[k] == pf[jb];
        if (!CRB_SELF_CULL || !one) return;
        int pa = ia, pb = jb;
        const double T = proxy(ia, na, pa) + proxy(jb, len, pb) + 2e-3;
        const float T2 = (float)(T * T * (1.0 + 1e-6));
        z = (uint32_t)pa | ((uint32_t)pb << 16);
        memcpy(&wv, &T2, 4);
    };
    // Two work-item tables over the same pairs: TO passes take whole runs (<= 511 partners: fewer,
    // longer items), IK passes runs cut into pieces of at most CRB_SELF_LEN partners (the random IK
    // seeds make penetrations uneven: finer items keep the warps' queue times balanced).  Ranks are
    // stored v-major per run ([v][u]), so a piece of a run indexes the same array: rank of pair
    // (u, v) of a block = rank[B.y + v * na + u].
    struct Blk { int ia, na, jb, len, rbase; };
    std::vector<Blk> full, cut;
    std::vector<uint16_t> ranks;
    for (int a = 0; a < M;) {
        const auto ra = runs_of(a);
        int na = 1;
        while (na < 4 && a + na < M && (!CRB_SELF_CULL || pf[a + na] == pf[a]) && runs_of(a + na) == ra) ++na;
        for (const auto &rn : ra) {
            const int base = (int)ranks.size(), len = rn.second - rn.first;
            for (int v = 0; v < len; ++v)
                for (int u = 0; u < na; ++u) ranks.push_back((uint16_t)rank_of[(size_t)(a + u) * M + rn.first + v]);
            for (int j0 = 0; j0 < len; j0 += 511)
                full.push_back({a, na, rn.first + j0, std::min(511, len - j0), base + j0 * na});
            for (int j0 = 0; j0 < len; j0 += CRB_SELF_LEN)
                cut.push_back({a, na, rn.first + j0, std::min(CRB_SELF_LEN, len - j0), base + j0 * na});
        }
        a += na;
    }
    // work-queue order: decreasing cost (~ len * (2 + 9 na) instructions), ties by position
    auto emit = [&](std::vector<Blk> &blks, std::vector<uint32_t> &bk) {
        std::stable_sort(blks.begin(), blks.end(), [&](const Blk &x, const Blk &y) {
            return x.len * (2 + 9 * x.na) > y.len * (2 + 9 * y.na);
        });
        for (const Blk &b : blks) {
            bk.push_back((uint32_t)b.ia | ((uint32_t)(b.na - 1) << 9) | ((uint32_t)b.jb << 11) | ((uint32_t)b.len << 20));
            bk.push_back((uint32_t)b.rbase);
            uint32_t z, wv;
            cull_of(b.ia, b.na, b.jb, b.len, z, wv);
            bk.push_back(z);
            bk.push_back(wv);
        }
    };
    std::vector<uint32_t> bk, bk_ik;
    emit(full, bk);
    emit(cut, bk_ik);
    const std::vector<Blk> &blks = full;
    rp.NB = (int)blks.size();
    rp.NB_ik = (int)cut.size();
    rp.P = npairs;
    rp.o_rself = w; w += r4(M);
    rp.o_blocks = w; w += r4((int)bk.size());
    rp.o_blocks_ik = w; w += r4((int)bk_ik.size());
    rp.o_rank = w; w += r4(((int)ranks.size() + 1) / 2);
    rp.o_lim = w; w += r4(5 * D);
    rp.o_doflink = w; w += r4(D);
    rp.o_desc = w; w += r4(NF);
    rp.o_perm = w; w += r4(M);
    rp.o_doff = w; w += r4(D);
    rp.words = r4(w);
    std::vector<uint32_t> blob(rp.words, 0);
    auto fput = [&](int o, float v) { memcpy(&blob[o], &v, 4); };
    for (int f = 0; f < NF; ++f) {
        for (int i = 0; i < 12; ++i) fput(rp.o_links + 16 * f + i, (float)fC[f][i]);
        blob[rp.o_links + 16 * f + 12] = (uint32_t)fparent[f];
        blob[rp.o_links + 16 * f + 13] = (uint32_t)ftype[f];
        blob[rp.o_links + 16 * f + 14] = (uint32_t)fdof[f];
    }
    for (int i = 0; i < 12; ++i) fput(rp.o_eeoff + i, (float)eeoff[i]);
    for (int k = 0; k < M; ++k) {
        const int m = ord[k];
        for (int i = 0; i < 3; ++i) fput(rp.o_sph + 4 * k + i, (float)scen[m][i]);
        fput(rp.o_sph + 4 * k + 3, r->spheres[4 * m + 3]);
        blob[rp.o_sphlink + k] = (uint32_t)sframe[m];
        blob[rp.o_perm + k] = (uint32_t)m;
    }
    for (int f = 1; f < NF; ++f) blob[rp.o_doff + fdof[f]] = (uint32_t)f | ((ftype[f] == 3 ? 1u : 0u) << 16);

    for (int f = 0, k = 0; f <= NF; ++f) {
        while (k < M && sframe[ord[k]] < f) ++k;
        blob[rp.o_sbeg + f] = (uint32_t)k;
    }
    for (int k = 0; k < M; ++k) fput(rp.o_rself + k, rself[k]);
    for (size_t i = 0; i < bk.size(); ++i) blob[rp.o_blocks + i] = bk[i];
    for (size_t i = 0; i < bk_ik.size(); ++i) blob[rp.o_blocks_ik + i] = bk_ik[i];
    if (!ranks.empty()) memcpy(&blob[rp.o_rank], ranks.data(), ranks.size() * 2);
    for (int d = 0; d < D; ++d) {
        fput(rp.o_lim + d, r->pos_lo[d]); fput(rp.o_lim + D + d, r->pos_hi[d]);
        fput(rp.o_lim + 2 * D + d, r->vel_max[d]); fput(rp.o_lim + 3 * D + d, r->acc_max[d]);
        fput(rp.o_lim + 4 * D + d, r->jerk_max[d]);
        blob[rp.o_doflink + d] = (uint32_t)frame_of[doflink[d]];
    }
    for (int f = 0; f < NF; ++f) {   // descendant masks over frames: walk every later frame up towards f
        uint32_t m = 1u << f;
        for (int c2 = f + 1; c2 < NF; ++c2) {
            int a = c2;
            while (a > f) a = fparent[a];
            if (a == f) m |= 1u << c2;
        }
        blob[rp.o_desc + f] = m;
    }
    cudaFree(ctx->d_robot);
    ctx->d_robot = nullptr;
    st = cuda_check(ctx, cudaMalloc(&ctx->d_robot, blob.size() * 4), "cudaMalloc robot");
    if (st != CRB_OK) return st;
    st = cuda_check(ctx, cudaMemcpy(ctx->d_robot, blob.data(), blob.size() * 4, cudaMemcpyHostToDevice), "upload robot");
    if (st != CRB_OK) return st;
    ctx->rp = rp;
    ctx->lo.assign(r->pos_lo, r->pos_lo + D);
    ctx->hi.assign(r->pos_hi, r->pos_hi + D);
    ctx->robot_ok = true;
    return CRB_OK;
}

crb_status crb_set_world(crb_ctx *ctx, int n_env, int k_max, const int *boxes_per_env, const crb_cuboid *boxes) {
    crb_status st = enter(ctx);
    if (st != CRB_OK) return st;
    if (n_env < 1 || k_max < 0 || !boxes_per_env || (k_max > 0 && !boxes)) return fail(ctx, CRB_E_ARG, "bad world arguments");
    // the large-world slow path packs (slot, sphere, cuboid) into 32 bits: 5 + 10 + 17
    if (k_max > CRB_MAX_CUBOIDS) return fail(ctx, CRB_E_SHAPE, "k_max > CRB_MAX_CUBOIDS (131071)");
    std::vector<float> packed((size_t)n_env * std::max(k_max, 1) * 16, 0.f);
    // world-frame AABB of each enabled cuboid (crb_device.cuh "World culling"): centre and half
    // extents e_i = sum_j |R_ij| h_j, widened by 1e-4 m + 1e-6 (|c| + e) (fp32 rounding of the
    // device-side test, far below the margin)
    std::vector<float4> aabb((size_t)n_env * std::max(k_max, 1) * 2, make_float4(0.f, 0.f, 0.f, 0.f));
    std::vector<int> count(n_env, 0);
    int kmax_en = 0;
    for (int e = 0; e < n_env; ++e) {
        if (boxes_per_env[e] < 0 || boxes_per_env[e] > k_max) return fail(ctx, CRB_E_SHAPE, "boxes_per_env > k_max");
        int k = 0;
        for (int i = 0; i < boxes_per_env[e]; ++i) {
            const crb_cuboid &b = boxes[(size_t)e * k_max + i];
            for (int j = 0; j < 3; ++j)
                if (!(b.dims[j] > 0.f) || !std::isfinite(b.dims[j]) || !std::isfinite(b.pos[j]))
                    return fail(ctx, CRB_E_WORLD, "cuboid with non-positive or non-finite extent/position");
            const double qn = std::sqrt((double)b.quat[0] * b.quat[0] + (double)b.quat[1] * b.quat[1] +
                                        (double)b.quat[2] * b.quat[2] + (double)b.quat[3] * b.quat[3]);
            if (!(qn > 1e-6)) return fail(ctx, CRB_E_WORLD, "cuboid quaternion of zero norm");
            if (!b.enabled) continue;   // Alg. 10 skips disabled boxes
            const double w = b.quat[0] / qn, x = b.quat[1] / qn, y = b.quat[2] / qn, z = b.quat[3] / qn;
            const double R[3][3] = {{1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)},
                                    {2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)},
                                    {2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)}};
            float *o = &packed[((size_t)e * k_max + k) * 16];
            for (int i2 = 0; i2 < 3; ++i2) {   // row i2 of R^T = column i2 of R, with -col . t
                o[4 * i2 + 0] = (float)R[0][i2];
                o[4 * i2 + 1] = (float)R[1][i2];
                o[4 * i2 + 2] = (float)R[2][i2];
                o[4 * i2 + 3] = (float)(-(R[0][i2] * b.pos[0] + R[1][i2] * b.pos[1] + R[2][i2] * b.pos[2]));
            }
            o[12] = 0.5f * b.dims[0]; o[13] = 0.5f * b.dims[1]; o[14] = 0.5f * b.dims[2];
            {
                double ext[3], cm = 0.0;
                for (int i2 = 0; i2 < 3; ++i2) {
                    ext[i2] = 0.0;
                    for (int j2 = 0; j2 < 3; ++j2) ext[i2] += std::fabs(R[i2][j2]) * 0.5 * (double)b.dims[j2];
                    cm = std::max(cm, std::fabs((double)b.pos[i2]) + ext[i2]);
                }
                const double mg = 1e-4 + 1e-6 * cm;
                aabb[((size_t)e * k_max + k) * 2] = make_float4(b.pos[0], b.pos[1], b.pos[2], 0.f);
                aabb[((size_t)e * k_max + k) * 2 + 1] =
                    make_float4((float)(ext[0] + mg), (float)(ext[1] + mg), (float)(ext[2] + mg), 0.f);
            }
            o[15] = 0.f;   // unused
            ++k;
        }
        count[e] = k;
        kmax_en = std::max(kmax_en, k);
    }
    cudaFree(ctx->d_boxes); cudaFree(ctx->d_box_count); cudaFree(ctx->d_boxes_ab);
    ctx->d_boxes = nullptr; ctx->d_box_count = nullptr; ctx->d_boxes_ab = nullptr;
    ctx->world_ok = false;
    st = cuda_check(ctx, cudaMalloc(&ctx->d_boxes_ab, aabb.size() * sizeof(float4)), "cudaMalloc boxes aabb");
    if (st != CRB_OK) return st;
    st = cuda_check(ctx, cudaMemcpy(ctx->d_boxes_ab, aabb.data(), aabb.size() * sizeof(float4), cudaMemcpyHostToDevice),
                    "upload boxes aabb");
    if (st != CRB_OK) return st;
    st = cuda_check(ctx, cudaMalloc(&ctx->d_boxes, packed.size() * 4), "cudaMalloc boxes");
    if (st != CRB_OK) return st;
    st = cuda_check(ctx, cudaMalloc(&ctx->d_box_count, n_env * sizeof(int)), "cudaMalloc box count");
    if (st != CRB_OK) return st;
    st = cuda_check(ctx, cudaMemcpy(ctx->d_boxes, packed.data(), packed.size() * 4, cudaMemcpyHostToDevice), "upload boxes");
    if (st != CRB_OK) return st;
    st = cuda_check(ctx, cudaMemcpy(ctx->d_box_count, count.data(), n_env * sizeof(int), cudaMemcpyHostToDevice), "upload counts");
    if (st != CRB_OK) return st;
    ctx->n_env = n_env;
    ctx->kmax = std::max(k_max, 1);
    ctx->kmax_enabled = kmax_en;
    ctx->world_ok = true;
    return CRB_OK;
}

crb_status crb_set_cost_params(crb_ctx *ctx, const crb_cost_params *p) {
    crb_status st = enter(ctx);
    if (st != CRB_OK) return st;
    if (!p) return fail(ctx, CRB_E_ARG, "null params");
    if (!(p->eta > 0) || !(p->eta_bound > 0) || !(p->dt > 0) || p->sweep_steps < 0 || p->sweep_steps > 64)
        return fail(ctx, CRB_E_ARG, "eta, eta_bound, dt must be > 0 and 0 <= sweep_steps <= 64");
    ctx->cp = *p;
    ctx->params_ok = true;
    return CRB_OK;
}

crb_status crb_fk(crb_ctx *ctx, const float *q, int B, float *spheres_out, float *ee_out, void *stream) {
    crb_status st = enter(ctx);
    if (st != CRB_OK) return st;
    if ((st = ready(ctx, false)) != CRB_OK) return st;
    if (B < 0 || (B > 0 && !q)) return fail(ctx, CRB_E_ARG, "bad fk arguments");
    if (B == 0) return CRB_OK;
    KParams kp = base_params(ctx);
    kp.kmax = 0;
    kp.B = B; kp.H = 1; kp.cp.H = 1; kp.mode = MODE_IK; kp.q_in = q; kp.spheres_out = spheres_out; kp.ee_out = ee_out;
    kp.q_stride = ctx->rp.D;
    const size_t bytes = make_layout(ctx->rp, 0, MODE_IK, 1, 1, 1, false, kp.lay);
    if (bytes > SMEM_MAX) return fail(ctx, CRB_E_LIMIT, "shared memory footprint too large");
    return launch(ctx, fk_kernel, (B + NC - 1) / NC, bytes, (cudaStream_t)stream, kp, "fk_kernel");
}

crb_status crb_evaluate_cost_grad(crb_ctx *ctx, const float *q, int B, int H, const int *env, const float *start,
                                  const float *goal, float *cost, float *grad, float *term_costs, void *stream) {
    return crb_evaluate_cost_grad_dt(ctx, q, B, H, env, start, goal, nullptr, cost, grad, term_costs, stream);
}

crb_status crb_evaluate_cost_grad_dt(crb_ctx *ctx, const float *q, int B, int H, const int *env, const float *start,
                                     const float *goal, const float *dt, float *cost, float *grad, float *term_costs,
                                     void *stream) {
    crb_status st = enter(ctx);
    if (st != CRB_OK) return st;
    if ((st = ready(ctx, true)) != CRB_OK) return st;
    if (B < 0 || (B > 0 && (!q || !goal || !cost))) return fail(ctx, CRB_E_ARG, "bad evaluate arguments");
    const int mode = H == 1 ? MODE_IK : MODE_TO;
    if (mode == MODE_TO && (H < 8 || H > 64 || H * ctx->rp.D > 512 || (B > 0 && !start)))
        return fail(ctx, H < 8 ? CRB_E_SHAPE : CRB_E_LIMIT, "TO mode needs 8 <= H <= 64, H*D <= 512 and start");
    KParams kp = base_params(ctx);
    kp.B = B; kp.H = H; kp.cp.H = H; kp.mode = mode; kp.q_in = q; kp.env = env; kp.start = start; kp.goal = goal;
    kp.cost_out = cost; kp.grad_out = grad; kp.terms_out = term_costs; kp.dt_arr = dt;
    const size_t bytes = make_layout(ctx->rp, use_gmem_world(ctx) ? 0 : ctx->kmax_enabled, mode, H, 1, 1, false, kp.lay);
    kp.lay.boxes_gmem = use_gmem_world(ctx) ? 1 : 0;
    if (bytes > SMEM_MAX) return fail(ctx, CRB_E_LIMIT, "shared memory footprint too large (robot + cuboids)");
    const bool wm = use_gmem_world(ctx);
    if (mode == MODE_TO)
        return launch_fn(ctx, H > NC ? (wm ? crb_gmem_kernel(KW_EVAL_TO_LONG) : (const void *)eval_to_kernel<false, true>)
                                     : (wm ? crb_gmem_kernel(KW_EVAL_TO) : (const void *)eval_to_kernel<false, false>), B, bytes,
                         (cudaStream_t)stream, kp,
                      "eval_to_kernel");
    return launch_fn(ctx, wm ? crb_gmem_kernel(KW_EVAL_IK) : (const void *)eval_ik_kernel<false>, (B + NC - 1) / NC, bytes,
                  (cudaStream_t)stream, kp, "eval_ik_kernel");
}

crb_status crb_lbfgs_solve(crb_ctx *ctx, const crb_solver_params *sp, int P, int S, int H, const float *seeds,
                           const int *env, const float *start, const float *goal, float *best_traj, float *best_cost,
                           int64_t *best_key, float *seed_best_cost, float *seed_best_traj, void *stream) {
    return crb_lbfgs_solve_dt(ctx, sp, P, S, H, seeds, env, start, goal, nullptr, best_traj, best_cost, best_key,
                              seed_best_cost, seed_best_traj, stream);
}

crb_status crb_lbfgs_solve_dt(crb_ctx *ctx, const crb_solver_params *sp, int P, int S, int H, const float *seeds,
                              const int *env, const float *start, const float *goal, const float *dt,
                              float *best_traj, float *best_cost, int64_t *best_key, float *seed_best_cost,
                              float *seed_best_traj, void *stream) {
    crb_status st = enter(ctx);
    if (st != CRB_OK) return st;
    if ((st = ready(ctx, true)) != CRB_OK) return st;
    if (!sp || P < 0 || S < 1 || (P > 0 && (!seeds || !goal))) return fail(ctx, CRB_E_ARG, "bad solve arguments");
    if (sp->history < 0 || sp->history > 32 || sp->n_alpha < 1 || sp->n_alpha > 8 || sp->iters < 0)
        return fail(ctx, CRB_E_LIMIT, "history must be in [0,32] (0 = gradient descent), n_alpha in [1,8], iters >= 0");
    if (sp->particle_iters < 0 ||
        (sp->particle_iters > 0 && (sp->n_particles < 1 || !(sp->particle_beta > 0.f) || !(sp->k_mu >= 0.f) ||
                                    !(sp->k_mu <= 1.f) || !(sp->k_sigma >= 0.f) || !(sp->k_sigma <= 1.f) ||
                                    !(sp->sigma0_frac >= 0.f))))
        return fail(ctx, CRB_E_ARG, "particle warm-up: iters >= 0, n >= 1, beta > 0, k_mu/k_sigma in [0,1], sigma0_frac >= 0");
    if (sp->check_every < 0 || !(sp->conv_rtol >= 0.f) || sp->cluster < -1 || sp->cluster > 1)
        return fail(ctx, CRB_E_ARG, "check_every >= 0, conv_rtol >= 0, cluster in {-1, 0, 1}");
    if (sp->trace && (sp->n_trace < 0 || sp->n_trace > 8))
        return fail(ctx, CRB_E_ARG, "trace: 0 <= n_trace <= 8");
    const int mode = H == 1 ? MODE_IK : MODE_TO;
    const int D = ctx->rp.D;
    if (mode == MODE_TO && (H < 8 || H > 64 || H * D > 512 || (P > 0 && !start)))
        return fail(ctx, H < 8 ? CRB_E_SHAPE : CRB_E_LIMIT, "TO mode needs 8 <= H <= 64, H*D <= 512 and start");
    if (P == 0) return CRB_OK;   // empty batch: validated, nothing launched
    const int N = H * D;
    cudaStream_t stream_ = (cudaStream_t)stream;
    float *sbc = seed_best_cost, *sbt = seed_best_traj;
    if (!sbc) { if ((st = grow(ctx, &ctx->ws_cost, &ctx->cap_cost, (size_t)P * S)) != CRB_OK) return st; sbc = ctx->ws_cost; }
    if (!sbt) { if ((st = grow(ctx, &ctx->ws_traj, &ctx->cap_traj, (size_t)P * S * N)) != CRB_OK) return st; sbt = ctx->ws_traj; }
    KParams kp = base_params(ctx);
    kp.P = P; kp.S = S; kp.H = H; kp.cp.H = H; kp.mode = mode; kp.q_in = seeds; kp.env = env; kp.start = start; kp.goal = goal;
    kp.dt_arr = mode == MODE_TO ? dt : nullptr;
    kp.iters = sp->iters; kp.m = sp->history; kp.A = sp->n_alpha; kp.ls_mode = sp->ls_mode;
    for (int i = 0; i < 8; ++i) kp.alpha[i] = sp->alpha[i];
    kp.c1 = sp->c1; kp.c2 = sp->c2; kp.seed_base = sp->global_seed_base;
    kp.pn_iters = sp->particle_iters; kp.pn = sp->particle_iters > 0 ? sp->n_particles : 1;
    kp.p_inv_beta = sp->particle_iters > 0 ? 1.f / sp->particle_beta : 0.f;
    kp.k_mu = sp->k_mu; kp.k_sigma = sp->k_sigma; kp.s0_frac = sp->sigma0_frac;
    kp.rng_key = sp->rng_key; kp.prob_base = sp->global_problem_base;
    kp.check_every = sp->check_every; kp.conv_rtol = sp->conv_rtol;
    kp.trace = sp->n_trace > 0 ? sp->trace : nullptr; kp.n_trace = sp->n_trace;
    for (int j = 0; j < 8; ++j) kp.trace_iter[j] = j < sp->n_trace ? sp->trace_iter[j] : -1;
    kp.seed_best_cost = sbc; kp.seed_best_traj = sbt;
    const size_t bytes = make_layout(ctx->rp, use_gmem_world(ctx) ? 0 : ctx->kmax_enabled, mode, H, sp->history, sp->n_alpha, true, kp.lay);
    kp.lay.boxes_gmem = use_gmem_world(ctx) ? 1 : 0;
    if (bytes > SMEM_MAX) return fail(ctx, CRB_E_LIMIT, "shared memory footprint too large (robot + cuboids + solver)");
    const bool wm = use_gmem_world(ctx);
    // latency mode: A CTAs per seed in a cluster when the whole batch fits one wave (2 CTAs / SM)
    const long long units = mode == MODE_TO ? (long long)P * S : (long long)P * ((S + NC - 1) / NC);
    // automatic choice (tools/cluster_vs_seq.py): the batch fits one wave in cluster mode; or the
    // particle warm-up (split A ways, not repeated) runs on at most 3 waves of units; or the
    // predicted wave count, ceil(A units / W) / A with ~15 % cluster overhead, beats the
    // sequential one by 5 % (a poorly filled last wave).  W = two CTAs per SM.
    const long long W = 2LL * ctx->sm_count, A_ = sp->n_alpha;
    const bool fits = units * A_ <= W;
    const bool parts = sp->particle_iters > 0 && units <= 3 * W;
    const bool waves = (double)((units * A_ + W - 1) / W) / (double)A_ * 1.15 < 0.95 * (double)((units + W - 1) / W);
    const bool clus = sp->n_alpha >= 2 && (sp->particle_iters == 0 || sp->n_particles >= sp->n_alpha) && !kp.trace &&
                      (sp->cluster == 1 || (sp->cluster == -1 && (fits || parts || waves)));
    if (clus && units > 0) {
        const void *kern = mode == MODE_TO
                               ? (H > NC ? (wm ? crb_gmem_kernel(KW_SOLVE_TO_CLUSTER_LONG) : (const void *)solve_to_cluster_kernel<false, true>)
                                         : (wm ? crb_gmem_kernel(KW_SOLVE_TO_CLUSTER) : (const void *)solve_to_cluster_kernel<false, false>))
                               : (wm ? crb_gmem_kernel(KW_SOLVE_IK_CLUSTER) : (const void *)solve_ik_cluster_kernel<false>);
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
        if (e != cudaSuccess) return cuda_check(ctx, e, "solve_cluster_kernel");
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3((unsigned)(units * sp->n_alpha));
        cfg.blockDim = dim3(NT);
        cfg.dynamicSmemBytes = bytes;
        cfg.stream = stream_;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = (unsigned)sp->n_alpha;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        void *args[] = {(void *)&kp};
        e = cudaLaunchKernelExC(&cfg, kern, args);
        ctx->launches++;
        if (e != cudaSuccess) return cuda_check(ctx, e, "solve_cluster_kernel");
        st = cuda_check(ctx, cudaGetLastError(), "solve_cluster_kernel");
    } else if (mode == MODE_TO) {
        // TO scheduling: the persistent chunked kernel when the seed
        // trajectories span >= 2 waves, 10 iteration chunks (measured best of 2..25 at cfg 2 / 4);
        // sp->persist = 0 forces one CTA per seed, k >= 1 k chunks.
        const void *kern = H > NC ? (wm ? crb_gmem_kernel(KW_SOLVE_TO_LONG) : (const void *)solve_to_kernel<false, true, false>)
                                  : (wm ? crb_gmem_kernel(KW_SOLVE_TO) : (const void *)solve_to_kernel<false, false, false>);
        const void *kern_p = H > NC ? (wm ? crb_gmem_kernel(KW_SOLVE_TO_LONG_PERSIST) : (const void *)solve_to_kernel<false, true, true>)
                                    : (wm ? crb_gmem_kernel(KW_SOLVE_TO_PERSIST) : (const void *)solve_to_kernel<false, false, true>);
        const long long NU = (long long)P * S;
        int chunks = sp->persist;
        int per_sm = 0;
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
        if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, NT, bytes);
        if (e != cudaSuccess || per_sm < 1) return cuda_check(ctx, e != cudaSuccess ? e : cudaErrorInvalidConfiguration, "occupancy");
        const long long Wr = (long long)per_sm * ctx->sm_count;
        if (chunks < 0) chunks = (NU >= 2 * Wr && sp->iters >= 8 && !kp.trace) ? 10 : 0;
        chunks = std::min(chunks, std::max(sp->iters, 1));
        if (chunks >= 1) {
            const int m = sp->history, Np = (N + 3) & ~3;
            const size_t swt = (size_t)6 * Np + (size_t)2 * (m + 1) * Np + 160 + 8;
            if ((st = grow(ctx, &ctx->ws_ik_state, &ctx->cap_ik_state, (size_t)NU * swt)) != CRB_OK) return st;
            if ((st = grow(ctx, &ctx->ws_ik_flags, &ctx->cap_ik_flags, (size_t)NU + 2)) != CRB_OK) return st;
            kp.ik_state = ctx->ws_ik_state; kp.ik_flags = ctx->ws_ik_flags; kp.ik_chunks = chunks;
            ik_persist_init_kernel<<<1, 256, 0, stream_>>>(nullptr, P, (int)NU, ctx->ws_ik_flags);
            ctx->launches++;
            if ((st = cuda_check(ctx, cudaGetLastError(), "ik_persist_init_kernel")) != CRB_OK) return st;
            e = cudaFuncSetAttribute(kern_p, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
            if (e != cudaSuccess) return cuda_check(ctx, e, "solve_to_kernel (persistent)");
            st = launch_fn(ctx, kern_p, (int)std::min<long long>(NU * chunks, Wr), bytes, stream_, kp,
                           "solve_to_kernel (persistent)");
        } else {
            st = launch_fn(ctx, kern, P * S, bytes, stream_, kp, "solve_to_kernel");
        }
    }
    else {
        // IK scheduling: the persistent chunked kernel when the batch
        // spans at least two waves of groups (sp->persist = -1: 16 iteration chunks, measured best
        // of 2..25 at cfg 3), else one CTA per 32-seed group.  sp->persist = 0 forces the latter,
        // k >= 1 k chunks.
        const int G = (S + NC - 1) / NC;
        const long long NGg = (long long)P * G;
        int chunks = sp->persist;
        if (chunks < 0) chunks = (NGg >= 2 * W && sp->iters >= 8) ? 16 : 0;
        chunks = std::min(chunks, std::max(sp->iters, 1));
        if (chunks >= 1) {
            const int m = sp->history, DC = D * NC;
            const size_t swt = (size_t)(6 + 2 * (m + 1)) * DC + 3 * (m + 1) * NC + (m + 5) * NC;
            if ((st = grow(ctx, &ctx->ws_ik_state, &ctx->cap_ik_state, (size_t)NGg * swt)) != CRB_OK) return st;
            if ((st = grow(ctx, &ctx->ws_ik_flags, &ctx->cap_ik_flags, (size_t)NGg + 2)) != CRB_OK) return st;
            kp.ik_state = ctx->ws_ik_state; kp.ik_flags = ctx->ws_ik_flags; kp.ik_chunks = chunks;
            ik_persist_init_kernel<<<1, 256, 0, stream_>>>(env, P, (int)NGg, ctx->ws_ik_flags);
            ctx->launches++;
            if ((st = cuda_check(ctx, cudaGetLastError(), "ik_persist_init_kernel")) != CRB_OK) return st;
            const void *kern = wm ? crb_gmem_kernel(KW_SOLVE_IK_PERSIST) : (const void *)solve_ik_kernel<false, true>;
            cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
            if (e != cudaSuccess) return cuda_check(ctx, e, "solve_ik_kernel (persistent)");
            int per_sm = 0;
            e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, NT, bytes);
            if (e != cudaSuccess || per_sm < 1) return cuda_check(ctx, e != cudaSuccess ? e : cudaErrorInvalidConfiguration, "occupancy");
            const long long grid = std::min<long long>(NGg * chunks, (long long)per_sm * ctx->sm_count);
            st = launch_fn(ctx, kern, (int)grid, bytes, stream_, kp, "solve_ik_kernel (persistent)");
        } else {
            kp.ik_chunks = 1;
            st = launch_fn(ctx, wm ? crb_gmem_kernel(KW_SOLVE_IK) : (const void *)solve_ik_kernel<false, false>, (int)NGg,
                           bytes, stream_, kp, "solve_ik_kernel");
        }
    }
    if (st != CRB_OK) return st;
    if (P > 0 && (best_traj || best_cost || best_key)) {
        select_kernel<<<P, 128, 0, stream_>>>(P, S, N, sbc, sbt, (long long)sp->global_seed_base, best_traj,
                                              best_cost, (long long *)best_key);
        ctx->launches++;
        st = cuda_check(ctx, cudaGetLastError(), "select_kernel");
    }
    return st;
}

crb_status crb_lbfgs_solve_host(crb_ctx *ctx, const crb_solver_params *sp, int P, int S, int H, const float *seeds,
                                const int *env, const float *start, const float *goal, float *best_traj,
                                float *best_cost, int64_t *best_key, void *stream) {
    crb_status st = enter(ctx);
    if (st != CRB_OK) return st;
    if ((st = ready(ctx, true)) != CRB_OK) return st;
    if (!sp || P < 0 || S < 1 || H < 1 || (P > 0 && (!seeds || !goal))) return fail(ctx, CRB_E_ARG, "bad solve arguments");
    if (P == 0)   // validate the parameters, copy nothing
        return crb_lbfgs_solve(ctx, sp, 0, S, H, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr,
                               nullptr, stream);
    const int D = ctx->rp.D, N = H * D;
    if (env)   // host buffer: the env indices can be checked here (the device path poisons them with NaN)
        for (int p = 0; p < P; ++p)
            if (env[p] < 0 || env[p] >= ctx->n_env) return fail(ctx, CRB_E_SHAPE, "env index outside [0, n_env)");
    cudaStream_t s = (cudaStream_t)stream;
    if ((st = grow(ctx, &ctx->h_seeds, &ctx->cap_h_seeds, (size_t)P * S * N)) != CRB_OK) return st;
    const int gw = (ctx->cp.flags & CRB_CSPACE) ? D : 7;
    if ((st = grow(ctx, &ctx->h_goal, &ctx->cap_h_goal, (size_t)P * gw)) != CRB_OK) return st;
    if ((st = grow(ctx, &ctx->h_best, &ctx->cap_h_best, (size_t)P * N)) != CRB_OK) return st;
    if ((st = grow(ctx, &ctx->h_bcost, &ctx->cap_h_bcost, (size_t)P)) != CRB_OK) return st;
    if ((st = grow(ctx, &ctx->h_key, &ctx->cap_h_key, (size_t)P)) != CRB_OK) return st;
    if (start && (st = grow(ctx, &ctx->h_start, &ctx->cap_h_start, (size_t)P * D)) != CRB_OK) return st;
    if (env && (st = grow(ctx, &ctx->h_env, &ctx->cap_h_env, (size_t)P)) != CRB_OK) return st;
    st = cuda_check(ctx, cudaMemcpyAsync(ctx->h_seeds, seeds, (size_t)P * S * N * 4, cudaMemcpyHostToDevice, s), "H2D seeds");
    if (st == CRB_OK) st = cuda_check(ctx, cudaMemcpyAsync(ctx->h_goal, goal, (size_t)P * gw * 4, cudaMemcpyHostToDevice, s), "H2D goal");
    if (st == CRB_OK && start) st = cuda_check(ctx, cudaMemcpyAsync(ctx->h_start, start, (size_t)P * D * 4, cudaMemcpyHostToDevice, s), "H2D start");
    if (st == CRB_OK && env) st = cuda_check(ctx, cudaMemcpyAsync(ctx->h_env, env, (size_t)P * 4, cudaMemcpyHostToDevice, s), "H2D env");
    if (st != CRB_OK) return st;
    st = crb_lbfgs_solve(ctx, sp, P, S, H, ctx->h_seeds, env ? ctx->h_env : nullptr, start ? ctx->h_start : nullptr,
                         ctx->h_goal, ctx->h_best, ctx->h_bcost, (int64_t *)ctx->h_key, nullptr, nullptr, stream);
    if (st != CRB_OK) return st;
    if (best_traj) st = cuda_check(ctx, cudaMemcpyAsync(best_traj, ctx->h_best, (size_t)P * N * 4, cudaMemcpyDeviceToHost, s), "D2H best");
    if (st == CRB_OK && best_cost) st = cuda_check(ctx, cudaMemcpyAsync(best_cost, ctx->h_bcost, (size_t)P * 4, cudaMemcpyDeviceToHost, s), "D2H cost");
    if (st == CRB_OK && best_key) st = cuda_check(ctx, cudaMemcpyAsync(best_key, ctx->h_key, (size_t)P * 8, cudaMemcpyDeviceToHost, s), "D2H key");
    if (st != CRB_OK) return st;
    return cuda_check(ctx, cudaStreamSynchronize(s), "solve_host synchronize");
}

crb_status crb_solver_occupancy(crb_ctx *ctx, int H, int history, int n_alpha, int *ctas_per_sm,
                                 int *smem_bytes) {
    crb_status st = enter(ctx);
    if (st != CRB_OK) return st;
    if ((st = ready(ctx, true)) != CRB_OK) return st;
    KParams kp = base_params(ctx);
    const int mode = H == 1 ? MODE_IK : MODE_TO;
    const size_t bytes = make_layout(ctx->rp, use_gmem_world(ctx) ? 0 : ctx->kmax_enabled, mode, H, history, n_alpha, true, kp.lay);
    kp.lay.boxes_gmem = use_gmem_world(ctx) ? 1 : 0;
    if (smem_bytes) *smem_bytes = (int)bytes;
    if (bytes > SMEM_MAX) { if (ctas_per_sm) *ctas_per_sm = 0; return CRB_OK; }
    int n = 0;
    const bool wm = use_gmem_world(ctx);
    const void *fn = mode == MODE_TO ? (H > NC ? (wm ? crb_gmem_kernel(KW_SOLVE_TO_LONG) : (const void *)solve_to_kernel<false, true, false>)
                                                : (wm ? crb_gmem_kernel(KW_SOLVE_TO) : (const void *)solve_to_kernel<false, false, false>))
                                     : (wm ? crb_gmem_kernel(KW_SOLVE_IK) : (const void *)solve_ik_kernel<false, false>);
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    st = cuda_check(ctx, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, fn, NT, bytes), "occupancy");
    if (ctas_per_sm) *ctas_per_sm = n;
    return st;
}

crb_status crb_ls_select(int n, int A, const float *alpha_host, const float *c0, const float *g0d, const float *ca,
                         const float *gda, float c1, float c2, int mode, int *out_idx, void *stream) {
    if (n < 0 || A < 1 || A > 8 || !alpha_host || !c0 || !g0d || !ca || !gda || !out_idx) return CRB_E_ARG;
    LsParams ap{};
    for (int a = 0; a < A; ++a) ap.alpha[a] = alpha_host[a];
    if (n == 0) return CRB_OK;
    ls_select_kernel<<<(n + 127) / 128, 128, 0, (cudaStream_t)stream>>>(n, A, ap, c0, g0d, ca, gda, c1, c2, mode, out_idx);
    return cudaGetLastError() == cudaSuccess ? CRB_OK : CRB_E_CUDA;
}

crb_status crb_argmin_keys(int P, int S, const float *cost, int64_t seed_base, int64_t *out_key, int *out_idx,
                           void *stream) {
    if (P < 0 || S < 1 || !cost) return CRB_E_ARG;
    if (P == 0) return CRB_OK;
    argmin_keys_kernel<<<(P + 127) / 128, 128, 0, (cudaStream_t)stream>>>(P, S, cost, (long long)seed_base,
                                                                        (long long *)out_key, out_idx);
    return cudaGetLastError() == cudaSuccess ? CRB_OK : CRB_E_CUDA;
}

crb_status crb_lbfgs_direction(int B, int n, int count, const float *S, const float *Y, const float *g, float *d,
                               void *stream) {
    if (B < 0 || n < 1 || n > 2 * NT || count < 0 || count > 32 || !g || !d || (count > 0 && (!S || !Y))) return CRB_E_ARG;
    if (B == 0) return CRB_OK;
    const int Np = (n + 3) & ~3;
    const size_t bytes = (size_t)(2 * count * Np + 2 * Np + 96 + 3 * NW + 32) * 4;
    if (cudaFuncSetAttribute(lbfgs_direction_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes) != cudaSuccess)
        return CRB_E_CUDA;
    lbfgs_direction_kernel<<<B, NT, bytes, (cudaStream_t)stream>>>(n, count, S, Y, g, d);
    return cudaGetLastError() == cudaSuccess ? CRB_OK : CRB_E_CUDA;
}

crb_status crb_mask_samples(crb_ctx *ctx, const float *q, int K, const int *env, int env_div, float margin,
                            uint8_t *valid, void *stream) {
    crb_status st = enter(ctx);
    if (st != CRB_OK) return st;
    if ((st = ready(ctx, true)) != CRB_OK) return st;
    if (K < 0 || (K > 0 && (!q || !valid)) || !(margin >= 0.f) || env_div < 1)
        return fail(ctx, CRB_E_ARG, "bad mask arguments");
    KParams kp = base_params(ctx);
    kp.B = K; kp.H = 1; kp.cp.H = 1; kp.mode = MODE_IK; kp.q_in = q; kp.env = env; kp.margin = margin;
    kp.mask_out = valid; kp.env_div = env_div;
    const size_t bytes = make_layout(ctx->rp, ctx->kmax_enabled, MODE_IK, 1, 1, 1, false, kp.lay);
    if (bytes > SMEM_MAX) return fail(ctx, CRB_E_LIMIT, "shared memory footprint too large (robot + cuboids)");
    return launch(ctx, mask_kernel, (K + NC - 1) / NC, bytes, (cudaStream_t)stream, kp, "mask_kernel");
}

crb_status crb_steer(crb_ctx *ctx, int E, const float *src, const float *dst, const float *dw, float r, int env,
                     float margin, int n_cap, int *n_out, int *h, float *v_new, float *dist, void *stream) {
    crb_status st = enter(ctx);
    if (st != CRB_OK) return st;
    if ((st = ready(ctx, true)) != CRB_OK) return st;
    if (E < 0 || (E > 0 && (!src || !dst || !dw || !h || !v_new || !dist)) || !(r > 0.f) || !(margin >= 0.f) ||
        n_cap < 1 || env < 0 || env >= ctx->n_env)
        return fail(ctx, CRB_E_ARG, "bad steer arguments");
    if (E == 0) return CRB_OK;
    const int D = ctx->rp.D;
    const size_t nw = (size_t)E * (n_cap + 1);
    if (nw > (size_t)1 << 31) return fail(ctx, CRB_E_LIMIT, "E * (n_cap + 1) too large");
    if ((st = grow(ctx, &ctx->ws_mask, &ctx->cap_mask, nw)) != CRB_OK) return st;
    if ((st = grow(ctx, &ctx->ws_n, &ctx->cap_n, (size_t)2)) != CRB_OK) return st;
    cudaStream_t s = (cudaStream_t)stream;
    steer_n_kernel<<<1, NT, 0, s>>>(E, D, src, dst, dw, r, n_cap, ctx->ws_n);
    ctx->launches++;
    if ((st = cuda_check(ctx, cudaGetLastError(), "steer_n_kernel")) != CRB_OK) return st;
    KParams kp = base_params(ctx);
    kp.H = 1; kp.cp.H = 1; kp.mode = MODE_IK; kp.margin = margin; kp.mask_out = ctx->ws_mask;
    kp.e_src = src; kp.e_dst = dst; kp.e_n = ctx->ws_n; kp.E = E; kp.e_env = env;
    const size_t bytes = make_layout(ctx->rp, ctx->kmax_enabled, MODE_IK, 1, 1, 1, false, kp.lay);
    if (bytes > SMEM_MAX) return fail(ctx, CRB_E_LIMIT, "shared memory footprint too large (robot + cuboids)");
    if ((st = launch(ctx, mask_kernel, (int)((nw + NC - 1) / NC), bytes, s, kp, "mask_kernel")) != CRB_OK) return st;
    steer_scan_kernel<<<(E + 7) / 8, 256, 0, s>>>(E, D, src, dst, dw, ctx->ws_n, ctx->ws_mask, h, v_new, dist);
    ctx->launches++;
    if ((st = cuda_check(ctx, cudaGetLastError(), "steer_scan_kernel")) != CRB_OK) return st;
    if (n_out)
        st = cuda_check(ctx, cudaMemcpyAsync(n_out, ctx->ws_n, 2 * sizeof(int), cudaMemcpyDeviceToDevice, s), "n copy");
    return st;
}

crb_status crb_retime(crb_ctx *ctx, int B, int H, const float *V, const float *start, int start_div, const float *dt,
                      float *scale, float *dt_opt, float *max_jerk, void *stream) {
    crb_status st = enter(ctx);
    if (st != CRB_OK) return st;
    if ((st = ready(ctx, false)) != CRB_OK) return st;
    if (B < 0 || H < 8 || (B > 0 && (!V || !start || !scale)) || start_div < 1)
        return fail(ctx, CRB_E_ARG, "bad retime arguments (H >= 8, start_div >= 1)");
    if (B == 0) return CRB_OK;
    const float *lim = reinterpret_cast<const float *>(ctx->d_robot) + ctx->rp.o_lim;
    retime_kernel<<<(B + 7) / 8, 256, 0, (cudaStream_t)stream>>>(B, H, ctx->rp.D, V, start, start_div, dt,
                                                                   ctx->params_ok ? ctx->cp.dt : 0.25f, lim, scale,
                                                                   dt_opt, max_jerk);
    ctx->launches++;
    return cuda_check(ctx, cudaGetLastError(), "retime_kernel");
}

crb_status crb_goal_error(crb_ctx *ctx, int B, const float *q, int q_stride, const float *goal, int goal_div,
                          float *pos_err, float *rot_err, void *stream) {
    crb_status st = enter(ctx);
    if (st != CRB_OK) return st;
    if ((st = ready(ctx, false)) != CRB_OK) return st;
    if (B < 0 || (B > 0 && (!q || !goal || !pos_err || !rot_err)) || q_stride < ctx->rp.D || goal_div < 1)
        return fail(ctx, CRB_E_ARG, "bad goal_error arguments");
    KParams kp = base_params(ctx);
    kp.kmax = 0;
    kp.B = B; kp.H = 1; kp.cp.H = 1; kp.mode = MODE_IK; kp.q_in = q; kp.q_stride = q_stride; kp.goal = goal;
    kp.pos_err_out = pos_err; kp.rot_err_out = rot_err; kp.goal_div = goal_div;
    const size_t bytes = make_layout(ctx->rp, 0, MODE_IK, 1, 1, 1, false, kp.lay);
    if (bytes > SMEM_MAX) return fail(ctx, CRB_E_LIMIT, "shared memory footprint too large");
    return launch(ctx, fk_kernel, (B + NC - 1) / NC, bytes, (cudaStream_t)stream, kp, "fk_kernel(goal_error)");
}

crb_status crb_ik_scores(int P, int S, int D, const float *q, const float *q0, const float *pos_err, const float *rot_err,
                         const uint8_t *valid, float pos_thr, float rot_thr, float w_pose, float w_dist, float penalty,
                         float *score, void *stream) {
    if (P < 0 || S < 1 || D < 1 || (P > 0 && (!q || !q0 || !pos_err || !rot_err || !score))) return CRB_E_ARG;
    if (P == 0) return CRB_OK;
    ik_scores_kernel<<<(P * S + 255) / 256, 256, 0, (cudaStream_t)stream>>>(P, S, D, q, q0, pos_err, rot_err, valid, pos_thr,
                                                                          rot_thr, w_pose, w_dist, penalty, score);
    return cudaGetLastError() == cudaSuccess ? CRB_OK : CRB_E_CUDA;
}

crb_status crb_to_scores(int P, int S, int H, const float *pos_err, const float *rot_err, const float *max_jerk,
                         const float *dt_opt, const uint8_t *valid, float pos_thr, float rot_thr, float w_pose,
                         float w_jerk, float w_time, float penalty, float *score, void *stream) {
    if (P < 0 || S < 1 || H < 1 || (P > 0 && (!pos_err || !rot_err || !max_jerk || !dt_opt || !score))) return CRB_E_ARG;
    if (P == 0) return CRB_OK;
    to_scores_kernel<<<(P * S + 255) / 256, 256, 0, (cudaStream_t)stream>>>(P, S, H, pos_err, rot_err, max_jerk, dt_opt,
                                                                          valid, pos_thr, rot_thr, w_pose, w_jerk, w_time,
                                                                          penalty, score);
    return cudaGetLastError() == cudaSuccess ? CRB_OK : CRB_E_CUDA;
}

crb_status crb_rank_seeds(int P, int S, const float *score, int k, int *idx, int *count, void *stream) {
    if (P < 0 || S < 1 || k < 1 || (P > 0 && (!score || !idx || !count))) return CRB_E_ARG;
    if (P == 0) return CRB_OK;
    rank_kernel<<<(P + 7) / 8, 256, 0, (cudaStream_t)stream>>>(P, S, score, k, idx, count);
    return cudaGetLastError() == cudaSuccess ? CRB_OK : CRB_E_CUDA;
}

crb_status crb_linear_seeds(int P, int S, int H, int D, const float *q0, const float *qT, int Sq, const int *idx,
                            float *seeds, void *stream) {
    if (P < 0 || S < 1 || H < 2 || D < 1 || Sq < 1 || (P > 0 && (!q0 || !qT || !seeds)) || (!idx && Sq < S))
        return CRB_E_ARG;
    if (P == 0) return CRB_OK;
    const size_t n = (size_t)P * S * H * D;
    const int grid = (int)std::min<size_t>((n + 255) / 256, 148 * 16);
    linear_seeds_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(P, S, H, D, q0, qT, Sq, idx, seeds);
    return cudaGetLastError() == cudaSuccess ? CRB_OK : CRB_E_CUDA;
}

crb_status crb_trajectory_states(int B, int H, int D, const float *V, const float *start, int start_div, float *x,
                                 void *stream) {
    if (B < 0 || H < 8 || D < 1 || start_div < 1 || (B > 0 && (!V || !start || !x))) return CRB_E_ARG;
    if (B == 0) return CRB_OK;
    const size_t n = (size_t)B * H * D;
    const int grid = (int)std::min<size_t>((n + 255) / 256, 148 * 16);
    states_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(B, H, D, V, start, start_div, x);
    return cudaGetLastError() == cudaSuccess ? CRB_OK : CRB_E_CUDA;
}

crb_status crb_interpolate(int B, int H, int D, const float *x, const float *dt, float dt_fine, int n_max, float *out,
                           int *n_out, void *stream) {
    if (B < 0 || H < 2 || D < 1 || !(dt_fine > 0.f) || n_max < 1 || (B > 0 && (!x || !dt || !out))) return CRB_E_ARG;
    if (B == 0) return CRB_OK;
    if (B > 65535) return CRB_E_LIMIT;
    const int gx = std::min((n_max * D + 255) / 256, 64);
    interp_kernel<<<dim3(gx, B), 256, 0, (cudaStream_t)stream>>>(B, H, D, x, dt, dt_fine, n_max, out, n_out);
    return cudaGetLastError() == cudaSuccess ? CRB_OK : CRB_E_CUDA;
}

crb_status crb_gather_rows(int P, int S, int n, const float *src, const int *idx, int idx_stride, float *dst,
                           void *stream) {
    if (P < 0 || S < 1 || n < 1 || idx_stride < 1 || (P > 0 && (!src || !idx || !dst))) return CRB_E_ARG;
    if (P == 0) return CRB_OK;
    const size_t tot = (size_t)P * n;
    const int grid = (int)std::min<size_t>((tot + 255) / 256, 148 * 16);
    gather_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(P, S, n, src, idx, idx_stride, dst);
    return cudaGetLastError() == cudaSuccess ? CRB_OK : CRB_E_CUDA;
}

crb_status crb_particle_normals(uint32_t key0, uint32_t key1, int n_var, int n_particles, int iter, uint32_t seed,
                                float *out, void *stream) {
    if (n_var < 0 || n_particles < 0 || iter < 0 || (!out && n_var * n_particles > 0)) return CRB_E_ARG;
    const int total = n_var * n_particles;
    if (total == 0) return CRB_OK;
    particle_normals_kernel<<<(total + 255) / 256, 256, 0, (cudaStream_t)stream>>>(key0, key1, n_var, n_particles,
                                                                                  iter, seed, out);
    return cudaGetLastError() == cudaSuccess ? CRB_OK : CRB_E_CUDA;
}

}  // extern "C"

#if CRB_STATS
// world-screen work counters (tools/world_stats.py only; not part of the product ABI)
extern "C" int crb_debug_stats(unsigned long long *out, int reset) {
    unsigned long long w[32];
    if (stats_copy(out, reset) != 0 || crb_gmem_stats(w, reset) != 0) return -1;
    for (int i = 0; i < 32; ++i) out[i] += w[i];   // the counters of both translation units
    return 0;
}
#endif

#endif  // CRB_PART == 0
