// K3: configuration evaluator (row a11): D20-D22 generalised to per-user
// partition points (R14: same-sub-task greedy batching, ALAP batch starts; R15:
// ASAP finishing time), with violation bits at a relative slack.
// One thread per instance; the O(N) batch-size and suffix tables live in the
// thread's local memory (this is a verification pass, not the inner loop).
#include <climits>

#include "jdob_dev.cuh"
#include "kernels.h"

namespace jdob {

// The user arrays of one instance: X[m] is user off + m's value (in global memory, or in the
// shared-memory window that holds the instance's users).
struct UserView {
    const double *z, *k, *f0, *f1, *R, *p, *T;
};

// One configuration (instance i), one thread: the reference form of the evaluator.
// (off, M64) = user_off[i] and the user count, loaded by the caller; uv.X[m] is user off + m's value.
__device__ __forceinline__ void eval_one(long long i, long long off, long long M64, const UserView &uv,
                                         const DevModel *models, const DevBatch &b, const int *partition,
                                         const int *plan_nt, const unsigned *plan_mask, const double *f_e,
                                         double slack, double *E_out, double *tf_out, double *f_user,
                                         unsigned *viol_out, int *status_out) {
    const int mid = b.model_id[i];
    const double t_free = b.t_free[i], fe_min = b.fe_min[i], fe_max = b.fe_max[i], rho = b.rho[i];
    const unsigned pmask = partition ? 0u : plan_mask[i];  // the identical plan, read once per instance
    const int pnt = partition ? 0 : plan_nt[i];
    int st = JDOB_ST_OK;
    if (mid < 0 || mid >= b.n_models) st = JDOB_ST_BADPARAM;
    const DevModel *mdp = (st == JDOB_ST_OK) ? &models[mid] : nullptr;
    if (st == JDOB_ST_OK && *mdp->valid == 0) st = JDOB_ST_BADMODEL;
    if (st == JDOB_ST_OK && (M64 < 1 || M64 > kMaxM || M64 > mdp->B1 - 1)) st = JDOB_ST_BADPARAM;
    const int M = (int)((M64 >= 1 && M64 <= kMaxM) ? M64 : 0);
    const int N = mdp ? mdp->N : 0;
    // one pass over the users: the box checks (BADPARAM), local feasibility, min T (Require,
    // P:259) and, for an identical plan, l_o = min T over its members; the statuses are then decided in
    // the oracle's precedence order (BADPARAM before LOCAL_INFEASIBLE before REQUIRE)
    double Tmin = dinf(), lo_plan = dinf();
    if (st == JDOB_ST_OK) {
        const double vN0 = mdp->v[N];
        bool bad = false, infeas = false;
        for (int m = 0; m < M; m++) {
            const double z = uv.z[m], k = uv.k[m], f0 = uv.f0[m], f1 = uv.f1[m], R = uv.R[m], p = uv.p[m],
                         T = uv.T[m];
            bool ok = dfinite(z) && dfinite(k) && dfinite(f0) && dfinite(f1) && dfinite(R) && dfinite(p) &&
                      dfinite(T) && (z >= 0.0) && (k >= 0.0) && (f0 > 0.0) && (f0 <= f1) && (R > 0.0) &&
                      (p >= 0.0) && (T > 0.0);
            const bool mem = (pmask >> m) & 1u;
            const int nm = partition ? partition[off + m] : (mem ? pnt : N);
            ok = ok && nm >= 0 && nm <= N;
            bad |= !ok;
            // RN(zeta v_N / f_max) > T; the fma sign proves "no" without the division
            const double zvN = z * vN0;
            if (ok && !(__fma_rn(T, f1, -zvN) > 0.0) && zvN / f1 > T) infeas = true;
            if (T < Tmin) Tmin = T;
            if (mem && T < lo_plan) lo_plan = T;
        }
        bool ok = dfinite(t_free) && dfinite(fe_min) && dfinite(fe_max) && dfinite(rho) && (t_free >= 0.0) &&
                  (fe_min > 0.0) && (fe_min <= fe_max) && (rho > 0.0);
        if (bad || !ok || grid_k(fe_min, fe_max, rho) > kMaxK) st = JDOB_ST_BADPARAM;
        else if (infeas) st = JDOB_ST_LOCAL_INFEASIBLE;
    }
    if (st == JDOB_ST_BADPARAM || st == JDOB_ST_BADMODEL) {
        E_out[i] = dnan();
        tf_out[i] = dnan();
        viol_out[i] = 0u;
        status_out[i] = st;
        return;
    }
    const DevModel &md = *mdp;
    const int B1 = md.B1;
    const double vN = md.v[N], uN = md.u[N];
    if (st == JDOB_ST_OK && Tmin < t_free) st = JDOB_ST_REQUIRE;
    unsigned viol = (Tmin < t_free) ? 16u : 0u;

    // batch sizes b_n = #{m : n_m < n} and suffix sums S_n = sum_{n' >= n} d_n'(b_n') A_n' (R14).
    // Identical plans (partition == NULL): b_n = B_o for n > n~, so S_{n~+1} and Psi are the
    // phi/psi aggregates of K0 (the same additions in the same order -> the same bits).
    int bcnt[kMaxN + 2];
    double S[kMaxN + 2];
    double Psi = 0.0, S_plan = 0.0;
    bool any = false;
    int nmin = N;
    double l_o = dinf();
    if (partition == nullptr) {
        const unsigned mk = pmask & (M >= 32 ? 0xffffffffu : ((1u << M) - 1u));
        const int nt = pnt;
        const int Bo = __popc(mk);
        if (Bo > 0 && nt < N) {
            any = true;
            nmin = nt;
            S_plan = md.phi[nt * B1 + Bo];
            Psi = md.psi[nt * B1 + Bo];
            l_o = lo_plan;
        }
    } else {
        for (int n = 1; n <= N; n++) bcnt[n] = 0;
        for (int m = 0; m < M; m++) {
            const int nm = partition[off + m];
            for (int n = nm + 1; n <= N; n++) bcnt[n]++;
        }
        S[N + 1] = 0.0;
        for (int n = N; n >= 1; n--) {
            const int bn = bcnt[n];
            S[n] = S[n + 1] + (bn > 0 ? md.dA[n * B1 + bn] : 0.0);
            Psi = Psi + (bn > 0 ? md.cA[n * B1 + bn] : 0.0);
        }
        for (int m = 0; m < M; m++) {
            const int nm = partition[off + m];
            if (nm < N) {
                any = true;
                if (nm < nmin) nmin = nm;
                const double T = uv.T[m];
                if (T < l_o) l_o = T;
            }
        }
    }
    const double fe = f_e[i];
    // f_e = 0 marks an all-local plan (R18); 1 / f_e is only used with members, so without members
    // the divisor is 1 (behind an opaque move: no slow-path division of 1 / 0)
    double fe_d;
    asm("mov.b64 %0, %1;" : "=d"(fe_d) : "d"(any ? fe : 1.0));
    const double inv = 1.0 / fe_d;
    const double tol = slack * fabs(l_o);
    double tf = t_free;
    if (any) {
        if (!(fe >= fe_min && fe <= fe_max)) viol |= 32u;
        double start = t_free + (partition ? S[nmin + 1] : S_plan) * inv;
        if (start > l_o + tol) viol |= 1u;
        tf = start;
    }
    double E = 0.0;
    for (int m = 0; m < M; m++) {
        const long long u = off + m;
        const int nm = partition ? partition[u] : (((pmask >> m) & 1u) ? pnt : N);
        double e, f;
        if (nm < N) {
            double OR = md.O[nm] / uv.R[m];
            double zv = uv.z[m] * md.v[nm];
            const double Sn = partition ? S[nm + 1] : S_plan;
            double budget = (l_o - OR) - Sn * inv;
            const double f0 = uv.f0[m];
            if (zv == 0.0) {
                if (budget < 0.0) viol |= 8u;
                f = f0;
            } else if (__fma_rn(f0, budget, -zv) > 0.0) {
                f = f0;  // f_min budget - zv > 0 exactly: budget > 0 and RN(zv / budget) <= f_min
            } else if (budget > 0.0) {
                f = clampf(zv / budget, f0, uv.f1[m]);
            } else {
                viol |= 8u;
                f = uv.f1[m];
            }
            e = ((uv.k[m] * md.u[nm]) * f) * f + OR * uv.p[m];
            double arr = div_z(zv, f) + OR;
            double fin = arr + Sn * inv;
            if (fin > l_o + tol) viol |= 2u;
            if (fin > tf) tf = fin;
        } else {
            double T = uv.T[m];
            const double zvN = uv.z[m] * vN, f0 = uv.f0[m];
            f = (__fma_rn(f0, T, -zvN) > 0.0) ? f0 : clampf(zvN / T, f0, uv.f1[m]);
            e = ((uv.k[m] * uN) * f) * f;
            if (d8_violated(uv.z[m] * vN, f, T + slack * fabs(T))) viol |= 4u;
        }
        if (f_user) f_user[u] = f;
        E = E + e;
    }
    E = E + (Psi * fe) * fe;
    E_out[i] = E;
    tf_out[i] = tf;
    viol_out[i] = viol;
    status_out[i] = st;
}

#ifndef JDOB_EVAL_WINDOW
#define JDOB_EVAL_WINDOW 1280  // users per shared-memory window (C2: 128 instances x 10 users, one pass)
#endif
constexpr int kEvalThreads = 128;                 // one thread per instance of the tile
constexpr int kEvalWin = JDOB_EVAL_WINDOW;        // even
constexpr int kEvalStride = kEvalWin + 2;         // per array: the window + alignment slack, 16-B multiple
static_assert(kEvalWin % 2 == 0, "window must be even");

__device__ __forceinline__ unsigned smem_u32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }

// Block-wide min/max of a 64-bit key (every thread gets the result).
__device__ __forceinline__ long long block_min_ll(long long x, long long *red) {
#pragma unroll
    for (int d = 16; d >= 1; d >>= 1) {
        const long long o = __shfl_xor_sync(0xffffffffu, x, d);
        x = o < x ? o : x;
    }
    __syncthreads();  // the previous reduction's reads of red[] are done
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = x;
    __syncthreads();
#pragma unroll
    for (int w = 0; w < kEvalThreads / 32; w++) x = red[w] < x ? red[w] : x;
    return x;
}

// K3 with the users staged in shared memory (see the header).  Persistent grid; tile t = instances
// [128 t, 128 t + 128).  `bulk`: the seven user arrays are 16-byte aligned, so every window is moved by
// seven cp.async.bulk copies issued by one thread; otherwise by the block's plain coalesced loads.
__global__ void __launch_bounds__(kEvalThreads) k_eval(const DevModel *models, DevBatch b, const int *partition,
                                                       const int *plan_nt, const unsigned *plan_mask,
                                                       const double *f_e, double slack, double *E_out,
                                                       double *tf_out, double *f_user, unsigned *viol_out,
                                                       int *status_out, int bulk) {
    extern __shared__ __align__(16) double ewin[];  // [7][kEvalStride]
    __shared__ __align__(8) unsigned long long bar;
    __shared__ long long red[kEvalThreads / 32];
    const int tid = threadIdx.x;
    const double *src[7] = {b.zeta, b.kappa, b.f_min, b.f_max, b.R, b.p_u, b.T};
    if (tid == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncthreads();
    unsigned phase = 0;
    const long long n_tiles = (b.n_inst + kEvalThreads - 1) / kEvalThreads;
    for (long long t = blockIdx.x; t < n_tiles; t += gridDim.x) {
        const long long i = t * kEvalThreads + tid;
        long long off = 0, M64 = 0;
        bool pending = false;
        if (i < b.n_inst) {
            off = b.user_off[i];
            M64 = b.user_off[i + 1] - off;
            // users are read only for an instance with 1 <= M <= 32 (otherwise BADPARAM before any read)
            pending = (M64 >= 1 && M64 <= kMaxM && off >= 0);
            if (!pending) {
                const UserView g{b.zeta + off, b.kappa + off, b.f_min + off, b.f_max + off, b.R + off,
                                 b.p_u + off, b.T + off};
                eval_one(i, off, M64, g, models, b, partition, plan_nt, plan_mask, f_e, slack, E_out, tf_out,
                         f_user, viol_out, status_out);
            }
        }
        for (bool first = true;; first = false) {
            // window [lo, hi): first the tile's whole user range when it fits (the common case, no
            // reduction), then from the smallest pending offset until every instance is served
            long long lo = 0, hi = 0;
            bool fast = false;
            if (first) {
                const long long i1 = (t + 1) * kEvalThreads < b.n_inst ? (t + 1) * kEvalThreads : b.n_inst;
                lo = b.user_off[t * kEvalThreads];
                hi = b.user_off[i1];
                fast = lo >= 0 && hi > lo && hi - lo <= kEvalWin;  // block-uniform
            } else if (!__syncthreads_or(pending)) {
                break;  // (the barrier also orders this pass's reads before the next tile's copies)
            }
            if (!fast) {
                lo = block_min_ll(pending ? off : LLONG_MAX, red);
                if (lo == LLONG_MAX) break;  // block-uniform
                hi = -block_min_ll(pending ? -(off + M64) : LLONG_MAX, red);
            }
            const long long w0 = lo & ~1ll;                                   // 16-byte aligned start
            const long long w1 = (hi - w0 <= kEvalWin) ? hi : w0 + kEvalWin;  // window end (exclusive)
            const long long nb = (w1 - w0) & ~1ll;                            // bulk part: 16-byte multiple
            JDOB_CHECK(w0 >= 0 && w1 > w0 && w1 - w0 <= kEvalWin && (w0 & 1) == 0);
            if (bulk) {
                if (tid == 0) {
                    const unsigned bytes = (unsigned)(nb * 8 * 7);
                    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar)),
                                 "r"(bytes)
                                 : "memory");
                    for (int a = 0; a < 7 && nb > 0; a++)  // (one instance of one user: tail only)
                        asm volatile(
                            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                                smem_u32(ewin + a * kEvalStride)),
                            "l"(src[a] + w0), "r"((unsigned)(nb * 8)), "r"(smem_u32(&bar))
                            : "memory");
                }
                if (tid < 7 && nb < w1 - w0) ewin[tid * kEvalStride + nb] = src[tid][w0 + nb];  // odd tail element
            } else {
                for (long long e = tid; e < w1 - w0; e += kEvalThreads)
#pragma unroll
                    for (int a = 0; a < 7; a++) ewin[a * kEvalStride + e] = src[a][w0 + e];
            }
            __syncthreads();
            if (bulk) {
                asm volatile(
                    "{\n .reg .pred P;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n"
                    " @!P bra WAIT_%=;\n}\n" ::"r"(smem_u32(&bar)),
                    "r"(phase)
                    : "memory");
                phase ^= 1u;
            }
#ifndef JDOB_EVAL_NO_L2PF
            if (first && bulk && tid == 0 && t + gridDim.x < n_tiles) {
                // the block's next tile: its user range is pulled into L2 while this one is evaluated
                const long long nt0 = (t + gridDim.x) * kEvalThreads;
                const long long nt1 = nt0 + kEvalThreads < b.n_inst ? nt0 + kEvalThreads : b.n_inst;
                const long long p0 = b.user_off[nt0] & ~1ll, p1 = b.user_off[nt1];
                if (p0 >= 0 && p1 - p0 >= 2 && p1 - p0 <= kEvalWin) {
                    const unsigned bytes = (unsigned)(((p1 - p0) & ~1ll) * 8);  // inside the arrays
                    for (int a = 0; a < 7; a++)
                        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src[a] + p0), "r"(bytes)
                                     : "memory");
                }
            }
#endif
            if (pending && off >= w0 && off + M64 <= w1) {
                const long long e = off - w0;
                JDOB_CHECK(e >= 0 && e + M64 <= kEvalStride && M64 >= 1 && M64 <= kMaxM);
                const UserView v{ewin + e, ewin + kEvalStride + e, ewin + 2 * kEvalStride + e,
                                 ewin + 3 * kEvalStride + e, ewin + 4 * kEvalStride + e, ewin + 5 * kEvalStride + e,
                                 ewin + 6 * kEvalStride + e};
                eval_one(i, off, M64, v, models, b, partition, plan_nt, plan_mask, f_e, slack, E_out, tf_out,
                         f_user, viol_out, status_out);
                pending = false;
            }
            // this thread's reads of the window are ordered before the async-proxy writes of the next
            // copy (issued after the next barrier)
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        }
    }
}

void launch_eval(const DevModel *models, const DevBatch &b, const int *partition, const int *plan_nt,
                 const unsigned *plan_mask, const double *f_e, double slack, double *E, double *tf, double *f_user,
                 unsigned *viol, int *status, cudaStream_t s) {
    if (b.n_inst <= 0) return;
    const size_t smem = sizeof(double) * 7 * kEvalStride;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_eval, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        attr = true;
    }
    int dev = 0, sms = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_eval, kEvalThreads, smem);
    if (per_sm < 1) per_sm = 1;
    const long long tiles = (b.n_inst + kEvalThreads - 1) / kEvalThreads;
    long long grid = (long long)sms * per_sm;
    if (tiles < grid) grid = tiles;
    int bulk = 1;
    const double *arr[7] = {b.zeta, b.kappa, b.f_min, b.f_max, b.R, b.p_u, b.T};
    for (int a = 0; a < 7; a++) bulk &= (((uintptr_t)arr[a] & 15u) == 0u) ? 1 : 0;
    k_eval<<<(unsigned)grid, kEvalThreads, smem, s>>>(models, b, partition, plan_nt, plan_mask, f_e, slack, E, tf,
                                                      f_user, viol, status, bulk);
}

}  // namespace jdob
