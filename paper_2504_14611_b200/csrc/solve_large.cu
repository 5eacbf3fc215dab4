// K1L: J-DOB for instances with more users than a warp has lanes (32 < M <= 1024;
// SURVEY NEXT-4, SPEC S:442's M = 1000 complexity case).  One 256-thread block per
// instance: users are spread over the threads for the per-n~ setup (gamma, the
// O(M^2/256) rank sort, thresholds), grid points over the threads for the Alg. 2 sweep,
// and the user-order energy sum of each configuration runs sequentially in its thread
// (that order is what makes the result bit-identical to the oracle).  The same readings,
// exact shortcuts and arithmetic contract as K1 (solve.cu).
//
// Launched after K1 over the whole batch; each block scans a contiguous instance range
// and solves only those K1 deferred (M > 32), so batches without such instances pay one
// short scan.
#include "jdob_dev.cuh"
#include "kernels.h"

namespace jdob {

constexpr int kLT = 256;  // threads per block
constexpr int kLInv = 192;

struct LargeView {
    double *gam, *L, *th, *gq, *T, *inv;
    int *rank, *order;
    double2 *et, *orzv, *kuup, *fmm;
};

__device__ __forceinline__ LargeView carve(char *p) {
    LargeView v;
    v.gam = (double *)p;
    v.L = v.gam + kMaxMLarge;
    v.th = v.L + kMaxMLarge;
    v.gq = v.th + kMaxMLarge;
    v.T = v.gq + kMaxMLarge;
    v.inv = v.T + kMaxMLarge;
    double2 *q = (double2 *)(v.inv + kLInv);
    v.et = q;
    v.orzv = q + kMaxMLarge;
    v.kuup = v.orzv + kMaxMLarge;
    v.fmm = v.kuup + kMaxMLarge;
    v.rank = (int *)(v.fmm + kMaxMLarge);
    v.order = v.rank + kMaxMLarge;
    return v;
}

size_t large_smem_bytes() { return (size_t)kMaxMLarge * (6 * 8 + 4 * 16 + 2 * 4) + kLInv * 8; }

// block-wide reductions through a small shared scratch
__device__ __forceinline__ double block_min_d(double v, double *scr) {
#pragma unroll
    for (int d = 16; d >= 1; d >>= 1) {
        const double o = __shfl_xor_sync(0xffffffffu, v, d);
        v = (o < v) ? o : v;
    }
    __syncthreads();
    if ((threadIdx.x & 31) == 0) scr[threadIdx.x >> 5] = v;
    __syncthreads();
    double r = scr[0];
    for (int w = 1; w < kLT / 32; w++) r = (scr[w] < r) ? scr[w] : r;
    __syncthreads();
    return r;
}

__device__ __forceinline__ double block_max_d(double v, double *scr) {
    return -block_min_d(-v, scr);
}

// ranks under (gamma desc, T asc, index asc) (R2); homogeneous users pass gam == null (key (T, index))
__device__ void large_sort(int M, const double *gam, LargeView &s) {
    for (int m = threadIdx.x; m < M; m += kLT) {
        const double g = gam ? gam[m] : 0.0, T = s.T[m];
        int r = 0;
        for (int t = 0; t < M; t++) {
            const double gt = gam ? gam[t] : 0.0, Tt = s.T[t];
            r += ((gt > g) || (gt == g && (Tt < T || (Tt == T && t < m)))) ? 1 : 0;
        }
        s.rank[m] = r;
        s.order[r] = m;
    }
    __syncthreads();
    if (threadIdx.x == 0) {  // suffix-min deadlines over sorted positions (Eq. fth's min, R1)
        double L = dinf();
        for (int q = M - 1; q >= 0; q--) {
            const double T = s.T[s.order[q]];
            if (T < L) L = T;
            s.L[q] = L;
        }
    }
    __syncthreads();
}

// Alg. 1 lines 4-6 for partition point nt; returns i^ (M if none)
__device__ int large_setup(const DevModel &md, int nt, int M, bool homog, double t_free, const DevBatch &b,
                           long long off, LargeView &s, int *iscr) {
    const double v_nt = md.v[nt], u_nt = md.u[nt], O_nt = md.O[nt];
    for (int m = threadIdx.x; m < M; m += kLT) {
        const long long u = off + m;
        const double OR = O_nt / b.R[u];  // Eq. (3)
        const double zv = b.zeta[u] * v_nt;
        s.gam[m] = OR + div_z(zv, b.f_max[u]);  // gamma
        s.orzv[m] = make_double2(OR, zv);
        s.kuup[m] = make_double2(b.kappa[u] * u_nt, OR * b.p_u[u]);  // Eq. (4)
    }
    __syncthreads();
    if (!homog) large_sort(M, s.gam, s);
    if (threadIdx.x == 0) iscr[0] = M;
    __syncthreads();
    for (int i = threadIdx.x; i < M; i += kLT) {
        const double gi = homog ? s.gam[0] : s.gam[s.order[i]];
        const double phi = md.phi[nt * md.B1 + (M - i)];
        const double th = phi / (s.L[i] - gi);  // Eq. (fth)
        s.th[i] = th;
        s.gq[i] = phi / (s.L[i] - t_free);      // D6 guard quotient of the set starting at i
        if (th >= 0.0) atomicMin(iscr, i);
    }
    __syncthreads();
    const int ihat = iscr[0];
    for (int m = threadIdx.x; m < M; m += kLT) {
        const int rm = s.rank[m];
        s.et[m].y = (rm >= ihat) ? s.th[rm] : dinf();
    }
    __syncthreads();
    return ihat;
}

template <bool COUNTS>
__device__ void large_instance(long long i, const DevModel *models, const DevBatch &b, const DevResult &r, int mode,
                               LargeView &s, double *dscr, int *iscr, long long *cscr) {
    const int tid = threadIdx.x;
    const long long off = b.user_off[i];
    const int M = (int)((b.user_end ? b.user_end[i] : b.user_off[i + 1]) - off);  // user_end: OG's views
    const DevModel &md = models[b.model_id[i]];
    const int N = md.N;
    const double t_free = b.t_free[i], fe_min = b.fe_min[i], fe_max = b.fe_max[i], rho = b.rho[i];
    const double vN = md.v[N], uN = md.u[N];
    // validation with the oracle's precedence (model id, validity and M were checked by K1)
    if (tid == 0) {
        iscr[0] = 0;  // bad user parameters
        iscr[1] = 0;  // local infeasibility
        iscr[2] = 1;  // homogeneous (R, zeta, f_max)
        iscr[3] = 1;  // uniform (+ f_min, kappa, p_u)
    }
    __syncthreads();
    double tmin = dinf();
    const long long u0 = off;
    for (int m = tid; m < M; m += kLT) {
        const long long u = off + m;
        const double z = b.zeta[u], k = b.kappa[u], f0 = b.f_min[u], f1 = b.f_max[u], R = b.R[u], p = b.p_u[u],
                     T = b.T[u];
        bool ok = dfinite(z) && dfinite(k) && dfinite(f0) && dfinite(f1) && dfinite(R) && dfinite(p) && dfinite(T);
        ok = ok && (z >= 0.0) && (k >= 0.0) && (f0 > 0.0) && (f0 <= f1) && (R > 0.0) && (p >= 0.0) && (T > 0.0);
        if (!ok) atomicOr(&iscr[0], 1);
        if (ok && (z * vN) / f1 > T) atomicOr(&iscr[1], 1);
        if (!(R == b.R[u0] && z == b.zeta[u0] && f1 == b.f_max[u0])) atomicAnd(&iscr[2], 0);
        if (!(f0 == b.f_min[u0] && k == b.kappa[u0] && p == b.p_u[u0])) atomicAnd(&iscr[3], 0);
        s.T[m] = T;
        tmin = (T < tmin) ? T : tmin;
    }
    tmin = block_min_d(tmin, dscr);
    const bool bad_user = iscr[0] != 0, linf = iscr[1] != 0, homog = iscr[2] != 0;
    const bool uni = homog && iscr[3] != 0;
    int st = JDOB_ST_OK;
    long long k = 0;
    if (bad_user) st = JDOB_ST_BADPARAM;
    else if (!(dfinite(t_free) && dfinite(fe_min) && dfinite(fe_max) && dfinite(rho) && (t_free >= 0.0) &&
               (fe_min > 0.0) && (fe_min <= fe_max) && (rho > 0.0)))
        st = JDOB_ST_BADPARAM;
    else {
        k = grid_k(fe_min, fe_max, rho);
        if (k > kMaxK) st = JDOB_ST_BADPARAM;
        else if (linf) st = JDOB_ST_LOCAL_INFEASIBLE;
        else if (tmin < t_free) st = JDOB_ST_REQUIRE;
    }
    if (st == JDOB_ST_BADPARAM) {
        if (tid == 0) {
            r.E[i] = dnan();
            r.E_lc[i] = dnan();
            r.t_free_next[i] = t_free;
            r.f_e[i] = 0.0;
            r.n_tilde[i] = N;
            r.j[i] = 0;
            r.status[i] = st;
            // jdob_eval gives no bits for a malformed instance; the others are not verified here
            if (r.viol) r.viol[i] = (st == JDOB_ST_BADPARAM || st == JDOB_ST_BADMODEL) ? 0u : 0x80000000u;
            r.mask[i] = 0u;
            if (r.counts) r.counts[3 * i] = r.counts[3 * i + 1] = r.counts[3 * i + 2] = 0;
            if (r.work) r.work[4 * i] = r.work[4 * i + 1] = r.work[4 * i + 2] = r.work[4 * i + 3] = 0;
        }
        for (int m = tid; m < M; m += kLT) {
            if (r.f_user) r.f_user[off + m] = dnan();
            if (r.partition) r.partition[off + m] = N;
        }
        __syncthreads();
        return;
    }
    // LC (row a2)
    for (int m = tid; m < M; m += kLT) {
        const long long u = off + m;
        const double floc = clampf((b.zeta[u] * vN) / b.T[u], b.f_min[u], b.f_max[u]);
        s.et[m].x = ((b.kappa[u] * uN) * floc) * floc;
        s.fmm[m] = make_double2(b.f_min[u], b.f_max[u]);
        s.gam[m] = floc;  // scratch: f_loc until the sweep
    }
    __syncthreads();
    if (tid == 0) {
        double E = 0.0;
        for (int m = 0; m < M; m++) E = E + s.et[m].x;  // user-index order
        dscr[8] = E;
    }
    __syncthreads();
    const double E_lc = dscr[8];
    auto write_local = [&](bool zero_counts) {
        if (tid == 0) {
            r.E[i] = E_lc;
            r.E_lc[i] = E_lc;
            r.t_free_next[i] = t_free;
            r.f_e[i] = 0.0;
            r.n_tilde[i] = N;
            r.j[i] = 0;
            r.status[i] = st;
            // jdob_eval gives no bits for a malformed instance; the others are not verified here
            if (r.viol) r.viol[i] = (st == JDOB_ST_BADPARAM || st == JDOB_ST_BADMODEL) ? 0u : 0x80000000u;
            r.mask[i] = 0u;
            if (r.counts && zero_counts) r.counts[3 * i] = r.counts[3 * i + 1] = r.counts[3 * i + 2] = 0;
            if (r.work && zero_counts) r.work[4 * i] = r.work[4 * i + 1] = r.work[4 * i + 2] = r.work[4 * i + 3] = 0;
        }
        for (int m = tid; m < M; m += kLT) {
            const long long u = off + m;
            if (r.f_user) r.f_user[u] = clampf((b.zeta[u] * vN) / b.T[u], b.f_min[u], b.f_max[u]);
            if (r.partition) r.partition[u] = N;
        }
        __syncthreads();
    };
    if (st != JDOB_ST_OK || mode == JDOB_MODE_LC) {
        write_local(true);
        return;
    }
    const long long kk = (mode == JDOB_MODE_NO_EDGE_DVFS) ? 1 : k;
    for (long long j = tid; j < kk && j < kLInv; j += kLT) s.inv[j] = 1.0 / grid_fe(fe_max, rho, j);
    if (homog) large_sort(M, nullptr, s);
    __syncthreads();
    double bE = dinf();
    int bN = 0x7fffffff, bJ = 0, bP = 0;
    int aN = N, aJ = 0;
    long long c_visit = 0, c_eval = 0, c_member = 0;
    for (int nt = 0; nt < N; nt++) {
        if (mode == JDOB_MODE_BINARY && nt != 0) break;
        const int ihat = large_setup(md, nt, M, homog, t_free, b, off, s, iscr);
        if (tid == 0) iscr[1] = (int)kk;  // first j with an empty set
        __syncthreads();
        for (long long j0 = 0; j0 < kk; j0 += kLT) {
            const long long j = j0 + tid;
            if (j >= kk) continue;
            const double fe = grid_fe(fe_max, rho, j);
            int lo = ihat, hi = M;
            while (lo < hi) {
                const int mm = (lo + hi) >> 1;
                if (fe < s.th[mm]) lo = mm + 1;
                else hi = mm;
            }
            const int p = lo;
            if (p == M) {  // empty set: Alg. 2's break point (monotone in j)
                atomicMin(&iscr[1], (int)j);
                continue;
            }
            if (COUNTS) c_visit += 1;
            if (!(fe >= s.gq[p])) continue;  // D6 guard
            if (COUNTS) {
                c_eval += 1;
                c_member += M - p;
            }
            const double inv = (j < kLInv) ? s.inv[j] : 1.0 / fe;
            const double lo_ = s.L[p];
            const double te = md.phi[nt * md.B1 + (M - p)] * inv;
            double E = 0.0;
            if (uni) {
                const double2 a0 = s.orzv[0], c0 = s.kuup[0], t0 = s.fmm[0];
                const double budget = (lo_ - a0.x) - te;
                double f = t0.x;
                if (!(__fma_rn(t0.x, budget, -a0.y) > 0.0) && a0.y != 0.0) f = clampf(a0.y / budget, t0.x, t0.y);
                const double em = ((c0.x * f) * f) + c0.y;
                for (int m = 0; m < M; m++) {
                    const double2 et = s.et[m];
                    E = E + ((!(fe < et.y)) ? em : et.x);
                }
            } else {
                for (int m = 0; m < M; m++) {
                    const double2 a = s.orzv[m], c = s.kuup[m], d = s.et[m], t = s.fmm[m];
                    const bool mem = !(fe < d.y);
                    double e = d.x;
                    if (mem) {
                        const double budget = (lo_ - a.x) - te;
                        double f = t.x;
                        if (!(__fma_rn(t.x, budget, -a.y) > 0.0) && a.y != 0.0) f = clampf(a.y / budget, t.x, t.y);
                        e = ((c.x * f) * f) + c.y;
                    }
                    E = E + e;
                }
            }
            E = E + (md.psi[nt * md.B1 + (M - p)] * fe) * fe;
            if (E < bE) {  // strict: thread keys ascend in (n~, j)
                bE = E;
                bN = nt;
                bJ = (int)j;
                bP = p;
            }
        }
        __syncthreads();
        const int jb = iscr[1];
        if (jb < kk) {
            if (aN == N) {
                aN = nt;
                aJ = jb;
            }
            if (COUNTS && tid == 0) {  // the all-local evaluation at jb
                c_visit += 1;
                c_eval += 1;
            }
        }
        __syncthreads();
    }
    // block argmin over (E, n~, j)
#pragma unroll
    for (int d = 16; d >= 1; d >>= 1) {
        const double oE = __shfl_xor_sync(0xffffffffu, bE, d);
        const int oN = __shfl_xor_sync(0xffffffffu, bN, d);
        const int oJ = __shfl_xor_sync(0xffffffffu, bJ, d);
        const int oP = __shfl_xor_sync(0xffffffffu, bP, d);
        if ((oE < bE) || (oE == bE && (oN < bN || (oN == bN && oJ < bJ)))) {
            bE = oE;
            bN = oN;
            bJ = oJ;
            bP = oP;
        }
    }
    if ((tid & 31) == 0) {
        dscr[tid >> 5] = bE;
        iscr[4 + 3 * (tid >> 5)] = bN;
        iscr[5 + 3 * (tid >> 5)] = bJ;
        iscr[6 + 3 * (tid >> 5)] = bP;
    }
    if (COUNTS) {
        if (tid == 0) cscr[0] = cscr[1] = cscr[2] = 0;
    }
    __syncthreads();
    if (COUNTS) {
        atomicAdd((unsigned long long *)&cscr[0], (unsigned long long)c_visit);
        atomicAdd((unsigned long long *)&cscr[1], (unsigned long long)c_eval);
        atomicAdd((unsigned long long *)&cscr[2], (unsigned long long)c_member);
    }
    bE = dscr[0];
    bN = iscr[4];
    bJ = iscr[5];
    bP = iscr[6];
    for (int w = 1; w < kLT / 32; w++) {
        const double oE = dscr[w];
        const int oN = iscr[4 + 3 * w], oJ = iscr[5 + 3 * w], oP = iscr[6 + 3 * w];
        if ((oE < bE) || (oE == bE && (oN < bN || (oN == bN && oJ < bJ)))) {
            bE = oE;
            bN = oN;
            bJ = oJ;
            bP = oP;
        }
    }
    __syncthreads();
    if (COUNTS && tid == 0 && r.counts) {
        r.counts[3 * i] = cscr[0];
        r.counts[3 * i + 1] = cscr[1];
        r.counts[3 * i + 2] = cscr[2];
    }
    if (COUNTS && tid == 0 && r.work) {  // no pruning on this path: executed = literal
        r.work[4 * i] = (mode == JDOB_MODE_BINARY) ? 1 : N;
        r.work[4 * i + 1] = cscr[0];
        r.work[4 * i + 2] = cscr[1];
        r.work[4 * i + 3] = cscr[2];
    }
    const bool offload_wins = (bE < E_lc) || (bE == E_lc && (bN < aN || (bN == aN && bJ < aJ)));
    if (!offload_wins) {
        write_local(false);
        return;
    }
    // winner: D20 per user and D22 (same arithmetic as the sweep)
    large_setup(md, bN, M, homog, t_free, b, off, s, iscr);
    const double lo_ = s.L[bP];
    const double fe = grid_fe(fe_max, rho, bJ);
    const double inv = 1.0 / fe;
    const double te = md.phi[bN * md.B1 + (M - bP)] * inv;
    double arr_max = t_free;
    for (int m = tid; m < M; m += kLT) {
        const long long u = off + m;
        const bool member = s.rank[m] >= bP;
        double f;
        if (member) {
            const double2 a = s.orzv[m], t = s.fmm[m];
            const double budget = (lo_ - a.x) - te;
            const bool low = (a.y == 0.0) || (__fma_rn(t.x, budget, -a.y) > 0.0);
            f = low ? t.x : clampf(div_z(a.y, budget), t.x, t.y);  // zv = 0 (n~ = 0): no slow-path 0 / budget
            const double arr = div_z(a.y, f) + a.x;
            arr_max = (arr > arr_max) ? arr : arr_max;
        } else {
            f = clampf((b.zeta[u] * vN) / b.T[u], b.f_min[u], b.f_max[u]);
        }
        if (r.f_user) r.f_user[u] = f;
        if (r.partition) r.partition[u] = member ? bN : N;
    }
    arr_max = block_max_d(arr_max, dscr);
    if (tid == 0) {
        r.E[i] = bE;
        r.E_lc[i] = E_lc;
        r.t_free_next[i] = arr_max + te;  // D22
        r.f_e[i] = fe;
        r.n_tilde[i] = bN;
        r.j[i] = bJ;
        r.status[i] = st;
        if (r.viol) r.viol[i] = 0x80000000u;  // not verified in this kernel (include/jdob.h)
        r.mask[i] = 0u;  // M > 32: see partition
    }
    __syncthreads();
}

template <bool COUNTS>
__global__ void __launch_bounds__(kLT) k_solve_large(const DevModel *models, DevBatch b, DevResult r, int mode) {
    extern __shared__ __align__(16) char lsm[];
    __shared__ double dscr[16];
    __shared__ int iscr[4 + 3 * (kLT / 32) + 4];
    __shared__ long long cscr[3];
    __shared__ int list[kLT];
    __shared__ int nlist;
    LargeView s = carve(lsm);
    const long long n = b.n_inst;
    const long long i0 = n * blockIdx.x / gridDim.x, i1 = n * (blockIdx.x + 1) / gridDim.x;
    for (long long base = i0; base < i1; base += kLT) {
        if (threadIdx.x == 0) nlist = 0;
        __syncthreads();
        const long long i = base + threadIdx.x;
        if (i < i1) {
            const long long M64 = (b.user_end ? b.user_end[i] : b.user_off[i + 1]) - b.user_off[i];
            const int mid = b.model_id[i];
            // the instances K1 deferred: valid model, 32 < M <= min(1024, B_max)
            if (M64 > kMaxM && M64 <= kMaxMLarge && mid >= 0 && mid < b.n_models && *models[mid].valid &&
                M64 <= models[mid].B1 - 1)
                list[atomicAdd(&nlist, 1)] = (int)(i - base);
        }
        __syncthreads();
        const int cnt = nlist;
        // ascending order is not needed (instances are independent); process the found ones
        for (int q = 0; q < cnt; q++) large_instance<COUNTS>(base + list[q], models, b, r, mode, s, dscr, iscr, cscr);
        __syncthreads();
    }
}

void launch_solve_large(const DevModel *models, const DevBatch &b, const DevResult &r, int mode, cudaStream_t s,
                        int num_sms) {
    if (b.n_inst <= 0) return;
    const size_t smem = large_smem_bytes();
    long long grid = 2LL * num_sms;
    if (b.n_inst < grid) grid = b.n_inst;
    if (r.counts || r.work) {
        cudaFuncSetAttribute(k_solve_large<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        k_solve_large<true><<<(unsigned)grid, kLT, smem, s>>>(models, b, r, mode);
    } else {
        cudaFuncSetAttribute(k_solve_large<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        k_solve_large<false><<<(unsigned)grid, kLT, smem, s>>>(models, b, r, mode);
    }
}

}  // namespace jdob
