// K1: J-DOB solve over a batch of independent instances (rows a2-a8).
//
// One warp per instance (persistent grid-stride loop).  Per partition point n~ the
// warp first works lane = user (gamma, hoists, all-pairs rank sort, suffix-min
// deadlines, thresholds), then lane = edge-grid point j for the Alg. 2 sweep:
// each lane finds its offloading set as the suffix of the sorted list starting at
// p(j) = min{i >= i^ : !(f_e(j) < th_i)} -- equal to Alg. 2's sequential pointer
// because the thresholds are exactly non-increasing from i^ (DESIGN.md §Sweep
// equivalence) -- checks the D6 guard, evaluates D20-D21 in user-index order and
// keeps a lane-local strict minimum.  A warp argmin over (E, n~, j) and the first
// all-local evaluation (R8) give the Alg. 1 answer; the winner's D20/D22 values
// are recomputed lane = user.
#include "jdob_dev.cuh"
#include "kernels.h"

namespace jdob {

struct SolveSmem {
    double eloc[kMaxM], fmin[kMaxM], fmax[kMaxM], T[kMaxM];
    double OR[kMaxM], zv[kMaxM], ku[kMaxM], up[kMaxM], gam[kMaxM];
    double th[kMaxM], L[kMaxM];
    int rank[kMaxM], order[kMaxM];
};

// Alg. 1 lines 4-6 for partition point nt.  Returns i^ (M if none).
__device__ __forceinline__ int setup_nt(const DevModel &md, int nt, int M, const InstRegs &x, SolveSmem &s,
                                        int lane) {
    const double v_nt = md.v[nt], u_nt = md.u[nt], O_nt = md.O[nt];
    double gam = 0.0;
    if (lane < M) {
        double OR = O_nt / x.R;                              // Eq. (3)
        double zv = x.z * v_nt;
        gam = OR + zv / x.f1;                                // gamma
        s.OR[lane] = OR;
        s.zv[lane] = zv;
        s.ku[lane] = x.k * u_nt;
        s.up[lane] = OR * x.p;                               // Eq. (4)
        s.gam[lane] = gam;
    }
    // rank under the key (gamma desc, T asc, index asc) (R2)
    int r = 0;
    for (int t = 0; t < M; t++) {
        double gt = __shfl_sync(0xffffffffu, gam, t);
        double Tt = __shfl_sync(0xffffffffu, x.T, t);
        bool before = (gt > gam) || (gt == gam && (Tt < x.T || (Tt == x.T && t < lane)));
        r += before ? 1 : 0;
    }
    if (lane < M) {
        s.rank[lane] = r;
        s.order[r] = lane;
    }
    __syncwarp();
    // suffix-min deadline and thresholds over sorted positions (Eq. fth, R1)
    double L = dinf(), gi = 0.0;
    if (lane < M) {
        int mi = s.order[lane];
        L = s.T[mi];
        gi = s.gam[mi];
    }
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        double o = __shfl_down_sync(0xffffffffu, L, d);
        if (lane + d < 32 && o < L) L = o;
    }
    double th = 0.0;
    if (lane < M) {
        th = md.phi[nt * md.B1 + (M - lane)] / (L - gi);
        s.th[lane] = th;
        s.L[lane] = L;
    }
    unsigned nn = __ballot_sync(0xffffffffu, lane < M && th >= 0.0);
    __syncwarp();
    return nn ? (__ffs(nn) - 1) : M;
}

__device__ __forceinline__ void write_bad(const DevResult &r, long long i, long long off, int M, int N, double t_free,
                                          int st, int lane) {
    if (lane == 0) {
        r.E[i] = dnan();
        r.E_lc[i] = dnan();
        r.t_free_next[i] = t_free;
        r.f_e[i] = 0.0;
        r.n_tilde[i] = N;
        r.j[i] = 0;
        r.status[i] = st;
        r.mask[i] = 0u;
        if (r.counts) {
            r.counts[3 * i] = 0;
            r.counts[3 * i + 1] = 0;
            r.counts[3 * i + 2] = 0;
        }
    }
    if (r.f_user && M >= 1 && M <= kMaxM && lane < M) r.f_user[off + lane] = dnan();
}

__device__ void solve_instance(long long i, const DevModel *models, const DevBatch &b, const DevResult &r, int mode,
                               SolveSmem &s, int lane) {
    __syncwarp();
    long long off, k;
    int M;
    const DevModel *mdp;
    InstRegs x;
    int st = warp_validate(models, b, i, lane, x, M, k, mdp, off);
    const double t_free = b.t_free[i], fe_min = b.fe_min[i], fe_max = b.fe_max[i], rho = b.rho[i];
    (void)fe_min;
    if (st == JDOB_ST_BADPARAM || st == JDOB_ST_BADMODEL) {
        write_bad(r, i, off, M, mdp ? mdp->N : 0, t_free, st, lane);
        return;
    }
    const DevModel &md = *mdp;
    const int N = md.N;
    const double vN = md.v[N], uN = md.u[N];

    // LC (row a2): f_loc = clamp(zeta v_N / T), e_loc = ((kappa u_N) f) f
    double floc = 0.0, eloc = 0.0;
    if (lane < M) {
        double G = (x.z * vN) / x.T;
        floc = clampf(G, x.f0, x.f1);
        eloc = ((x.k * uN) * floc) * floc;
        s.eloc[lane] = eloc;
        s.fmin[lane] = x.f0;
        s.fmax[lane] = x.f1;
    }
    s.T[lane] = x.T;  // +inf beyond M
    double E_lc = 0.0;
    for (int t = 0; t < M; t++) E_lc = E_lc + __shfl_sync(0xffffffffu, eloc, t);  // user-index order
    __syncwarp();

    if (st != JDOB_ST_OK || mode == JDOB_MODE_LC) {
        if (lane == 0) {
            r.E[i] = E_lc;
            r.E_lc[i] = E_lc;
            r.t_free_next[i] = t_free;
            r.f_e[i] = 0.0;
            r.n_tilde[i] = N;
            r.j[i] = 0;
            r.status[i] = st;
            r.mask[i] = 0u;
            if (r.counts) {
                r.counts[3 * i] = 0;
                r.counts[3 * i + 1] = 0;
                r.counts[3 * i + 2] = 0;
            }
        }
        if (r.f_user && lane < M) r.f_user[off + lane] = floc;
        return;
    }

    const long long kk = (mode == JDOB_MODE_NO_EDGE_DVFS) ? 1 : k;
    const int B1 = md.B1;
    double bE = dinf();
    int bN = 0x7fffffff, bP = 0;
    long long bJ = 0;
    int aN = N;          // first all-local evaluation key (R8); n~ = N at j = 0 by default (R4)
    long long aJ = 0;
    long long c_visit = 0, c_eval = 0, c_member = 0;

    for (int nt = 0; nt < N; nt++) {
        if (mode == JDOB_MODE_BINARY && nt != 0) break;
        const int ihat = setup_nt(md, nt, M, x, s, lane);
        // first j whose offloading set is empty: f_e(j) < th_{M-1} (or j = 0 if i^ = NAN)
        long long jb;
        if (ihat == M) {
            jb = 0;
        } else {
            const double thl = s.th[M - 1];
            long long lo = 0, hi = kk;
            while (lo < hi) {
                long long md2 = (lo + hi) >> 1;
                if (grid_fe(fe_max, rho, md2) < thl) hi = md2;
                else lo = md2 + 1;
            }
            jb = lo;
        }
        if (jb < kk) {
            if (aN == N) {
                aN = nt;
                aJ = jb;
            }
            if (lane == 0) {  // the all-local evaluation at jb (guard passes: 0 / inf = 0)
                c_visit += 1;
                c_eval += 1;
            }
        }
        const long long jend = (jb < kk) ? jb : kk;
        const double *phi_row = md.phi + nt * B1;
        const double *psi_row = md.psi + nt * B1;
        for (long long j0 = 0; j0 < jend; j0 += 32) {
            const long long j = j0 + lane;
            if (j < jend) {
                const double fe = grid_fe(fe_max, rho, j);
                const double inv = 1.0 / fe;
                int lo = ihat, hi = M;
                while (lo < hi) {
                    int mm = (lo + hi) >> 1;
                    if (fe < s.th[mm]) lo = mm + 1;
                    else hi = mm;
                }
                const int p = lo;
                const int Bo = M - p;
                const double lo_ = s.L[p];
                const double phib = phi_row[Bo];
                c_visit += 1;
                if (fe >= phib / (lo_ - t_free)) {  // D6 guard
                    c_eval += 1;
                    c_member += Bo;
                    const double te = phib * inv;
                    double E = 0.0;
                    for (int m = 0; m < M; m++) {
                        double e;
                        if (s.rank[m] >= p) {
                            const double zv = s.zv[m];
                            double f;
                            if (zv == 0.0) {
                                f = s.fmin[m];  // R9
                            } else {
                                const double budget = (lo_ - s.OR[m]) - te;
                                f = clampf(zv / budget, s.fmin[m], s.fmax[m]);  // D20
                            }
                            e = ((s.ku[m] * f) * f) + s.up[m];  // D21 offloader term
                        } else {
                            e = s.eloc[m];
                        }
                        E = E + e;
                    }
                    E = E + (psi_row[Bo] * fe) * fe;
                    if (E < bE) {  // strict: lane keys ascend in (n~, j)
                        bE = E;
                        bN = nt;
                        bJ = j;
                        bP = p;
                    }
                }
            }
        }
        __syncwarp();
    }
    // warp argmin over (E, n~, j)
#pragma unroll
    for (int d = 16; d >= 1; d >>= 1) {
        double oE = __shfl_xor_sync(0xffffffffu, bE, d);
        int oN = __shfl_xor_sync(0xffffffffu, bN, d);
        long long oJ = __shfl_xor_sync(0xffffffffu, bJ, d);
        int oP = __shfl_xor_sync(0xffffffffu, bP, d);
        bool take = (oE < bE) || (oE == bE && (oN < bN || (oN == bN && oJ < bJ)));
        if (take) {
            bE = oE;
            bN = oN;
            bJ = oJ;
            bP = oP;
        }
    }
    if (r.counts) {
#pragma unroll
        for (int d = 16; d >= 1; d >>= 1) {
            c_visit += __shfl_xor_sync(0xffffffffu, c_visit, d);
            c_eval += __shfl_xor_sync(0xffffffffu, c_eval, d);
            c_member += __shfl_xor_sync(0xffffffffu, c_member, d);
        }
        if (lane == 0) {
            r.counts[3 * i] = c_visit;
            r.counts[3 * i + 1] = c_eval;
            r.counts[3 * i + 2] = c_member;
        }
    }
    const bool offload_wins = (bE < E_lc) || (bE == E_lc && (bN < aN || (bN == aN && bJ < aJ)));
    if (!offload_wins) {
        if (lane == 0) {
            r.E[i] = E_lc;
            r.E_lc[i] = E_lc;
            r.t_free_next[i] = t_free;
            r.f_e[i] = 0.0;
            r.n_tilde[i] = N;
            r.j[i] = 0;
            r.status[i] = st;
            r.mask[i] = 0u;
        }
        if (r.f_user && lane < M) r.f_user[off + lane] = floc;
        return;
    }
    // winner: recompute D20 and D22 lane = user (same arithmetic as the sweep)
    setup_nt(md, bN, M, x, s, lane);
    const int Bo = M - bP;
    const double lo_ = s.L[bP];
    const double fe = grid_fe(fe_max, rho, bJ);
    const double inv = 1.0 / fe;
    const double te = md.phi[bN * B1 + Bo] * inv;
    const bool member = (lane < M) && (s.rank[lane] >= bP);
    double f = floc, arr = t_free;
    if (member) {
        const double zv = s.zv[lane];
        if (zv == 0.0) f = x.f0;
        else f = clampf(zv / ((lo_ - s.OR[lane]) - te), x.f0, x.f1);
        arr = zv / f + s.OR[lane];
        if (arr < t_free) arr = t_free;
    }
#pragma unroll
    for (int d = 16; d >= 1; d >>= 1) {
        double o = __shfl_xor_sync(0xffffffffu, arr, d);
        arr = (o > arr) ? o : arr;
    }
    const unsigned mask = __ballot_sync(0xffffffffu, member);
    if (lane == 0) {
        r.E[i] = bE;
        r.E_lc[i] = E_lc;
        r.t_free_next[i] = arr + te;  // D22
        r.f_e[i] = fe;
        r.n_tilde[i] = bN;
        r.j[i] = (int)bJ;
        r.status[i] = st;
        r.mask[i] = mask;
    }
    if (r.f_user && lane < M) r.f_user[off + lane] = f;
}

__global__ void __launch_bounds__(kSolveWarps * 32) k_solve(const DevModel *models, DevBatch b, DevResult r, int mode) {
    __shared__ SolveSmem smem[kSolveWarps];
    const int lane = threadIdx.x & 31;
    const int w = threadIdx.x >> 5;
    const long long gw = (long long)blockIdx.x * kSolveWarps + w;
    const long long nw = (long long)gridDim.x * kSolveWarps;
    for (long long i = gw; i < b.n_inst; i += nw) solve_instance(i, models, b, r, mode, smem[w], lane);
}

void launch_solve(const DevModel *models, const DevBatch &b, const DevResult &r, int mode, cudaStream_t s,
                  int num_sms) {
    if (b.n_inst <= 0) return;
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_solve, kSolveWarps * 32, 0);
    if (per_sm < 1) per_sm = 1;
    long long want = (b.n_inst + kSolveWarps - 1) / kSolveWarps;
    long long grid = (long long)num_sms * per_sm;
    if (want < grid) grid = want;
    k_solve<<<(unsigned)grid, kSolveWarps * 32, 0, s>>>(models, b, r, mode);
}

}  // namespace jdob
