// K2: exhaustive search over partition-point vectors x edge-grid points (rows a9-a10).
//
// Candidate idx = vec * k + j.  General space: vec = sum_m n_m (N+1)^(M-1-m) (user 0
// most significant), n_m = N local.  Identical space ((P1)): vec = n~ 2^M + mask.
// Objective and constraints: DESIGN.md reading R14 (same-sub-task greedy batching,
// Fig. 1 caption P:75; ALAP batch starts; exact D6'/D7'/D13 feasibility, R10).
//
// Kernels: bf_setup (one warp: validation, k, LC terms, per-(n, user) hoists, 1/f_e
// table) -> bf_main (persistent; lane = vector, inner loop over j; a vector's scan
// stops at its first infeasible j, which is exact because D6' and D7' are monotone
// in j -- DESIGN.md §Brute-force monotone stop) -> bf_final (fixed-order fold of the
// per-block (E, idx) partials; lexicographic min = lowest index on ties).
#include "jdob_dev.cuh"
#include "kernels.h"

namespace jdob {

constexpr int kInvTab = 256;   // 1/f_e(j) cached in shared memory for j < kInvTab (C4: k = 64, C5: <= 191)
constexpr int kBfThreads = kBfWarps * 32;

#ifndef JDOB_BF_PRUNE
#define JDOB_BF_PRUNE 1
#endif

// setup output, in the workspace
struct BfHeader {
    int status, M, N, B1;
    long long k;
    unsigned long long size;   // index-space size (0 when too big)
    double t_free, fe_max, rho;
    unsigned long long best_bits;  // incumbent energy (bits of a double >= 0), shared by every block
};

// Per-(n, user) tables are stored user-major, element m (N + 1) + n: the brute force gathers them with
// a lane-dependent n for a fixed user, so consecutive n must fall in distinct shared-memory banks.
// NP = the row length: N + 1, or 16 when the kernel is specialised for N <= 15 (PAD: every shared-memory
// offset is then a compile-time constant of the M = 8 kernel, so no registers hold table pointers).
__device__ __forceinline__ int tix(int n, int m, int NP) { return m * NP + n; }

// Base-(N+1) digits of a lane's block index (users 0 .. M-2).  (Packing them as 6-bit fields of one
// 64-bit word frees registers but costs more instructions than the spills it removes: measured.)
template <int MAXM>
struct Digits {
    int a[MAXM];
    __device__ __forceinline__ int get(int m) const { return a[m]; }
    __device__ __forceinline__ void set(int m, int v) { a[m] = v; }
};

__global__ void k_bf_setup(const DevModel *models, DevBatch b, int space, int NP, BfHeader *hdr, double *tab /*[5][M][NP]*/,
                           double *user /*[4][32]: eloc fmin fmax T*/, double *invtab) {
    const int lane = threadIdx.x & 31;
    long long off, k;
    int M;
    const DevModel *mdp;
    InstRegs x;
    int st = warp_validate(models, b, 0, lane, x, M, k, mdp, off);
    if (st == kStDefer) {  // more than 32 users: outside the brute-force index encoding
        st = JDOB_ST_TOOBIG;
        M = 0;
    }
    if (lane == 0) {
        hdr->status = st;
        hdr->M = M;
        hdr->N = mdp ? mdp->N : 0;
        hdr->B1 = mdp ? mdp->B1 : 0;
        hdr->k = k;
        hdr->size = 0ull;
        hdr->t_free = b.t_free[0];
        hdr->fe_max = b.fe_max[0];
        hdr->rho = b.rho[0];
        hdr->best_bits = (unsigned long long)__double_as_longlong(dinf());
    }
    if (st != JDOB_ST_OK && st != JDOB_ST_REQUIRE) return;
    const DevModel &md = *mdp;
    const int N = md.N;
    // index-space size (< 2^62)
    if (lane == 0) {
        const unsigned long long lim = 1ull << 62;
        unsigned long long s = (unsigned long long)k;
        bool big = false;
        if (space == 0) {
            for (int m = 0; m < M && !big; m++) {
                if (s > lim / (unsigned long long)(N + 1)) big = true;
                else s *= (unsigned long long)(N + 1);
            }
        } else {
            unsigned long long f = (unsigned long long)(N + 1) << M;
            if (s > lim / f) big = true;
            else s *= f;
        }
        hdr->size = big ? 0ull : s;
        if (big) hdr->status = JDOB_ST_TOOBIG;
    }
    const double vN = md.v[N], uN = md.u[N];
    // all 32 entries are written (zeros beyond M) so the main kernel's tile copy reads initialised memory
    user[0 * 32 + lane] = 0.0;
    user[1 * 32 + lane] = 0.0;
    user[2 * 32 + lane] = 0.0;
    user[3 * 32 + lane] = 0.0;
    if (lane < M) {
        const double floc = clampf((x.z * vN) / x.T, x.f0, x.f1);
        user[0 * 32 + lane] = ((x.k * uN) * floc) * floc;
        user[1 * 32 + lane] = x.f0;
        user[2 * 32 + lane] = x.f1;
        user[3 * 32 + lane] = x.T;
        const int NM = NP * M;
        for (int n = 0; n <= N; n++) {
            const double OR = md.O[n] / x.R;
            const int t = tix(n, lane, NP);
            tab[0 * NM + t] = OR;                  // O_n / R_m
            tab[1 * NM + t] = x.z * md.v[n];       // zeta_m v_n
            tab[2 * NM + t] = x.k * md.u[n];       // kappa_m u_n
            tab[3 * NM + t] = OR * x.p;            // (O_n / R_m) p_m
            // energy lower bound of user m at partition point n: the f_min offloader
            // term for n < N, e_loc for n = N -- the same expressions as the kernel's bound
            tab[4 * NM + t] = (n < N) ? (((x.k * md.u[n]) * x.f0) * x.f0) + OR * x.p : user[0 * 32 + lane];
        }
    }
    const long long kt = k < kInvTab ? k : kInvTab;
    for (long long j = lane; j < kt; j += 32) invtab[j] = 1.0 / grid_fe(b.fe_max[0], b.rho[0], j);
}

// EXACT: M == MAXM, so every per-user guard folds at compile time (the C4 case, M = 8).
// WORK: count the work the pruned scan executes (diagnostic instantiation, launched only when the
// caller asks for the counters; the product instantiation carries no counter code):
//   [0] vectors visited  [1] past the user-term bound  [2] past the n_min-only bound
//   [3] past the exact vector bound (j loop entered)    [4] candidates evaluated (j iterations,
//   including the one that ends a scan)  [5] Gamma divisions executed  [6] candidates skipped by
//   the edge-only j skip  [7] vectors whose D6' fails at the first grid point  [8] offloaders
//   summed over the evaluated candidates
// GEN: the general space (blocks of N + 1 vectors per lane) or the identical space (one vector per
// lane), a compile-time choice so that each kernel carries only its own space's code.
template <int MAXM, bool EXACT, bool WORK, bool GEN, bool PAD>
#ifndef JDOB_BF_MINB
#define JDOB_BF_MINB 3
#endif
__global__ void __launch_bounds__(kBfWarps * 32, JDOB_BF_MINB) k_bf_main(const DevModel *models, int model_id, int space,
                                                           unsigned long long idx_begin, unsigned long long idx_end,
                                                           BfHeader *hdr, const double *tab,
                                                           const double *user, const double *invtab,
                                                           double *part_E, long long *part_idx,
                                                           unsigned long long *work) {
    extern __shared__ double sm[];
    unsigned long long wk[9] = {0ull, 0ull, 0ull, 0ull, 0ull, 0ull, 0ull, 0ull, 0ull};
    const int st = hdr->status;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    __shared__ double wE[kBfWarps];
    __shared__ long long wI[kBfWarps];
    double bestE = dinf();
    long long bestI = -1;
    if (st == JDOB_ST_OK || st == JDOB_ST_REQUIRE) {
        const int M = EXACT ? MAXM : hdr->M, N = hdr->N, B1 = hdr->B1;
        const long long k = hdr->k;
        const unsigned long long size = hdr->size;
        const double t_free = hdr->t_free, fe_max = hdr->fe_max, rho = hdr->rho;
        const DevModel &md = models[model_id];
        const int NP = PAD ? 16 : N + 1, NR = PAD ? 16 : N + 1;  // table row length, d/c table rows
        const int NM = NP * M;
        double *sOR = sm, *sZV = sm + NM, *sKU = sm + 2 * NM, *sUP = sm + 3 * NM;
        double *sLB = sm + 4 * NM;  // [M][N+1] per-user bound terms (tix)
        double *sEl = sm + 5 * NM, *sFmin = sEl + 32, *sFmax = sEl + 64, *sT = sEl + 96;
        double *sInv = sEl + 128;
        double *sSuf = sInv + kInvTab;  // [17][kBfThreads] per-lane suffix sums (N <= 15 path)
        double *sSlb = sSuf + 17 * kBfThreads, *sPlb = sSlb + 64;  // [nmin] lower bounds of S_{nmin+1}, Psi
        double *sG = sPlb + 64;  // [M][N+1] lower bound of user m's arrival O/R + zv/f* when offloading at n
        // d_n(b) A_n and c_n(b) A_n for b = 0..M (row stride M + 1): the batch sums gather them with a
        // lane-dependent b, consecutive b in distinct banks
        double *sDA = sG + NP * M, *sCA = sDA + NR * (M + 1);
        const long long kt = k < kInvTab ? k : kInvTab;
        for (int x = threadIdx.x; x < 5 * NM; x += blockDim.x) sm[x] = tab[x];
        for (int x = threadIdx.x; x < 128; x += blockDim.x) sEl[x] = user[x];
        for (long long x = threadIdx.x; x < kt; x += blockDim.x) sInv[x] = invtab[x];
        for (int x = threadIdx.x; x < (N + 1) * (M + 1); x += blockDim.x) {
            const int n = x / (M + 1), bb = x % (M + 1);
            sDA[x] = md.dA[n * B1 + bb];
            sCA[x] = md.cA[n * B1 + bb];
        }
        if (threadIdx.x == 0) {
            // For a vector whose first offloaded sub-task is nmin + 1, b_n >= 1 exactly for n > nmin and
            // b_n = 0 below, so S_{nmin+1} = RN-sum_{n=N..nmin+1} d_n(b_n) A_n >= the same RN-sum of
            // d_n(1) A_n (d non-decreasing in b, R19; RN monotone) and Psi >= the RN-sum of
            // min_{1<=b<=M} c_n(b) A_n, in the literal loop's order (descending n).
            double S = 0.0, P = 0.0;
            sSlb[N] = 0.0;
            sPlb[N] = 0.0;
            for (int n = N; n >= 1; n--) {
                double cm = md.cA[n * B1 + 1];
                for (int bb = 2; bb <= M; bb++) cm = (md.cA[n * B1 + bb] < cm) ? md.cA[n * B1 + bb] : cm;
                S = S + md.dA[n * B1 + 1];
                P = P + cm;
                sSlb[n - 1] = S;
                sPlb[n - 1] = P;
            }
        }
        __syncthreads();
#if JDOB_BF_PRUNE
        // Arrival lower bounds for the D7' f_e bound.  A feasible candidate has budget > 0 (>= 0 when
        // zv = 0) and RN(zv / budget) <= f_max, which with budget = RN(RN(l_o - O/R) - RN(S RN(1/f_e)))
        // gives S / f_e <= ((l_o - O/R)(1 + u) - (zv / f_max)(1 - 2u)) / (1 - u)^2 (u = 2^-53).  With
        // G = RN(O/R + RN(zv RD(1/f_max))) (1 - 2^-46) <= (O/R + zv/f_max)(1 - 2^-47) and the margins
        // of X below, S / X <= f_e for every feasible candidate.
        for (int y = threadIdx.x; y < N * M; y += blockDim.x) {
            const int m = y % M, x = tix(y / M, m, NP);
#ifndef JDOB_BF_NO_D7_FE
            sG[x] = (sOR[x] + sZV[x] * recip_rd(sFmax[m])) * (1.0 - 0x1p-46);
#else
            sG[x] = 0.0;
#endif
        }
        __syncthreads();
#endif
#if JDOB_BF_PRUNE && !defined(JDOB_BF_NO_DVFS_LB)
        // Offloader terms of the user bound with the deadline-driven device frequency (exact for the
        // brute force, whose infeasible candidates are skipped): an evaluated candidate with user m
        // offloading at n has budget = RN(RN(l_o - O/R) - RN(S_{n+1} RN(1/f_e))) <= X =
        // RN(RN(T_m - O/R) - RN(Slb[n] RN(1/f_e,max))) (l_o <= T_m, S_{n+1} >= Slb[n], f_e <=
        // f_e,max), and either f* = f_min with zv / X < f_min, or f* = RN(zv / budget) >=
        // RN(zv / X) with 0 < budget <= X; X <= 0 or RN(zv / X) > f_max leave no feasible candidate.
        {
            const double inv_max = sInv[0];  // RN(1 / f_e(0)) = RN(1 / f_e,max)
            for (int y = threadIdx.x; y < N * M; y += blockDim.x) {
                const int n = y / M, m = y % M, x = tix(n, m, NP);
                const double zv = sZV[x];
                if (zv == 0.0) continue;  // f* = f_min (R9): the f_min term stands
                const double X = (sT[m] - sOR[x]) - sSlb[n] * inv_max;
                double t;
                if (!(X > 0.0)) {
                    t = dinf();
                } else {
                    const double g = zv / X, fm = sFmin[m];
                    if (g > sFmax[m]) {
                        t = dinf();
                    } else {
                        const double f = (g > fm) ? g : fm;
                        t = ((sKU[x] * f) * f) + sUP[x];
                    }
                }
                sLB[x] = t;
            }
        }
        __syncthreads();
#endif
        if (idx_end > size) idx_end = size;
        if (idx_begin < idx_end) {
            const unsigned long long uk = (unsigned long long)k;
            const unsigned long long vb = idx_begin / uk, ve = (idx_end + uk - 1) / uk;
            // General space: a lane takes a block of radix consecutive vectors that differ only in the
            // last user's digit (the least significant one), so the other digits, their bound terms and
            // their n_min / l_o are formed once per block; blocks advance by 32 nw per step through a
            // mixed-radix add of the stride's digits (64-bit division only here).  Identical space:
            // one vector per lane and step.  Either way a lane visits its vectors in increasing order.
            const int radix = N + 1;
            constexpr bool blk = GEN;
            const int L = blk ? radix : 1;
            const unsigned long long ubeg = blk ? vb / (unsigned long long)radix : vb;
            const unsigned long long uend = blk ? (ve + radix - 1) / (unsigned long long)radix : ve;
            const unsigned long long nchunks = (uend - ubeg + 31) / 32;
            const unsigned long long gw = (unsigned long long)blockIdx.x * kBfWarps + w;
            const unsigned long long nw = (unsigned long long)gridDim.x * kBfWarps;
            const double *dA = sDA, *cA = sCA;
            const int B1s = M + 1;  // row stride of the staged tables
            Digits<MAXM> dig, sdig;  // digits of the block index and of the stride: users 0 .. M-2
            {
                unsigned long long t = ubeg + gw * 32 + lane, u = 32ull * nw;
#pragma unroll
                for (int m = MAXM - 1; m >= 0; m--) {
                    dig.set(m, 0);
                    sdig.set(m, 0);
                    if (m < M - 1 && blk) {
                        dig.set(m, (int)(t % (unsigned long long)radix));
                        t /= (unsigned long long)radix;
                        sdig.set(m, (int)(u % (unsigned long long)radix));
                        u /= (unsigned long long)radix;
                    }
                }
            }
            auto advance = [&]() {  // dig += sdig (mod radix^(M-1))
                if (!blk) return;
                int carry = 0;
#pragma unroll
                for (int m = MAXM - 1; m >= 0; m--) {
                    if (m < M - 1) {
                        const int d = dig.get(m) + sdig.get(m) + carry;
                        carry = d >= radix ? 1 : 0;
                        dig.set(m, carry ? d - radix : d);
                    }
                }
            };
            for (unsigned long long c = gw; c < nchunks; c += nw, advance()) {
                const unsigned long long unit = ubeg + c * 32 + lane;
                if (unit >= uend) continue;
                // users 0 .. M-2 of the block (general space): bound terms in user order, n_min, l_o
                double lbu_hi = 0.0, lo_hi = dinf(), gmax_hi = t_free;
                int nmin_hi = N;
                unsigned long long hist_hi = 0ull;  // digit histogram of users 0 .. M-2 (4-bit fields)
                if (blk) {
#pragma unroll
                    for (int m = 0; m < MAXM; m++)
                        if (m < M - 1) {
#if JDOB_BF_PRUNE
                            lbu_hi = lbu_hi + sLB[tix(dig.get(m), m, NP)];
#endif
                            const int dm = dig.get(m);
                            if (M <= 15 && N <= 15) hist_hi += 1ull << (4 * dm);
                            if (dm < N) {
                                if (dm < nmin_hi) nmin_hi = dm;
                                lo_hi = (sT[m] < lo_hi) ? sT[m] : lo_hi;
                            }
                        }
#if 1  // D7' arrival maximum hoisted per block (-3 % on C4)
                    // the D7' arrival maximum over users 0 .. M-2 offloading at nmin_hi (max is exact in any
                    // order): per vector only the last user is added
                    if (nmin_hi < N) {
#pragma unroll
                        for (int m = 0; m < MAXM; m++)
                            if (m < M - 1 && dig.get(m) == nmin_hi) {
                                const double g = sG[tix(nmin_hi, m, NP)];
                                gmax_hi = (g > gmax_hi) ? g : gmax_hi;
                            }
                    }
#endif
                }
#if JDOB_BF_PRUNE
                // the incumbent, read once per block of vectors (it only decides how much is skipped)
                const double inc = __longlong_as_double(*(volatile long long *)&hdr->best_bits);
#endif
                for (int t = 0; t < L; t++) {
                const unsigned long long vec = blk ? unit * (unsigned long long)radix + t : unit;
                if (vec < vb || vec >= ve) continue;
                if constexpr (WORK) wk[0]++;
                // the partition vector
                int nv[MAXM];
                if (blk) {
#pragma unroll
                    for (int m = 0; m < MAXM; m++) nv[m] = (m == M - 1) ? t : dig.get(m);
                } else {
                    const unsigned long long mask = vec & ((1ull << M) - 1ull);
                    const int nt = (int)(vec >> M);
#pragma unroll
                    for (int m = 0; m < MAXM; m++) nv[m] = (nt < N && ((mask >> m) & 1ull)) ? nt : N;
                }
#if JDOB_BF_PRUNE
                // user terms of the vector bound first (table lookups, in user order): most vectors
                // stop here
                double lbu = 0.0;
                if (blk) {
                    lbu = lbu_hi + sLB[tix(t, M - 1, NP)];
                } else {
#pragma unroll
                    for (int m = 0; m < MAXM; m++)
                        if (m < M) lbu = lbu + sLB[tix(nv[m], m, NP)];
                }
                if (lbu >= bestE || lbu > inc) continue;  // the edge term only adds (>= 0)
                if constexpr (WORK) wk[1]++;
#endif
                int nmin = N;
                double l_o = dinf();
                if (blk) {
                    nmin = nmin_hi;
                    l_o = lo_hi;
                    if (t < N) {
                        if (t < nmin) nmin = t;
                        l_o = (sT[M - 1] < l_o) ? sT[M - 1] : l_o;
                    }
                } else {
#pragma unroll
                    for (int m = 0; m < MAXM; m++) {
                        if (m < M && nv[m] < N) {
                            if (nv[m] < nmin) nmin = nv[m];
                            const double T = sT[m];
                            if (T < l_o) l_o = T;
                        }
                    }
                }
                const unsigned long long jlo = (vec == vb) ? idx_begin - vb * uk : 0ull;
                const unsigned long long jhi = (vec == ve - 1) ? idx_end - (ve - 1) * uk : uk;
                double Xd7 = 0.0;  // the D6'/D7' denominator of this vector (set when it has offloaders)
#if JDOB_BF_PRUNE
                // The vector bound below with S_{nmin+1} and Psi replaced by their lower bounds from
                // nmin alone (sSlb, sPlb): skips most vectors before the batch-size and suffix sums
                {
                    const double Slo = sSlb[nmin], Plo = sPlb[nmin];
                    double fel = grid_fe(fe_max, rho, (long long)(jhi - 1));
                    if (nmin < N) {
                        // D6' (t_free) and D7' of the users offloading at nmin (their arrival): f_e >=
                        // S_{nmin+1} / (l_o - max(t_free, arrival)) up to rounding, covered by the margins
                        double gmax = t_free;
#if 1  // D7' arrival maximum hoisted per block (-3 % on C4)
                        if (blk) {
                            gmax = (t < nmin_hi) ? t_free : gmax_hi;  // t < nmin_hi: only the last user at nmin = t
                            if (t == nmin) {
                                const double g = sG[tix(t, M - 1, NP)];
                                gmax = (g > gmax) ? g : gmax;
                            }
                        } else
#endif
                        {
#pragma unroll
                            for (int m = 0; m < MAXM; m++)
                                if (m < M && nv[m] == nmin)
                                    gmax = (sG[tix(nmin, m, NP)] > gmax) ? sG[tix(nmin, m, NP)] : gmax;
                        }
                        Xd7 = __dmul_ru(__dadd_ru(__dmul_ru(l_o, 1.0 + 0x1p-48), -gmax), 1.0 + 0x1p-48);
                        const double fd = div_lb(Slo, Xd7);  // <= S_{nmin+1} / X
                        fel = (fd > fel) ? fd : fel;
                    }
                    const double LB = lbu + (Plo * fel) * fel;
                    if (LB >= bestE || LB > inc) continue;
                }
                if constexpr (WORK) wk[2]++;
#endif
                // batch sizes, suffix sums S_n and Psi (descending n), per-user S_{n_m + 1}
                double Sm[MAXM];
#pragma unroll
                for (int m = 0; m < MAXM; m++) Sm[m] = 0.0;
                double S = 0.0, Psi = 0.0, Smin = 0.0;
                const bool HIST = (M <= 15 && N <= 15);
                unsigned long long hist = 0ull;
                if (HIST) {
                    // digit histogram in 4-bit fields: b_n = M - #{m : n_m >= n}, accumulated while n
                    // descends.  Below n_min + 1 every b_n is 0 and the literal loop adds +0.0, which
                    // leaves S and Psi unchanged, so the sums stop there: S = Psi's partner S_{nmin+1}.
                    // The per-user S_{n_m+1} are formed only for vectors that pass the bound below.
                    if (blk) {
                        hist = hist_hi + (1ull << (4 * t));  // the block's histogram plus the last user
                    } else {
#pragma unroll
                        for (int m = 0; m < MAXM; m++)
                            if (m < M) hist += 1ull << (4 * nv[m]);
                    }
                    int ge = 0;
                    for (int n = N; n > nmin; n--) {
                        ge += (int)((hist >> (4 * n)) & 0xfull);
                        const int bn = M - ge;
                        S = S + ((bn > 0) ? dA[n * B1s + bn] : 0.0);
                        Psi = Psi + ((bn > 0) ? cA[n * B1s + bn] : 0.0);
                    }
                    Smin = S;
                } else {
                    for (int n = N; n >= 1; n--) {
                        int bn = 0;
#pragma unroll
                        for (int m = 0; m < MAXM; m++) bn += (m < M && nv[m] < n) ? 1 : 0;
                        if (bn > 0) {
                            S = S + dA[n * B1s + bn];
                            Psi = Psi + cA[n * B1s + bn];
                        } else {
                            S = S + 0.0;
                            Psi = Psi + 0.0;
                        }
#pragma unroll
                        for (int m = 0; m < MAXM; m++)
                            if (m < M && nv[m] + 1 == n) Sm[m] = S;
                        if (nmin + 1 == n) Smin = S;
                    }
                }
                const bool any = nmin < N;
#if JDOB_BF_PRUNE
                // Vector bound (exact, DESIGN.md §4 "brute-force bound").  Every candidate the literal
                // scan evaluates passes D6': RN(t_free + RN(Smin RN(1/f_e))) <= l_o, which implies
                // f_e >= Smin / ((l_o (1 + u) - t_free)(1 + u)(1 + 2u)) (u = 2^-53) >= fl, computed
                // below with directed rounding; f_e >= f_e(jhi - 1) as well.  Each offloader term is
                // >= its f_min value, a local term is e_loc, and RN is monotone, so
                //   E(j) >= RN(RN-sum_m(term lower bounds) + (Psi fl) fl) = LB.
                // The vector is skipped when LB >= this lane's best (its candidates have larger
                // indices, so an equal E cannot win) or LB > the incumbent shared by all blocks.
                {
                    double fel = grid_fe(fe_max, rho, (long long)(jhi - 1));
                    if (any) {
                        const double fe0 = grid_fe(fe_max, rho, (long long)jlo);
                        const double inv0 = (jlo < (unsigned long long)kt) ? sInv[jlo] : 1.0 / fe0;
                        if (!(t_free + Smin * inv0 <= l_o)) {  // D6' fails at once: no candidate
                            if constexpr (WORK) wk[7]++;
                            continue;
                        }
                        const double fd = div_lb(Smin, Xd7);  // <= Smin / X (X of the n_min-only bound)
                        fel = (fd > fel) ? fd : fel;
                    }
                    const double LB = lbu + (Psi * fel) * fel;
                    if (LB >= bestE || LB > inc) continue;
                }
                if constexpr (WORK) wk[3]++;
                const double best_before = bestE;
#endif
                if (HIST) {  // the per-user S_{n_m+1} of a vector that reaches the grid loop (same sums again)
                    double *Sa = sSuf + threadIdx.x;
                    double S2 = 0.0;
                    int ge = 0;
                    Sa[(N + 1) * kBfThreads] = 0.0;
                    for (int n = N; n > nmin; n--) {
                        ge += (int)((hist >> (4 * n)) & 0xfull);
                        const int bn = M - ge;
                        S2 = S2 + ((bn > 0) ? dA[n * B1s + bn] : 0.0);
                        Sa[n * kBfThreads] = S2;
                    }
#pragma unroll
                    for (int m = 0; m < MAXM; m++)
                        if (m < M && nv[m] < N) Sm[m] = Sa[(nv[m] + 1) * kBfThreads];
                }
                // per-vector hoists: REG (M <= 8) keeps l_o - O/R, zeta v, kappa u, (O/R) p per user in
                // registers, so the candidate loop reads no shared memory for offloaders
                constexpr bool REG = MAXM <= 8;
                double lo[REG ? MAXM : 1], zvr[REG ? MAXM : 1], kur[REG ? MAXM : 1], upr[REG ? MAXM : 1];
                unsigned offm = 0u;
#pragma unroll
                for (int m = 0; m < MAXM; m++) {
                    if (m < M && nv[m] < N) {
                        offm |= 1u << m;
                        if constexpr (REG) {
                            const int x = tix(nv[m], m, NP);
                            lo[m] = l_o - sOR[x];
                            zvr[m] = sZV[x];
                            kur[m] = sKU[x];
                            upr[m] = sUP[x];
                        }
                    }
                }
                unsigned long long j0 = jlo;
#if JDOB_BF_PRUNE && !defined(JDOB_BF_NO_JSKIP)
                // Edge-only skip of the high-f_e prefix: E(j) >= RN(lbu + RN(RN(Psi f_e(j)) f_e(j))),
                // non-increasing in j, so the j with that bound >= the lane's best (larger indices lose
                // ties) or > the incumbent form a prefix of [jlo, jhi); binary search for its end.
                {
                    const double thr = (bestE < inc) ? bestE : inc;  // skip iff b >= bestE or b > inc
                    auto skip = [&](unsigned long long j) {
                        const double fe = grid_fe(fe_max, rho, (long long)j);
                        const double b = lbu + (Psi * fe) * fe;
                        return b >= bestE || b > inc;
                    };
                    if (thr < dinf() && skip(jlo)) {
                        unsigned long long lo = jlo + 1, hi = jhi;  // first non-skipped j in [lo, hi]
                        while (lo < hi) {
                            const unsigned long long mid = (lo + hi) >> 1;
                            if (skip(mid)) lo = mid + 1;
                            else hi = mid;
                        }
                        j0 = lo;
                    }
                }
                if constexpr (WORK) wk[6] += j0 - jlo;
#endif
                if constexpr (REG) {
                    // M <= 8: (A) budgets and the exact low-clamp test for every offloader, no
                    // branches; (B) the rare literal divisions / feasibility checks; (C) the energies
                    // in user order.  Keeping the branch out of the straight-line code lets the
                    // users' dependency chains overlap.
                    for (unsigned long long j = j0; j < jhi; j++) {
                        const double fe = grid_fe(fe_max, rho, (long long)j);
                        const double inv = (j < (unsigned long long)kt) ? sInv[j] : 1.0 / fe;
                        if constexpr (WORK) {
                            wk[4]++;
                            wk[8] += __popc(offm);
                        }
                        if (any && !(t_free + Smin * inv <= l_o)) break;  // D6' (monotone in j)
                        double bud[MAXM], fv[MAXM];
                        unsigned need = 0u;
#pragma unroll
                        for (int m = 0; m < MAXM; m++) {
                            bud[m] = lo[m] - Sm[m] * inv;  // (l_o - O/R) - S_{n_m+1}/f_e
                            fv[m] = sFmin[m];
                            // exact low clamp: fmin*budget > zv exactly => budget > 0 and
                            // RN(zv/budget) <= f_min <= f_max: feasible with f* = f_min (R9 when zv = 0)
                            if (((offm >> m) & 1u) && !(__fma_rn(fv[m], bud[m], -zvr[m]) > 0.0)) need |= 1u << m;
                        }
                        bool feas = true;
                        if (need) {
#pragma unroll
                            for (int m = 0; m < MAXM; m++) {
                                if ((need >> m) & 1u) {
                                    if (zvr[m] == 0.0) {
                                        if (!(bud[m] >= 0.0)) feas = false;
                                    } else if (!(bud[m] > 0.0)) {
                                        feas = false;
                                    } else {
                                        if constexpr (WORK) wk[5]++;
                                        const double G = zvr[m] / bud[m];
                                        if (G > sFmax[m]) feas = false;  // D7' with D13 (exact, R10)
                                        fv[m] = (G < fv[m]) ? fv[m] : G;
                                    }
                                }
                            }
                        }
                        if (!feas) break;  // D7' (monotone in j)
                        double E = 0.0;
#pragma unroll
                        for (int m = 0; m < MAXM; m++) {
                            if (m < M) {
                                const double em = ((kur[m] * fv[m]) * fv[m]) + upr[m];
                                E = E + (((offm >> m) & 1u) ? em : sEl[m]);
                            }
                        }
                        E = E + (Psi * fe) * fe;
                        if (E < bestE) {
                            bestE = E;
                            bestI = (long long)(vec * uk + j);
                        }
                    }
                } else {
                for (unsigned long long j = j0; j < jhi; j++) {
                        const double fe = grid_fe(fe_max, rho, (long long)j);
                        const double inv = (j < (unsigned long long)kt) ? sInv[j] : 1.0 / fe;
                        if constexpr (WORK) {
                            wk[4]++;
                            wk[8] += __popc(offm);
                        }
                        if (any && !(t_free + Smin * inv <= l_o)) break;  // D6' (monotone in j)
                        double E = 0.0;
                        bool feas = true;
    #pragma unroll
                        for (int m = 0; m < MAXM; m++) {
                            if (m >= M) break;
                            double e;
                            if ((offm >> m) & 1u) {
                                double lom, zv, ku, up;
                                if constexpr (REG) {
                                    lom = lo[m];
                                    zv = zvr[m];
                                    ku = kur[m];
                                    up = upr[m];
                                } else {
                                    const int x = tix(nv[m], m, NP);
                                    lom = l_o - sOR[x];
                                    zv = sZV[x];
                                    ku = sKU[x];
                                    up = sUP[x];
                                }
                                const double budget = lom - Sm[m] * inv;  // (l_o - O/R) - S_{n_m+1}/f_e
                                double f = sFmin[m];
                                // exact low clamp: fmin*budget > zv exactly => budget > 0 and
                                // RN(zv/budget) <= f_min <= f_max: feasible with f* = f_min (R9 when zv = 0)
                                if (!(__fma_rn(f, budget, -zv) > 0.0)) {
                                    if (zv == 0.0) {
                                        if (!(budget >= 0.0)) {
                                            feas = false;
                                            break;
                                        }
                                    } else {
                                        if (!(budget > 0.0)) {
                                            feas = false;
                                            break;
                                        }
                                        if constexpr (WORK) wk[5]++;
                                        const double G = zv / budget;
                                        if (G > sFmax[m]) {  // D7' with D13 (exact, R10)
                                            feas = false;
                                            break;
                                        }
                                        f = (G < f) ? f : G;
                                    }
                                }
                                e = ((ku * f) * f) + up;
                            } else {
                                e = sEl[m];
                            }
                            E = E + e;
                        }
                        if (!feas) break;  // D7' (monotone in j)
                        E = E + (Psi * fe) * fe;
                        if (E < bestE) {
                            bestE = E;
                            bestI = (long long)(vec * uk + j);
                        }
                }
                }
#if JDOB_BF_PRUNE
                if (bestE < best_before)  // publish the lane's new best as the shared incumbent
                    atomicMin(&hdr->best_bits, (unsigned long long)__double_as_longlong(bestE));
#endif
                }  // t: the vectors of the lane's block
            }
        }
    }
    if constexpr (WORK) {
#pragma unroll
        for (int q = 0; q < 9; q++) {
            unsigned long long v = wk[q];
            for (int d = 16; d >= 1; d >>= 1) v += __shfl_xor_sync(0xffffffffu, v, d);
            if (lane == 0 && v) atomicAdd(&work[q], v);
        }
    }
    // warp, then block argmin over (E, idx)
#pragma unroll
    for (int d = 16; d >= 1; d >>= 1) {
        double oE = __shfl_xor_sync(0xffffffffu, bestE, d);
        long long oI = __shfl_xor_sync(0xffffffffu, bestI, d);
        bool take = (oE < bestE) || (oE == bestE && oI >= 0 && (bestI < 0 || oI < bestI));
        if (take) {
            bestE = oE;
            bestI = oI;
        }
    }
    if (lane == 0) {
        wE[w] = bestE;
        wI[w] = bestI;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double E = wE[0];
        long long I = wI[0];
        for (int q = 1; q < kBfWarps; q++) {
            if (wE[q] < E || (wE[q] == E && wI[q] >= 0 && (I < 0 || wI[q] < I))) {
                E = wE[q];
                I = wI[q];
            }
        }
        part_E[blockIdx.x] = E;
        part_idx[blockIdx.x] = I;
    }
}

__global__ void k_bf_final(const BfHeader *hdr, const double *part_E, const long long *part_idx, int nblocks,
                           double *E_min, long long *idx_min, int *status) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    double E = dinf();
    long long I = -1;
    for (int q = 0; q < nblocks; q++) {
        if (part_E[q] < E || (part_E[q] == E && part_idx[q] >= 0 && (I < 0 || part_idx[q] < I))) {
            E = part_E[q];
            I = part_idx[q];
        }
    }
    *E_min = E;
    *idx_min = I;
    *status = hdr->status;
}

size_t bf_workspace_bytes() {
    return 256 + sizeof(double) * (5 * 64 * 32 + 4 * 32 + kInvTab) + (sizeof(double) + sizeof(long long)) * kBfBlocks +
           1024;
}

// one wave of the persistent grid: JDOB_BF_GRID blocks per SM (at most kBfBlocks in all)
#ifndef JDOB_BF_GRID
#define JDOB_BF_GRID 3
#endif
static int bf_grid() {
    static const int g = [] {
        int dev = 0, n = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        if (n <= 0) n = 148;
        long long want = (long long)n * JDOB_BF_GRID / grid_divisor();
        if (want < 1) want = 1;
        return (int)(want < kBfBlocks ? want : kBfBlocks);
    }();
    return g;
}

template <int MAXM, bool EXACT = false, bool PAD = false>
static void launch_main(const DevModel *models, int model_id, int space, unsigned long long ib, unsigned long long ie,
                        BfHeader *hdr, const double *tab, const double *user, const double *inv,
                        double *part_E, long long *part_idx, unsigned long long *work, size_t smem, cudaStream_t s) {
    if (work) cudaMemsetAsync(work, 0, 9 * sizeof(unsigned long long), s);
    auto go = [&](auto kern, unsigned long long *w) {  // (the PAD choice is the caller's template argument)
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        kern<<<bf_grid(), kBfWarps * 32, smem, s>>>(models, model_id, space, ib, ie, hdr, tab, user, inv, part_E,
                                                    part_idx, w);
    };
    if (space == 0) {
        if (work) go(k_bf_main<MAXM, EXACT, true, true, PAD>, work);
        else go(k_bf_main<MAXM, EXACT, false, true, PAD>, nullptr);
    } else {
        if (work) go(k_bf_main<MAXM, EXACT, true, false, PAD>, work);
        else go(k_bf_main<MAXM, EXACT, false, false, PAD>, nullptr);
    }
}

void launch_bruteforce_impl(const DevModel *models, const DevBatch &b, int model_id, int N, int M, int space,
                            unsigned long long idx_begin, unsigned long long idx_end, void *ws, double *E_min,
                            long long *idx_min, int *status, unsigned long long *work, cudaStream_t s) {
    char *p = (char *)ws;
    BfHeader *hdr = (BfHeader *)p;
    p += 256;
    double *tab = (double *)p;
    p += sizeof(double) * 5 * 64 * 32;
    double *user = (double *)p;
    p += sizeof(double) * 4 * 32;
    double *inv = (double *)p;
    p += sizeof(double) * kInvTab;
    double *part_E = (double *)p;
    p += sizeof(double) * kBfBlocks;
    long long *part_idx = (long long *)p;
    const int Mc = (M >= 1 && M <= kMaxM) ? M : 1;
#ifndef JDOB_BF_NO_PAD
    const bool pad = (Mc == 8 && N <= 15);  // M = 8, N <= 15: the constant-layout kernel (C4: N = 11)
#else
    const bool pad = false;
#endif
    const size_t NP = pad ? 16 : (size_t)N + 1;
    k_bf_setup<<<1, 32, 0, s>>>(models, b, space, (int)NP, hdr, tab, user, inv);
    const size_t smem = sizeof(double) * (5 * NP * Mc + 128 + kInvTab + 17 * kBfThreads + 128 + NP * Mc +
                                          2 * NP * (Mc + 1));
    if (pad)
        launch_main<8, true, true>(models, model_id, space, idx_begin, idx_end, hdr, tab, user, inv, part_E, part_idx,
                                   work, smem, s);
    else if (Mc == 8)
        launch_main<8, true>(models, model_id, space, idx_begin, idx_end, hdr, tab, user, inv, part_E, part_idx, work, smem,
                             s);
    else if (Mc <= 8)
        launch_main<8>(models, model_id, space, idx_begin, idx_end, hdr, tab, user, inv, part_E, part_idx, work, smem, s);
    else if (Mc <= 16)
        launch_main<16>(models, model_id, space, idx_begin, idx_end, hdr, tab, user, inv, part_E, part_idx, work, smem, s);
    else
        launch_main<32>(models, model_id, space, idx_begin, idx_end, hdr, tab, user, inv, part_E, part_idx, work, smem, s);
    k_bf_final<<<1, 32, 0, s>>>(hdr, part_E, part_idx, bf_grid(), E_min, idx_min, status);
}

}  // namespace jdob
