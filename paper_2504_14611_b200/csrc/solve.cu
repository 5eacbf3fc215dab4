// K1: J-DOB solve over a batch of independent instances (rows a2-a8).
//
// One warp per instance (persistent grid-stride loop).  Per partition point n~ the
// warp first works lane = user (gamma, hoists, all-pairs rank sort, suffix-min
// deadlines, thresholds), then lane = edge-grid point j for the Alg. 2 sweep.
//
// Sweep equivalence (DESIGN.md §Sweep equivalence): the thresholds are exactly
// non-increasing from i^, so Alg. 2's sequential pointer at grid point j equals
// p(j) = min{i >= i^ : !(f_e(j) < th_i)}, and user m (sorted position r_m) is in
// the offloading set iff r_m >= i^ and !(f_e(j) < th_{r_m}).  Each lane therefore
// finds B_o and l_o by a binary search over the thresholds, decides membership per
// user with one comparison against the user's own threshold, checks the D6 guard,
// evaluates D20-D21 in user-index order and keeps a lane-local strict minimum.  The
// first j with an empty set (Alg. 2's break) is found by a ballot inside the chunk
// loop.  A warp argmin over (E, n~, j) and the first all-local evaluation (R8) give
// the Alg. 1 answer; the winner's D20/D22 values are recomputed lane = user.
//
// Division is the expensive operation on sm_100a (MUFU.RCP64H-bound, ~4.6/clk/SM
// measured vs 64 DFMA/clk/SM), so the sweep avoids it where that is exact
// (DESIGN.md §4): the D20 low clamp RN(zv/budget) <= f_min is implied by
// fma(f_min, budget, -zv) > 0 (a correctly rounded fma is > 0 only if the exact
// value is, and the exact inequality implies the rounded one), otherwise the literal
// division runs; the D6 guard quotient phi(B_o)/(l_o - t_free) depends only on the
// set start p, so it is formed once per (n~, p) in setup, not per grid point.  1/f_e(j) is
// computed once per instance and cached in shared memory.  When every user of an
// instance has the same (R, zeta, f_max) -- the paper's Table I setting -- gamma
// is equal for all users at every n~, so the sort key reduces to (T, index) and
// the order and suffix-min deadlines are computed once per instance; if moreover
// f_min, kappa and p_u agree ("uniform users": all of Table I's experiments, where
// only deadlines differ), every member of a configuration has the same budget, f*
// and offloader energy, which are then formed once per (n~, j) instead of per user.
// Uniform-user instances are solved by their own kernels (UNI = true), compiled once for
// equal deadlines (TIGHT = false: every user identical; members are the users m >= p,
// summed from a prefix of the e_loc terms) and once for differing deadlines (TIGHT =
// true: with the batch-coupled bound below); each defers the other class, and the
// general kernel takes the rest.  Small per-class code keeps K1 fast (it is sensitive
// to its code size and register allocation); deferral flags let a kernel with nothing
// deferred to it return at once.  k_solve_multi answers J-DOB, no edge DVFS and binary
// J-DOB from one sweep (NEXT-2).
//
// Branch and bound over n~ (DESIGN.md §4 "n~ pruning"): a lower bound of every
// configuration's energy is formed per n~ (lane = n~); n~ are visited in ascending
// order and one whose bound is not below the best energy so far is skipped.  The
// differing-deadline kernel also bounds each candidate n~ per set start p (members at
// f_min, the edge energy at the lowest f_e that passes the guard and the membership
// threshold of p) and skips it when that is not below the best or above E_LC.  An
// exact tie of the best offloading energy with E_LC after pruning re-sweeps the
// instance literally (the all-local key of a skipped n~ could matter, R8).
#include "jdob_dev.cuh"
#include "kernels.h"

namespace jdob {

#ifndef JDOB_INV_CACHE
#define JDOB_INV_CACHE 192
#endif
constexpr int kInvCache = JDOB_INV_CACHE;  // 1/f_e(j) cached for j < kInvCache

// Order of the pruned n~ sweep (DESIGN.md §4 "n~ pruning"): 0 ascending n~ (the literal order),
// 1 ascending with the bound also capped at E_LC, 2 best first (smallest lower bound first).
#ifndef JDOB_PRUNE_ORDER
#define JDOB_PRUNE_ORDER 0
#endif

struct SolveSmem {
    // per-user values as 16-byte pairs (lane stride 16 B: 4-way store conflicts at most)
    double2 orzv[kMaxM];                 // O_n~/R_m, zeta_m v_n~
    double2 kuup[kMaxM];                 // kappa_m u_n~, (O_n~/R_m) p_m
    double2 et[kMaxM];                   // e_loc,m, th_{r_m} if r_m >= i^ else +inf
    double2 fmm[kMaxM];                  // f_m,min, f_m,max
    double R[kMaxM], z[kMaxM], f1[kMaxM], kap[kMaxM], pu[kMaxM];  // user parameters (lane = user)
    double T[kMaxM], gam[kMaxM];
    double th[kMaxM];
    double2 Lg[kMaxM];                   // per sorted position p: {l_o = L_p, guard threshold phi/(L_p - t_free)}
    double2 pp[kMaxM];                   // per sorted position p: {phi_n~(M - p), psi_n~(M - p)}
    int rank[kMaxM], order[kMaxM];
    double inv[kInvCache];
    double2 inv_key;                     // (f_e,max, rho) of the cached 1/f_e(j), j < inv_n
    int inv_n;
    GridKCache kc;                       // k of the last (f_e,min, f_e,max, rho)
    double rinv[kMaxM];                  // general kernel: RD(1 / R_m), lower-bound upload term; differing-
                                         // deadline kernel: RD sum of e_loc over sorted positions >= p (p < M)
    double lbem[64];                     // per n~: the lower bound's member term (uniform users)
    int defer;                           // this warp deferred an instance (uniform kernels)
    double pre[kMaxM + 1];               // equal-deadline kernel: P[p] = user-order sum of the first p e_loc;
                                         // differing-deadline kernel: RD sum of e_loc over sorted positions < p
    double lb[64];                       // per n~: lower bound of every configuration's energy
    // uniform users (UNI kernel, N <= kUniCache): the per-n~ values that depend only on the model and
    // the users' shared (R, zeta, f_max, kappa, f_min, p_u) -- O/R, zeta v, gamma and the lower-bound
    // member term -- formed once per warp for consecutive instances with the same key (Table I: all)
    long long ukey[8];
    double uOR[32], uZV[32], uG[32], uEM[32];
};
#ifndef JDOB_NO_UNI_CACHE
constexpr int kUniCache = 32;
#endif

// Ranks under the key (gamma desc, T asc, index asc) (R2), then order[] and the
// suffix-min deadlines L_i = min_{i' >= i} T_order[i'] (Eq. fth's min, R1).
__device__ __forceinline__ void sort_users(int M, double gam, double T, SolveSmem &s, int lane) {
    int r = 0;
    for (int t = 0; t < M; t++) {
        const double gt = __shfl_sync(0xffffffffu, gam, t);
        const double Tt = __shfl_sync(0xffffffffu, T, t);
        const bool before = (gt > gam) || (gt == gam && (Tt < T || (Tt == T && t < lane)));
        r += before ? 1 : 0;
    }
    if (lane < M) {
        s.rank[lane] = r;
        s.order[r] = lane;
    }
    __syncwarp();
    double L = lane < M ? s.T[s.order[lane]] : dinf();
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const double o = __shfl_down_sync(0xffffffffu, L, d);
        if (lane + d < 32 && o < L) L = o;
    }
    if (lane < M) s.Lg[lane].x = L;
    __syncwarp();
}

// Homogeneous users (equal gamma): ranks under the key (T asc, index asc) from the deadlines in
// shared memory (broadcast reads, no shuffles), then order[] and the suffix minima (= sorted T).
__device__ __noinline__ void sort_users_T(int M, double T, SolveSmem &s, int lane) {
    int r = 0;
    for (int t = 0; t < M; t++) {
        const double Tt = s.T[t];
        r += (Tt < T || (Tt == T && t < lane)) ? 1 : 0;
    }
    if (lane < M) {
        s.rank[lane] = r;
        s.order[r] = lane;
        s.Lg[r].x = T;  // ascending deadlines: the suffix minimum at position r is T itself
    }
    __syncwarp();
}

// Alg. 1 lines 4-6 for partition point nt.  Returns i^ (M if none).
// need_et = false: the caller does not read the per-user thresholds et.y (the equal-deadline kernel sums
// members from the prefix P[p]).
__device__ __forceinline__ int setup_nt(const DevModel &md, int nt, int M, bool homog, bool uni, double t_free,
                                        SolveSmem &s, int lane, bool uc = false, bool need_et = true) {
    const double v_nt = md.v[nt], u_nt = md.u[nt], O_nt = md.O[nt];
    double gam = 0.0;
    if (lane < M) {
        // uc: the same expressions, formed once per warp for this key (uniform users)
        const double OR = uc ? s.uOR[nt] : O_nt / s.R[lane];  // Eq. (3)
        const double zv = uc ? s.uZV[nt] : s.z[lane] * v_nt;
        gam = uc ? s.uG[nt] : OR + div_z(zv, s.f1[lane]);      // gamma
        if (!uni || lane == 0) {             // uniform users: one copy serves every member
            s.orzv[lane] = make_double2(OR, zv);
            s.kuup[lane] = make_double2(s.kap[lane] * u_nt, OR * s.pu[lane]);  // Eq. (4)
        }
        if (!homog) s.gam[lane] = gam;  // (homogeneous: every user's gamma is this lane's)
    }
    if (!homog) sort_users(M, gam, s.T[lane], s, lane);  // homogeneous: order fixed per instance
    double th = 0.0;
    if (lane < M) {
        const double gi = homog ? gam : s.gam[s.order[lane]];
        const double phi = md.phi[nt * md.B1 + (M - lane)], psi = md.psi[nt * md.B1 + (M - lane)];
        const double L = s.Lg[lane].x;
        th = phi / (L - gi);                          // Eq. (fth)
        s.th[lane] = th;
        s.Lg[lane].y = phi / (L - t_free);            // D6 guard threshold of the set starting at p = lane
        s.pp[lane] = make_double2(phi, psi);
    }
    const unsigned nn = __ballot_sync(0xffffffffu, lane < M && th >= 0.0);
    const int ihat = nn ? (__ffs(nn) - 1) : M;
    __syncwarp();
    if (need_et) {
        if (lane < M) {
            const int rm = s.rank[lane];
            s.et[lane].y = (rm >= ihat) ? s.th[rm] : dinf();
        }
        __syncwarp();
    }
    return ihat;
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
        if (r.work) r.work[4 * i] = r.work[4 * i + 1] = r.work[4 * i + 2] = r.work[4 * i + 3] = 0;
        if (r.viol) r.viol[i] = 0u;  // jdob_eval reports no bits for a malformed instance
    }
    if (r.f_user && M >= 1 && M <= kMaxM && lane < M) r.f_user[off + lane] = dnan();
    if (r.partition && M >= 1 && M <= kMaxM && lane < M) r.partition[off + lane] = N;
}

// The all-local plan re-verified with jdob_eval's formulas (row a11): Require (bit 4) and each
// local user's D8 at relative slack (bit 2); the eval call's own status does not enter the bits.
__device__ __forceinline__ unsigned verify_local(const InstRegs &x, double vN, double floc, int M, unsigned vflags,
                                                 double slack, int lane) {
    unsigned vb = (vflags & kVRequire) ? 16u : 0u;
    if (lane < M && d8_violated(x.z * vN, floc, x.T + slack * fabs(x.T))) vb |= 4u;
    return __reduce_or_sync(0xffffffffu, vb);
}

__device__ __forceinline__ void write_local(const DevResult &r, long long i, long long off, int M, int N,
                                            double E_lc, double t_free, double floc, int st, int lane,
                                            bool zero_counts) {
    if (lane == 0) {
        r.E[i] = E_lc;
        r.E_lc[i] = E_lc;
        r.t_free_next[i] = t_free;
        r.f_e[i] = 0.0;
        r.n_tilde[i] = N;
        r.j[i] = 0;
        r.status[i] = st;
        r.mask[i] = 0u;
        if (r.counts && zero_counts) {
            r.counts[3 * i] = 0;
            r.counts[3 * i + 1] = 0;
            r.counts[3 * i + 2] = 0;
        }
        if (r.work && zero_counts) r.work[4 * i] = r.work[4 * i + 1] = r.work[4 * i + 2] = r.work[4 * i + 3] = 0;
    }
    if (r.f_user && lane < M) r.f_user[off + lane] = floc;
    if (r.partition && lane < M) r.partition[off + lane] = N;
}

// COUNTS: per-instance work counters.  PRUNE: skip every n~ whose energy lower bound is not below
// the best energy found so far (exact, DESIGN.md §4 "n~ pruning").  <true, false> = literal Alg. 2
// counters (r.counts), <true, true> = executed-work counters of the pruned sweep (r.work),
// <false, true> = the product path.
// UNI: the instance class this kernel solves.  true = uniform users (Table I; the other instances
// are marked kStDefer), false = the rest (only instances marked kStDefer by the kernels before).
// Specialised kernels keep each one's code, and so its instruction-cache footprint, small.
// TIGHT (uniform kernels only): false = the kernel of equal deadlines (Table I's identical-deadline
// setting; instances whose deadlines differ are marked kStDefer), true = the kernel of differing deadlines,
// which adds the batch-coupled n~ bound (it prunes 43-66 % of the set-ups there, little with equal
// deadlines, and its code costs the other kernel 2-6 % when compiled in).
// MULTI (NEXT-2, k_solve_multi): one pass answers JDOB_MODE_FULL into r and, from the same sweep,
// JDOB_MODE_NO_EDGE_DVFS (the candidates at j = 0) and JDOB_MODE_BINARY (the candidates at n~ = 0) into
// rx[0] and rx[1]; every mode's (E, n~, j) tie rule and all-local key are kept as in its own pass.
template <bool COUNTS, bool PRUNE, bool UNI, bool VERIFY, bool TIGHT, bool MULTI = false>
__device__ __forceinline__ void solve_instance(long long i, long long off, long long M64, int mid,
                                               const DevModel *models, const DevBatch &b, const DevResult &r,
                                               int mode, SolveSmem &s, int lane, long long nx_off = 0,
                                               long long nx_end = 0, const DevResult *rx = nullptr) {
    __syncwarp();
    long long k;
    int M;
    const DevModel *mdp;
    InstRegs x;
    unsigned vflags = 0u;
    // (without edge DVFS the differing-deadline kernel takes every uniform instance: its batch-coupled
    // bound, exact at the one grid point f_e,max, skips the set-ups of the n~ that cannot beat LC)
    const bool noedge = mode == JDOB_MODE_NO_EDGE_DVFS;
    const int st = warp_validate_pre(models, b, i, lane, off, M64, mid, x, M, k, mdp, &s.kc, &vflags,
                                     UNI ? (TIGHT ? (noedge ? 0 : 2) : (noedge ? 3 : 1)) : 0);
#ifndef JDOB_L1PF
#define JDOB_L1PF 1
#endif
#if JDOB_L1PF
    // the next instance's users (nx_off, nx_end: the head the kernel loop loaded ahead) are pulled toward
    // the SM while this one is solved, so its validation loads hit the cache
    const long long nx_M = nx_end - nx_off;
    if (lane < nx_M && nx_M <= kMaxM) {
        const long long u = nx_off + lane;
        const double *pp[7] = {b.zeta + u, b.kappa + u, b.f_min + u, b.f_max + u, b.R + u, b.p_u + u, b.T + u};
#pragma unroll
        for (int q = 0; q < 7; q++) {
#if JDOB_L1PF == 2
            asm volatile("prefetch.global.L2 [%0];" ::"l"(pp[q]));
#else
            asm volatile("prefetch.global.L1 [%0];" ::"l"(pp[q]));
#endif
        }
    }
#endif
    if (st == kStDefer) {  // the other uniform kernel, or M > 32: k_solve_large (solve_large.cu)
        if (UNI && lane == 0) {
            r.status[i] = kStDefer;
            s.defer = 1;  // published once per warp when the kernel ends
        }
        return;
    }
    const double t_free = x.t_free, fe_max = x.fe_max, rho = x.rho;
    if (st == JDOB_ST_BADPARAM || st == JDOB_ST_BADMODEL) {
        write_bad(r, i, off, M, mdp ? mdp->N : 0, t_free, st, lane);
        if (MULTI) {
            write_bad(rx[0], i, off, M, mdp ? mdp->N : 0, t_free, st, lane);
            write_bad(rx[1], i, off, M, mdp ? mdp->N : 0, t_free, st, lane);
        }
        return;
    }
    // the uniform kernels leave non-uniform instances, whatever their status, to the general kernel
    const bool homog_ = !(vflags & kNotHomog);
    const bool uni_ = homog_ && !(vflags & kNotUni);
    if (UNI && !uni_) {
        if (lane == 0) {
            r.status[i] = kStDefer;
            s.defer = 1;  // published once per warp when the kernel ends
        }
        return;
    }
    const DevModel &md = *mdp;
    const int N = md.N;
    const double vN = md.v[N], uN = md.u[N];

    // LC (row a2): f_loc = clamp(zeta v_N / T), e_loc = ((kappa u_N) f) f
    double floc = 0.0, eloc = 0.0;
    if (lane < M) {
        // D20 local branch; f_min T - zeta v_N > 0 exactly => RN(zeta v_N / T) <= f_min => f_min
        const double zvN = x.z * vN;
        floc = (__fma_rn(x.f0, x.T, -zvN) > 0.0) ? x.f0 : clampf(zvN / x.T, x.f0, x.f1);
        eloc = ((x.k * uN) * floc) * floc;
        s.et[lane].x = eloc;
        s.fmm[lane] = make_double2(x.f0, x.f1);
        s.R[lane] = x.R;
        s.z[lane] = x.z;
        s.f1[lane] = x.f1;
        s.kap[lane] = x.k;
        s.pu[lane] = x.p;
    }
    s.T[lane] = x.T;  // +inf beyond M
    __syncwarp();
    double E_lc = 0.0;
    // equal-deadline kernel (uniform users, equal deadlines): every user's e_loc is the same bits
    const bool same_el = UNI && !TIGHT;
    const double el0 = __shfl_sync(0xffffffffu, eloc, 0);
    for (int t = 0; t < M; t++) {
        E_lc = E_lc + (same_el ? el0 : s.et[t].x);  // user-index order
#ifndef JDOB_NO_PREFIX
        if (UNI && !TIGHT && lane == 0) s.pre[t + 1] = E_lc;  // P[t + 1]: the sum of the first t + 1 terms
#endif
    }
    if (st != JDOB_ST_OK || mode == JDOB_MODE_LC) {
        if (MULTI) {
            write_local(rx[0], i, off, M, N, E_lc, t_free, floc, st, lane, true);
            write_local(rx[1], i, off, M, N, E_lc, t_free, floc, st, lane, true);
        }
        write_local(r, i, off, M, N, E_lc, t_free, floc, st, lane, true);
        if (VERIFY) {
            const unsigned vb = verify_local(x, vN, floc, M, vflags, r.slack, lane);
            if (lane == 0) r.viol[i] = vb;
        }
        return;
    }

    const int kk = (mode == JDOB_MODE_NO_EDGE_DVFS) ? 1 : (int)k;  // k <= kMaxK (validated)
    const int kc = kk < kInvCache ? kk : kInvCache;
    // 1/f_e(j) cache per warp: the hit test is read by every lane before any lane rewrites it
    const bool inv_hit = __all_sync(0xffffffffu, fe_max == s.inv_key.x && rho == s.inv_key.y && kc <= s.inv_n);
    if (!inv_hit) {  // warp-uniform
        __syncwarp();
        for (int j = lane; j < kc; j += 32) s.inv[j] = 1.0 / grid_fe(fe_max, rho, (long long)j);
        if (lane == 0) {
            s.inv_key = make_double2(fe_max, rho);
            s.inv_n = (int)kc;
        }
        __syncwarp();
    }
    // instance-level flags (warp-uniform)
    const double R0 = s.R[0], z0 = s.z[0], f10 = s.f1[0];  // user 0's values
    // (from the validation's single warp reduction)
    const double f00 = s.fmm[0].x, k0 = s.kap[0], p0 = s.pu[0];
    const bool homog = UNI ? true : homog_, uni = UNI ? true : uni_;
    // (the uniform kernels know the deadline class: equal in the first, differing in the second)
    if (homog && (UNI ? !TIGHT : !(vflags & kNotSameT))) {
        // equal gamma and equal deadlines (Table I identical-deadline setting): the key (T asc,
        // index asc) is the index order and every suffix minimum is T
        if (lane < M) {
            s.rank[lane] = lane;
            s.order[lane] = lane;
            s.Lg[lane].x = x.T;
        }
    } else if (homog) {
        sort_users_T(M, x.T, s, lane);  // equal gamma: key (T asc, index asc)
    }
    __syncwarp();

    const int B1 = md.B1;
    bool uc = false;  // per-warp cache of the uniform users' per-n~ values
#ifndef JDOB_NO_UNI_CACHE
    if (UNI && N <= kUniCache) {
        const long long key[7] = {(long long)mid, __double_as_longlong(R0), __double_as_longlong(z0),
                                  __double_as_longlong(f10), __double_as_longlong(k0), __double_as_longlong(f00),
                                  __double_as_longlong(p0)};
        bool same = true;
#pragma unroll
        for (int q = 0; q < 7; q++) same = same && s.ukey[q] == key[q];
        if (!__all_sync(0xffffffffu, same)) {  // every lane has read the key before lane 0 rewrites it
            __syncwarp();
            if (lane < N) {
                const double O_nt = md.O[lane], v_nt = md.v[lane];
                const double OR = O_nt / R0, zv = z0 * v_nt;  // the expressions of setup_nt and the bound
                s.uOR[lane] = OR;
                s.uZV[lane] = zv;
                s.uG[lane] = OR + div_z(zv, f10);
                s.uEM[lane] = (((k0 * md.u[lane]) * f00) * f00) + __dmul_rd(O_nt, recip_rd(R0)) * p0;
            }
            if (lane == 0) {
#pragma unroll
                for (int q = 0; q < 7; q++) s.ukey[q] = key[q];
            }
            __syncwarp();
        }
        uc = true;
    }
#endif
    const bool use_lb = PRUNE && mode != JDOB_MODE_BINARY;
    if (use_lb) {
        // Lower bound of E over every configuration at n~: a member's term
        // ((kappa u) f*) f* + (O/R) p >= ((kappa u) f_min) f_min + RN(RD(O RD(1/R)) p) (f* >= f_min, RN
        // monotone), a non-member's term is e_loc, so each term >= the min of the two; the user-order
        // RN sum of the minima is <= the sum of the terms, and the edge term (psi f_e) f_e >= 0.
        if (UNI) {  // every user has user 0's kappa, f_min, p_u and R: one bound term per n~
            const double rv = uc ? 0.0 : recip_rd(R0), kv = k0, fv = f00, pv = p0;  // user 0's values
            const double cM = 1.0 - (double)(M - 1) * 0x1p-53;  // (1 - (M-1) u), exact
            if (TIGHT) {
                // differing deadlines: e_loc along the sorted positions (deadline ascending) is non-increasing
                // (uniform users: f_loc = clamp(RN(zeta v_N / T)) is non-increasing in T, e_loc non-decreasing
                // in f_loc, RN monotone); its RD prefix / suffix sums (each <= the exact sum) serve both bounds
                JDOB_CHECK(M >= 1 && M <= kMaxM);
                if (lane < M) s.gam[lane] = s.et[s.order[lane]].x;  // (gamma is not stored for equal-gamma users)
                __syncwarp();
                if (lane < M) {
                    double pr = 0.0, sf = 0.0;
                    for (int t = 0; t < M; t++) {
                        const double v = s.gam[t];
                        if (t < lane) pr = __dadd_rd(pr, v);
                        else sf = __dadd_rd(sf, v);
                    }
                    s.pre[lane] = pr;
                    s.rinv[lane] = sf;
                }
                __syncwarp();
            }
            for (int nt = lane; nt < N; nt += 32) {
                const double em = uc ? s.uEM[nt] : (((kv * md.u[nt]) * fv) * fv) + __dmul_rd(md.O[nt], rv) * pv;
#ifndef JDOB_NO_TIGHT_LB
                if (TIGHT || MULTI) s.lbem[nt] = em;
#endif
                double S = 0.0;
                if (!TIGHT) {
                    // equal deadlines: every user's e_loc is the same bits, so every term is t; the RN sum of
                    // M copies of t >= M t (1 - u)^(M-1) >= M t (1 - (M-1) u) (u = 2^-53, each RN step
                    // >= (1 - u) times its exact sum), bounded below by two RD products (a valid, slightly
                    // weaker bound: pruning stays exact)
                    const double el = s.et[0].x, t = (em < el) ? em : el;
                    S = __dmul_rd(__dmul_rd((double)M, t), 1.0 - (double)(M - 1) * 0x1p-53);
                } else {
                    // every term >= min(em, e_loc_m), whose exact sum is c em + (the e_loc of the sorted
                    // positions >= c), c = #{q : e_loc(q) >= em} (a prefix: e_loc non-increasing); the RN sum of
                    // non-negative terms in any order is >= (1 - (M-1) u) times the exact sum
                    int lo = 0, hi = M;
                    while (lo < hi) {
                        const int mm = (lo + hi) >> 1;
                        if (s.gam[mm] >= em) lo = mm + 1;
                        else hi = mm;
                    }
                    JDOB_CHECK(lo >= 0 && lo <= M && nt < 64);
                    S = __dmul_rd(__dadd_rd(__dmul_rd((double)lo, em), (lo < M) ? s.rinv[lo] : 0.0), cM);
                }
                s.lb[nt] = S;
            }
        } else {
            if (lane < M) s.rinv[lane] = recip_rd(x.R);
            __syncwarp();
            for (int nt = lane; nt < N; nt += 32) {
                const double u_nt = md.u[nt], O_nt = md.O[nt];
                double S = 0.0;
                for (int m = 0; m < M; m++) {
                    const double ku = s.kap[m] * u_nt;
                    const double up = __dmul_rd(O_nt, s.rinv[m]) * s.pu[m];
                    const double fm = s.fmm[m].x;
                    const double em = ((ku * fm) * fm) + up;
                    const double el = s.et[m].x;
                    S = S + ((em < el) ? em : el);
                }
                s.lb[nt] = S;
            }
        }
        __syncwarp();
    }
    double bE;
    int bN, bP, bJ, aN, aJ;
    // MULTI: the no-edge-DVFS mode's best (candidates at j = 0: lane 0's first point) and all-local key,
    // and the binary mode's (candidates at n~ = 0)
    double gE = dinf(), hE = dinf();
    int gN = 0x7fffffff, gP = 0, gaN = N, gaJ = 0, hJ = 0, hP = 0, haN = N, haJ = 0;
    long long c_setup = 0, c_visit = 0, c_eval = 0, c_member = 0;
    int last_nt = -1;  // the n~ whose set-up is in shared memory
    for (int pass = 0;; pass++) {
        // pass 1 (rare): an exact tie with E_LC after pruning -- the all-local key (aN, aJ) of the
        // skipped n~ may matter (R8), so the instance is swept again without pruning
        const bool prune = use_lb && pass == 0;
        bool pruned = false;
        double bEw = dinf();  // warp-uniform best energy so far
        double bEwG = dinf();  // MULTI: the no-edge-DVFS mode's
        bE = dinf();
        bN = 0x7fffffff;
        bP = 0;
        bJ = 0;
        aN = N;  // first all-local evaluation key (R8); n~ = N at j = 0 by default (R4)
        aJ = 0;
        if (MULTI) {
            gE = hE = dinf();
            gN = 0x7fffffff;
            gP = hJ = hP = 0;
            gaN = haN = N;
            gaJ = haJ = 0;
        }

#if JDOB_PRUNE_ORDER == 2
        unsigned long long done = 0ull;  // n~ swept in this pass (best-first order)
#endif
        for (int nt = -1;;) {
            int kkn = kk;  // this n~'s grid length (MULTI: 1 when only the no-edge-DVFS mode needs the n~)
            if (!prune) {
                if (++nt >= N || (mode == JDOB_MODE_BINARY && nt != 0)) break;
            } else {
#if JDOB_PRUNE_ORDER == 2
                // best first: the unswept n~ with the smallest lower bound (ties: smallest n~) among those
                // whose bound is <= min(best so far, E_LC).  A configuration at a skipped n~ has E >= lb >
                // the best (it cannot win) or > E_LC (LC beats it); bounds equal to the best are swept, so
                // exact ties are decided by the (E, n~, j) key as in the literal loop.
                const double Bd = (bEw < E_lc) ? bEw : E_lc;
                const double l0 = (lane < N && !((done >> lane) & 1ull) && s.lb[lane] <= Bd) ? s.lb[lane] : dinf();
                const double l1 = (lane + 32 < N && !((done >> (lane + 32)) & 1ull) && s.lb[lane + 32] <= Bd)
                                      ? s.lb[lane + 32] : dinf();
                const double lm = warp_min_nonneg((l1 < l0) ? l1 : l0);  // bounds are >= 0
                if (!(lm < dinf())) {
                    pruned |= __popcll(done) < N;
                    break;
                }
                unsigned long long hit = __ballot_sync(0xffffffffu, l0 == lm);
                if (N > 32) hit |= (unsigned long long)__ballot_sync(0xffffffffu, l1 == lm) << 32;
                nt = __ffsll((long long)hit) - 1;
                done |= 1ull << nt;
#else
                // next n~ (ascending) whose lower bound is below the best so far (every configuration at
                // a skipped n~ has E >= lb >= bEw, so none of them can win; an equal E at a later n~
                // loses the (E, n~, j) tie-break).  JDOB_PRUNE_ORDER 1 also caps the bound at E_LC: a
                // configuration with E > E_LC loses to LC.
#if JDOB_PRUNE_ORDER == 1
                unsigned long long cand = __ballot_sync(0xffffffffu, lane < N && s.lb[lane] < bEw && s.lb[lane] <= E_lc);
                if (N > 32) cand |= (unsigned long long)__ballot_sync(0xffffffffu, lane + 32 < N && s.lb[lane + 32] < bEw &&
                                                                                s.lb[lane + 32] <= E_lc) << 32;
#else
                // (MULTI: an n~ is visited when either pruned mode may still improve there)
                const double bEs = MULTI ? ((bEwG > bEw) ? bEwG : bEw) : bEw;
                unsigned long long cand = __ballot_sync(0xffffffffu, lane < N && s.lb[lane] < bEs);
                if (N > 32) cand |= (unsigned long long)__ballot_sync(0xffffffffu, lane + 32 < N &&
                                                                                s.lb[lane + 32] < bEs) << 32;
#endif
                cand &= ~0ull << (nt + 1);
                if (cand == 0ull) {
                    pruned |= nt + 1 < N;
                    break;
                }
                const int nx = __ffsll((long long)cand) - 1;
                pruned |= nx > nt + 1;
                nt = nx;
                if (MULTI && !(s.lb[nt] < bEw) && kk > 1) {
                    // the full mode skips this n~ (its configurations cannot win there); the no-edge-DVFS
                    // mode needs its j = 0 only.  A partial sweep counts as pruning for the R8 re-sweep.
                    kkn = 1;
                    pruned = true;
                    if (homog) {
                        // the j = 0 configurations' bound (f_e = f_e,max exactly): set start p needs f_e,max >=
                        // th_p and >= the guard quotient (the set-up's own expressions), members' terms >=
                        // their lower-bound terms, the edge term is the sweep's; skip the n~ when no such
                        // configuration can beat the no-edge-DVFS best so far or LC (homogeneous users:
                        // the ranks and suffix-min deadlines are the instance's)
                        const double O_nt = md.O[nt], v_nt = md.v[nt], u_nt = md.u[nt];
                        const double ORg = O_nt / s.R[0];
                        const double gamg = ORg + div_z(s.z[0] * v_nt, s.f1[0]);
                        double lbp = dinf();
                        if (lane < M) {
                            double S = 0.0;
                            if (UNI) {
                                // uniform users: the members' term bound em is common; the RD sum of the
                                // non-members' e_loc (the sorted positions < p) plus (M - p) em, times
                                // (1 - (M-1) u), bounds the RN sum (as the batch-coupled bound)
                                const double em = s.lbem[nt];
                                const double pel = TIGHT ? s.pre[lane] : __dmul_rd((double)lane, s.et[0].x);
                                S = __dmul_rd(__dadd_rd(pel, __dmul_rd((double)(M - lane), em)),
                                              1.0 - (double)(M - 1) * 0x1p-53);
                            } else {
                                for (int m = 0; m < M; m++) {
                                    const double fm = s.fmm[m].x;
                                    const double emm = (((s.kap[m] * u_nt) * fm) * fm) +
                                                       __dmul_rd(O_nt, s.rinv[m]) * s.pu[m];
                                    S = S + ((s.rank[m] >= lane) ? emm : s.et[m].x);
                                }
                            }
                            const double phi = md.phi[nt * B1 + (M - lane)], psi = md.psi[nt * B1 + (M - lane)];
                            const double L = s.Lg[lane].x;
                            const double thp = phi / (L - gamg), gp = phi / (L - t_free);
                            if (!(fe_max < thp) && fe_max >= gp) lbp = S + (psi * fe_max) * fe_max;
                        }
                        const double lg = warp_min_nonneg(lbp);
                        if (!(lg < bEwG) || lg > E_lc) continue;
                    }
                }
#ifndef JDOB_NO_TIGHT_LB
                // (not in the equal-deadline kernel: there it removes 28 % of C2's set-ups, mostly of the
                // instances LC wins, but its code costs that kernel 2 % more than the set-ups it saves)
                if (UNI && TIGHT) {
                    // batch-coupled bound of the candidate n~: a configuration with set start p
                    // has the members {m : r_m >= p} (terms >= the member term em of lb) and B = M - p; its f_e
                    // passes the guard, f_e >= RN(phi(B) / RN(L_p - t_free)), and the membership threshold of p,
                    // f_e >= th_p = RN(phi(B) / RN(L_p - gamma)) (uniform users: one gamma), so f_e >= g_p =
                    // RD(phi(B) max(RD(1 / (L_p - t_free)), RD(1 / (L_p - gamma)))) (the second only when
                    // L_p - gamma > 0).  Hence E >= RN(S_p + RD(RD(psi(B) g_p) g_p)), S_p the user-order RN
                    // sum of the terms.  The minimum over p bounds every configuration at n~; the n~ is
                    // skipped when it is not below the best so far, or above E_LC (LC wins)
                    const double em = s.lbem[nt];
                    const double gam = uc ? s.uG[nt] : dinf();  // gamma of n~ (cached for N <= 32)
                    double lbp = dinf();
                    if (lane < M) {
                        // the members' terms >= em, the others' are e_loc: the exact sum is >= the RD sum of
                        // e_loc over the sorted positions < p plus (M - p) em; the RN sum >= (1 - (M-1) u) times it
                        const double S = __dmul_rd(__dadd_rd(s.pre[lane], __dmul_rd((double)(M - lane), em)),
                                                   1.0 - (double)(M - 1) * 0x1p-53);
                        const double L = s.Lg[lane].x;
                        const double r1 = recip_rd(L - t_free);  // L_p >= t_free (Require); +inf iff L_p = t_free:
                        const double dg = L - gam;               // then no f_e passes the guard
                        const double r2 = (dg > 0.0) ? recip_rd(dg) : 0.0;
                        const double g = __dmul_rd(md.phi[nt * B1 + (M - lane)], (r2 > r1) ? r2 : r1);
                        // g > f_e,max: no grid point reaches set start p.  With one grid point (no edge
                        // DVFS) f_e = f_e,max exactly, and the edge term is the sweep's own expression
                        const double psi = md.psi[nt * B1 + (M - lane)];
                        if (r1 != dinf() && !(g > fe_max))
                            lbp = S + ((kk == 1) ? (psi * fe_max) * fe_max : __dmul_rd(__dmul_rd(psi, g), g));
                    }
                    const double lt = warp_min_nonneg(lbp);
                    if (!(lt < (MULTI ? ((bEwG > bEw) ? bEwG : bEw) : bEw)) || lt > E_lc) {
                        pruned = true;
                        continue;
                    }
                }
#endif
#endif
            }
            if (COUNTS) c_setup += 1;
            last_nt = nt;
            const int ihat = setup_nt(md, nt, M, homog, uni, t_free, s, lane, uc, !(UNI && !TIGHT));
            // two grid points per lane (j0 + lane and j0 + 32 + lane): the two energy chains are
            // independent, which doubles the instruction-level parallelism of the sweep and lets both
            // share each user's shared-memory loads
            for (int j0 = 0; j0 < kkn; j0 += 64) {
                const int jA = j0 + lane, jB = jA + 32;
                const bool vA = jA < kkn, vB = jB < kkn;
                const double feA = grid_fe(fe_max, rho, jA), feB = grid_fe(fe_max, rho, jB);
                // p(j): first sorted position >= i^ with !(f_e < th_i)  (M if the set is empty)
                int loA = ihat, hiA = M, loB = ihat, hiB = M;
                while (loA < hiA) {
                    const int mm = (loA + hiA) >> 1;
                    if (feA < s.th[mm]) loA = mm + 1;
                    else hiA = mm;
                }
                while (loB < hiB) {
                    const int mm = (loB + hiB) >> 1;
                    if (feB < s.th[mm]) loB = mm + 1;
                    else hiB = mm;
                }
                const int pA = loA, pB = loB;
                // Alg. 2's break: the first j with an empty set ends this n~'s sweep
                const unsigned empA = __ballot_sync(0xffffffffu, vA && pA == M);
                const unsigned empB = __ballot_sync(0xffffffffu, vB && pB == M);
                const int jb = empA ? j0 + (__ffs(empA) - 1) : (empB ? j0 + 32 + (__ffs(empB) - 1) : kkn);
                const bool emp = (empA | empB) != 0u;
                if (emp && nt < aN) {  // the first all-local evaluation in the literal (n~, j) order
                    aN = nt;
                    aJ = (int)jb;
                }
                if (MULTI && emp) {
                    if (jb == 0 && nt < gaN) {  // no edge DVFS: the set at j = 0 is empty
                        gaN = nt;
                        gaJ = 0;
                    }
                    if (nt == 0 && haN == N) {  // binary: the first all-local evaluation at n~ = 0
                        haN = 0;
                        haJ = (int)jb;
                    }
                }
                if (COUNTS && emp && lane == 0) {  // the all-local evaluation at jb (guard passes: 0 / inf = 0)
                    c_visit += 1;
                    c_eval += 1;
                }
                const bool actA = vA && jA < jb, actB = vB && jB < jb;
                const int qA = actA ? pA : 0, qB = actB ? pB : 0;  // p < M for active grid points
                const double2 lgA = s.Lg[qA], lgB = s.Lg[qB];     // l_o, phi / (l_o - t_free)
                const double2 pqA = s.pp[qA], pqB = s.pp[qB];     // phi_n~(B_o), psi_n~(B_o)
                // D6 guard: f_e >= phi / (l_o - t_free); the quotient depends only on p
                const bool passA = actA && feA >= lgA.y, passB = actB && feB >= lgB.y;
                if (COUNTS) {
                    c_visit += (actA ? 1 : 0) + (actB ? 1 : 0);
                    c_eval += (passA ? 1 : 0) + (passB ? 1 : 0);
                    c_member += (passA ? M - pA : 0) + (passB ? M - pB : 0);
                }
                if (!(passA || passB)) {
                    if (emp) break;
                    continue;
                }
                const double invA = (jA < kInvCache) ? s.inv[jA] : 1.0 / feA;
                const double invB = (jB < kInvCache) ? s.inv[jB] : 1.0 / feB;
                const double teA = pqA.x * invA, teB = pqB.x * invB;
                double EA = 0.0, EB = 0.0;
                if (uni) {
                    // Uniform users (same R, zeta, f_min, f_max, kappa, p_u; Table I): every member
                    // has the same budget, f* and offloader term, so D20/D21 are formed once and
                    // only the user-order sum runs over M.  Same operations, same bits.
                    const double2 a0 = s.orzv[0], c0 = s.kuup[0], t0 = s.fmm[0];
                    const double budA = (lgA.x - a0.x) - teA, budB = (lgB.x - a0.x) - teB;
                    double fA = t0.x, fB = t0.x;
                    if (passA && !(__fma_rn(t0.x, budA, -a0.y) > 0.0) && a0.y != 0.0)
                        fA = clampf(a0.y / budA, t0.x, t0.y);  // D20 (R9 when zv = 0)
                    if (passB && !(__fma_rn(t0.x, budB, -a0.y) > 0.0) && a0.y != 0.0)
                        fB = clampf(a0.y / budB, t0.x, t0.y);
                    const double emA = ((c0.x * fA) * fA) + c0.y;  // D21 offloader term
                    const double emB = ((c0.x * fB) * fB) + c0.y;
#ifndef JDOB_NO_PREFIX
                    if (UNI && !TIGHT) {  // (the equal-deadline kernel: members are the users m >= p)
                        // equal deadlines: the ranks are the user indices, so the members are the users
                        // m >= p (thresholds non-increasing from i^) and the user-order sum is the prefix
                        // P[p] of the e_loc terms (formed with E_LC) followed by M - p member terms
                        JDOB_CHECK(pA >= 0 && pA <= M && pB >= 0 && pB <= M);
                        EA = s.pre[pA];
                        EB = s.pre[pB];
                        for (int m = (pA < pB) ? pA : pB; m < M; m++) {
                            if (m >= pA) EA = EA + emA;
                            if (m >= pB) EB = EB + emB;
                        }
                    } else
#endif
                    {
#pragma unroll 4
                        for (int m = 0; m < M; m++) {
                            const double2 et = s.et[m];  // eloc, thu
                            EA = EA + ((!(feA < et.y)) ? emA : et.x);
                            EB = EB + ((!(feB < et.y)) ? emB : et.x);
                        }
                    }
                } else {
                    const long long fbA = __double_as_longlong(feA), fbB = __double_as_longlong(feB);
#pragma unroll 2
                    for (int m = 0; m < M; m++) {
                        const double2 a = s.orzv[m];  // OR, zv
                        const double2 c = s.kuup[m];  // ku, up
                        const double2 d = s.et[m];    // eloc, thu
                        const double2 t = s.fmm[m];   // fmin, fmax
                        // f_e, th >= 0 (or +inf): IEEE order = integer order of the bit patterns
                        const long long thb = __double_as_longlong(d.y);
                        const bool memA = fbA >= thb, memB = fbB >= thb;
                        const double budA = (lgA.x - a.x) - teA, budB = (lgB.x - a.x) - teB;
                        double fA = t.x, fB = t.x;  // f_min unless f_min budget > zv fails exactly
                        const bool needA = passA && memA && !(__fma_rn(t.x, budA, -a.y) > 0.0);
                        const bool needB = passB && memB && !(__fma_rn(t.x, budB, -a.y) > 0.0);
                        if (needA || needB) {
                            // R9 (zv = 0 -> f_min) tested on the bits, inside the rare branch
                            const bool nz = (__double_as_longlong(a.y) << 1) != 0;
                            if (needA && nz) fA = clampf(a.y / budA, t.x, t.y);  // D20
                            if (needB && nz) fB = clampf(a.y / budB, t.x, t.y);
                        }
                        const double emA = ((c.x * fA) * fA) + c.y;  // D21 offloader term
                        const double emB = ((c.x * fB) * fB) + c.y;
                        EA = EA + (memA ? emA : d.x);
                        EB = EB + (memB ? emB : d.x);
                    }
                }
                EA = EA + (pqA.y * feA) * feA;
                EB = EB + (pqB.y * feB) * feB;
                // strict in (E, n~, j): within an n~ a lane's j ascend; n~ may be swept out of order
                if (passA && (EA < bE || (EA == bE && nt < bN))) {
                    bE = EA;
                    bN = nt;
                    bJ = (int)jA;
                    bP = pA;
                }
                if (passB && (EB < bE || (EB == bE && nt < bN))) {
                    bE = EB;
                    bN = nt;
                    bJ = (int)jB;
                    bP = pB;
                }
                if (MULTI) {
                    if (j0 == 0 && lane == 0 && passA && (EA < gE || (EA == gE && nt < gN))) {  // j = 0
                        gE = EA;
                        gN = nt;
                        gP = pA;
                    }
                    if (nt == 0) {  // binary: n~ = 0 only; a lane's j ascend
                        if (passA && EA < hE) {
                            hE = EA;
                            hJ = (int)jA;
                            hP = pA;
                        }
                        if (passB && EB < hE) {
                            hE = EB;
                            hJ = (int)jB;
                            hP = pB;
                        }
                    }
                }
                if (emp) break;
            }
            if (prune) {  // warp minimum of the lane bests (energies are >= 0)
                const double w = warp_min_nonneg(bE);
                bEw = (w < bEw) ? w : bEw;
                if (MULTI) bEwG = __shfl_sync(0xffffffffu, gE, 0);
            }
            __syncwarp();
        }
        // warp argmin over (E, n~, j): E >= 0, so the minimum energy comes from two integer
        // reductions of its bits; among the lanes holding it, the smallest packed key
        // n~ << 22 | j << 5 | p (n~ < 64, j < 2^16, p < 32) is the smallest (n~, j)
        {
            const double Emin = warp_min_nonneg(bE);
            const unsigned key = (bE == Emin && bE < dinf())
                                     ? (((unsigned)bN << 22) | ((unsigned)bJ << 5) | (unsigned)bP)
                                     : 0xffffffffu;
            const unsigned mk = __reduce_min_sync(0xffffffffu, key);
            bE = Emin;
            if (mk != 0xffffffffu) {
                bN = (int)(mk >> 22);
                bJ = (int)((mk >> 5) & 0xffffu);
                bP = (int)(mk & 31u);
            } else {  // no candidate in any lane (bE = +inf)
                bN = 0x7fffffff;
                bJ = 0;
                bP = 0;
            }
        }
        if (MULTI) {
            // binary: the same argmin at n~ = 0; no edge DVFS: lane 0 holds its best
            const double Hmin = warp_min_nonneg(hE);
            const unsigned key = (hE == Hmin && hE < dinf()) ? (((unsigned)hJ << 5) | (unsigned)hP) : 0xffffffffu;
            const unsigned mk = __reduce_min_sync(0xffffffffu, key);
            hE = Hmin;
            hJ = (mk != 0xffffffffu) ? (int)((mk >> 5) & 0xffffu) : 0;
            hP = (mk != 0xffffffffu) ? (int)(mk & 31u) : 0;
            gE = __shfl_sync(0xffffffffu, gE, 0);
            gN = __shfl_sync(0xffffffffu, gN, 0);
            gP = __shfl_sync(0xffffffffu, gP, 0);
        }
        if (!(pruned && (bE == E_lc || (MULTI && gE == E_lc)))) break;
    }
    if (COUNTS) {
#pragma unroll
        for (int d = 16; d >= 1; d >>= 1) {
            c_visit += __shfl_xor_sync(0xffffffffu, c_visit, d);
            c_eval += __shfl_xor_sync(0xffffffffu, c_eval, d);
            c_member += __shfl_xor_sync(0xffffffffu, c_member, d);
        }
        if (lane == 0 && !PRUNE) {
            r.counts[3 * i] = c_visit;
            r.counts[3 * i + 1] = c_eval;
            r.counts[3 * i + 2] = c_member;
        }
        if (lane == 0 && PRUNE) {
            r.work[4 * i] = c_setup;
            r.work[4 * i + 1] = c_visit;
            r.work[4 * i + 2] = c_eval;
            r.work[4 * i + 3] = c_member;
        }
    }
    // the answer of one mode (the winner re-evaluated lane = user, or the all-local plan)
    auto emit = [&](const DevResult &rr, const double bE, const int bN, const int bJ, const int bP, const int aN,
                    const int aJ) {
        const bool offload_wins = (bE < E_lc) || (bE == E_lc && (bN < aN || (bN == aN && bJ < aJ)));
        if (!offload_wins) {
            write_local(rr, i, off, M, N, E_lc, t_free, floc, st, lane, false);
            if (VERIFY) {
                const unsigned vb = verify_local(x, vN, floc, M, vflags, rr.slack, lane);
                if (lane == 0) rr.viol[i] = vb;
            }
            return;
        }
        // winner: recompute D20 and D22 lane = user (same arithmetic as the sweep)
#ifdef JDOB_WIN_SETUP
        const bool win_direct = false;
#else
        // homogeneous users: ranks and sorted deadlines are per instance, only (O/R, zv) depend on n~,
        // so the winner's are formed directly (same expressions as setup_nt) instead of a new set-up
        const bool win_direct = homog;
#endif
        if (!win_direct && bN != last_nt) {
            setup_nt(md, bN, M, homog, uni, t_free, s, lane, uc);
            last_nt = bN;
        }
        const int Bo = M - bP;
        const double lo_ = s.Lg[bP].x;
        const double fe = grid_fe(fe_max, rho, bJ);
        const double inv = (bJ < kInvCache) ? s.inv[bJ] : 1.0 / fe;  // the sweep's cached 1/f_e(j), same bits
        const double te = md.phi[bN * B1 + Bo] * inv;
        const bool member = (lane < M) && (s.rank[lane] >= bP);
        double f = floc, arr = t_free;
        unsigned vbits = 0u;  // the plan re-verified with jdob_eval's formulas (row a11)
        if (VERIFY) {
            if (lane == 0) {
                if (!(fe >= x.fe_min && fe <= fe_max)) vbits |= 32u;
                if (t_free + te > lo_ + rr.slack * fabs(lo_)) vbits |= 1u;  // D6: the ASAP start of batch n~ + 1
            }
            if (!member && lane < M && d8_violated(x.z * vN, floc, x.T + rr.slack * fabs(x.T))) vbits |= 4u;  // D8
        }
        if (member) {
            const double2 a = (win_direct && uc) ? make_double2(s.uOR[bN], s.uZV[bN])
                              : win_direct ? make_double2(md.O[bN] / s.R[lane], s.z[lane] * md.v[bN])
                                         : s.orzv[uni ? 0 : lane];  // (O/R, zv)
            const double2 t = s.fmm[lane];                          // (f_min, f_max)
            const double budget = (lo_ - a.x) - te;
            const bool low = (a.y == 0.0) || (__fma_rn(t.x, budget, -a.y) > 0.0);
            f = low ? t.x : clampf(a.y / budget, t.x, t.y);
            arr = div_z(a.y, f) + a.x;
            if (VERIFY) {
                // jdob_eval's D20 branches (bit 3 and the f of an infeasible budget) and its D7 finish test
                double fev = f;
                if (a.y == 0.0) {
                    if (budget < 0.0) vbits |= 8u;
                } else if (!(__fma_rn(t.x, budget, -a.y) > 0.0) && !(budget > 0.0)) {
                    vbits |= 8u;
                    fev = t.y;
                }
                double fin = arr;  // eval's arrival div_z(zv, f) + O/R: arr unless eval took f_max
                if (fev != f) fin = div_z(a.y, fev) + a.x;
                fin = fin + te;
                if (fin > lo_ + rr.slack * fabs(lo_)) vbits |= 2u;
            }
            if (arr < t_free) arr = t_free;
        }
        arr = warp_max_nonneg(arr);  // arrivals >= t_free >= 0
        const unsigned mask = __ballot_sync(0xffffffffu, member);
        if (VERIFY) {
            vbits = __reduce_or_sync(0xffffffffu, vbits);
            if (lane == 0) rr.viol[i] = vbits;
        }
        if (lane == 0) {
            rr.E[i] = bE;
            rr.E_lc[i] = E_lc;
            rr.t_free_next[i] = arr + te;  // D22
            rr.f_e[i] = fe;
            rr.n_tilde[i] = bN;
            rr.j[i] = (int)bJ;
            rr.status[i] = st;
            rr.mask[i] = mask;
        }
        if (rr.f_user && lane < M) rr.f_user[off + lane] = f;
        if (rr.partition && lane < M) rr.partition[off + lane] = member ? bN : N;
    };
    if (MULTI) {
        emit(rx[0], gE, gN, 0, gP, gaN, gaJ);                                  // no edge DVFS
        emit(rx[1], hE, (hE < dinf()) ? 0 : 0x7fffffff, hJ, hP, haN, haJ);      // binary
    }
    emit(r, bE, bN, bJ, bP, aN, aJ);
}

#ifndef JDOB_SOLVE_MINB
#define JDOB_SOLVE_MINB 5
#endif

#ifndef JDOB_SOLVE_MINB_U
#define JDOB_SOLVE_MINB_U 5
#endif

// VERIFY: the instantiation with row a11 in the epilogue (r.viol != NULL); the product kernel without
// it carries none of that code (K1's speed is sensitive to its code size)
template <bool COUNTS, bool PRUNE, bool UNI, bool VERIFY, bool TIGHT>
__global__ void __launch_bounds__(kSolveWarps * 32, UNI ? JDOB_SOLVE_MINB_U : JDOB_SOLVE_MINB)
    k_solve(const DevModel *models, DevBatch b, DevResult r, int mode) {
    __shared__ SolveSmem smem[kSolveWarps];
    const int lane = threadIdx.x & 31;
    SolveSmem &s = smem[threadIdx.x >> 5];
    if (lane == 0) {
        s.inv_key = make_double2(0.0, 0.0);  // rho > 0 in every valid instance: no false hit
        s.inv_n = 0;
        s.kc = GridKCache{0.0, 0.0, 0.0, 0};  // rho > 0 in every valid instance: no false hit
        s.ukey[0] = -1;                       // no model id -1: no false hit
        s.defer = 0;
        s.pre[0] = 0.0;
    }
    __syncwarp();
    const long long gw = (long long)blockIdx.x * kSolveWarps + (threadIdx.x >> 5);
    const long long nw = (long long)gridDim.x * kSolveWarps;
    if (UNI && !TIGHT) {
        // (user_off, user count, model id) of the warp's next instance are loaded while it solves the
        // current one, so each instance's user loads issue at once (one HBM latency less per instance)
        // (the user count is formed when the instance starts, not next to the loads: the subtraction
        // would wait for them there)
        auto head = [&](long long i, long long &o, long long &e, int &id) {
            if (i < b.n_inst) {
                o = b.user_off[i];
                e = b.user_end ? b.user_end[i] : b.user_off[i + 1];
                id = b.model_id[i];
            }
        };
        long long o = 0, e = 0;
        int id = 0;
#ifndef JDOB_STRIDED
        // dynamic hand-out of 32-instance chunks from a counter in the workspace (the warps that drew
        // expensive instances take fewer chunks: no tail of a few late warps); the next chunk is drawn
        // when the current one starts
        // (a batch with fewer than 8 chunks per warp keeps the static grid-stride order: chunks of one
        // instance, gw, gw + nw, ...; the chunks' granularity would otherwise leave a tail)
#ifndef JDOB_CHUNK
#define JDOB_CHUNK 8
#endif
        const bool dyn = r.flags && b.n_inst >= 8ll * JDOB_CHUNK * nw;
        unsigned long long *ctr = dyn ? (unsigned long long *)(r.flags + 2) : nullptr;
        const int csz = dyn ? JDOB_CHUNK : 1;
        long long kst = 0;
        auto grab = [&]() -> long long {
            if (!ctr) return gw + nw * (kst++);
            long long v = 0;
            if (lane == 0) v = (long long)atomicAdd(ctr, 1ull);
            return __shfl_sync(0xffffffffu, v, 0);
        };
        long long nchunk = grab();
        long long i = nchunk * csz;
        nchunk = grab();
        int q = 0;
        head(i, o, e, id);
        while (i < b.n_inst) {
            const long long co = o, cm = e - o;
            const int cid = id;
            const long long inext = (q < csz - 1) ? i + 1 : nchunk * csz;
            head(inext, o, e, id);
            solve_instance<COUNTS, PRUNE, UNI, VERIFY, TIGHT>(i, co, cm, cid, models, b, r, mode, s, lane, o, e);
            if (q < csz - 1) {
                q++;
            } else {
                q = 0;
                nchunk = grab();
            }
            i = inext;
        }
#else
        head(gw, o, e, id);
        for (long long i = gw; i < b.n_inst; i += nw) {
            const long long co = o, cm = e - o;
            const int cid = id;
            head(i + nw, o, e, id);
            // (o, e: the next instance's head; for a warp's last instance the current one's, whose users
            // the prefetch then touches again -- valid addresses, no select waiting on the loads)
            solve_instance<COUNTS, PRUNE, UNI, VERIFY, TIGHT>(i, co, cm, cid, models, b, r, mode, s, lane, o, e);
        }
#endif
        __syncwarp();
        if (lane == 0 && s.defer && r.flags) r.flags[0] = 1;  // one store per warp, not per deferral
    } else {
        // nothing deferred by the kernel before: no instance to visit
        if (r.flags && r.flags[UNI ? 0 : 1] == 0) return;
        // only the instances the kernels before left (kStDefer), 32 statuses per load.  Groups of 32
        // consecutive instances are handed out dynamically from a counter in the workspace (a warp that
        // drew expensive instances takes fewer groups); without one, lane l of round t looks at instance
        // gw + (32 t + l) nw, the deferred instances spread over the warps as in a grid-stride loop
        // (dynamic groups only for a batch of at least 8 groups per warp, as in the kernel before)
        unsigned long long *ctr = (r.flags && b.n_inst >= 8ll * 32 * nw) ? (unsigned long long *)(r.flags + (UNI ? 4 : 6))
                                                                        : nullptr;
        for (long long t = 0;; t++) {
            long long base, step;
            if (ctr) {
                long long g = 0;
                if (lane == 0) g = (long long)atomicAdd(ctr, 1ull);
                base = __shfl_sync(0xffffffffu, g, 0) * 32;
                step = 1;
            } else {
                base = gw + t * 32 * nw;
                step = nw;
            }
            if (base >= b.n_inst) break;
            const long long ii = base + lane * step;
            const bool in = ii < b.n_inst;
            unsigned def = __ballot_sync(0xffffffffu, in && r.status[ii] == kStDefer);
            // the heads (user_off, user count, model id) of the group's instances, one coalesced load each,
            // handed to the instance's solve by shuffles (no dependent load per instance)
            long long ho = 0, hm = 0;
            int hid = 0;
            if (def && in) {
                ho = b.user_off[ii];
                hm = (b.user_end ? b.user_end[ii] : b.user_off[ii + 1]) - ho;
                hid = b.model_id[ii];
            }
            while (def) {
                const int q = __ffs(def) - 1;
                def &= def - 1u;
                const long long o = __shfl_sync(0xffffffffu, ho, q), m = __shfl_sync(0xffffffffu, hm, q);
                const int id = __shfl_sync(0xffffffffu, hid, q);
                solve_instance<COUNTS, PRUNE, UNI, VERIFY, TIGHT>(base + q * step, o, m, id, models, b, r, mode, s,
                                                                  lane);
            }
        }
        __syncwarp();
        if (UNI && lane == 0 && s.defer && r.flags) r.flags[1] = 1;  // the differing-deadline kernel's deferrals
    }
}

template <bool COUNTS, bool PRUNE, bool UNI, bool VERIFY, bool TIGHT>
static void launch_solve_t(const DevModel *models, const DevBatch &b, const DevResult &r, int mode, cudaStream_t s,
                           int num_sms) {
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_solve<COUNTS, PRUNE, UNI, VERIFY, TIGHT>,
                                                  kSolveWarps * 32, 0);
    if (per_sm < 1) per_sm = 1;
    const long long want = (b.n_inst + kSolveWarps - 1) / kSolveWarps;
    long long grid = (long long)num_sms * per_sm / grid_divisor();
    if (grid < 1) grid = 1;
    if (want < grid) grid = want;
    k_solve<COUNTS, PRUNE, UNI, VERIFY, TIGHT><<<(unsigned)grid, kSolveWarps * 32, 0, s>>>(models, b, r, mode);
}

template <bool COUNTS, bool PRUNE, bool VERIFY = false>
static void launch_pair(const DevModel *models, const DevBatch &b, const DevResult &r, int mode, cudaStream_t s,
                        int num_sms) {
    launch_solve_t<COUNTS, PRUNE, true, VERIFY, false>(models, b, r, mode, s, num_sms);  // uniform, equal deadlines
    launch_solve_t<COUNTS, PRUNE, true, VERIFY, true>(models, b, r, mode, s, num_sms);   // uniform, differing ones
    launch_solve_t<COUNTS, PRUNE, false, VERIFY, false>(models, b, r, mode, s, num_sms); // the rest
}

// NEXT-2 in one pass (k_solve's structure with MULTI solve_instance): JDOB_MODE_FULL into r0,
// JDOB_MODE_NO_EDGE_DVFS into r1, JDOB_MODE_BINARY into r2
template <bool UNI, bool TIGHT>
__global__ void __launch_bounds__(kSolveWarps * 32, UNI ? JDOB_SOLVE_MINB_U : JDOB_SOLVE_MINB)
    k_solve_multi(const DevModel *models, DevBatch b, DevResult r0, DevResult r1, DevResult r2) {
    __shared__ SolveSmem smem[kSolveWarps];
    const int lane = threadIdx.x & 31;
    SolveSmem &s = smem[threadIdx.x >> 5];
    if (lane == 0) {
        s.inv_key = make_double2(0.0, 0.0);
        s.inv_n = 0;
        s.kc = GridKCache{0.0, 0.0, 0.0, 0};
        s.ukey[0] = -1;
        s.pre[0] = 0.0;
        s.defer = 0;
    }
    __syncwarp();
    const DevResult rx[2] = {r1, r2};
    const long long gw = (long long)blockIdx.x * kSolveWarps + (threadIdx.x >> 5);
    const long long nw = (long long)gridDim.x * kSolveWarps;
    if (UNI && !TIGHT) {  // every instance (the equal-deadline kernel defers the others)
        for (long long i = gw; i < b.n_inst; i += nw) {
            const long long o = b.user_off[i];
            const long long m = (b.user_end ? b.user_end[i] : b.user_off[i + 1]) - o;
            solve_instance<false, true, UNI, false, TIGHT, true>(i, o, m, b.model_id[i], models, b, r0,
                                                                 JDOB_MODE_FULL, s, lane, 0, 0, rx);
        }
        __syncwarp();
        if (lane == 0 && s.defer && r0.flags) r0.flags[0] = 1;
    } else {  // the deferred ones, spread like a grid-stride loop (as k_solve)
        if (r0.flags && r0.flags[UNI ? 0 : 1] == 0) return;
        for (long long base = gw; base < b.n_inst; base += 32 * nw) {
            const long long ii = base + lane * nw;
            const bool in = ii < b.n_inst;
            unsigned def = __ballot_sync(0xffffffffu, in && r0.status[ii] == kStDefer);
            long long ho = 0, hm = 0;
            int hid = 0;
            if (def && in) {
                ho = b.user_off[ii];
                hm = (b.user_end ? b.user_end[ii] : b.user_off[ii + 1]) - ho;
                hid = b.model_id[ii];
            }
            while (def) {
                const int q = __ffs(def) - 1;
                def &= def - 1u;
                const long long o = __shfl_sync(0xffffffffu, ho, q), m = __shfl_sync(0xffffffffu, hm, q);
                const int id = __shfl_sync(0xffffffffu, hid, q);
                solve_instance<false, true, UNI, false, TIGHT, true>(base + q * nw, o, m, id, models, b, r0,
                                                                     JDOB_MODE_FULL, s, lane, 0, 0, rx);
            }
        }
        __syncwarp();
        if (UNI && lane == 0 && s.defer && r0.flags) r0.flags[1] = 1;
    }
}

template <bool UNI, bool TIGHT>
static void launch_multi_t(const DevModel *models, const DevBatch &b, const DevResult &r0, const DevResult &r1,
                           const DevResult &r2, cudaStream_t s, int num_sms) {
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_solve_multi<UNI, TIGHT>, kSolveWarps * 32, 0);
    if (per_sm < 1) per_sm = 1;
    const long long want = (b.n_inst + kSolveWarps - 1) / kSolveWarps;
    long long grid = (long long)num_sms * per_sm / grid_divisor();
    if (grid < 1) grid = 1;
    if (want < grid) grid = want;
    k_solve_multi<UNI, TIGHT><<<(unsigned)grid, kSolveWarps * 32, 0, s>>>(models, b, r0, r1, r2);
}

// NEXT-2 in one pass through the same three-kernel chain as launch_solve (equal-deadline uniform,
// differing-deadline uniform, general; r0.flags zeroed by the caller): J-DOB into r0, no edge DVFS into r1,
// binary into r2; M > 32 is left to k_solve_large, one launch per mode
void launch_solve_multi(const DevModel *models, const DevBatch &b, const DevResult &r0, const DevResult &r1,
                        const DevResult &r2, cudaStream_t s, int num_sms) {
    if (b.n_inst <= 0) return;
    launch_multi_t<true, false>(models, b, r0, r1, r2, s, num_sms);
    launch_multi_t<true, true>(models, b, r0, r1, r2, s, num_sms);
    launch_multi_t<false, false>(models, b, r0, r1, r2, s, num_sms);
}

void launch_solve(const DevModel *models, const DevBatch &b, const DevResult &r, int mode, cudaStream_t s,
                  int num_sms) {
    if (b.n_inst <= 0) return;
    if (r.counts) launch_pair<true, false>(models, b, r, mode, s, num_sms);      // literal counters
    else if (r.work) launch_pair<true, true>(models, b, r, mode, s, num_sms);    // executed counters
    else if (r.viol) launch_pair<false, true, true>(models, b, r, mode, s, num_sms);  // + row a11 in the epilogue
    else launch_pair<false, true>(models, b, r, mode, s, num_sms);
}

}  // namespace jdob
