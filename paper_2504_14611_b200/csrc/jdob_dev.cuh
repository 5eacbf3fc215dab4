// jdob_dev.cuh -- device-side data layout and helpers shared by the libjdob kernels.
//
// Compiled with --fmad=false: every double expression below rounds each operation
// separately (IEEE-754 binary64, round-to-nearest-even), in the order fixed by
// DESIGN.md §Arithmetic contract, so results are bit-identical to the CPU oracle.
// Explicit __fma_rn() is used only where DESIGN.md §Exact shortcuts proves the
// result bit-identical to the contract's plain expression.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/jdob.h"

namespace jdob {

// Bounds checks of the shared-memory and workspace indexing, compiled in only for the checking build
// (-DJDOB_BOUNDS: tools/bounds_check.sh runs the GPU suite on it; compute-sanitizer is closed on the
// GPU pool).  A failed check traps the kernel, which fails the calling test.
#ifdef JDOB_BOUNDS
#define JDOB_CHECK(cond) \
    do {                 \
        if (!(cond)) __trap(); \
    } while (0)
#else
#define JDOB_CHECK(cond) \
    do {                 \
    } while (0)
#endif

constexpr int kMaxM = JDOB_MAX_M;
constexpr int kMaxMLarge = JDOB_MAX_M_LARGE;
constexpr int kStDefer = -1;  // internal status: M > 32, handled by k_solve_large
constexpr int kMaxN = JDOB_MAX_N;
constexpr int kMaxK = JDOB_MAX_K;
constexpr int kStatsF = JDOB_STATS_FIELDS;

// Device-side model descriptor: user tables + aggregate tables built by K0 in the
// caller's workspace (DESIGN.md §Data layout).  All tables are row-major by n.
struct DevModel {
    int N, B1;                                // B1 = B_max + 1
    const double *A, *O, *g, *q, *d, *c;      // inputs
    double *u, *v;                            // [N+1]  prefix sums
    double *phi, *psi;                        // [(N+1)*B1] phi_n~(b), psi_n~(b)
    double *dA, *cA;                          // [(N+1)*B1] d_n(b) A_n, c_n(b) A_n
    int *valid;                               // 1 = model passed validation
};

struct DevBatch {
    long long n_inst;
    int n_models;
    const int *model_id;
    const long long *user_off;
    const long long *user_end;  // internal: if set, instance i's users end at user_end[i] (overlapping views)
    const double *zeta, *kappa, *f_min, *f_max, *R, *p_u, *T;
    const double *t_free, *fe_min, *fe_max, *rho;
    const int *bucket;
};

struct DevResult {
    double *E, *E_lc, *t_free_next, *f_e;
    int *n_tilde, *j, *status;
    unsigned *mask;
    double *f_user;
    long long *counts;
    int *partition = nullptr;   // per user n~* or N, or NULL
    long long *work = nullptr;  // [4 n_inst] executed-work counters of the pruned sweep, or NULL
    unsigned *viol = nullptr;   // [n_inst] the plan re-verified in the epilogue (jdob_eval bits), or NULL
    int *flags = nullptr;       // [8] zeroed before K1: [0..1] set when the equal- / differing-deadline kernel
                                // defers an instance (a later kernel with nothing to do returns at once);
                                // [2..7] three 64-bit work counters (dynamic hand-out of instance chunks)
    double slack = 0.0;
};

__device__ __forceinline__ double dinf() { return __longlong_as_double(0x7ff0000000000000LL); }

// Warp min / max of NON-NEGATIVE doubles (+0 .. +inf): their IEEE order is the integer order of the
// bit patterns, so two 32-bit redux.sync steps (high word, then low word among the lanes holding the
// extreme high word) give the exact extreme value.
__device__ __forceinline__ double warp_min_nonneg(double x) {
    const unsigned long long b = (unsigned long long)__double_as_longlong(x);
    const unsigned hi = (unsigned)(b >> 32), lo = (unsigned)b;
    const unsigned mh = __reduce_min_sync(0xffffffffu, hi);
    const unsigned ml = __reduce_min_sync(0xffffffffu, (hi == mh) ? lo : 0xffffffffu);
    return __longlong_as_double((long long)(((unsigned long long)mh << 32) | ml));
}
__device__ __forceinline__ double warp_max_nonneg(double x) {
    const unsigned long long b = (unsigned long long)__double_as_longlong(x);
    const unsigned hi = (unsigned)(b >> 32), lo = (unsigned)b;
    const unsigned mh = __reduce_max_sync(0xffffffffu, hi);
    const unsigned ml = __reduce_max_sync(0xffffffffu, (hi == mh) ? lo : 0u);
    return __longlong_as_double((long long)(((unsigned long long)mh << 32) | ml));
}
__device__ __forceinline__ double dnan() { return __longlong_as_double(0x7ff8000000000000LL); }
__device__ __forceinline__ bool dfinite(double x) { return isfinite(x); }

// D20 clamp: min{max{G, f_min}, f_max} -- same comparison order as the oracle.
__device__ __forceinline__ double clampf(double G, double fmin, double fmax) {
    double x = (G < fmin) ? fmin : G;
    return (x > fmax) ? fmax : x;
}

// a / b for b > 0 finite.  A zero numerator sends the correctly rounded division to its slow
// path (~140 instructions: the fast path's exponent test fails for a zero quotient), and
// 0 / b = 0 with a's sign, i.e. a itself: same bits, no division.  zeta v_0 = 0 at n~ = 0.
// (The compiler if-converts "a == 0 ? a : a / b" and divides anyway, and it folds a numerator
// select back to a / b, so the zero numerator is replaced by 1 behind an opaque move before the
// division and that quotient discarded.)
__device__ __forceinline__ double div_z(double a, double b) {
    const bool z = (a == 0.0);
    double n;
    asm("mov.b64 %0, %1;" : "=d"(n) : "d"(z ? 1.0 : a));
    const double q = n / b;
    return z ? a : q;
}

// a / b where a zero numerator over a positive finite b returns a (the quotient's exact value)
// without the slow path; every other case is the literal a / b (0 / 0 = NaN, x / 0 = inf, ...).
__device__ __forceinline__ double div_z0(double a, double b) {
    const bool z = (a == 0.0) && (b > 0.0) && (b <= 1.7976931348623157e308);
    double n;
    asm("mov.b64 %0, %1;" : "=d"(n) : "d"(z ? 1.0 : a));
    const double q = n / b;
    return z ? a : q;
}

// RD(1 / x) for x > 0 (the bound of DESIGN.md §4 "n~ pruning"), without the div_rd subroutine:
// q = RN(1 / x); if q x - 1 > 0 exactly (the sign of the fma) then q > 1/x and RD(1/x) is q's
// predecessor (no representable number lies strictly between RD and RN when they differ),
// otherwise q <= 1/x and q = RD(1/x).  q = +inf (x subnormal) gives DBL_MAX = RD; q = +0 gives
// +0 = RD (1/x below half the smallest subnormal).
__device__ __forceinline__ double recip_rd(double x) {
    const double q = 1.0 / x;
    return (__fma_rn(q, x, -1.0) > 0.0) ? __longlong_as_double(__double_as_longlong(q) - 1) : q;
}

// A lower bound of a / b for a >= 0, b > 0, at most RD(a / b)'s predecessor below it, without the
// div_rd subroutine: q = RN(a / b) and the sign of a - q b (exact in the fma) tells whether q
// exceeds the quotient; if it may (<= 0), q's predecessor is returned.  Only bounds use it.
__device__ __forceinline__ double div_lb(double a, double b) {
    const double q = a / b;
    return (q > 0.0 && !(__fma_rn(-q, b, a) > 0.0)) ? __longlong_as_double(__double_as_longlong(q) - 1) : q;
}

// jdob_eval's D8 test RN(zvN / f) > lim, lim = RN(T + slack |T|), f > 0: when lim f - zvN >= 0 exactly
// (the sign of the correctly rounded fma) the quotient is <= lim, so RN(quotient) <= lim and the test
// fails without the division; otherwise the literal division decides.
__device__ __forceinline__ bool d8_violated(double zvN, double f, double lim) {
    if (__fma_rn(lim, f, -zvN) >= 0.0) return false;
    return zvN / f > lim;
}

// Test hook (results independent of the grid size): the environment variable
// JDOB_GRID_DIV = d > 1 divides the persistent grids of K1 and K2 by d.  Host-side, read once.
int grid_divisor();

// Edge grid (R7): f_e(j) = f_e,max - j*rho, one multiply then one subtract.
__device__ __forceinline__ double grid_fe(double fe_max, double rho, long long j) {
    return __dsub_rn(fe_max, __dmul_rn((double)j, rho));
}
__device__ __forceinline__ double grid_fe(double fe_max, double rho, int j) {  // same value: j < 2^31
    return __dsub_rn(fe_max, __dmul_rn((double)j, rho));
}

// k = #{j >= 0 : f_e(j) >= f_e,min}; the predicate is monotone in j (RN(j rho) is
// non-decreasing, so is the subtraction's complement), so k is its first failing j in
// [0, kMaxK + 1].  Start from the estimate (f_e,max - f_e,min)/rho + 1 and step until
// pred(k - 1) holds and pred(k) fails -- the same k as the oracle's literal walk.
// Returns kMaxK + 1 when the grid is longer than kMaxK.
__device__ __forceinline__ long long grid_k(double fe_min, double fe_max, double rho) {
    if (grid_fe(fe_max, rho, kMaxK + 1) >= fe_min) return kMaxK + 1;
    const double est = (fe_max - fe_min) / rho;
    long long j = (est < 0.0) ? 0 : (est < (double)kMaxK ? (long long)est + 1 : kMaxK + 1);
    while (j <= kMaxK && grid_fe(fe_max, rho, j) >= fe_min) j++;
    while (j > 0 && !(grid_fe(fe_max, rho, j - 1) >= fe_min)) j--;
    return j;
}

// Per-warp cache of the grid length k for the last (f_e,min, f_e,max, rho) seen (shared memory).
struct GridKCache {
    double fe_min, fe_max, rho;
    long long k;
};

struct InstRegs {  // lane-resident user parameters (lane = user)
    double z, k, f0, f1, R, p, T;
    double t_free, fe_min, fe_max, rho;  // the instance's scalars (every lane)
};

// Warp-cooperative load and validation of instance i (lane = user), with the same
// predicates and precedence as the oracle's check_inst: BADMODEL, then BADPARAM
// (model id, M range, user boxes, edge boxes, grid length), then LOCAL_INFEASIBLE
// (P:127), then REQUIRE.  Lanes >= M get T = +inf and zeros.
// (off, M64, mid) = user_off[i], the user count and model_id[i], loaded by the caller (K1 loads
// the next instance's while it solves the current one).  The user loads are issued before the
// model checks so that their latency overlaps the model-table loads.
// The per-user predicates (box check, local feasibility P:127, T < t_free for Require P:259) and, when
// `flags` is given, the instance flags (users differ from user 0 in (R, zeta, f_max) -> kNotHomog, in
// (f_min, kappa, p_u) -> kNotUni, in T -> kNotSameT) are combined by ONE warp OR-reduction; the
// statuses are then decided in the oracle's precedence order.
constexpr unsigned kVBad = 1u, kVInfeas = 2u, kVRequire = 4u, kNotHomog = 8u, kNotUni = 16u, kNotSameT = 32u;

// tmode (K1's kernel split by deadlines): 1 = return kStDefer when the users' deadlines differ, 2 = when
// they are all equal, 3 = always; tested right after the loads, before the other checks (the next
// kernel decides).
__device__ __forceinline__ int warp_validate_pre(const DevModel *models, const DevBatch &b, long long i, int lane,
                                                 long long off, long long M64, int mid, InstRegs &x, int &M,
                                                 long long &k, const DevModel *&mdp, GridKCache *kc = nullptr,
                                                 unsigned *flags = nullptr, int tmode = 0) {
    M = (M64 >= 1 && M64 <= kMaxM) ? (int)M64 : 0;
    k = 0;
    x.z = x.k = x.f0 = x.f1 = x.R = x.p = 0.0;
    x.T = dinf();
    // the instance scalars are loaded with the users' values, so that both latencies overlap
    x.t_free = b.t_free[i];
    x.fe_min = b.fe_min[i];
    x.fe_max = b.fe_max[i];
    x.rho = b.rho[i];
#ifndef JDOB_LATE_USERS
    if (lane < M) {  // users of an instance rejected below are loaded but not used
        const long long u = off + lane;
        x.z = b.zeta[u];
        x.k = b.kappa[u];
        x.f0 = b.f_min[u];
        x.f1 = b.f_max[u];
        x.R = b.R[u];
        x.p = b.p_u[u];
        x.T = b.T[u];
    }
#endif
    if (mid < 0 || mid >= b.n_models) {
        mdp = nullptr;
        return JDOB_ST_BADPARAM;
    }
    mdp = &models[mid];
    if (*mdp->valid == 0) return JDOB_ST_BADMODEL;
    if (M64 < 1 || M64 > kMaxMLarge || M64 > mdp->B1 - 1) return JDOB_ST_BADPARAM;
    if (M64 > kMaxM) return kStDefer;  // more users than lanes: the block-per-instance path
    if (tmode == 3) return kStDefer;  // (every instance to the next kernel)
    if (tmode) {
        const double T0 = __shfl_sync(0xffffffffu, x.T, 0);
        const bool differ = __any_sync(0xffffffffu, lane < M && !(x.T == T0));
        if (differ == (tmode == 1)) return kStDefer;
    }
    bool ok = true;
    unsigned bits = 0u;
    if (lane < M) {
#ifdef JDOB_LATE_USERS
        const long long u = off + lane;
        x.z = b.zeta[u];
        x.k = b.kappa[u];
        x.f0 = b.f_min[u];
        x.f1 = b.f_max[u];
        x.R = b.R[u];
        x.p = b.p_u[u];
        x.T = b.T[u];
#endif
        ok = dfinite(x.z) && dfinite(x.k) && dfinite(x.f0) && dfinite(x.f1) && dfinite(x.R) && dfinite(x.p) &&
             dfinite(x.T);
        ok = ok && (x.z >= 0.0) && (x.k >= 0.0) && (x.f0 > 0.0) && (x.f0 <= x.f1) && (x.R > 0.0) &&
             (x.p >= 0.0) && (x.T > 0.0);
        bits |= ok ? 0u : kVBad;
    }
    const double vN = mdp->v[mdp->N];
    if (lane < M) {
        // P:127 literally RN(zeta v_N / f_max) > T; when T f_max - zeta v_N > 0 exactly (the fma's sign)
        // the quotient is < T, so RN(.) <= T and the test fails without the division
        const double zvN = x.z * vN;
        if (!(__fma_rn(x.T, x.f1, -zvN) > 0.0) && (zvN / x.f1 > x.T)) bits |= kVInfeas;
        if (x.T < x.t_free) bits |= kVRequire;  // min_m T_m < t_free <=> some T_m < t_free
    }
    if (flags) {
        auto sb = [](double a, double c) { return __double_as_longlong(a) == __double_as_longlong(c); };
        const double R0 = __shfl_sync(0xffffffffu, x.R, 0), z0 = __shfl_sync(0xffffffffu, x.z, 0),
                     f10 = __shfl_sync(0xffffffffu, x.f1, 0), f00 = __shfl_sync(0xffffffffu, x.f0, 0),
                     k0 = __shfl_sync(0xffffffffu, x.k, 0), p0 = __shfl_sync(0xffffffffu, x.p, 0),
                     T0 = __shfl_sync(0xffffffffu, x.T, 0);
        if (lane < M) {
            if (!(sb(x.R, R0) && sb(x.z, z0) && sb(x.f1, f10))) bits |= kNotHomog;
            if (!(sb(x.f0, f00) && sb(x.k, k0) && sb(x.p, p0))) bits |= kNotUni;
            if (!(x.T == T0)) bits |= kNotSameT;
        }
    }
    bits = __reduce_or_sync(0xffffffffu, bits);
    if (flags) *flags = bits;
    if (bits & kVBad) return JDOB_ST_BADPARAM;
    const double t_free = x.t_free, fe_min = x.fe_min, fe_max = x.fe_max, rho = x.rho;
    if (!(dfinite(t_free) && dfinite(fe_min) && dfinite(fe_max) && dfinite(rho) && (t_free >= 0.0) &&
          (fe_min > 0.0) && (fe_min <= fe_max) && (rho > 0.0)))
        return JDOB_ST_BADPARAM;
    if (kc) {  // warp-uniform: every lane reads the cache before lane 0 may rewrite it
        const bool hit = __all_sync(0xffffffffu, kc->fe_min == fe_min && kc->fe_max == fe_max && kc->rho == rho);
        if (hit) {
            k = kc->k;
        } else {
            __syncwarp();
            k = grid_k(fe_min, fe_max, rho);
            if (lane == 0) *kc = GridKCache{fe_min, fe_max, rho, k};
        }
    } else {
        k = grid_k(fe_min, fe_max, rho);
    }
    if (k > kMaxK) return JDOB_ST_BADPARAM;
    if (bits & kVInfeas) return JDOB_ST_LOCAL_INFEASIBLE;
    if (bits & kVRequire) return JDOB_ST_REQUIRE;
    return JDOB_ST_OK;
}

__device__ __forceinline__ int warp_validate(const DevModel *models, const DevBatch &b, long long i, int lane,
                                             InstRegs &x, int &M, long long &k, const DevModel *&mdp,
                                             long long &off) {
    off = b.user_off[i];
    const long long M64 = (b.user_end ? b.user_end[i] : b.user_off[i + 1]) - off;
    return warp_validate_pre(models, b, i, lane, off, M64, b.model_id[i], x, M, k, mdp);
}

__device__ __forceinline__ double shfl_d(double x, int src, unsigned mask = 0xffffffffu) {
    return __shfl_sync(mask, x, src);
}

}  // namespace jdob
