// K4: energy-saving statistics (row a12; "average energy consumption per user",
// P:407; reduction vs LC; R16), bucketed, with a FIXED reduction tree
// defined on the GLOBAL batch of n_total instances: leaf w of W = 1024 (one warp) owns the
// contiguous instance range [w n / W, (w+1) n / W); each lane accumulates its fixed
// subsequence of it into lane-private shared memory, the lanes are folded in lane order,
// and the leaves are folded by the dyadic (pairwise) tree over w.  Counts are exact
// integers.  A shard [r n / P, (r+1) n / P) of a power-of-two P is a subtree, so the
// per-rank roots folded pairwise over r (paper_2504_14611_b200.dist.fold_stats) give the
// same bits as one GPU over the whole batch.
#include "jdob_dev.cuh"
#include "kernels.h"

namespace jdob {

__device__ __forceinline__ bool is_max_field(int f) { return f == 3; }
__device__ __forceinline__ bool is_min_field(int f) { return f == 4; }

__device__ __forceinline__ double field_init(int f) {
    return is_max_field(f) ? -dinf() : (is_min_field(f) ? dinf() : 0.0);
}

__device__ __forceinline__ double combine(int f, double a, double b) {
    if (is_max_field(f)) return (b > a) ? b : a;
    if (is_min_field(f)) return (b < a) ? b : a;
    return a + b;
}

// Field slots kept per lane in floating point (the sums, whose bits depend on the order): sum r,
// sum r^2, sum E/M, sum E_lc/M.  max r and min r are exact in any order: integer atomics on the bits of
// the non-negative r (E <= E_LC), NaN (a zero-energy instance's 0/0) never taking part, as in the
// comparison form.
constexpr int kLaneF = 4;
__device__ __forceinline__ int lane_slot(int f) {  // field -> per-lane slot, -1 = not a lane slot
    return (f == 1) ? 0 : (f == 2) ? 1 : (f == 5) ? 2 : (f == 6) ? 3 : -1;
}

// One warp per block.  Lane l of warp w owns the instances i0 + l, i0 + l + 32, ... of the warp's fixed
// range and accumulates them IN THAT ORDER into its own shared-memory slots (no shuffles, no atomics on
// floating point); integer counters use shared-memory integer atomics (exact, order-free).  The lanes
// are then folded in lane order, so the result is identical run to run.
// One pass accumulates the buckets [b_lo, b_lo + n_buckets) of n_all (at most kBucketGroup, the shared
// memory of one warp); more buckets take one pass per group over the same instances.
#ifndef JDOB_STATS_GROUP
#define JDOB_STATS_GROUP 16
#endif
constexpr int kBucketGroup = JDOB_STATS_GROUP;

__global__ void __launch_bounds__(32) k_stats_partial(DevBatch b, DevResult r, double *partials, double *stats,
                                                      int n_buckets, long long n_total, long long begin, long long w0,
                                                      int b_lo, int n_all) {
    // leaf w of the global tree = instances [n_total w / W, n_total (w + 1) / W); this block is w0 + blockIdx.x
    extern __shared__ double sh[];
    double *fs = sh;                                                        // [n_buckets][kLaneF][32]
    unsigned long long *mxb = (unsigned long long *)(sh + (size_t)n_buckets * kLaneF * 32);  // [n_buckets]
    unsigned long long *mnb = mxb + n_buckets;                              // [n_buckets]
    int *cnt = (int *)(mnb + n_buckets);                                    // [n_buckets][kStatsF]
    const int lane = threadIdx.x;
    for (int x = lane; x < n_buckets * kLaneF * 32; x += 32) fs[x] = 0.0;
    for (int x = lane; x < n_buckets; x += 32) {
        mxb[x] = 0ull;                    // +0; cnt field 3 says whether any r was seen
        mnb[x] = 0x7ff0000000000000ull;   // +inf
    }
    for (int x = lane; x < n_buckets * kStatsF; x += 32) cnt[x] = 0;
    __syncwarp();
    const long long W = kStatsBlocks;
    const long long gw = w0 + blockIdx.x;  // global leaf
    const long long i0 = n_total * gw / W - begin, i1 = n_total * (gw + 1) / W - begin;
    // the lane's instances i0 + lane, + 32, ... in that order, four per step: the loads of the four are
    // issued together (latency overlap), the accumulation keeps the order (same bits)
    constexpr int U = 4;
    for (long long i = i0 + lane; i < i1; i += 32 * U) {
        int Mq[U], bq[U], sq[U], nq[U];
        double Eq[U], Lq[U], Fq[U];
#pragma unroll
        for (int q = 0; q < U; q++) {
            const long long ii = i + 32 * q;
            sq[q] = JDOB_ST_BADPARAM;
            bq[q] = -1;
            if (ii < i1) {
                Mq[q] = (int)(b.user_off[ii + 1] - b.user_off[ii]);
                // default bucket M - 1; instances with M > n_all are not counted; local index in the group
                const int bg = b.bucket ? b.bucket[ii] : ((Mq[q] >= 1 && Mq[q] <= n_all) ? Mq[q] - 1 : -1);
                bq[q] = (bg >= 0 && bg < n_all) ? bg - b_lo : -1;
                sq[q] = r.status[ii];
                Eq[q] = r.E[ii];
                Lq[q] = r.E_lc[ii];
                Fq[q] = r.f_e[ii];
                nq[q] = r.n_tilde[ii];
            }
        }
#pragma unroll
        for (int q = 0; q < U; q++) {
            const int bk = bq[q];
            if (bk < 0 || bk >= n_buckets) continue;  // also: beyond the range
            JDOB_CHECK(bk < kBucketGroup);
            int *c = cnt + bk * kStatsF;
            if (sq[q] != JDOB_ST_OK) {
                atomicAdd(c + 8, 1);
                continue;
            }
            const double E = Eq[q], El = Lq[q];
            const int M = Mq[q];
            const double rr = div_z0(100.0 * (El - E), El);  // E = E_LC: 0 without the slow path
            double *a = fs + (size_t)bk * kLaneF * 32 + lane;
            a[0 * 32] = a[0 * 32] + rr;
            a[1 * 32] = a[1 * 32] + rr * rr;
            a[2 * 32] = a[2 * 32] + E / (double)M;
            a[3 * 32] = a[3 * 32] + El / (double)M;
            if (rr == rr) {  // not NaN
                const unsigned long long rb = (unsigned long long)__double_as_longlong(rr);
                atomicMax(mxb + bk, rb);
                atomicMin(mnb + bk, rb);
                c[3] = 1;  // some r seen (a benign same-value race)
            }
            atomicAdd(c + 0, 1);
            if (Fq[q] > 0.0) atomicAdd(c + 7, 1);  // the plan offloads (f_e* = 0 only when all-local, R18)
            const int nt = nq[q];
            if (nt >= 0 && nt < 64) atomicAdd(c + 9 + nt, 1);
        }
    }
    __syncwarp();
    // the exact fields go straight to the output: counts by integer-valued double atomics (exact in any
    // order below 2^53), max r / min r by integer atomics on their bits (max stored as bits + 1, 0 = none,
    // decoded by k_stats_max_decode); only the four floating-point sums go through the fixed tree
    double *out = stats + (size_t)b_lo * kStatsF;
    for (int x = lane; x < n_buckets * kStatsF; x += 32) {
        const int f = x % kStatsF, bk = x / kStatsF;
        if (f == 3) {
            if (cnt[bk * kStatsF + 3]) atomicMax((unsigned long long *)(out + x), mxb[bk] + 1ull);
        } else if (f == 4) {
            if (mnb[bk] != 0x7ff0000000000000ull) atomicMin((unsigned long long *)(out + x), mnb[bk]);
        } else if ((f == 0 || f == 7 || f == 8 || (f >= 9 && f < 9 + 64)) && cnt[x] != 0) {
            atomicAdd(out + x, (double)cnt[x]);
        }
    }
    double *dst = partials + (size_t)blockIdx.x * n_buckets * kLaneF;
    for (int x = lane; x < n_buckets * kLaneF; x += 32) {
        const int slot = x % kLaneF, bk = x / kLaneF;
        const int f = (slot == 0) ? 1 : (slot == 1) ? 2 : (slot == 2) ? 5 : 6;
        const double *q = fs + ((size_t)bk * kLaneF + slot) * 32;
        double v = field_init(f);
        for (int l = 0; l < 32; l++) v = combine(f, v, q[l]);
        dst[x] = v;
    }
}

// The output's initial values (every field of every bucket): 0 for the sums and counts, the max slot's
// "none" code 0, +inf for the min.
__global__ void k_stats_init(double *stats, int n) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    if (x < n) stats[x] = (x % kStatsF == 4) ? dinf() : 0.0;
}

// max r: the atomics' code (bits + 1, 0 = no r seen) back to the double (-inf when none, field_init)
__global__ void k_stats_max_decode(double *stats, int n_buckets) {
    const int bk = blockIdx.x * blockDim.x + threadIdx.x;
    if (bk >= n_buckets) return;
    const unsigned long long u = (unsigned long long)__double_as_longlong(stats[(size_t)bk * kStatsF + 3]);
    stats[(size_t)bk * kStatsF + 3] = u ? __longlong_as_double((long long)(u - 1ull)) : -dinf();
}

// One warp per output element: the dyadic tree over the nl (a power of two) leaves.  Lane l folds
// its consecutive block of s = max(nl / 32, 1) leaves pairwise (a binary-counter stack: the same tree),
// then an xor butterfly with d = 1, 2, 4, ... combines neighbouring blocks -- combine() is commutative
// bit for bit, so lane l and lane l ^ d hold the same subtree value at every level.
__global__ void k_stats_final(const double *partials, int nl, int n_buckets, double *stats) {
    const int lane = threadIdx.x & 31;
    const int x = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;  // (bucket, floating-point slot)
    if (x >= n_buckets * kLaneF) return;
    const int slot = x % kLaneF, bk = x / kLaneF;
    const int f = (slot == 0) ? 1 : (slot == 1) ? 2 : (slot == 2) ? 5 : 6;
    const int s = nl >= 32 ? nl / 32 : 1;
    double stack[11];
    double v = field_init(f);
    if (lane < nl) {
        for (int i = 0; i < s; i++) {
            double y = partials[(size_t)(lane * s + i) * n_buckets * kLaneF + x];
            int lev = 0;
            for (; (i >> lev) & 1; lev++) y = combine(f, stack[lev], y);
            stack[lev] = y;
        }
        v = stack[__ffs(s) - 1];  // s is a power of two: the root of the lane's block
    }
    const int lanes = nl >= 32 ? 32 : nl;
    for (int d = 1; d < lanes; d <<= 1) v = combine(f, v, __shfl_xor_sync(0xffffffffu, v, d));
    if (lane == 0) stats[(size_t)bk * kStatsF + f] = v;
}

bool launch_stats(const DevBatch &b, const DevResult &r, double *partials, double *stats, int n_buckets,
                  long long n_total, int parts, int part, cudaStream_t s) {
    const long long W = kStatsBlocks;
    if (parts < 1 || parts > W || (parts & (parts - 1)) || part < 0 || part >= parts || n_total < 0) return false;
    const long long begin = n_total * part / parts, end = n_total * (part + 1) / parts;
    if (b.n_inst != end - begin) return false;
    const long long nl = W / parts, w0 = nl * part;  // leaf w0 starts at n_total w0 / W = begin
    cudaFuncSetAttribute(k_stats_partial, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)((size_t)kBucketGroup * (kLaneF * 32 * sizeof(double) + 2 * sizeof(long long) +
                                                       kStatsF * sizeof(int))));
    const int n_out = n_buckets * kStatsF;
    k_stats_init<<<(n_out + 255) / 256, 256, 0, s>>>(stats, n_out);
    for (int b_lo = 0; b_lo < n_buckets; b_lo += kBucketGroup) {  // partials reused group after group
        const int nb = (n_buckets - b_lo < kBucketGroup) ? n_buckets - b_lo : kBucketGroup;
        const size_t smem = (size_t)nb * kLaneF * 32 * sizeof(double) + 2 * (size_t)nb * sizeof(long long) +
                            (size_t)nb * kStatsF * sizeof(int);
        k_stats_partial<<<(unsigned)nl, 32, smem, s>>>(b, r, partials, stats, nb, n_total, begin, w0, b_lo,
                                                       n_buckets);
        const int warps = nb * kLaneF;
        k_stats_final<<<(warps * 32 + 255) / 256, 256, 0, s>>>(partials, (int)nl, nb, stats + (size_t)b_lo * kStatsF);
    }
    k_stats_max_decode<<<(n_buckets + 255) / 256, 256, 0, s>>>(stats, n_buckets);
    return true;
}

}  // namespace jdob
