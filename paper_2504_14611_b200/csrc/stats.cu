// K4: energy-saving statistics (row a12; "average energy consumption per user",
// P:407; reduction vs LC; R16), bucketed, with a FIXED reduction tree:
// block w of the fixed grid (one warp) owns the contiguous instance range
// [w n / W, (w+1) n / W); each lane accumulates its fixed subsequence of it into
// lane-private shared memory, the lanes are folded in lane order, and a final kernel
// folds the per-block partials in a fixed tree.  Counts are exact integers.  Results are
// therefore identical run to run for a given n_inst.
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

// Field slots kept per lane in floating point: sum r, sum r^2, max r, min r, sum E/M, sum E_lc/M.
constexpr int kLaneF = 6;
__device__ __forceinline__ int lane_slot(int f) {  // field -> per-lane slot, -1 = integer counter
    return (f == 1) ? 0 : (f == 2) ? 1 : (f == 3) ? 2 : (f == 4) ? 3 : (f == 5) ? 4 : (f == 6) ? 5 : -1;
}

// One warp per block.  Lane l of warp w owns the instances i0 + l, i0 + l + 32, ... of the warp's fixed
// range and accumulates them IN THAT ORDER into its own shared-memory slots (no shuffles, no atomics on
// floating point); integer counters use shared-memory integer atomics (exact, order-free).  The lanes
// are then folded in lane order, so the result is identical run to run.
__global__ void __launch_bounds__(32) k_stats_partial(DevBatch b, DevResult r, double *partials, int n_buckets) {
    extern __shared__ double sh[];
    double *fs = sh;                                                        // [n_buckets][kLaneF][32]
    int *cnt = (int *)(sh + (size_t)n_buckets * kLaneF * 32);               // [n_buckets][kStatsF]
    const int lane = threadIdx.x;
    for (int x = lane; x < n_buckets * kLaneF * 32; x += 32) {
        const int slot = (x / 32) % kLaneF;
        fs[x] = (slot == 2) ? -dinf() : (slot == 3) ? dinf() : 0.0;
    }
    for (int x = lane; x < n_buckets * kStatsF; x += 32) cnt[x] = 0;
    __syncwarp();
    const long long W = gridDim.x;
    const long long gw = blockIdx.x;
    const long long i0 = b.n_inst * gw / W, i1 = b.n_inst * (gw + 1) / W;
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
                // default bucket M - 1; instances with M > n_buckets are not counted
                bq[q] = b.bucket ? b.bucket[ii] : ((Mq[q] >= 1 && Mq[q] <= n_buckets) ? Mq[q] - 1 : -1);
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
            a[2 * 32] = (rr > a[2 * 32]) ? rr : a[2 * 32];
            a[3 * 32] = (rr < a[3 * 32]) ? rr : a[3 * 32];
            a[4 * 32] = a[4 * 32] + E / (double)M;
            a[5 * 32] = a[5 * 32] + El / (double)M;
            atomicAdd(c + 0, 1);
            if (Fq[q] > 0.0) atomicAdd(c + 7, 1);  // the plan offloads (f_e* = 0 only when all-local, R18)
            const int nt = nq[q];
            if (nt >= 0 && nt < 64) atomicAdd(c + 9 + nt, 1);
        }
    }
    __syncwarp();
    double *dst = partials + (size_t)blockIdx.x * n_buckets * kStatsF;
    for (int x = lane; x < n_buckets * kStatsF; x += 32) {
        const int f = x % kStatsF, bk = x / kStatsF;
        const int slot = lane_slot(f);
        double v;
        if (slot < 0) {
            v = (f == 0 || f == 7 || f == 8 || (f >= 9 && f < 9 + 64)) ? (double)cnt[x] : field_init(f);
        } else {
            const double *q = fs + ((size_t)bk * kLaneF + slot) * 32;
            v = field_init(f);
            for (int l = 0; l < 32; l++) v = combine(f, v, q[l]);
        }
        dst[x] = v;
    }
}

// one warp per output element: lane l folds partials l, l+32, ... in order, then a fixed
// xor-butterfly combines the lanes -- a fixed tree, so the result is run-to-run identical
__global__ void k_stats_final(const double *partials, int n_blocks, int n_buckets, double *stats) {
    const int lane = threadIdx.x & 31;
    const int x = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (x >= n_buckets * kStatsF) return;
    const int f = x % kStatsF;
    double v = field_init(f);
#pragma unroll 8
    for (int blk = lane; blk < n_blocks; blk += 32) v = combine(f, v, partials[(size_t)blk * n_buckets * kStatsF + x]);
#pragma unroll
    for (int d = 16; d >= 1; d >>= 1) v = combine(f, v, __shfl_xor_sync(0xffffffffu, v, d));
    if (lane == 0) stats[x] = v;
}

void launch_stats(const DevBatch &b, const DevResult &r, double *partials, double *stats, int n_buckets,
                  cudaStream_t s) {
    const size_t smem = (size_t)n_buckets * kLaneF * 32 * sizeof(double) + (size_t)n_buckets * kStatsF * sizeof(int);
    cudaFuncSetAttribute(k_stats_partial, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)((size_t)JDOB_MAX_BUCKETS * (kLaneF * 32 * sizeof(double) + kStatsF * sizeof(int))));
    k_stats_partial<<<kStatsBlocks, 32, smem, s>>>(b, r, partials, n_buckets);
    const int warps = n_buckets * kStatsF;
    k_stats_final<<<(warps * 32 + 255) / 256, 256, 0, s>>>(partials, kStatsBlocks, n_buckets, stats);
}

}  // namespace jdob
