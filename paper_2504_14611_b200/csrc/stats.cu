// K4: energy-saving statistics (row a12; "average energy consumption per user",
// P:407; reduction vs LC; R16), bucketed, with a FIXED reduction tree:
// warp w of the fixed grid owns the contiguous instance range [w n / W, (w+1) n / W),
// accumulates it sequentially into warp-private shared memory (lane f owns fields
// f, f+32, f+64 -> no atomics), warps of a block are combined in warp order, and a
// final one-block kernel folds the per-block partials in block order.  Results are
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

__global__ void __launch_bounds__(kStatsWarps * 32) k_stats_partial(DevBatch b, DevResult r, double *partials,
                                                                      int n_buckets) {
    extern __shared__ double acc[];  // [kStatsWarps][n_buckets][kStatsF]
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    double *my = acc + (size_t)w * n_buckets * kStatsF;
    for (int x = lane; x < n_buckets * kStatsF; x += 32) my[x] = field_init(x % kStatsF);
    __syncwarp();
    const long long W = (long long)gridDim.x * kStatsWarps;
    const long long gw = (long long)blockIdx.x * kStatsWarps + w;
    const long long i0 = b.n_inst * gw / W, i1 = b.n_inst * (gw + 1) / W;
    for (long long base = i0; base < i1; base += 32) {
        const long long i = base + lane;
        bool valid = i < i1;
        int bk = -1, ok = 0, nt = 0, offl = 0;
        double rr = 0.0, eM = 0.0, elM = 0.0;
        if (valid) {
            const int M = (int)(b.user_off[i + 1] - b.user_off[i]);
            bk = b.bucket ? b.bucket[i] : ((M >= 1 && M <= kMaxM) ? M - 1 : 0);
            if (bk < 0 || bk >= n_buckets) bk = -1;
            ok = (r.status[i] == JDOB_ST_OK);
            if (ok) {
                const double E = r.E[i], El = r.E_lc[i];
                rr = 100.0 * (El - E) / El;
                eM = E / (double)M;
                elM = El / (double)M;
                nt = r.n_tilde[i];
                offl = r.mask[i] != 0u;
            }
        }
        const int cnt = (int)((i1 - base) < 32 ? (i1 - base) : 32);
        for (int t = 0; t < cnt; t++) {
            const int tb = __shfl_sync(0xffffffffu, bk, t);
            const int tok = __shfl_sync(0xffffffffu, ok, t);
            const double tr = __shfl_sync(0xffffffffu, rr, t);
            const double te = __shfl_sync(0xffffffffu, eM, t);
            const double tl = __shfl_sync(0xffffffffu, elM, t);
            const int tn = __shfl_sync(0xffffffffu, nt, t);
            const int to = __shfl_sync(0xffffffffu, offl, t);
            if (tb < 0) continue;
            double *a = my + (size_t)tb * kStatsF;
            if (!tok) {
                if (lane == 8) a[8] = a[8] + 1.0;
                continue;
            }
#pragma unroll
            for (int q = 0; q < 3; q++) {
                const int f = lane + 32 * q;
                if (f >= kStatsF) break;
                double v;
                switch (f) {
                    case 0: v = 1.0; break;
                    case 1: v = tr; break;
                    case 2: v = tr * tr; break;
                    case 3: v = tr; break;
                    case 4: v = tr; break;
                    case 5: v = te; break;
                    case 6: v = tl; break;
                    case 7: v = to ? 1.0 : 0.0; break;
                    case 8: v = 0.0; break;
                    default: v = (f - 9 == tn) ? 1.0 : 0.0; break;
                }
                if (f == 8 || (f >= 9 + 64)) continue;
                a[f] = combine(f, a[f], v);
            }
        }
    }
    __syncthreads();
    // combine warps in order, write this block's partial
    double *dst = partials + (size_t)blockIdx.x * n_buckets * kStatsF;
    for (int x = threadIdx.x; x < n_buckets * kStatsF; x += blockDim.x) {
        const int f = x % kStatsF;
        double v = acc[x];
        for (int ww = 1; ww < kStatsWarps; ww++) v = combine(f, v, acc[(size_t)ww * n_buckets * kStatsF + x]);
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
    for (int blk = lane; blk < n_blocks; blk += 32) v = combine(f, v, partials[(size_t)blk * n_buckets * kStatsF + x]);
#pragma unroll
    for (int d = 16; d >= 1; d >>= 1) v = combine(f, v, __shfl_xor_sync(0xffffffffu, v, d));
    if (lane == 0) stats[x] = v;
}

void launch_stats(const DevBatch &b, const DevResult &r, double *partials, double *stats, int n_buckets,
                  cudaStream_t s) {
    size_t smem = (size_t)kStatsWarps * n_buckets * kStatsF * sizeof(double);
    cudaFuncSetAttribute(k_stats_partial, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         kStatsWarps * JDOB_MAX_BUCKETS * kStatsF * (int)sizeof(double));
    k_stats_partial<<<kStatsBlocks, kStatsWarps * 32, smem, s>>>(b, r, partials, n_buckets);
    const int warps = n_buckets * kStatsF;
    k_stats_final<<<(warps * 32 + 255) / 256, 256, 0, s>>>(partials, kStatsBlocks, n_buckets, stats);
}

}  // namespace jdob
