// K6: the seeded C5 Monte Carlo workload generated on the device (SURVEY §8(d) C5 "generated
// in-kernel", §8(e) "each rank generates its own instances ... no input traffic").
//
// INPUT PLUMBING, not the method: this file draws random numbers and writes input arrays; it holds
// none of J-DOB's arithmetic.  It is the device twin of jdobgen.config_c5 (DESIGN.md §5 Input
// recipe): the same counter-based SplitMix64 draws keyed by (seed, instance id,
// user, field), the same integer choice and uniform formulas in the same operation order, so every
// array is bit-identical to the host generator's (tests/test_gpu_gen.py, T9).  The host passes the
// recipe's constants (Table I users, per-model minimum local latency, the rho choices) so both sides
// use the same doubles.
#include "jdob_dev.cuh"
#include "kernels.h"

namespace jdob {

// jdobgen field ids
constexpr unsigned kFM = 0, kFModel = 1, kFRegime = 2, kFRho = 3, kFBetaUser = 4, kFRHet = 6, kFKHet = 7;

__device__ __forceinline__ unsigned long long mix64(unsigned long long x) {
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}
__device__ __forceinline__ unsigned long long draw(unsigned long long seed, unsigned long long inst,
                                                   unsigned long long user, unsigned long long fld) {
    return mix64(mix64(mix64(seed) ^ inst) ^ ((user << 8) | fld));
}
__device__ __forceinline__ double u01(unsigned long long d) { return __dmul_rn((double)(d >> 11), 0x1p-53); }
__device__ __forceinline__ double uniform(unsigned long long d, double lo, double hi) {
    return __dadd_rn(lo, __dmul_rn(__dsub_rn(hi, lo), u01(d)));
}
__device__ __forceinline__ long long choice(unsigned long long d, long long a, long long b) {
    return a + (long long)(((d >> 32) * (unsigned long long)(b - a + 1)) >> 32);
}

// per instance: M, model, regime, rho; model_id, bucket and the instance scalars are written, M is
// kept in user_off[i + 1] until the scan turns the counts into offsets
__global__ void k_gen_inst(GenParams p, long long n, int *model_id, long long *user_off, double *t_free,
                           double *fe_min, double *fe_max, double *rho, int *bucket, int *regime) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const unsigned long long id = (unsigned long long)(p.inst_begin + i);
    const long long M = choice(draw(p.seed, id, 0, kFM), 1, 32);
    const int mid = (int)choice(draw(p.seed, id, 0, kFModel), 0, 2);
    const int reg = (int)choice(draw(p.seed, id, 0, kFRegime), 0, 4);
    const int rc = (int)choice(draw(p.seed, id, 0, kFRho), 0, 2);
    model_id[i] = mid;
    user_off[i + 1] = M;
    if (i == 0) user_off[0] = 0;
    t_free[i] = 0.0;
    fe_min[i] = p.fe_min;
    fe_max[i] = p.fe_max;
    rho[i] = p.rho[rc];
    bucket[i] = (mid * 5 + reg) * 32 + (int)(M - 1);  // (model, regime, M): 480 buckets
    regime[i] = reg;
}

// inclusive scan of user_off[1..n] in place (counts -> offsets): block sums, a one-block scan of
// them, then the block-local scans with their offsets
constexpr int kScanBlock = 1024;
__global__ void k_gen_scan_blocks(long long *user_off, long long n, long long *bsum) {
    __shared__ long long s[kScanBlock];
    const long long i = (long long)blockIdx.x * kScanBlock + threadIdx.x;
    s[threadIdx.x] = (i < n) ? user_off[i + 1] : 0;
    __syncthreads();
    for (int d = kScanBlock / 2; d >= 1; d >>= 1) {
        if (threadIdx.x < d) s[threadIdx.x] += s[threadIdx.x + d];
        __syncthreads();
    }
    if (threadIdx.x == 0) bsum[blockIdx.x] = s[0];
}
__global__ void k_gen_scan_sums(long long *bsum, long long nb) {  // one thread: exclusive scan
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    long long acc = 0;
    for (long long b = 0; b < nb; b++) {
        const long long v = bsum[b];
        bsum[b] = acc;
        acc += v;
    }
    bsum[nb] = acc;
}
__global__ void k_gen_scan_final(long long *user_off, long long n, const long long *bsum) {
    __shared__ long long s[kScanBlock];
    const long long i = (long long)blockIdx.x * kScanBlock + threadIdx.x;
    s[threadIdx.x] = (i < n) ? user_off[i + 1] : 0;
    __syncthreads();
    for (int d = 1; d < kScanBlock; d <<= 1) {  // Hillis-Steele inclusive scan (integers: exact)
        const long long v = (threadIdx.x >= d) ? s[threadIdx.x - d] : 0;
        __syncthreads();
        s[threadIdx.x] += v;
        __syncthreads();
    }
    if (i < n) user_off[i + 1] = bsum[blockIdx.x] + s[threadIdx.x];
}

// per user (one warp per instance, lane = user): deadlines from the regime's beta, Table I users
__global__ void k_gen_users(GenParams p, long long n, const int *model_id, const long long *user_off,
                            const int *regime, double *zeta, double *kappa, double *f_min, double *f_max, double *R,
                            double *p_u, double *T) {
    const int lane = threadIdx.x & 31;
    const long long i = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (i >= n) return;
    const long long o = user_off[i], M = user_off[i + 1] - o;
    if (lane >= M) return;
    const unsigned long long id = (unsigned long long)(p.inst_begin + i);
    const int reg = regime[i], mid = model_id[i];
    const double lo = (reg == 0) ? 2.13 : (reg == 1) ? 30.25 : (reg == 2) ? 4.5 : (reg == 3) ? 2.0 : 0.0;
    const double hi = (reg == 0) ? 2.13 : (reg == 1) ? 30.25 : (reg == 2) ? 5.5 : (reg == 3) ? 8.0 : 10.0;
    const double beta = (reg < 2) ? lo : uniform(draw(p.seed, id, (unsigned long long)lane, kFBetaUser), lo, hi);
    const long long u = o + lane;
    zeta[u] = p.zeta;
    double kap = p.kappa, r = p.R;
    if (p.hetero) {
        r = __dmul_rn(r, uniform(draw(p.seed, id, (unsigned long long)lane, kFRHet), 0.5, 2.0));
        kap = __dmul_rn(kap, uniform(draw(p.seed, id, (unsigned long long)lane, kFKHet), 0.5, 2.0));
    }
    kappa[u] = kap;
    f_min[u] = p.f_min;
    f_max[u] = p.f_max;
    R[u] = r;
    p_u[u] = p.p_u;
    T[u] = __dmul_rn(__dadd_rn(1.0, beta), p.lat[mid]);  // T = (1 + beta) * zeta v_N / f_max
}

size_t gen_workspace_bytes(long long n) {
    return (size_t)((n + kScanBlock - 1) / kScanBlock + 2) * sizeof(long long) + (size_t)n * sizeof(int) + 512;
}

void launch_gen_inst(const GenParams &p, long long n, int *model_id, long long *user_off, double *t_free,
                     double *fe_min, double *fe_max, double *rho, int *bucket, void *ws, cudaStream_t s) {
    if (n <= 0) return;
    long long *bsum = (long long *)ws;
    const long long nb = (n + kScanBlock - 1) / kScanBlock;
    int *regime = (int *)((char *)ws + ((nb + 2) * sizeof(long long) + 255) / 256 * 256);
    k_gen_inst<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(p, n, model_id, user_off, t_free, fe_min, fe_max, rho,
                                                           bucket, regime);
    k_gen_scan_blocks<<<(unsigned)nb, kScanBlock, 0, s>>>(user_off, n, bsum);
    k_gen_scan_sums<<<1, 32, 0, s>>>(bsum, nb);
    k_gen_scan_final<<<(unsigned)nb, kScanBlock, 0, s>>>(user_off, n, bsum);
}

void launch_gen_users(const GenParams &p, long long n, const int *model_id, const long long *user_off, double *zeta,
                      double *kappa, double *f_min, double *f_max, double *R, double *p_u, double *T, void *ws,
                      cudaStream_t s) {
    if (n <= 0) return;
    const long long nb = (n + kScanBlock - 1) / kScanBlock;
    const int *regime = (const int *)((char *)ws + ((nb + 2) * sizeof(long long) + 255) / 256 * 256);
    k_gen_users<<<(unsigned)((n * 32 + 255) / 256), 256, 0, s>>>(p, n, model_id, user_off, regime, zeta, kappa, f_min,
                                                                f_max, R, p_u, T);
}

}  // namespace jdob
