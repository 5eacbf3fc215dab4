// K5: outer grouping (reading R21).
//
// The paper wraps J-DOB in the optimal-grouping dynamic program of its reference
// [shi2022multiuser] for different deadlines without printing it;
// we follow SPEC S:295-303: users sorted by deadline (ties by index), cell i keeps the
// lexicographically best (energy, t_free) of the first i sorted users, transition
// j -> i is the group {j..i-1} solved by the inner J-DOB at t_free = cell j's t_free
// (strict improvement: ties keep the smallest j).
//
// GPU mapping: the users of every instance are first copied in deadline order, so a
// group is a contiguous slice [off + j, off + i) of the sorted arrays.  Stage i of the
// DP solves, for every instance at once, the i groups ending at i as one batch of
// overlapping views (DevBatch.user_end) through K1, then a per-instance update picks
// cell i.  After the last stage the chosen groups are re-solved as one batch and the
// schedule (group of each user, partition point, f*, per-group f_e) is written in the
// input's user order.
#include "jdob_dev.cuh"
#include "kernels.h"

namespace jdob {

// sort each instance's users by (T asc, index asc); copy them in that order
__global__ void k_og_prep(const DevModel *models, DevBatch b, OgWork w) {
    const int lane = threadIdx.x & 31;
    const long long i = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (i >= b.n_inst) return;
    long long off, k;
    int M;
    const DevModel *mdp;
    InstRegs x;
    int st = warp_validate(models, b, i, lane, x, M, k, mdp, off);
    if (st == kStDefer) st = JDOB_ST_BADPARAM;   // grouping takes M <= 32
    if (st == JDOB_ST_REQUIRE) st = JDOB_ST_OK;  // the DP costs a failed Require per group
    const long long M64 = b.user_off[i + 1] - off;
    if (st != JDOB_ST_OK) {
        // identity copy (the final pass then returns the solver's status answer in input order)
        for (long long q = lane; q < M64; q += 32) {
            const long long u = off + q;
            w.sz[u] = b.zeta[u];
            w.sk[u] = b.kappa[u];
            w.sf0[u] = b.f_min[u];
            w.sf1[u] = b.f_max[u];
            w.sR[u] = b.R[u];
            w.sp[u] = b.p_u[u];
            w.sT[u] = b.T[u];
            w.perm[u] = u;
        }
        if (lane == 0) w.status[i] = st;
        return;
    }
    int r = 0;
    for (int t = 0; t < M; t++) {
        const double Tt = __shfl_sync(0xffffffffu, x.T, t);
        r += (Tt < x.T || (Tt == x.T && t < lane)) ? 1 : 0;
    }
    if (lane < M) {
        const long long u = off + r;
        w.sz[u] = x.z;
        w.sk[u] = x.k;
        w.sf0[u] = x.f0;
        w.sf1[u] = x.f1;
        w.sR[u] = x.R;
        w.sp[u] = x.p;
        w.sT[u] = x.T;
        w.perm[u] = off + lane;
    }
    if (lane == 0) {
        w.status[i] = st;
        w.cE[i * kCells] = 0.0;
        w.cT[i * kCells] = b.t_free[i];
        w.from[i * kCells] = -1;
        atomicMax(w.mmax, M);
    }
}

// stage i: slot s = inst * i + j is the group {j..i-1} of instance inst
__global__ void k_og_build(DevBatch b, OgWork w, int stage) {
    const long long s = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= b.n_inst * stage) return;
    const long long inst = s / stage;
    const int j = (int)(s % stage);
    const long long off = b.user_off[inst];
    const long long M = b.user_off[inst + 1] - off;
    const bool active = w.status[inst] == JDOB_ST_OK && M >= stage;
    w.s_off[s] = off + (active ? j : 0);
    w.s_end[s] = active ? off + stage : off;  // empty view (M = 0) for inactive slots
    w.s_model[s] = b.model_id[inst];
    w.s_tfree[s] = active ? w.cT[inst * kCells + j] : 0.0;
    w.s_femin[s] = b.fe_min[inst];
    w.s_femax[s] = b.fe_max[inst];
    w.s_rho[s] = b.rho[inst];
}

__global__ void k_og_update(DevBatch b, OgWork w, int stage) {
    const long long inst = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (inst >= b.n_inst) return;
    const long long M = b.user_off[inst + 1] - b.user_off[inst];
    if (w.status[inst] != JDOB_ST_OK || M < stage) return;
    double bE = dinf(), bT = dinf();
    int bj = -1;
    for (int j = 0; j < stage; j++) {
        const long long s = inst * stage + j;
        const double E = w.cE[inst * kCells + j] + w.r_E[s];
        const double tf = w.r_tf[s];
        if (E < bE || (E == bE && tf < bT)) {
            bE = E;
            bT = tf;
            bj = j;
        }
    }
    w.cE[inst * kCells + stage] = bE;
    w.cT[inst * kCells + stage] = bT;
    w.from[inst * kCells + stage] = bj;
}

// final pass: the chosen groups of every instance (slot inst * 32 + g), or the whole
// instance (slot inst * 32) for a non-OK status
__global__ void k_og_final_build(DevBatch b, OgWork w) {
    const long long inst = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (inst >= b.n_inst) return;
    const long long off = b.user_off[inst];
    const long long M = b.user_off[inst + 1] - off;
    const long long s0 = inst * kMaxM;
    int ng = 0;
    int starts[kMaxM + 1];
    if (w.status[inst] == JDOB_ST_OK) {
        for (int i = (int)M; i > 0; i = w.from[inst * kCells + i]) starts[ng++] = w.from[inst * kCells + i];
    }
    for (int g = 0; g < kMaxM; g++) {
        const long long s = s0 + g;
        w.s_model[s] = b.model_id[inst];
        w.s_femin[s] = b.fe_min[inst];
        w.s_femax[s] = b.fe_max[inst];
        w.s_rho[s] = b.rho[inst];
        if (g < ng) {
            const int a = starts[ng - 1 - g];
            const int e = (g + 1 < ng) ? starts[ng - 2 - g] : (int)M;
            w.s_off[s] = off + a;
            w.s_end[s] = off + e;
            w.s_tfree[s] = w.cT[inst * kCells + a];
        } else if (g == 0) {  // non-OK status: the whole instance (identity order) reports it
            w.s_off[s] = off;
            w.s_end[s] = off + M;
            w.s_tfree[s] = b.t_free[inst];
        } else {
            w.s_off[s] = off;
            w.s_end[s] = off;
            w.s_tfree[s] = 0.0;
        }
    }
    w.ngroups[inst] = ng;
}

__global__ void k_og_final_write(const DevModel *models, DevBatch b, OgWork w, GroupedOut o) {
    const int lane = threadIdx.x & 31;
    const long long inst = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (inst >= b.n_inst) return;
    const long long off = b.user_off[inst];
    const long long M = b.user_off[inst + 1] - off;
    const int st = w.status[inst];
    const int ng = w.ngroups[inst];
    const long long s0 = inst * kMaxM;
    const int mid = b.model_id[inst];
    const int N = (mid >= 0 && mid < b.n_models) ? models[mid].N : 0;
    // M > 32 (K1 deferred it; grouping takes M <= 32): the final pass solved the whole instance in LC
    // mode on the block path; report BADPARAM with that LC answer unless the instance is malformed
    // or locally infeasible (the oracle's precedence)
    int st_out = (st == JDOB_ST_OK) ? JDOB_ST_OK : w.r_st[s0];
    if (st != JDOB_ST_OK && M > kMaxM && st_out != JDOB_ST_LOCAL_INFEASIBLE) st_out = JDOB_ST_BADPARAM;
    if (lane == 0) {
        o.status[inst] = st_out;
        o.n_groups[inst] = ng;
        o.E[inst] = (st == JDOB_ST_OK) ? w.cE[inst * kCells + M] : w.r_E[s0];
        o.t_free_next[inst] = (st == JDOB_ST_OK) ? w.cT[inst * kCells + M] : b.t_free[inst];
    }
    for (int g = lane; g < kMaxM; g += 32) o.group_fe[s0 + g] = (g < ng) ? w.r_fe[s0 + g] : 0.0;
    if (st != JDOB_ST_OK) {
        for (long long q = lane; q < M; q += 32) {
            o.group_of[off + q] = 0;
            o.partition[off + q] = N;
            if (o.f_user) o.f_user[off + q] = w.fs[off + q];
        }
        return;
    }
    for (int g = 0; g < ng; g++) {
        const long long a = w.s_off[s0 + g] - off, e = w.s_end[s0 + g] - off;
        const int nt = w.r_nt[s0 + g];
        const unsigned mask = w.r_mask[s0 + g];
        for (long long q = a + lane; q < e; q += 32) {
            const long long orig = w.perm[off + q];
            o.group_of[orig] = g;
            o.partition[orig] = ((mask >> (q - a)) & 1u) ? nt : N;
            if (o.f_user) o.f_user[orig] = w.fs[off + q];
        }
    }
}

static DevBatch stage_batch(const DevBatch &b, const OgWork &w, long long n_slots) {
    DevBatch sb = b;
    sb.n_inst = n_slots;
    sb.model_id = w.s_model;
    sb.user_off = w.s_off;
    sb.user_end = w.s_end;
    sb.zeta = w.sz;
    sb.kappa = w.sk;
    sb.f_min = w.sf0;
    sb.f_max = w.sf1;
    sb.R = w.sR;
    sb.p_u = w.sp;
    sb.T = w.sT;
    sb.t_free = w.s_tfree;
    sb.fe_min = w.s_femin;
    sb.fe_max = w.s_femax;
    sb.rho = w.s_rho;
    sb.bucket = nullptr;
    return sb;
}

static DevResult stage_result(const OgWork &w, double *f_user) {
    DevResult r;
    r.E = w.r_E;
    r.E_lc = w.r_Elc;
    r.t_free_next = w.r_tf;
    r.f_e = w.r_fe;
    r.n_tilde = w.r_nt;
    r.j = w.r_j;
    r.status = w.r_st;
    r.mask = w.r_mask;
    r.f_user = f_user;
    r.counts = nullptr;
    r.partition = nullptr;
    return r;
}

int launch_grouped(const DevModel *models, const DevBatch &b, int mode, const OgWork &w, const GroupedOut &o,
                   cudaStream_t s, int num_sms, bool wide) {
    const long long n = b.n_inst;
    if (n <= 0) return 0;
    cudaMemsetAsync(w.mmax, 0, sizeof(int), s);
    const int bs = 128;
    k_og_prep<<<(unsigned)((n * 32 + bs - 1) / bs), bs, 0, s>>>(models, b, w);
    int mmax = 0;
    cudaMemcpyAsync(&mmax, w.mmax, sizeof(int), cudaMemcpyDeviceToHost, s);
    if (cudaStreamSynchronize(s) != cudaSuccess) return 1;
    for (int stage = 1; stage <= mmax; stage++) {
        const long long slots = n * stage;
        k_og_build<<<(unsigned)((slots + bs - 1) / bs), bs, 0, s>>>(b, w, stage);
        launch_solve(models, stage_batch(b, w, slots), stage_result(w, nullptr), mode, s, num_sms);
        k_og_update<<<(unsigned)((n + bs - 1) / bs), bs, 0, s>>>(b, w, stage);
    }
    k_og_final_build<<<(unsigned)((n + bs - 1) / bs), bs, 0, s>>>(b, w);
    launch_solve(models, stage_batch(b, w, n * kMaxM), stage_result(w, w.fs), mode, s, num_sms);
    // instances with 32 < M <= B_max (K1 defers them; grouping is defined for M <= 32): the whole
    // instance, in slot inst * 32, gets its LC answer from the block-per-instance kernel
    if (wide) launch_solve_large(models, stage_batch(b, w, n * kMaxM), stage_result(w, w.fs), JDOB_MODE_LC, s, num_sms);
    k_og_final_write<<<(unsigned)((n * 32 + bs - 1) / bs), bs, 0, s>>>(models, b, w, o);
    return 0;
}

}  // namespace jdob
