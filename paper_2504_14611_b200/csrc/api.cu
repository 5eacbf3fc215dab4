// api.cu -- the C ABI of libjdob.so (include/jdob.h): argument checks, workspace
// layout, model-aggregate setup (K0) and kernel launches.  No torch types, no
// exceptions across the boundary, nothing allocated beyond a call.
#include <cstdarg>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>

#include "jdob_dev.cuh"
#include "kernels.h"
#include <nvtx3/nvToolsExt.h>

namespace jdob {
void launch_bruteforce_impl(const DevModel *models, const DevBatch &b, int model_id, int N, int M, int space,
                            unsigned long long idx_begin, unsigned long long idx_end, void *ws, double *E_min,
                            long long *idx_min, int *status, unsigned long long *work, cudaStream_t s);
size_t bf_workspace_bytes();
}  // namespace jdob

using namespace jdob;

static thread_local std::string g_err;

static int fail(int code, const char *fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}

static int cuda_check(const char *where) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(JDOB_ECUDA, "%s: %s", where, cudaGetErrorString(e));
    return JDOB_OK;
}

static size_t al(size_t x) { return (x + 255) & ~(size_t)255; }

static size_t model_table_bytes(const jdob_model &m) {
    const size_t n1 = (size_t)m.N + 1, b1 = (size_t)m.B_max + 1;
    return 2 * al(n1 * sizeof(double)) + 4 * al(n1 * b1 * sizeof(double)) + al(sizeof(int));
}

static size_t stats_partial_bytes() {
    return al((size_t)kStatsBlocks * 64 * kStatsF * sizeof(double));  // one group (<= 64 buckets, stats.cu)
}

static int check_models(const jdob_model *models, int32_t n_models) {
    if (!models) return fail(JDOB_EINVAL, "models is NULL");
    if (n_models < 1) return fail(JDOB_EINVAL, "n_models = %d < 1", n_models);
    for (int i = 0; i < n_models; i++) {
        const jdob_model &m = models[i];
        if (m.N < 1 || m.N > JDOB_MAX_N) return fail(JDOB_EINVAL, "model %d: N = %d outside [1, %d]", i, m.N, JDOB_MAX_N);
        if (m.B_max < 1 || m.B_max > JDOB_MAX_M_LARGE)
            return fail(JDOB_EINVAL, "model %d: B_max = %d outside [1, %d]", i, m.B_max, JDOB_MAX_M_LARGE);
        if (!m.A || !m.O || !m.g || !m.q || !m.d || !m.c) return fail(JDOB_EINVAL, "model %d: NULL table", i);
    }
    return JDOB_OK;
}

constexpr size_t kFlagBytes = 8 * sizeof(int);  // K1's deferral flags [2] and its three kernels' work counters

static size_t models_bytes(const jdob_model *models, int32_t n_models) {
    size_t s = al((size_t)n_models * sizeof(DevModel));
    for (int i = 0; i < n_models; i++) s += model_table_bytes(models[i]);
    return s;
}

// Lays out the model part of the workspace and launches K0 (validation + aggregates).
static int prepare_models(const jdob_model *models, int32_t n_models, char *ws, DevModel **dev_models,
                          cudaStream_t s) {
    DevModel *dst = (DevModel *)ws;
    char *p = ws + al((size_t)n_models * sizeof(DevModel));
    ModelChunk chunk;
    chunk.count = 0;
    chunk.dst = dst;
    for (int i = 0; i < n_models; i++) {
        const jdob_model &m = models[i];
        const size_t n1 = (size_t)m.N + 1, b1 = (size_t)m.B_max + 1;
        DevModel d;
        d.N = m.N;
        d.B1 = m.B_max + 1;
        d.A = m.A;
        d.O = m.O;
        d.g = m.g;
        d.q = m.q;
        d.d = m.d;
        d.c = m.c;
        d.u = (double *)p;
        p += al(n1 * sizeof(double));
        d.v = (double *)p;
        p += al(n1 * sizeof(double));
        d.phi = (double *)p;
        p += al(n1 * b1 * sizeof(double));
        d.psi = (double *)p;
        p += al(n1 * b1 * sizeof(double));
        d.dA = (double *)p;
        p += al(n1 * b1 * sizeof(double));
        d.cA = (double *)p;
        p += al(n1 * b1 * sizeof(double));
        d.valid = (int *)p;
        p += al(sizeof(int));
        chunk.m[chunk.count++] = d;
        if (chunk.count == kChunkModels || i == n_models - 1) {
            launch_aggregates(chunk, s);
            chunk.dst += chunk.count;
            chunk.count = 0;
        }
    }
    *dev_models = dst;
    return cuda_check("aggregates");
}

static int check_batch(const jdob_batch *b, int32_t n_models) {
    if (!b) return fail(JDOB_EINVAL, "batch is NULL");
    if (b->n_inst < 0) return fail(JDOB_EINVAL, "n_inst < 0");
    if (b->n_models != n_models) return fail(JDOB_EINVAL, "batch n_models %d != %d", b->n_models, n_models);
    if (b->n_inst > 0 && (!b->model_id || !b->user_off || !b->zeta || !b->kappa || !b->f_min || !b->f_max || !b->R ||
                          !b->p_u || !b->T || !b->t_free || !b->fe_min || !b->fe_max || !b->rho))
        return fail(JDOB_EINVAL, "batch has a NULL array");
    return JDOB_OK;
}

static DevBatch to_dev(const jdob_batch *b) {
    DevBatch d;
    d.n_inst = b->n_inst;
    d.n_models = b->n_models;
    d.model_id = b->model_id;
    d.user_off = (const long long *)b->user_off;
    d.user_end = nullptr;
    d.zeta = b->zeta;
    d.kappa = b->kappa;
    d.f_min = b->f_min;
    d.f_max = b->f_max;
    d.R = b->R;
    d.p_u = b->p_u;
    d.T = b->T;
    d.t_free = b->t_free;
    d.fe_min = b->fe_min;
    d.fe_max = b->fe_max;
    d.rho = b->rho;
    d.bucket = b->bucket;
    return d;
}

// Keep the device's default memory pool from returning memory to the OS at every
// synchronisation, so jdob_solve_batch_host's stream-ordered buffers are reused.
// Library-private stream-ordered memory pool per device for the host API: its release threshold is
// the maximum, so a call's footprint stays mapped for the next call (no per-call map/unmap); the
// device's default pool (and so other cudaMallocAsync users in the process) is left untouched.
// jdob_release_pool() trims it.
static cudaMemPool_t g_pool[64];
static bool g_pool_made[64];

static cudaMemPool_t host_pool() {
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) return nullptr;
    if (!g_pool_made[dev]) {
        cudaMemPoolProps pp = {};
        pp.allocType = cudaMemAllocationTypePinned;
        pp.location.type = cudaMemLocationTypeDevice;
        pp.location.id = dev;
        if (cudaMemPoolCreate(&g_pool[dev], &pp) != cudaSuccess) {
            cudaGetLastError();
            return nullptr;
        }
        unsigned long long thr = ~0ull;
        cudaMemPoolSetAttribute(g_pool[dev], cudaMemPoolAttrReleaseThreshold, &thr);
        g_pool_made[dev] = true;
    }
    return g_pool[dev];
}

int jdob_release_pool(void) {
    g_err.clear();
    for (int d = 0; d < 64; d++)
        if (g_pool_made[d] && cudaMemPoolTrimTo(g_pool[d], 0) != cudaSuccess) return cuda_check("release_pool");
    return JDOB_OK;
}

namespace jdob {
int grid_divisor() {
    static const int d = [] {
        const char *e = getenv("JDOB_GRID_DIV");
        const int v = e ? atoi(e) : 1;
        return v > 1 ? v : 1;
    }();
    return d;
}
}  // namespace jdob

static int num_sms() {
    int dev = 0, n = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return n > 0 ? n : 148;
}

// NVTX range around each entry point (header-only NVTX v3: a no-op unless a profiler is attached)
struct NvtxRange {
    explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
};

extern "C" {

const char *jdob_last_error(void) { return g_err.c_str(); }

const char *jdob_version(void) { return "jdob-b200 0.1 (sm_100a)"; }

size_t jdob_workspace_bytes(const jdob_model *models, int32_t n_models, int32_t which) {
    if (which == 2) return stats_partial_bytes();  // jdob_stats: no model part
    if (!models || n_models < 1) return 0;
    for (int i = 0; i < n_models; i++)
        if (models[i].N < 1 || models[i].N > JDOB_MAX_N || models[i].B_max < 1 ||
            models[i].B_max > JDOB_MAX_M_LARGE)
            return 0;
    size_t s = models_bytes(models, n_models);
    if (which == 0) return s + stats_partial_bytes() + al(kFlagBytes);  // + K1's deferral flags
    if (which == 1) return s + al(bf_workspace_bytes());
    return 0;
}

uint64_t jdob_bf_space_size(int32_t space, int32_t N, int32_t M, int64_t k) {
    if (N < 1 || M < 1 || M > JDOB_MAX_M || k < 1) return 0;
    const unsigned long long lim = 1ull << 62;
    unsigned long long s = (unsigned long long)k;
    if (space == 0) {
        for (int m = 0; m < M; m++) {
            if (s > lim / (unsigned long long)(N + 1)) return 0;
            s *= (unsigned long long)(N + 1);
        }
    } else if (space == 1) {
        unsigned long long f = (unsigned long long)(N + 1) << M;
        if (s > lim / f) return 0;
        s *= f;
    } else {
        return 0;
    }
    return s;
}

static int solve_prepared(const jdob_model *models, int32_t n_models, const DevModel *dm, const jdob_batch *b,
                          int32_t mode, const jdob_result *out, void *ws, cudaStream_t s);

int jdob_solve_batch(const jdob_model *models, int32_t n_models, const jdob_batch *b, int32_t mode,
                     const jdob_result *out, void *ws, size_t ws_bytes, void *stream) {
    NvtxRange nvtx_("jdob_solve_batch");
    g_err.clear();
    int rc = check_models(models, n_models);
    if (rc) return rc;
    if ((rc = check_batch(b, n_models))) return rc;
    if (mode < JDOB_MODE_FULL || mode > JDOB_MODE_BINARY) return fail(JDOB_EINVAL, "bad mode %d", mode);
    if (!out) return fail(JDOB_EINVAL, "out is NULL");
    if (b->n_inst > 0 && (!out->E || !out->E_lc || !out->t_free_next || !out->f_e || !out->n_tilde || !out->j ||
                          !out->status || !out->mask))
        return fail(JDOB_EINVAL, "result has a NULL required array");
    if (out->violations && (out->counts || out->work))
        return fail(JDOB_EINVAL, "violations cannot be combined with the counts/work diagnostics");
    if (out->stats && (out->n_buckets < 1 || out->n_buckets > JDOB_MAX_BUCKETS))
        return fail(JDOB_EINVAL, "n_buckets = %d outside [1, %d]", out->n_buckets, JDOB_MAX_BUCKETS);
    const size_t need = jdob_workspace_bytes(models, n_models, 0);
    if (!ws || ws_bytes < need) return fail(JDOB_EINVAL, "workspace %zu bytes < %zu", ws_bytes, need);
    cudaStream_t s = (cudaStream_t)stream;
    DevModel *dm = nullptr;
    if ((rc = prepare_models(models, n_models, (char *)ws, &dm, s))) return rc;
    return solve_prepared(models, n_models, dm, b, mode, out, ws, s);
}

// jdob_solve_batch after the model tables are prepared (K0) in ws: K1 (+ K1L), optional K4
static int solve_prepared(const jdob_model *models, int32_t n_models, const DevModel *dm, const jdob_batch *b,
                          int32_t mode, const jdob_result *out, void *ws, cudaStream_t s) {
    int rc = JDOB_OK;
    DevBatch db = to_dev(b);
    DevResult dr;
    dr.E = out->E;
    dr.E_lc = out->E_lc;
    dr.t_free_next = out->t_free_next;
    dr.f_e = out->f_e;
    dr.n_tilde = out->n_tilde;
    dr.j = out->j;
    dr.status = out->status;
    dr.mask = out->mask;
    dr.f_user = out->f_user;
    dr.counts = (long long *)out->counts;
    dr.partition = out->partition;
    dr.work = (long long *)out->work;
    dr.viol = out->violations;
    dr.slack = out->slack;
    dr.flags = (int *)((char *)ws + models_bytes(models, n_models) + stats_partial_bytes());
    cudaMemsetAsync(dr.flags, 0, kFlagBytes, s);
    launch_solve(dm, db, dr, mode, s, num_sms());
    // instances with 32 < M <= B_max (block per instance); M > B_max is BADPARAM, so the launch is
    // needed only when some model admits batches wider than a warp
    bool wide = false;
    for (int i = 0; i < n_models; i++) wide |= models[i].B_max > JDOB_MAX_M;
    if (wide) launch_solve_large(dm, db, dr, mode, s, num_sms());
    if ((rc = cuda_check("solve"))) return rc;
    if (out->stats) {
        double *partials = (double *)((char *)ws + models_bytes(models, n_models));
        launch_stats(db, dr, partials, out->stats, out->n_buckets, b->n_inst, 1, 0, s);
        if ((rc = cuda_check("stats"))) return rc;
    }
    return JDOB_OK;
}

static DevResult dev_result(const jdob_result *out) {
    DevResult dr;
    dr.E = out->E;
    dr.E_lc = out->E_lc;
    dr.t_free_next = out->t_free_next;
    dr.f_e = out->f_e;
    dr.n_tilde = out->n_tilde;
    dr.j = out->j;
    dr.status = out->status;
    dr.mask = out->mask;
    dr.f_user = out->f_user;
    dr.counts = nullptr;
    dr.partition = out->partition;
    dr.work = nullptr;
    dr.viol = nullptr;
    dr.slack = out->slack;
    return dr;
}

int jdob_solve_batch_modes(const jdob_model *models, int32_t n_models, const jdob_batch *b, const jdob_result *out,
                           void *ws, size_t ws_bytes, void *stream) {
    NvtxRange nvtx_("jdob_solve_batch_modes");
    g_err.clear();
    int rc = check_models(models, n_models);
    if (rc) return rc;
    if ((rc = check_batch(b, n_models))) return rc;
    if (!out) return fail(JDOB_EINVAL, "out is NULL");
    for (int m = 0; m < 3; m++) {
        const jdob_result *o = &out[m];
        if (b->n_inst > 0 && (!o->E || !o->E_lc || !o->t_free_next || !o->f_e || !o->n_tilde || !o->j || !o->status ||
                              !o->mask))
            return fail(JDOB_EINVAL, "result %d has a NULL required array", m);
        if (o->counts || o->work || o->violations)
            return fail(JDOB_EINVAL, "result %d: counts/work/violations are not produced by the one-pass call", m);
        if (o->stats && (o->n_buckets < 1 || o->n_buckets > JDOB_MAX_BUCKETS))
            return fail(JDOB_EINVAL, "result %d: n_buckets = %d outside [1, %d]", m, o->n_buckets, JDOB_MAX_BUCKETS);
    }
    const size_t need = jdob_workspace_bytes(models, n_models, 0);
    if (!ws || ws_bytes < need) return fail(JDOB_EINVAL, "workspace %zu bytes < %zu", ws_bytes, need);
    cudaStream_t s = (cudaStream_t)stream;
    DevModel *dm = nullptr;
    if ((rc = prepare_models(models, n_models, (char *)ws, &dm, s))) return rc;
    const DevBatch db = to_dev(b);
    DevResult r0 = dev_result(&out[0]);
    const DevResult r1 = dev_result(&out[1]), r2 = dev_result(&out[2]);
    r0.flags = (int *)((char *)ws + models_bytes(models, n_models) + stats_partial_bytes());  // deferral flags
    cudaMemsetAsync(r0.flags, 0, kFlagBytes, s);
    launch_solve_multi(dm, db, r0, r1, r2, s, num_sms());
    bool wide = false;  // instances with 32 < M <= B_max: the block-per-instance kernel, once per mode
    for (int i = 0; i < n_models; i++) wide |= models[i].B_max > JDOB_MAX_M;
    if (wide) {
        launch_solve_large(dm, db, r0, JDOB_MODE_FULL, s, num_sms());
        launch_solve_large(dm, db, r1, JDOB_MODE_NO_EDGE_DVFS, s, num_sms());
        launch_solve_large(dm, db, r2, JDOB_MODE_BINARY, s, num_sms());
    }
    if ((rc = cuda_check("solve_modes"))) return rc;
    const DevResult *rs[3] = {&r0, &r1, &r2};
    for (int m = 0; m < 3; m++) {
        if (!out[m].stats) continue;
        double *partials = (double *)((char *)ws + models_bytes(models, n_models));
        launch_stats(db, *rs[m], partials, out[m].stats, out[m].n_buckets, b->n_inst, 1, 0, s);
        if ((rc = cuda_check("stats"))) return rc;
    }
    return JDOB_OK;
}

int jdob_stats(const jdob_batch *b, const jdob_result *res, void *ws, size_t ws_bytes, void *stream) {
    return jdob_stats_part(b, res, b ? b->n_inst : 0, 1, 0, ws, ws_bytes, stream);
}

int jdob_stats_part(const jdob_batch *b, const jdob_result *res, int64_t n_total, int32_t parts, int32_t part,
                    void *ws, size_t ws_bytes, void *stream) {
    NvtxRange nvtx_("jdob_stats_part");
    g_err.clear();
    if (!b || !res) return fail(JDOB_EINVAL, "stats: NULL batch or result");
    if (b->n_inst < 0) return fail(JDOB_EINVAL, "n_inst < 0");
    if (!res->stats) return fail(JDOB_EINVAL, "stats: NULL stats array");
    if (res->n_buckets < 1 || res->n_buckets > JDOB_MAX_BUCKETS)
        return fail(JDOB_EINVAL, "n_buckets = %d outside [1, %d]", res->n_buckets, JDOB_MAX_BUCKETS);
    if (b->n_inst > 0 && (!b->user_off || !res->E || !res->E_lc || !res->f_e || !res->n_tilde || !res->status))
        return fail(JDOB_EINVAL, "stats: NULL input array");
    if (!ws || ws_bytes < stats_partial_bytes())
        return fail(JDOB_EINVAL, "workspace %zu bytes < %zu", ws_bytes, stats_partial_bytes());
    DevResult dr;
    dr.E = res->E;
    dr.E_lc = res->E_lc;
    dr.t_free_next = res->t_free_next;
    dr.f_e = res->f_e;
    dr.n_tilde = res->n_tilde;
    dr.j = res->j;
    dr.status = res->status;
    dr.mask = res->mask;
    dr.f_user = nullptr;
    dr.counts = nullptr;
    dr.partition = nullptr;
    dr.work = nullptr;
    if (!launch_stats(to_dev(b), dr, (double *)ws, res->stats, res->n_buckets, n_total, parts, part,
                      (cudaStream_t)stream))
        return fail(JDOB_EINVAL, "stats: the batch (%lld instances) is not part %d of %d of %lld instances (parts a "
                    "power of two <= %d)", (long long)b->n_inst, part, parts, (long long)n_total, kStatsBlocks);
    return cuda_check("stats");
}

static GenParams gen_params(const jdob_gen_params *p) {
    GenParams g;
    g.seed = p->seed;
    g.inst_begin = p->inst_begin;
    g.hetero = p->hetero;
    g.zeta = p->zeta;
    g.kappa = p->kappa;
    g.f_min = p->f_min;
    g.f_max = p->f_max;
    g.R = p->R;
    g.p_u = p->p_u;
    g.fe_min = p->fe_min;
    g.fe_max = p->fe_max;
    for (int i = 0; i < 3; i++) {
        g.rho[i] = p->rho[i];
        g.lat[i] = p->lat[i];
    }
    return g;
}

size_t jdob_generate_workspace_bytes(int64_t n_inst) { return n_inst < 0 ? 0 : gen_workspace_bytes(n_inst); }

int jdob_generate_c5_instances(const jdob_gen_params *p, const jdob_batch *b, int64_t *n_users, void *ws,
                               size_t ws_bytes, void *stream) {
    NvtxRange nvtx_("jdob_generate_c5_instances");
    g_err.clear();
    if (!p || !b || !n_users) return fail(JDOB_EINVAL, "generate: NULL argument");
    if (b->n_inst < 0) return fail(JDOB_EINVAL, "n_inst < 0");
    if (b->n_inst > 0 && (!b->model_id || !b->user_off || !b->t_free || !b->fe_min || !b->fe_max || !b->rho ||
                          !b->bucket))
        return fail(JDOB_EINVAL, "generate: NULL instance array");
    if (!ws || ws_bytes < gen_workspace_bytes(b->n_inst)) return fail(JDOB_EINVAL, "generate: small workspace");
    cudaStream_t s = (cudaStream_t)stream;
    *n_users = 0;
    if (b->n_inst == 0) return JDOB_OK;
    launch_gen_inst(gen_params(p), b->n_inst, (int *)b->model_id, (long long *)b->user_off, (double *)b->t_free,
                    (double *)b->fe_min, (double *)b->fe_max, (double *)b->rho, (int *)b->bucket, ws, s);
    long long nu = 0;
    cudaMemcpyAsync(&nu, b->user_off + b->n_inst, sizeof(nu), cudaMemcpyDeviceToHost, s);
    if (cudaStreamSynchronize(s) != cudaSuccess) return cuda_check("generate: read n_users");
    *n_users = nu;
    return cuda_check("generate instances");
}

int jdob_generate_c5_users(const jdob_gen_params *p, const jdob_batch *b, void *ws, size_t ws_bytes, void *stream) {
    NvtxRange nvtx_("jdob_generate_c5_users");
    g_err.clear();
    if (!p || !b) return fail(JDOB_EINVAL, "generate: NULL argument");
    if (b->n_inst > 0 && (!b->model_id || !b->user_off || !b->zeta || !b->kappa || !b->f_min || !b->f_max ||
                          !b->R || !b->p_u || !b->T))
        return fail(JDOB_EINVAL, "generate: NULL user array");
    if (!ws || ws_bytes < gen_workspace_bytes(b->n_inst)) return fail(JDOB_EINVAL, "generate: small workspace");
    launch_gen_users(gen_params(p), b->n_inst, b->model_id, (const long long *)b->user_off, (double *)b->zeta,
                     (double *)b->kappa, (double *)b->f_min, (double *)b->f_max, (double *)b->R, (double *)b->p_u,
                     (double *)b->T, ws, (cudaStream_t)stream);
    return cuda_check("generate users");
}

static size_t og_work_bytes(int64_t n, int64_t nu) {
    const size_t ns = (size_t)n * kMaxM, nc = (size_t)n * kCells;
    return 9 * al(nu * 8) + 2 * al(nc * 8) + al(nc * 4) + 2 * al(n * 4) + al(8) + 2 * al(ns * 8) + al(ns * 4) +
           4 * al(ns * 8) + 4 * al(ns * 8) + 4 * al(ns * 4);
}

size_t jdob_grouped_workspace_bytes(const jdob_model *models, int32_t n_models, int64_t n_inst, int64_t n_users) {
    const size_t base = jdob_workspace_bytes(models, n_models, 0);
    if (base == 0 || n_inst < 0 || n_users < 0) return 0;
    return base + og_work_bytes(n_inst, n_users);
}

int jdob_solve_grouped(const jdob_model *models, int32_t n_models, const jdob_batch *b, int32_t mode,
                       const jdob_grouped_result *out, void *ws, size_t ws_bytes, void *stream) {
    NvtxRange nvtx_("jdob_solve_grouped");
    g_err.clear();
    int rc = check_models(models, n_models);
    if (rc) return rc;
    if ((rc = check_batch(b, n_models))) return rc;
    if (mode < JDOB_MODE_FULL || mode > JDOB_MODE_BINARY) return fail(JDOB_EINVAL, "bad mode %d", mode);
    if (!out || (b->n_inst > 0 && (!out->E || !out->t_free_next || !out->n_groups || !out->status ||
                                   !out->group_of || !out->partition || !out->group_fe)))
        return fail(JDOB_EINVAL, "grouped result has a NULL required array");
    cudaStream_t s = (cudaStream_t)stream;
    const long long n = b->n_inst;
    if (n == 0) return JDOB_OK;
    long long nu = 0;
    cudaMemcpyAsync(&nu, b->user_off + n, sizeof(long long), cudaMemcpyDeviceToHost, s);
    if (cudaStreamSynchronize(s) != cudaSuccess) return cuda_check("grouped: read user_off");
    const size_t need = jdob_grouped_workspace_bytes(models, n_models, n, nu);
    if (!ws || ws_bytes < need) return fail(JDOB_EINVAL, "workspace %zu bytes < %zu", ws_bytes, need);
    DevModel *dm = nullptr;
    if ((rc = prepare_models(models, n_models, (char *)ws, &dm, s))) return rc;
    char *p = (char *)ws + jdob_workspace_bytes(models, n_models, 0);
    auto take = [&](size_t nb) -> char * {
        char *d = p;
        p += al(nb);
        return d;
    };
    const size_t ns = (size_t)n * kMaxM, nc = (size_t)n * kCells;
    OgWork w;
    w.sz = (double *)take(nu * 8);
    w.sk = (double *)take(nu * 8);
    w.sf0 = (double *)take(nu * 8);
    w.sf1 = (double *)take(nu * 8);
    w.sR = (double *)take(nu * 8);
    w.sp = (double *)take(nu * 8);
    w.sT = (double *)take(nu * 8);
    w.perm = (long long *)take(nu * 8);
    w.fs = (double *)take(nu * 8);
    w.cE = (double *)take(nc * 8);
    w.cT = (double *)take(nc * 8);
    w.from = (int *)take(nc * 4);
    w.status = (int *)take(n * 4);
    w.ngroups = (int *)take(n * 4);
    w.mmax = (int *)take(8);
    w.s_off = (long long *)take(ns * 8);
    w.s_end = (long long *)take(ns * 8);
    w.s_model = (int *)take(ns * 4);
    w.s_tfree = (double *)take(ns * 8);
    w.s_femin = (double *)take(ns * 8);
    w.s_femax = (double *)take(ns * 8);
    w.s_rho = (double *)take(ns * 8);
    w.r_E = (double *)take(ns * 8);
    w.r_Elc = (double *)take(ns * 8);
    w.r_tf = (double *)take(ns * 8);
    w.r_fe = (double *)take(ns * 8);
    w.r_nt = (int *)take(ns * 4);
    w.r_j = (int *)take(ns * 4);
    w.r_st = (int *)take(ns * 4);
    w.r_mask = (unsigned *)take(ns * 4);
    GroupedOut o;
    o.E = out->E;
    o.t_free_next = out->t_free_next;
    o.n_groups = out->n_groups;
    o.status = out->status;
    o.group_of = out->group_of;
    o.partition = out->partition;
    o.f_user = out->f_user;
    o.group_fe = out->group_fe;
    bool wide = false;  // some model admits M > 32: such instances are reported with their LC answer
    for (int i = 0; i < n_models; i++) wide |= models[i].B_max > JDOB_MAX_M;
    if (launch_grouped(dm, to_dev(b), mode, w, o, s, num_sms(), wide)) return cuda_check("grouped");
    return cuda_check("grouped");
}

int jdob_eval(const jdob_model *models, int32_t n_models, const jdob_batch *b, const int32_t *partition,
              const int32_t *plan_n_tilde, const uint32_t *plan_mask, const double *f_e, double slack, double *E,
              double *t_free_next, double *f_user, uint32_t *violations, int32_t *status, void *ws, size_t ws_bytes,
              void *stream) {
    NvtxRange nvtx_("jdob_eval");
    g_err.clear();
    int rc = check_models(models, n_models);
    if (rc) return rc;
    if ((rc = check_batch(b, n_models))) return rc;
    if (b->n_inst > 0 && ((!partition && (!plan_n_tilde || !plan_mask)) || !f_e || !E || !t_free_next ||
                          !violations || !status))
        return fail(JDOB_EINVAL, "eval: NULL array");
    const size_t need = jdob_workspace_bytes(models, n_models, 0);
    if (!ws || ws_bytes < need) return fail(JDOB_EINVAL, "workspace %zu bytes < %zu", ws_bytes, need);
    cudaStream_t s = (cudaStream_t)stream;
    DevModel *dm = nullptr;
    if ((rc = prepare_models(models, n_models, (char *)ws, &dm, s))) return rc;
    launch_eval(dm, to_dev(b), partition, plan_n_tilde, plan_mask, f_e, slack, E, t_free_next, f_user, violations,
                status, s);
    return cuda_check("eval");
}

int jdob_bruteforce(const jdob_model *models, int32_t n_models, const jdob_batch *b, int32_t space,
                    uint64_t idx_begin, uint64_t idx_end, double *E_min, int64_t *idx_min, int32_t *status,
                    int64_t *work, void *ws, size_t ws_bytes, void *stream) {
    NvtxRange nvtx_("jdob_bruteforce");
    g_err.clear();
    int rc = check_models(models, n_models);
    if (rc) return rc;
    if ((rc = check_batch(b, n_models))) return rc;
    if (b->n_inst != 1) return fail(JDOB_EINVAL, "bruteforce needs n_inst == 1 (got %lld)", (long long)b->n_inst);
    if (space != 0 && space != 1) return fail(JDOB_EINVAL, "bad space %d", space);
    if (idx_begin > idx_end) return fail(JDOB_EINVAL, "idx_begin > idx_end");
    if (!E_min || !idx_min || !status) return fail(JDOB_EINVAL, "bruteforce: NULL output");
    const size_t need = jdob_workspace_bytes(models, n_models, 1);
    if (!ws || ws_bytes < need) return fail(JDOB_EINVAL, "workspace %zu bytes < %zu", ws_bytes, need);
    cudaStream_t s = (cudaStream_t)stream;
    // one small synchronous read: M and the model id select the kernel specialisation
    long long off[2] = {0, 0};
    int mid = 0;
    cudaMemcpyAsync(off, b->user_off, sizeof(off), cudaMemcpyDeviceToHost, s);
    cudaMemcpyAsync(&mid, b->model_id, sizeof(int), cudaMemcpyDeviceToHost, s);
    if (cudaStreamSynchronize(s) != cudaSuccess) return cuda_check("bruteforce: read user_off");
    const int M = (int)(off[1] - off[0]);
    const int N = (mid >= 0 && mid < n_models) ? models[mid].N : 1;
    DevModel *dm = nullptr;
    if ((rc = prepare_models(models, n_models, (char *)ws, &dm, s))) return rc;
    void *bws = (char *)ws + models_bytes(models, n_models);
    launch_bruteforce_impl(dm, to_dev(b), (mid >= 0 && mid < n_models) ? mid : 0, N, M, space, idx_begin, idx_end,
                           bws, E_min, (long long *)idx_min, status, (unsigned long long *)work, s);
    return cuda_check("bruteforce");
}

}  // extern "C"

// Users of one instance given with shared device parameters (jdob_shared_batch): expanded, per chunk,
// into the struct-of-arrays layout the kernels read (one warp per instance, lane = user).
__global__ void k_expand_shared(long long n, const long long *user_off, const double *z, const double *k,
                                const double *f0, const double *f1, const double *R, const double *p, double *uz,
                                double *uk, double *uf0, double *uf1, double *uR, double *up) {
    const long long i = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (i >= n) return;
    const long long o = user_off[i], e = user_off[i + 1];
    for (long long u = o + lane; u < e; u += 32) {
        uz[u] = z[i];
        uk[u] = k[i];
        uf0[u] = f0[i];
        uf1[u] = f1[i];
        uR[u] = R[i];
        up[u] = p[i];
    }
}

// The host API's copy-in, compute and copy-out streams and its events, created once per device (the
// host API's calls on one device are serialised through them; each call joins them into the caller's
// stream before it returns).
struct HostStreams {
    static constexpr int kMaxChunks = 70;
    cudaStream_t h2d, compute, d2h;
    cudaEvent_t start, hdone, kdone, ddone, in[kMaxChunks], solved[kMaxChunks];
};
static HostStreams g_hs[64];
static bool g_hs_made[64];

static std::mutex g_hs_mutex[64];  // one host call per device at a time (the streams and events are shared)

static HostStreams &host_streams() {
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) dev = 0;
    HostStreams &h = g_hs[dev];
    if (!g_hs_made[dev]) {
        cudaStreamCreateWithFlags(&h.h2d, cudaStreamNonBlocking);
        cudaStreamCreateWithFlags(&h.compute, cudaStreamNonBlocking);
        cudaStreamCreateWithFlags(&h.d2h, cudaStreamNonBlocking);
        cudaEvent_t *ev[4] = {&h.start, &h.hdone, &h.kdone, &h.ddone};
        for (auto e : ev) cudaEventCreateWithFlags(e, cudaEventDisableTiming);
        for (int c = 0; c < HostStreams::kMaxChunks; c++) {
            cudaEventCreateWithFlags(&h.in[c], cudaEventDisableTiming);
            cudaEventCreateWithFlags(&h.solved[c], cudaEventDisableTiming);
        }
        g_hs_made[dev] = true;
    }
    return h;
}

// jdob_solve_batch_host and jdob_solve_shared_host: exactly one of b (users as arrays) and sb (users
// sharing their device parameters within an instance) is given
static int solve_host_impl(const jdob_model *models, int32_t n_models, const jdob_batch *b_full,
                           const jdob_shared_batch *sb, int32_t mode, const jdob_result *out, void *stream,
                           int64_t *h2d_bytes, int64_t *d2h_bytes) {
    // the instance-level fields of either form, in a jdob_batch (user arrays: T only for sb)
    jdob_batch bv;
    if (b_full) {
        bv = *b_full;
    } else {
        bv.n_inst = sb->n_inst;
        bv.n_models = sb->n_models;
        bv.model_id = sb->model_id;
        bv.user_off = sb->user_off;
        bv.zeta = bv.kappa = bv.f_min = bv.f_max = bv.R = bv.p_u = sb->T;  // placeholders: not copied
        bv.T = sb->T;
        bv.t_free = sb->t_free;
        bv.fe_min = sb->fe_min;
        bv.fe_max = sb->fe_max;
        bv.rho = sb->rho;
        bv.bucket = sb->bucket;
    }
    const jdob_batch *b = &bv;
    const bool shared = (sb != nullptr);
    if (!models || n_models < 1) return fail(JDOB_EINVAL, "models");
    for (int i = 0; i < n_models; i++) {
        if (models[i].N < 1 || models[i].N > JDOB_MAX_N || models[i].B_max < 1 ||
            models[i].B_max > JDOB_MAX_M_LARGE)
            return fail(JDOB_EINVAL, "model %d: N/B_max out of range", i);
        if (!models[i].A || !models[i].O || !models[i].g || !models[i].q || !models[i].d || !models[i].c)
            return fail(JDOB_EINVAL, "model %d: NULL table", i);
    }
    int rc = check_batch(b, n_models);
    if (rc) return rc;
    if (shared && b->n_inst > 0 && (!sb->zeta || !sb->kappa || !sb->f_min || !sb->f_max || !sb->R || !sb->p_u))
        return fail(JDOB_EINVAL, "shared batch has a NULL parameter array");
    if (!out || !out->E || !out->E_lc || !out->t_free_next || !out->f_e || !out->n_tilde || !out->j ||
        !out->status || !out->mask)
        return fail(JDOB_EINVAL, "result has a NULL required array");
    if (out->stats && (out->n_buckets < 1 || out->n_buckets > JDOB_MAX_BUCKETS))
        return fail(JDOB_EINVAL, "n_buckets = %d outside [1, %d]", out->n_buckets, JDOB_MAX_BUCKETS);
    if (mode < JDOB_MODE_FULL || mode > JDOB_MODE_BINARY) return fail(JDOB_EINVAL, "bad mode %d", mode);
    cudaStream_t s = (cudaStream_t)stream;
    cudaMemPool_t pool = host_pool();
    const long long n = b->n_inst;
    if (n > 0 && b->user_off[0] < 0) return fail(JDOB_EINVAL, "user_off[0] = %lld < 0", (long long)b->user_off[0]);
    const long long nu = n > 0 ? (long long)b->user_off[n] : 0;
    // device layout: model tables | batch | outputs | workspace
    size_t bytes = 0;
    for (int i = 0; i < n_models; i++) {
        const size_t n1 = (size_t)models[i].N + 1, b1 = (size_t)models[i].B_max + 1;
        bytes += 4 * al(n1 * 8) + 2 * al(n1 * b1 * 8);
    }
    const size_t in_inst = al(n * 4) + al((n + 1) * 8) + 4 * al(n * 8) + (b->bucket ? al(n * 4) : 0);
    const size_t in_user = 7 * al(nu * 8) + (shared ? 6 * al(n * 8) : 0);
    const size_t outb = 4 * al(n * 8) + 4 * al(n * 4) + (out->f_user ? al(nu * 8) : 0) +
                        (out->partition ? al(nu * 4) : 0) +
                        (out->counts ? al(n * 3 * 8) : 0) +
                        (out->stats ? al((size_t)out->n_buckets * JDOB_STATS_FIELDS * 8) : 0);
    const size_t wsb = jdob_workspace_bytes(models, n_models, 0);
    bytes += in_inst + in_user + outb + al(wsb);
    char *base = nullptr;
    if ((pool ? cudaMallocFromPoolAsync((void **)&base, bytes, pool, s) : cudaMallocAsync((void **)&base, bytes, s)) !=
        cudaSuccess)
        return cuda_check("cudaMallocAsync");
    char *p = base;
    long long h2d = 0, d2h = 0;
    auto take = [&](size_t nb) -> char * {
        char *d = p;
        p += al(nb);
        return d;
    };
    jdob_model dmods[64];
    jdob_model *dm = n_models <= 64 ? dmods : new jdob_model[n_models];
    for (int i = 0; i < n_models; i++) {
        const size_t n1 = (size_t)models[i].N + 1, b1 = (size_t)models[i].B_max + 1;
        const double *src[6] = {models[i].A, models[i].O, models[i].g, models[i].q, models[i].d, models[i].c};
        const size_t nb[6] = {n1 * 8, n1 * 8, n1 * 8, n1 * 8, n1 * b1 * 8, n1 * b1 * 8};
        const double *dst[6];
        for (int t = 0; t < 6; t++) {
            char *d = take(nb[t]);
            cudaMemcpyAsync(d, src[t], nb[t], cudaMemcpyHostToDevice, s);
            h2d += (long long)nb[t];
            dst[t] = (const double *)d;
        }
        dm[i].N = models[i].N;
        dm[i].B_max = models[i].B_max;
        dm[i].A = dst[0];
        dm[i].O = dst[1];
        dm[i].g = dst[2];
        dm[i].q = dst[3];
        dm[i].d = dst[4];
        dm[i].c = dst[5];
    }
    // full-size device arrays; chunks are views (user indices stay global)
    jdob_batch db = *b;
    db.model_id = (const int32_t *)take(n * 4);
    db.user_off = (const int64_t *)take((n + 1) * 8);
    const double **uf[7] = {&db.zeta, &db.kappa, &db.f_min, &db.f_max, &db.R, &db.p_u, &db.T};
    const double *uh[7] = {b->zeta, b->kappa, b->f_min, b->f_max, b->R, b->p_u, b->T};
    for (int t = 0; t < 7; t++) *uf[t] = (const double *)take(nu * 8);
    const double **inf[4] = {&db.t_free, &db.fe_min, &db.fe_max, &db.rho};
    const double *ih[4] = {b->t_free, b->fe_min, b->fe_max, b->rho};
    for (int t = 0; t < 4; t++) *inf[t] = (const double *)take(n * 8);
    db.bucket = b->bucket ? (const int32_t *)take(n * 4) : nullptr;
    double *sh_dev[6] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};  // shared parameters [n]
    const double *sh_host[6] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
    if (shared) {
        const double *hs[6] = {sb->zeta, sb->kappa, sb->f_min, sb->f_max, sb->R, sb->p_u};
        for (int t = 0; t < 6; t++) {
            sh_dev[t] = (double *)take(n * 8);
            sh_host[t] = hs[t];
        }
    }
    jdob_result dr = *out;
    dr.E = (double *)take(n * 8);
    dr.E_lc = (double *)take(n * 8);
    dr.t_free_next = (double *)take(n * 8);
    dr.f_e = (double *)take(n * 8);
    dr.n_tilde = (int32_t *)take(n * 4);
    dr.j = (int32_t *)take(n * 4);
    dr.status = (int32_t *)take(n * 4);
    dr.mask = (uint32_t *)take(n * 4);
    dr.f_user = out->f_user ? (double *)take(nu * 8) : nullptr;
    dr.counts = out->counts ? (int64_t *)take(n * 3 * 8) : nullptr;
    dr.stats = out->stats ? (double *)take((size_t)out->n_buckets * JDOB_STATS_FIELDS * 8) : nullptr;
    dr.partition = out->partition ? (int32_t *)take(nu * 4) : nullptr;
    dr.work = nullptr;  // device-API diagnostic only
    dr.violations = nullptr;
    void *ws = take(wsb);

    // pipeline on three streams of the library (HostStreams): the copy-ins of every chunk back to back on
    // one stream, each chunk's solve on a second stream once its copy-ins are done, its copy-outs on a
    // third once its solve is done -- the H2D engine never waits for a solve or a copy-out, and the solve
    // of chunk c overlaps the copy-ins of the chunks after it and the copy-outs of those before it
    int hdev = 0;
    cudaGetDevice(&hdev);
    std::lock_guard<std::mutex> hs_lock(g_hs_mutex[(hdev >= 0 && hdev < 64) ? hdev : 0]);
    HostStreams &hs = host_streams();
    cudaStream_t sh = hs.h2d, sk = hs.compute, sd = hs.d2h;
    cudaEventRecord(hs.start, s);
    cudaStreamWaitEvent(sh, hs.start, 0);
    cudaStreamWaitEvent(sk, hs.start, 0);
    cudaStreamWaitEvent(sd, hs.start, 0);
    // the model tables were copied on s (above): K0 runs once on the compute stream, every chunk's solve
    // uses its tables
    DevModel *dmod = nullptr;
    if ((rc = prepare_models(dm, n_models, (char *)ws, &dmod, sk))) {
        cudaEventRecord(hs.kdone, sk);
        cudaStreamWaitEvent(s, hs.kdone, 0);
        cudaFreeAsync(base, s);
        if (dm != dmods) delete[] dm;
        return rc;
    }
#ifndef JDOB_HOST_CHUNK
#define JDOB_HOST_CHUNK 131072
#endif
    // chunk boundaries: JDOB_HOST_CHUNK instances each, then a geometric tail (halving, >= 16384) so
    // that the solve and copy-out left after the last copy-in are short
    long long per = JDOB_HOST_CHUNK;
    if (n > 48 * per) per = (n + 47) / 48;
    long long bounds[HostStreams::kMaxChunks + 2];
    int nchunks = 0;
    bounds[0] = 0;
    for (long long pos = 0; pos < n && nchunks < HostStreams::kMaxChunks;) {
        const long long rem = n - pos;
        long long sz = per;
#ifdef JDOB_HOST_RAMP
        // geometric ramp-up: the first solve starts after a small copy-in
        if (nchunks < 8 && (JDOB_HOST_RAMP << nchunks) < per) sz = (long long)JDOB_HOST_RAMP << nchunks;
#endif
#ifndef JDOB_HOST_NO_TAIL
        if (rem <= 2 * per) sz = (rem / 2 > 16384) ? rem / 2 : 16384;
#endif
        if (sz > rem || nchunks == HostStreams::kMaxChunks - 1) sz = rem;
        pos += sz;
        bounds[++nchunks] = pos;
    }
    for (int c = 0; c < nchunks && rc == JDOB_OK; c++) {
        const long long i0 = bounds[c], i1 = bounds[c + 1];
        if (i1 <= i0) continue;
        // the host offsets size this chunk's copies: a decreasing pair would wrap a byte count, so
        // the chunk is checked before anything of it is submitted (the chunks before it are valid)
        bool mono = true;
        for (long long q = i0; q < i1; q++) mono &= b->user_off[q] <= b->user_off[q + 1];
        mono &= b->user_off[i1] <= nu;  // within the arrays sized by user_off[n_inst]
        if (!mono) {
            rc = fail(JDOB_EINVAL, "user_off decreases inside instances [%lld, %lld]", i0, i1);
            break;
        }
        const long long u0 = b->user_off[i0], u1 = b->user_off[i1];
        // the chunk's copy-ins: one cudaMemcpyAsync per array on the copy-in stream
        auto h2 = [&](const void *dst, const void *src, size_t nb) {
            if (nb) cudaMemcpyAsync((void *)dst, src, nb, cudaMemcpyHostToDevice, sh);
            h2d += (long long)nb;
        };
        h2(db.model_id + i0, b->model_id + i0, (i1 - i0) * 4);
        // user_off[i0..i1] (the shared boundary element is written with identical bytes by both chunks)
        h2(db.user_off + i0, b->user_off + i0, (i1 - i0 + 1) * 8);
        if (!shared) {
            for (int t = 0; t < 7; t++) h2(*uf[t] + u0, uh[t] + u0, (u1 - u0) * 8);
        } else {
            h2(db.T + u0, b->T + u0, (u1 - u0) * 8);
            for (int t = 0; t < 6; t++) h2(sh_dev[t] + i0, sh_host[t] + i0, (i1 - i0) * 8);
        }
        for (int t = 0; t < 4; t++) h2(*inf[t] + i0, ih[t] + i0, (i1 - i0) * 8);
        if (b->bucket) h2(db.bucket + i0, b->bucket + i0, (i1 - i0) * 4);
        cudaEventRecord(hs.in[c], sh);
        cudaStreamWaitEvent(sk, hs.in[c], 0);
        if (shared)  // the users' arrays of this chunk from the instances' shared values
            k_expand_shared<<<(unsigned)(((i1 - i0) * 32 + 255) / 256), 256, 0, sk>>>(
                i1 - i0, (const long long *)db.user_off + i0, sh_dev[0] + i0, sh_dev[1] + i0, sh_dev[2] + i0,
                sh_dev[3] + i0, sh_dev[4] + i0, sh_dev[5] + i0, (double *)db.zeta, (double *)db.kappa,
                (double *)db.f_min, (double *)db.f_max, (double *)db.R, (double *)db.p_u);
        jdob_batch cb = db;
        cb.n_inst = i1 - i0;
        cb.model_id = db.model_id + i0;
        cb.user_off = db.user_off + i0;
        cb.t_free = db.t_free + i0;
        cb.fe_min = db.fe_min + i0;
        cb.fe_max = db.fe_max + i0;
        cb.rho = db.rho + i0;
        cb.bucket = db.bucket ? db.bucket + i0 : nullptr;
        jdob_result cr = dr;
        cr.E = dr.E + i0;
        cr.E_lc = dr.E_lc + i0;
        cr.t_free_next = dr.t_free_next + i0;
        cr.f_e = dr.f_e + i0;
        cr.n_tilde = dr.n_tilde + i0;
        cr.j = dr.j + i0;
        cr.status = dr.status + i0;
        cr.mask = dr.mask + i0;
        cr.counts = dr.counts ? dr.counts + 3 * i0 : nullptr;
        cr.stats = nullptr;
        rc = solve_prepared(dm, n_models, dmod, &cb, mode, &cr, ws, sk);
        if (rc != JDOB_OK) break;
        cudaEventRecord(hs.solved[c], sk);
        cudaStreamWaitEvent(sd, hs.solved[c], 0);
        auto d2 = [&](void *dst, const void *src, size_t nb) {
            if (nb) cudaMemcpyAsync(dst, src, nb, cudaMemcpyDeviceToHost, sd);
            d2h += (long long)nb;
        };
        d2(out->E + i0, cr.E, (i1 - i0) * 8);
        d2(out->E_lc + i0, cr.E_lc, (i1 - i0) * 8);
        d2(out->t_free_next + i0, cr.t_free_next, (i1 - i0) * 8);
        d2(out->f_e + i0, cr.f_e, (i1 - i0) * 8);
        d2(out->n_tilde + i0, cr.n_tilde, (i1 - i0) * 4);
        d2(out->j + i0, cr.j, (i1 - i0) * 4);
        d2(out->status + i0, cr.status, (i1 - i0) * 4);
        d2(out->mask + i0, cr.mask, (i1 - i0) * 4);
        if (out->f_user) d2(out->f_user + u0, dr.f_user + u0, (u1 - u0) * 8);
        if (out->partition) d2(out->partition + u0, dr.partition + u0, (u1 - u0) * 4);
        if (out->counts) d2(out->counts + 3 * i0, cr.counts, (i1 - i0) * 3 * 8);
    }
    // join: s waits for the three streams (the copy-in stream's work precedes every solve it fed)
    cudaEventRecord(hs.hdone, sh);
    cudaEventRecord(hs.kdone, sk);
    cudaEventRecord(hs.ddone, sd);
    cudaStreamWaitEvent(s, hs.hdone, 0);
    cudaStreamWaitEvent(s, hs.kdone, 0);
    cudaStreamWaitEvent(s, hs.ddone, 0);
    if (rc == JDOB_OK && out->stats && n > 0) {
        DevResult r2;
        r2.E = dr.E;
        r2.E_lc = dr.E_lc;
        r2.t_free_next = dr.t_free_next;
        r2.f_e = dr.f_e;
        r2.n_tilde = dr.n_tilde;
        r2.j = dr.j;
        r2.status = dr.status;
        r2.mask = dr.mask;
        r2.f_user = dr.f_user;
        r2.counts = (long long *)dr.counts;
        r2.partition = dr.partition;
        double *partials = (double *)((char *)ws + models_bytes(models, n_models));
        launch_stats(to_dev(&db), r2, partials, dr.stats, out->n_buckets, n, 1, 0, s);
        cudaMemcpyAsync(out->stats, dr.stats, (size_t)out->n_buckets * JDOB_STATS_FIELDS * 8,
                        cudaMemcpyDeviceToHost, s);
        d2h += (long long)out->n_buckets * JDOB_STATS_FIELDS * 8;
    }
    if (dm != dmods) delete[] dm;
    cudaFreeAsync(base, s);
    cudaError_t e = cudaStreamSynchronize(s);
    if (rc != JDOB_OK) return rc;
    if (e != cudaSuccess) return fail(JDOB_ECUDA, "solve_batch_host: %s", cudaGetErrorString(e));
    if (h2d_bytes) *h2d_bytes = h2d;
    if (d2h_bytes) *d2h_bytes = d2h;
    return JDOB_OK;
}

extern "C" {

int jdob_solve_batch_host(const jdob_model *models, int32_t n_models, const jdob_batch *b, int32_t mode,
                          const jdob_result *out, void *stream, int64_t *h2d_bytes, int64_t *d2h_bytes) {
    NvtxRange nvtx_("jdob_solve_batch_host");
    g_err.clear();
    if (!b) return fail(JDOB_EINVAL, "batch is NULL");
    return solve_host_impl(models, n_models, b, nullptr, mode, out, stream, h2d_bytes, d2h_bytes);
}

int jdob_solve_shared_host(const jdob_model *models, int32_t n_models, const jdob_shared_batch *b, int32_t mode,
                           const jdob_result *out, void *stream, int64_t *h2d_bytes, int64_t *d2h_bytes) {
    NvtxRange nvtx_("jdob_solve_shared_host");
    g_err.clear();
    if (!b) return fail(JDOB_EINVAL, "batch is NULL");
    return solve_host_impl(models, n_models, nullptr, b, mode, out, stream, h2d_bytes, d2h_bytes);
}

}  // extern "C"
