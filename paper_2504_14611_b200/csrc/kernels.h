// kernels.h -- internal launch interface between the C-ABI layer (api.cu) and the kernels.
#pragma once

#include <cuda_runtime.h>

#include "jdob_dev.cuh"

namespace jdob {

constexpr int kChunkModels = 8;  // model descriptors passed by value per K0 launch

struct ModelChunk {
    int count;
    DevModel m[kChunkModels];
    DevModel *dst;  // where K0 publishes the descriptors (workspace)
};

// Launch geometry of the solve kernel (one warp per instance, persistent grid).
constexpr int kSolveWarps = 4;
constexpr int kStatsBlocks = 1024;   // leaves of the fixed dyadic statistics tree (power of two)
constexpr int kBfBlocks = 148 * 8;   // persistent brute-force grid
constexpr int kBfWarps = 4;

// outer grouping (K5) work arrays, all in the caller's workspace
constexpr int kCells = kMaxM + 1;
struct OgWork {
    double *sz, *sk, *sf0, *sf1, *sR, *sp, *sT;  // [users] user parameters in deadline order
    long long *perm;                             // [users] sorted position -> input user index
    double *fs;                                  // [users] f* of the final pass (sorted order)
    double *cE, *cT;                             // [n_inst * kCells] DP cells
    int *from;                                   // [n_inst * kCells]
    int *status, *ngroups;                       // [n_inst]
    int *mmax;                                   // [1]
    long long *s_off, *s_end;                    // [n_inst * kMaxM] stage views
    int *s_model;
    double *s_tfree, *s_femin, *s_femax, *s_rho;
    double *r_E, *r_Elc, *r_tf, *r_fe;           // [n_inst * kMaxM] stage results
    int *r_nt, *r_j, *r_st;
    unsigned *r_mask;
};
struct GroupedOut {
    double *E, *t_free_next;
    int *n_groups, *status;
    int *group_of, *partition;
    double *f_user, *group_fe;
};

void launch_aggregates(const ModelChunk &chunk, cudaStream_t s);
int launch_grouped(const DevModel *models, const DevBatch &b, int mode, const OgWork &w, const GroupedOut &o,
                   cudaStream_t s, int num_sms, bool wide);  // wide: some model has B_max > 32
void launch_solve(const DevModel *models, const DevBatch &b, const DevResult &r, int mode, cudaStream_t s,
                  int num_sms);
void launch_solve_multi(const DevModel *models, const DevBatch &b, const DevResult &r0, const DevResult &r1,
                        const DevResult &r2, cudaStream_t s, int num_sms);
void launch_solve_large(const DevModel *models, const DevBatch &b, const DevResult &r, int mode, cudaStream_t s,
                        int num_sms);
// Statistics of the local batch b = part `part` of `parts` (a power of two <= kStatsBlocks) of a batch
// of n_total instances, i.e. its instances [n_total part / parts, n_total (part + 1) / parts): the
// leaves [part W / parts, (part + 1) W / parts) of the global dyadic tree folded into their subtree
// root.  Returns false (nothing launched) when the arguments do not describe such a part.
bool launch_stats(const DevBatch &b, const DevResult &r, double *partials, double *stats, int n_buckets,
                  long long n_total, int parts, int part, cudaStream_t s);
void launch_eval(const DevModel *models, const DevBatch &b, const int *partition, const int *plan_nt,
                 const unsigned *plan_mask, const double *f_e, double slack,
                 double *E, double *tf, double *f_user, unsigned *viol, int *status, cudaStream_t s);
// K6 (gen.cu): the C5 workload generated on the device -- input plumbing (jdobgen's device twin)
struct GenParams {
    unsigned long long seed;
    long long inst_begin;
    int hetero;
    double zeta, kappa, f_min, f_max, R, p_u, fe_min, fe_max;
    double rho[3], lat[3];
};
size_t gen_workspace_bytes(long long n);
void launch_gen_inst(const GenParams &p, long long n, int *model_id, long long *user_off, double *t_free,
                     double *fe_min, double *fe_max, double *rho, int *bucket, void *ws, cudaStream_t s);
void launch_gen_users(const GenParams &p, long long n, const int *model_id, const long long *user_off, double *zeta,
                      double *kappa, double *f_min, double *f_max, double *R, double *p_u, double *T, void *ws,
                      cudaStream_t s);
void launch_bruteforce(const DevModel *models, const DevBatch &b, int space, unsigned long long idx_begin,
                       unsigned long long idx_end, double *part_E, long long *part_idx, double *E_min,
                       long long *idx_min, int *status, cudaStream_t s);

}  // namespace jdob
