/*
 * jdob.h -- C ABI of the B200-native J-DOB hot path (libjdob.so).
 *
 * Method: Xu, Zhou, Niu, "Joint Optimization of Offloading, Batching and DVFS for
 * Multiuser Co-Inference" (arXiv 2504.14611).  "P:n" cites /root/reference/PAPER.md
 * line n; R1..R16 are the readings listed in DESIGN.md §Readings; the arithmetic
 * contract (operation order, no FMA contraction, IEEE division) is DESIGN.md
 * §Arithmetic contract.  Every entry point is asynchronous on the caller's stream
 * unless stated otherwise.
 *
 * Conventions for every entry point
 *  - Plain C types only.  Pointers documented "device" must point to device memory
 *    valid on the current device; "host" pointers to host memory.
 *  - The caller owns every buffer.  The library allocates no buffer that outlives a
 *    call (the host calls allocate and free their own stream-ordered device buffers
 *    inside the call, from a private pool that jdob_release_pool() trims); the host
 *    calls' three streams and their events are created once per device and kept.
 *  - Return value: JDOB_OK, or a call-level error (JDOB_EINVAL bad shape/pointer/
 *    limit detectable on the host, JDOB_ECUDA a CUDA launch/runtime failure).  The
 *    message of the last error of the calling thread is jdob_last_error().
 *  - Value errors inside the data are reported per instance in `status`
 *    (JDOB_ST_*), never by aborting: the instance's outputs are then the local-
 *    computing (LC) answer (n~* = N, j* = 0, mask 0), or NaN energies when the
 *    instance or its model is malformed.
 *  - No exceptions cross the ABI; the library never calls exit/abort.
 *  - Frequencies in Hz, times in s, data sizes in bits, workloads in MAC/FLOP,
 *    powers in W, energies in J (§II).
 */
#ifndef JDOB_H
#define JDOB_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define JDOB_API __attribute__((visibility("default")))
#else
#define JDOB_API
#endif

#define JDOB_MAX_M 32          /* users per instance on the warp path; offload mask width */
#define JDOB_MAX_M_LARGE 1024  /* users per instance (M' of Alg. 1), block path above 32 */
#define JDOB_MAX_N 63          /* sub-tasks per DNN (N)                        */
#define JDOB_MAX_K 65536       /* edge-frequency grid points per instance (k) */
#define JDOB_STATS_FIELDS 80   /* doubles per statistics bucket (a12)               */
#define JDOB_MAX_BUCKETS 512   /* (M, regime, model) of C5: 32 x 5 x 3 = 480 */

/* call-level return codes */
enum { JDOB_OK = 0, JDOB_EINVAL = 1, JDOB_ETOOBIG = 2, JDOB_ECUDA = 3 };

/* per-instance status codes (same numbering as the oracle) */
enum {
    JDOB_ST_OK = 0,
    JDOB_ST_LOCAL_INFEASIBLE = 1, /* zeta sum(gA)/f_max > T for some user        */
    JDOB_ST_REQUIRE = 2,          /* min_m T_m < t_free: Alg. 1 Require violated  */
    JDOB_ST_BADPARAM = 3,         /* M out of [1, min(32, B_max)], non-finite or out-of-box
                                     user/edge parameters, k > JDOB_MAX_K                 */
    JDOB_ST_BADMODEL = 4,         /* model tables invalid (A_0 != 0, A_n <= 0, d not
                                     positive non-decreasing in b, c < 0, ...)           */
    JDOB_ST_TOOBIG = 5            /* brute-force index space >= 2^62                      */
};

/* solver modes (§IV benchmarks) */
enum {
    JDOB_MODE_FULL = 0,         /* Alg. 1 + Alg. 2                                         */
    JDOB_MODE_LC = 1,           /* local computing only (benchmark (i))                    */
    JDOB_MODE_NO_EDGE_DVFS = 2, /* f_e fixed at f_e,max (k = 1)                            */
    JDOB_MODE_BINARY = 3        /* n~ restricted to {0, N}                                 */
};

/*
 * One DNN profile (§II-B, Eq. (5)).  Host struct whose
 * array members are DEVICE pointers.
 *   A, O, g, q : [N+1] doubles; index 0 is the virtual input layer (A[0] = 0,
 *                O[0] = input size).  A_n workload, O_n output bits, g_n/q_n
 *                latency/energy block factors of Eqs. (1)-(2).
 *   d, c       : row-major [(N+1) x (B_max+1)] doubles, element n*(B_max+1)+b =
 *                d_n(b), c_n(b) of Eq. (5); rows n = 0 and columns b = 0 unused.
 */
typedef struct {
    int32_t N, B_max; /* 1 <= N <= 63, 1 <= B_max <= 1024 */
    const double *A, *O, *g, *q;
    const double *d, *c;
} jdob_model;

/*
 * A batch of independent co-inference instances, users in CSR layout (struct of
 * arrays; DESIGN.md §Data layout).  All array members are DEVICE pointers.
 *   model_id [n_inst]      : index into the models[] array of the call.
 *   user_off [n_inst+1]    : users of instance i are user_off[i] .. user_off[i+1]-1;
 *                            M_i = user_off[i+1] - user_off[i] must be in [1, min(1024, B_max)].
 *                            jdob_solve_batch solves M_i <= 32 one warp per instance and
 *                            M_i > 32 one thread block per instance; the other
 *                            entry points take M_i <= 32.
 *   zeta, kappa, f_min, f_max, R, p_u, T [user_off[n_inst]] : per-user zeta_m
 *                            (cycles/workload), kappa_m (switched capacitance),
 *                            f_m,min/max (Hz), R_m (bit/s), p_m^u (W), T_m^(d) (s)
 *                            (P:116-138).
 *   t_free, fe_min, fe_max, rho [n_inst] : GPU-available time t_free, edge
 *                            frequency box and sweep step rho of Alg. 2 (P:155,
 *                            P:326-348).
 *   bucket [n_inst]        : optional statistics bucket in [0, n_buckets); NULL =
 *                            bucket M_i - 1.
 */
typedef struct {
    int64_t n_inst;
    int32_t n_models;
    const int32_t *model_id;
    const int64_t *user_off;
    const double *zeta, *kappa, *f_min, *f_max, *R, *p_u, *T;
    const double *t_free, *fe_min, *fe_max, *rho;
    const int32_t *bucket;
} jdob_batch;

/*
 * Outputs of jdob_solve_batch, DEVICE pointers, caller-allocated.
 *   E [n_inst]           : E_* of Alg. 1, the (P1) objective of the plan.
 *   E_lc [n_inst]        : local-computing energy (benchmark (i)).
 *   t_free_next [n_inst] : t_free,* (D22); t_free when all-local.
 *   f_e [n_inst]         : chosen edge frequency; 0.0 when all-local.
 *   n_tilde [n_inst]     : identical partition point n~*; N when all-local (R4, R8).
 *   j [n_inst]           : grid index of f_e (f_e = fe_max - j*rho); 0 when all-local.
 *   status [n_inst]      : JDOB_ST_*.
 *   mask [n_inst]        : offloading set M'_o, bit m = user m of the instance (M_i <= 32;
 *                          0 for M_i > 32 -- use `partition`).
 *   f_user [user_off[n_inst]] : optional (NULL = skip) device frequencies f_m* (D20).
 *   counts [3*n_inst]    : optional (NULL = skip) literal Alg. 2 work counters per
 *                          instance: (n~, j) pairs visited, pairs evaluated (guard
 *                          passed), sum of B_o over evaluated pairs.  Requesting them
 *                          turns off the exact n~ pruning (every n~ is swept literally);
 *                          results are identical either way.
 *   stats [n_buckets * JDOB_STATS_FIELDS] : optional (NULL = skip) energy-saving
 *                          statistics (a12, R16), fields per bucket:
 *                          [0] #OK instances, [1] sum r, [2] sum r^2, [3] max r,
 *                          [4] min r, [5] sum E/M, [6] sum E_lc/M, [7] #offloading
 *                          plans (f_e* > 0: some user offloads, R18; valid for any M),
 *                          [8] #status != OK, [9+n] #instances with n~* = n (n <= 63);
 *                          r = 100 (E_lc - E) / E_lc.  Deterministic for a given
 *                          n_inst (fixed reduction tree, see jdob_stats_part).  Default buckets (bucket == NULL):
 *                          bucket M_i - 1; instances with M_i > n_buckets are not counted.
 */
typedef struct {
    double *E, *E_lc, *t_free_next, *f_e;
    int32_t *n_tilde, *j, *status;
    uint32_t *mask;
    double *f_user;
    int64_t *counts;
    double *stats;
    int32_t n_buckets;  /* 1 .. JDOB_MAX_BUCKETS when stats != NULL */
    int32_t *partition; /* optional [user_off[n_inst]]: n~* for offloaders, N for local users */
    int64_t *work;      /* optional [4*n_inst], ignored when counts != NULL and by the host API:
                           work the pruned sweep executed per instance -- n~ set-ups, visited
                           pairs, evaluated pairs, member evaluations */
    uint32_t *violations; /* optional [n_inst] (NULL = skip; ignored by the host API): the plan
                           re-verified in the solver's epilogue with jdob_eval's formulas and
                           bits at relative slack `slack` (row a11: D6 bit 0, D7 bit 1, D8 bit 2,
                           non-positive budget bit 3, Require bit 4, f_e box bit 5) -- the same
                           bits jdob_eval returns for the (n_tilde, mask, f_e) outputs; 0 for
                           BADPARAM/BADMODEL; bit 31 only ("not verified") for M_i > 32 */
    double slack;
} jdob_result;

/*
 * Bytes of caller-provided device workspace needed by jdob_solve_batch /
 * jdob_eval (which = 0) or jdob_bruteforce (which = 1) for these models (a HOST
 * array of n_models descriptors; only N and B_max are read), or by jdob_stats
 * (which = 2; models may be NULL).  Returns 0 on bad arguments.
 */
JDOB_API size_t jdob_workspace_bytes(const jdob_model *models, int32_t n_models, int32_t which);

/*
 * J-DOB over a batch of independent instances (rows a1-a8, a12 of DESIGN.md §Scope):
 * model aggregates u, v, phi, psi; per instance LC energy (P:296,
 * P:303), then Alg. 1: for n~ = 0..N-1 gamma, the sort by
 * descending gamma (R2 tie-break), thresholds Eq. (fth) (R1), the Alg. 2
 * edge-frequency sweep with greedy-batching set updates, the D6
 * guard, closed forms D20-D22 and strict-minimum updates; n~ = N is
 * local computing (R4).  Results are bit-identical to the CPU oracle under the
 * arithmetic contract.
 *   models   : HOST array of n_models descriptors (device table pointers).
 *   b        : HOST struct of DEVICE arrays; b->n_models == n_models.
 *   mode     : JDOB_MODE_*.
 *   out      : HOST struct of DEVICE output arrays.
 *   ws, ws_bytes : DEVICE workspace of >= jdob_workspace_bytes(models, n_models, 0).
 *   stream   : cudaStream_t as void* (NULL = legacy default stream).
 * Errors: JDOB_EINVAL (NULL required pointer, n_models < 1, N/B_max out of range,
 * small workspace, bad mode, n_buckets out of range), JDOB_ECUDA.
 */
JDOB_API int jdob_solve_batch(const jdob_model *models, int32_t n_models, const jdob_batch *b, int32_t mode,
                     const jdob_result *out, void *ws, size_t ws_bytes, void *stream);

/*
 * The paper's comparison set minus IP-SSA (NEXT-2) in ONE pass: J-DOB (JDOB_MODE_FULL) into
 * out[0], J-DOB without edge DVFS (JDOB_MODE_NO_EDGE_DVFS: f_e fixed at f_e,max, the j = 0
 * configurations) into out[1], and binary J-DOB (JDOB_MODE_BINARY: n~ in {0, N}, the n~ = 0
 * configurations) into out[2], from one validation, one LC evaluation and one pruned sweep per
 * instance (an n~ is visited while either pruned mode may still improve there; each mode keeps its own
 * strict (E, n~, j) minimum and all-local key, R8).  LC is every result's E_lc.  Every output is
 * bit-identical to jdob_solve_batch with that mode.
 *   models, b, ws, ws_bytes, stream : as jdob_solve_batch.
 *   out      : HOST array of 3 structs of DEVICE output arrays, each as jdob_solve_batch's `out`
 *              (f_user, partition and stats optional per mode); counts, work and violations must be
 *              NULL (JDOB_EINVAL otherwise).
 * Errors: as jdob_solve_batch.
 */
JDOB_API int jdob_solve_batch_modes(const jdob_model *models, int32_t n_models, const jdob_batch *b,
                                    const jdob_result *out, void *ws, size_t ws_bytes, void *stream);

/*
 * Energy-saving statistics (row a12; R16) of solved instances, as a call of
 * its own: the same bucketed fields, the same fixed reduction tree and the same bits as the
 * `stats` output of jdob_solve_batch (described there).
 *   b    : HOST struct; n_inst, user_off (device) and the optional bucket (device) are read.
 *   res  : HOST struct of DEVICE arrays: E, E_lc, f_e, n_tilde, status are read (the outputs of
 *          jdob_solve_batch for b); stats [n_buckets * JDOB_STATS_FIELDS] and n_buckets are
 *          written / read; the other members are ignored.
 *   ws   : DEVICE workspace of >= jdob_workspace_bytes(NULL, 0, 2) bytes.
 * Errors: JDOB_EINVAL (NULL arrays, n_buckets out of range, small workspace), JDOB_ECUDA.
 */
JDOB_API int jdob_stats(const jdob_batch *b, const jdob_result *res, void *ws, size_t ws_bytes, void *stream);

/*
 * The statistics of one part of a larger batch, for a multi-GPU fold with the same bits as one call
 * over the whole batch.  The fixed reduction tree of jdob_stats is defined on the
 * whole batch of n_total instances: 1024 leaves, leaf w = instances [n_total w / 1024,
 * n_total (w + 1) / 1024), folded pairwise (a dyadic tree; fields 0-2 and 5-9+ add, 3 max, 4 min).
 * `b` must hold exactly the instances [n_total part / parts, n_total (part + 1) / parts) with parts a
 * power of two <= 1024; the call writes the root of that part's subtree to res->stats.  Folding the
 * parts' roots pairwise in part order (paper_2504_14611_b200.dist.fold_stats) gives the same bits as
 * jdob_stats over the whole batch.  jdob_stats(b, ...) is jdob_stats_part(b, ..., b->n_inst, 1, 0, ...).
 * Errors: as jdob_stats, plus JDOB_EINVAL when (n_total, parts, part) does not describe `b`.
 */
JDOB_API int jdob_stats_part(const jdob_batch *b, const jdob_result *res, int64_t n_total, int32_t parts,
                             int32_t part, void *ws, size_t ws_bytes, void *stream);

/*
 * Same computation from HOST buffers (the end-to-end public call): copies the
 * model tables and the batch host->device, solves, copies E, E_lc, t_free_next,
 * f_e, n_tilde, j, status, mask (and f_user/stats when non-NULL) back to the host
 * arrays of `out`, and synchronises `stream` before returning.  Every pointer in
 * models/b/out is a HOST pointer (pinned memory gives asynchronous copies).
 * Device memory is stream-ordered, allocated from a memory pool private to the library
 * (cudaMallocFromPoolAsync) and returned to that pool before returning; the pool keeps the
 * largest call's footprint mapped for the next call (the device's default pool and the
 * caller's allocators are not touched) until jdob_release_pool() trims it.
 * Errors: as jdob_solve_batch, plus JDOB_EINVAL when the host user_off is not a
 * non-decreasing sequence starting at >= 0 (checked per chunk before its copies).
 * If `h2d_bytes`/`d2h_bytes` are non-NULL they receive the bytes copied.  The batch is processed in
 * chunks on three streams of the library (every chunk's copy-ins on one, each chunk's solve on a
 * second after its copy-ins, its copy-outs on a third after its solve), joined into `stream`
 * before the call returns; a chunk's copy-ins are one cudaMemcpyAsync per array.  The library's
 * streams are per device: host calls on one device from several threads are serialised by a lock.
 */
JDOB_API int jdob_solve_batch_host(const jdob_model *models, int32_t n_models, const jdob_batch *b, int32_t mode,
                          const jdob_result *out, void *stream, int64_t *h2d_bytes, int64_t *d2h_bytes);

/*
 * A batch whose users share their device parameters within each instance -- identical devices, the
 * setting of every experiment of the paper (Table I), where only the deadlines differ --
 * given with one copy of (zeta, kappa, f_min, f_max, R, p_u) per INSTANCE and T per user.  HOST
 * pointers (jdob_solve_shared_host).  Same meaning as jdob_batch otherwise.
 */
typedef struct {
    int64_t n_inst;
    int32_t n_models;
    const int32_t *model_id;
    const int64_t *user_off;
    const double *zeta, *kappa, *f_min, *f_max, *R, *p_u;  /* [n_inst]: the instance's users' values */
    const double *T;                                        /* [user_off[n_inst]] */
    const double *t_free, *fe_min, *fe_max, *rho;           /* [n_inst] */
    const int32_t *bucket;
} jdob_shared_batch;

/*
 * jdob_solve_batch_host for a jdob_shared_batch: the same computation and outputs (bit-identical to
 * jdob_solve_batch_host on the equivalent per-user arrays); a chunk's users are expanded on the device
 * from the instances' values (one small kernel), so the host->device traffic is 8 B per user + 48 B per
 * instance for the user parameters instead of 56 B per user.  Errors: as jdob_solve_batch_host.
 */
JDOB_API int jdob_solve_shared_host(const jdob_model *models, int32_t n_models, const jdob_shared_batch *b,
                                    int32_t mode, const jdob_result *out, void *stream, int64_t *h2d_bytes,
                                    int64_t *d2h_bytes);

/*
 * Release the device memory the library's private pool keeps between jdob_solve_batch_host
 * calls (cudaMemPoolTrimTo(pool, 0) on every device the library has used).  Host call; safe
 * when no jdob_solve_batch_host call is in flight.  Returns JDOB_OK or JDOB_ECUDA.
 */
JDOB_API int jdob_release_pool(void);

/*
 * Exhaustive search (rows a9-a10): argmin of the energy over candidate indices
 * [idx_begin, idx_end) of ONE instance (b->n_inst == 1), lowest index on ties.
 *   space 0 (general, reading R14): idx = vec*k + j with vec = sum_m n_m (N+1)^(M-1-m),
 *           n_m in {0..N} the partition point of user m (N = local), same-sub-task
 *           greedy batching b_n = #{m : n_m < n} (Fig. 1 caption P:75), ALAP batch
 *           starts, exact D6'/D7'/D13 feasibility.
 *   space 1 (identical, the (P1) space of P:224): idx = ((n~ 2^M + mask) k + j);
 *           n~ = N means all local.
 *   k = number of grid points f_e(j) = fe_max - j*rho >= fe_min.
 * Outputs (DEVICE scalars): *E_min (+inf if no feasible candidate in range),
 * *idx_min (-1 if none), *status (JDOB_ST_*; the search runs for OK and REQUIRE).
 * work (DEVICE int64[9], or NULL = skip): counters of the work the pruned scan executed
 * over the range: [0] vectors visited, [1] vectors past the user-term
 * bound, [2] past the n_min-only bound, [3] past the exact vector bound (grid loop
 * entered), [4] candidates evaluated (grid iterations, including the one that ends a
 * vector's scan), [5] device-frequency divisions executed, [6] candidates skipped by the
 * edge-only grid skip, [7] vectors whose D6' fails at the first grid point, [8] offloading
 * users summed over the evaluated candidates.  Requesting
 * them runs a counting instantiation of the same kernel (same result; the counts depend
 * on the order in which lanes publish their incumbents, so they vary slightly run to run).
 * Ranges beyond the space size are clipped.  Deterministic.  Unlike the other entry
 * points this call performs one small synchronous device->host read (user_off[0..1]
 * and model_id[0], 20 bytes) on `stream` to select the kernel specialisation for M;
 * the search itself is asynchronous.
 * Errors: JDOB_EINVAL (n_inst != 1, NULL pointers, idx_begin > idx_end, small
 * workspace), JDOB_ECUDA.
 */
JDOB_API int jdob_bruteforce(const jdob_model *models, int32_t n_models, const jdob_batch *b, int32_t space,
                    uint64_t idx_begin, uint64_t idx_end, double *E_min, int64_t *idx_min, int32_t *status,
                    int64_t *work, void *ws, size_t ws_bytes, void *stream);

/*
 * Host helper: size of the brute-force index space of an instance with N, M, k
 * (0 when >= 2^62).  Pure host arithmetic.
 */
JDOB_API uint64_t jdob_bf_space_size(int32_t space, int32_t N, int32_t M, int64_t k);

/*
 * Configuration evaluator (row a11): for given partition vectors and edge
 * frequencies, E (D21 generalised), t_free_next (D22 generalised, ASAP, R15),
 * device frequencies f* (D20) and violation bits: bit0 D6, bit1 any D7, bit2 any
 * D8, bit3 non-positive device budget, bit4 Require, bit5 f_e out of box.  A
 * constraint lhs <= rhs is violated when lhs > rhs + slack*|rhs|.
 * Used to re-verify every plan jdob_solve_batch returns.
 *   partition [user_off[n_inst]] (device int32): n_m in {0..N}, N = local; or NULL,
 *     in which case the configurations are identical-offloading plans given by
 *     plan_n_tilde [n_inst] and plan_mask [n_inst] (the n_tilde/mask outputs of
 *     jdob_solve_batch: user m offloads after block n~ iff bit m of mask is set).
 *   f_e [n_inst] (device): edge frequency per instance (ignored if all local).
 *   E, t_free_next [n_inst], f_user [users] (may be NULL), violations [n_inst],
 *   status [n_inst]: device outputs.
 *   ws: workspace of >= jdob_workspace_bytes(models, n_models, 0) bytes.
 * Errors: JDOB_EINVAL (NULL arrays, small workspace), JDOB_ECUDA.
 */
JDOB_API int jdob_eval(const jdob_model *models, int32_t n_models, const jdob_batch *b, const int32_t *partition,
                       const int32_t *plan_n_tilde, const uint32_t *plan_mask, const double *f_e, double slack,
                       double *E, double *t_free_next, double *f_user, uint32_t *violations, int32_t *status,
                       void *ws, size_t ws_bytes, void *stream);

/*
 * Outputs of jdob_solve_grouped (DEVICE pointers, caller-allocated).
 *   E [n_inst]            : total energy of the grouped schedule.
 *   t_free_next [n_inst]  : GPU-available time after the last group.
 *   n_groups [n_inst]     : number of groups (0 for a non-OK status).
 *   status [n_inst]       : JDOB_ST_* (a failed Require is costed inside the DP, so REQUIRE is
 *                           never reported here).
 *   group_of [users]      : group of each user, numbered in execution order (ascending deadlines).
 *   partition [users]     : partition point of each user (N = local).
 *   f_user [users]        : device frequency f* of each user (may be NULL).
 *   group_fe [n_inst*32]  : edge frequency of group g at [i*32 + g] (0.0 = all-local group).
 */
typedef struct {
    double *E, *t_free_next;
    int32_t *n_groups, *status;
    int32_t *group_of, *partition;
    double *f_user, *group_fe;
} jdob_grouped_result;

/* Workspace bytes of jdob_solve_grouped for a batch of n_inst instances and n_users users. */
JDOB_API size_t jdob_grouped_workspace_bytes(const jdob_model *models, int32_t n_models, int64_t n_inst,
                                            int64_t n_users);

/*
 * Outer grouping over deadline-sorted users with J-DOB as the inner module (
 * PAPER.md: "an outer module that groups users by deadline similarity" P:183, the optimal-
 * grouping DP of the different-deadline experiments P:430-431, reading R21 = SPEC S:295-303):
 * users sorted by deadline (ties by index); cell i of a DP over prefixes keeps the
 * lexicographically best (energy, t_free) of the first i users; the transition j -> i is the
 * group of sorted users j..i-1 solved by jdob (mode `mode`) at t_free = cell j's t_free; a
 * group whose earliest deadline is below that t_free is costed all-local (Alg. 1's Require,
 * P:259).  Bit-identical to the CPU oracle.  Performs one small synchronous device->host read
 * (the largest M, 4 bytes) to size the DP stages.
 * Errors: JDOB_EINVAL (NULL pointers, small workspace), JDOB_ECUDA.
 */
JDOB_API int jdob_solve_grouped(const jdob_model *models, int32_t n_models, const jdob_batch *b, int32_t mode,
                                const jdob_grouped_result *out, void *ws, size_t ws_bytes, void *stream);

/*
 * The C5 Monte Carlo workload generated on the device, so that a rank
 * solves instances it made itself with no input traffic.  INPUT PLUMBING, not the
 * method: the device twin of the host generator jdobgen.config_c5, bit-identical to
 * it (counter-based SplitMix64 draws keyed by (seed, instance id, user, field); per instance M ~
 * U{1..32}, model ~ U{0,1,2}, deadline regime ~ U{0..4}, rho from rho[3]; per user beta = 2.13 or
 * 30.25 (regimes 0, 1) or ~ U[4.5, 5.5], U[2, 8], U[0, 10] (regimes 2-4) and T = (1 + beta) lat[model]
 * (P:361); Table I users, optionally R and kappa scaled by U[0.5, 2]).  The host supplies the recipe's
 * constants so both generators use the same doubles.
 */
typedef struct {
    uint64_t seed;
    int64_t inst_begin;      /* global id of the first instance (shards generate their own range) */
    int32_t hetero;          /* 1: R and kappa scaled by U[0.5, 2] per user                       */
    double zeta, kappa, f_min, f_max, R, p_u;  /* Table I users                                    */
    double fe_min, fe_max;   /* edge frequency box                                                  */
    double rho[3];           /* the three sweep steps                                              */
    double lat[3];           /* per model: zeta v_N / f_max, the beta denominator of P:361         */
} jdob_gen_params;

/* Device workspace bytes of the two generator calls for n_inst instances (kept between them). */
JDOB_API size_t jdob_generate_workspace_bytes(int64_t n_inst);

/*
 * Generator phase 1: writes b->model_id, user_off [n_inst + 1], t_free, fe_min, fe_max, rho and
 * bucket (model * 5 + regime) of instances [p->inst_begin, p->inst_begin + b->n_inst) (DEVICE arrays
 * of `b`, caller-allocated; bucket = (model * 5 + regime) * 32 + M - 1), and the total user count user_off[n_inst] to the HOST *n_users (one
 * synchronous 8-byte read on `stream`), so the caller can size the user arrays.
 * Errors: JDOB_EINVAL (NULL arrays or n_users, small workspace), JDOB_ECUDA.
 */
JDOB_API int jdob_generate_c5_instances(const jdob_gen_params *p, const jdob_batch *b, int64_t *n_users, void *ws,
                                        size_t ws_bytes, void *stream);

/*
 * Generator phase 2: writes the user arrays zeta, kappa, f_min, f_max, R, p_u, T [n_users] of `b`
 * (DEVICE, caller-allocated), reading the model_id and user_off phase 1 wrote and its workspace.
 * Asynchronous.  Errors: JDOB_EINVAL (NULL arrays, small workspace), JDOB_ECUDA.
 */
JDOB_API int jdob_generate_c5_users(const jdob_gen_params *p, const jdob_batch *b, void *ws, size_t ws_bytes,
                                    void *stream);

/* Message of the last call-level error on this thread ("" if none). */
JDOB_API const char *jdob_last_error(void);

/* Library version string. */
JDOB_API const char *jdob_version(void);

#ifdef __cplusplus
}
#endif
#endif /* JDOB_H */
