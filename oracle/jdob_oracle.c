/*
 * jdob_oracle.c -- plain, slow, obviously-correct CPU oracle for the J-DOB hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  It shares no code,
 * header, table or constant with the CUDA path (paper_2504_14611_b200/csrc) and
 * must never be called from the product path.
 *
 * Source of truth: /root/reference/PAPER.md ("P:n" = line n) -- arXiv 2504.14611,
 * "Joint Optimization of Offloading, Batching and DVFS for Multiuser Co-Inference".
 * Readings where the paper is silent/ambiguous are R1..R16 of DESIGN.md §Readings.
 *
 * Build: gcc -O2 -std=c11 -ffp-contract=off -fno-fast-math (IEEE-754 binary64, RNE,
 * no FMA contraction).  Every floating-point expression is written in the order
 * fixed by DESIGN.md §Arithmetic contract; nothing is blocked, fused or reordered.
 *
 * Pins (tests/test_oracle_*.py): hand-derived golden values (tests/golden/), closed
 * forms, D20 vs. numeric minimisation, invariants (J-DOB <= LC, thresholds
 * non-increasing, plan feasibility, BF-general <= BF-identical <= J-DOB,
 * J-DOB == BF-identical at M = 1), independent brute force on tiny inputs.
 * "parity unpinned": absolute BF-general values on non-identical vectors beyond the
 * toy-4 hand check (the paper never evaluates that space).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ---- status codes (numbering documented in DESIGN.md §Status) ---- */
#define O_ST_OK 0
#define O_ST_LOCAL_INFEASIBLE 1
#define O_ST_REQUIRE 2
#define O_ST_BADPARAM 3
#define O_ST_BADMODEL 4
#define O_ST_TOOBIG 5

#define O_MAXM 32          /* brute force, grouping, offload mask */
#define O_MAXM_LARGE 1024  /* J-DOB, LC, eval (NEXT-4: M > 32) */
#define O_MAXN 63
#define O_MAXK 65536

typedef struct {
    int N, B_max;
    const double *A, *O, *g, *q; /* [N+1] */
    const double *d, *c;         /* [(N+1)*(B_max+1)], element n*(B_max+1)+b */
} o_model;

typedef struct {
    int M;
    const double *zeta, *kappa, *f_min, *f_max, *R, *p_u, *T; /* [M] */
    double t_free, fe_min, fe_max, rho;
} o_inst;

typedef struct {
    double E, E_lc, t_free_next, f_e;
    int n_tilde, j, status;
    unsigned mask;
    double f_user[O_MAXM_LARGE];
    int part[O_MAXM_LARGE]; /* per user: partition point n~* if offloading, else N */
    /* algorithmic work counters: the literal Alg. 1/2 loop counts */
    long long n_visit;   /* (n~, j) pairs visited by the sweep (guard evaluated)            */
    long long n_eval;    /* (n~, j) pairs that passed the guard and were evaluated (D20-D22) */
    long long n_member;  /* sum over evaluated pairs of B_o (one Gamma division each)         */
} o_result;

static const double O_INF = HUGE_VAL;

/* ------------------------------------------------------------------ */
/* Model access and aggregates.                            */
/* ------------------------------------------------------------------ */
static double o_d(const o_model *m, int n, int b) { return m->d[n * (m->B_max + 1) + b]; }
static double o_c(const o_model *m, int n, int b) { return m->c[n * (m->B_max + 1) + b]; }

/* u_n~ = sum_{n=0}^{n~} q_n A_n, ascending n. */
static double o_u(const o_model *m, int nt) {
    double s = 0.0;
    for (int n = 0; n <= nt; n++) s = s + m->q[n] * m->A[n];
    return s;
}
/* v_n~ = sum_{n=0}^{n~} g_n A_n, ascending n. */
static double o_v(const o_model *m, int nt) {
    double s = 0.0;
    for (int n = 0; n <= nt; n++) s = s + m->g[n] * m->A[n];
    return s;
}
/* phi_n~(b) = sum_{n=n~+1}^{N} d_n(b) A_n; accumulated from n = N downward.
 * phi(0) = 0 (R5). */
static double o_phi(const o_model *m, int nt, int b) {
    if (b == 0) return 0.0;
    double s = 0.0;
    for (int n = m->N; n >= nt + 1; n--) s = s + o_d(m, n, b) * m->A[n];
    return s;
}
/* psi_n~(b) = sum_{n=n~+1}^{N} c_n(b) A_n; accumulated from n = N downward. */
static double o_psi(const o_model *m, int nt, int b) {
    if (b == 0) return 0.0;
    double s = 0.0;
    for (int n = m->N; n >= nt + 1; n--) s = s + o_c(m, n, b) * m->A[n];
    return s;
}

/* Frequency clamp of D20: min{max{G, f_min}, f_max}. */
static double o_clamp(double G, double fmin, double fmax) {
    double x = (G < fmin) ? fmin : G;
    return (x > fmax) ? fmax : x;
}

/* Edge grid f_e(j) = f_e,max - j*rho (R7: one multiply, one subtract). */
static double o_fe(const o_inst *in, long long j) { return in->fe_max - (double)j * in->rho; }

/* Grid size k: number of j with f_e(j) >= f_e,min (the literal while-condition of Alg. 2,
 * P:328), counted by walking the grid. Returns -1 above O_MAXK. */
static long long o_grid_k(const o_inst *in) {
    long long k = 0;
    while (o_fe(in, k) >= in->fe_min) {
        k++;
        if (k > O_MAXK) return -1;
    }
    return k;
}

static int o_finite(double x) { return isfinite(x); }

/* Model validation: A_0 = 0, A_n > 0 (n >= 1), O, g, q >= 0,
 * d_n(b) > 0 and non-decreasing in b, c_n(b) >= 0 (Fig. 3 trend). */
int oracle_check_model(const o_model *m) {
    if (m->N < 1 || m->N > O_MAXN || m->B_max < 1 || m->B_max > O_MAXM_LARGE) return O_ST_BADMODEL;
    if (!(m->A[0] == 0.0)) return O_ST_BADMODEL;
    for (int n = 0; n <= m->N; n++) {
        if (!o_finite(m->A[n]) || !o_finite(m->O[n]) || !o_finite(m->g[n]) || !o_finite(m->q[n]))
            return O_ST_BADMODEL;
        if (n >= 1 && !(m->A[n] > 0.0)) return O_ST_BADMODEL;
        if (!(m->O[n] >= 0.0) || !(m->g[n] >= 0.0) || !(m->q[n] >= 0.0)) return O_ST_BADMODEL;
    }
    for (int n = 1; n <= m->N; n++) {
        for (int b = 1; b <= m->B_max; b++) {
            double d = o_d(m, n, b), c = o_c(m, n, b);
            if (!o_finite(d) || !o_finite(c) || !(d > 0.0) || !(c >= 0.0)) return O_ST_BADMODEL;
            if (b >= 2 && !(d >= o_d(m, n, b - 1))) return O_ST_BADMODEL;
        }
    }
    return O_ST_OK;
}

/* Instance validation: parameter boxes, local feasibility,
 * Require of Alg. 1. */
int oracle_check_inst(const o_model *m, const o_inst *in) {
    if (oracle_check_model(m) != O_ST_OK) return O_ST_BADMODEL;
    if (in->M < 1 || in->M > O_MAXM_LARGE || in->M > m->B_max) return O_ST_BADPARAM;
    for (int i = 0; i < in->M; i++) {
        double z = in->zeta[i], k = in->kappa[i], f0 = in->f_min[i], f1 = in->f_max[i];
        double R = in->R[i], p = in->p_u[i], T = in->T[i];
        if (!o_finite(z) || !o_finite(k) || !o_finite(f0) || !o_finite(f1) || !o_finite(R) ||
            !o_finite(p) || !o_finite(T))
            return O_ST_BADPARAM;
        if (!(z >= 0.0) || !(k >= 0.0) || !(f0 > 0.0) || !(f0 <= f1) || !(R > 0.0) || !(p >= 0.0) ||
            !(T > 0.0))
            return O_ST_BADPARAM;
    }
    if (!o_finite(in->t_free) || !o_finite(in->fe_min) || !o_finite(in->fe_max) || !o_finite(in->rho))
        return O_ST_BADPARAM;
    if (!(in->t_free >= 0.0) || !(in->fe_min > 0.0) || !(in->fe_min <= in->fe_max) || !(in->rho > 0.0))
        return O_ST_BADPARAM;
    if (o_grid_k(in) < 0) return O_ST_BADPARAM;
    double vN = o_v(m, m->N);
    for (int i = 0; i < in->M; i++) {
        /* zeta sum g A / f_max <= T */
        if ((in->zeta[i] * vN) / in->f_max[i] > in->T[i]) return O_ST_LOCAL_INFEASIBLE;
    }
    double Tmin = O_INF;
    for (int i = 0; i < in->M; i++)
        if (in->T[i] < Tmin) Tmin = in->T[i];
    if (Tmin < in->t_free) return O_ST_REQUIRE; /* Require: min T >= t_free */
    return O_ST_OK;
}

/* ------------------------------------------------------------------ */
/* Local computing (LC), P:388 benchmark (i); D20/D21 local branch. */
/* f_m = clamp(zeta_m v_N / T_m, f_min, f_max); e_m = kappa_m u_N f_m^2.           */
/* ------------------------------------------------------------------ */
double oracle_lc(const o_model *m, const o_inst *in, double *f_loc, double *e_loc) {
    double uN = o_u(m, m->N), vN = o_v(m, m->N);
    double E = 0.0;
    for (int i = 0; i < in->M; i++) {
        double G = (in->zeta[i] * vN) / in->T[i];
        double f = o_clamp(G, in->f_min[i], in->f_max[i]);
        double e = ((in->kappa[i] * uN) * f) * f;
        if (f_loc) f_loc[i] = f;
        if (e_loc) e_loc[i] = e;
        E = E + e; /* user-index order (R13) */
    }
    return E;
}

/* ------------------------------------------------------------------ */
/* Alg. 1 lines 4-6 for one partition point n~.            */
/* gamma_m = O_n~/R_m + zeta_m v_n~ / f_m,max                  */
/* list = users sorted by descending gamma; ties: T ascending, then     */
/* user index ascending (R2).                                           */
/* th_i = phi_n~(M - i) / (min_{i' >= i} T_list[i'] - gamma_list[i])    */
/*   (Eq. fth; 0-based i, R1).                                    */
/* ------------------------------------------------------------------ */
static int o_key_before(const o_inst *in, const double *gamma, int a, int b) {
    /* returns 1 iff user a precedes user b in list(M') */
    if (gamma[a] > gamma[b]) return 1;
    if (gamma[a] < gamma[b]) return 0;
    if (in->T[a] < in->T[b]) return 1;
    if (in->T[a] > in->T[b]) return 0;
    return a < b;
}

void oracle_thresholds(const o_model *m, const o_inst *in, int nt, double *gamma, int *list, double *th) {
    int M = in->M;
    double vn = o_v(m, nt);
    for (int i = 0; i < M; i++) gamma[i] = m->O[nt] / in->R[i] + (in->zeta[i] * vn) / in->f_max[i];
    /* plain insertion sort by the key (O(M^2), M <= 32) */
    for (int i = 0; i < M; i++) list[i] = i;
    for (int i = 1; i < M; i++) {
        int x = list[i], p = i - 1;
        while (p >= 0 && o_key_before(in, gamma, x, list[p])) {
            list[p + 1] = list[p];
            p--;
        }
        list[p + 1] = x;
    }
    for (int i = 0; i < M; i++) {
        double Lmin = O_INF;
        for (int k = i; k < M; k++)
            if (in->T[list[k]] < Lmin) Lmin = in->T[list[k]];
        th[i] = o_phi(m, nt, M - i) / (Lmin - gamma[list[i]]);
    }
}

/* ------------------------------------------------------------------ */
/* D20-D22 for identical offloading at (n~, set, f_e).       */
/* budget_m = (l_o - O_n~/R_m) - phi_n~(B_o) * (1/f_e)      (R13, Eq. 5)  */
/* Gamma_m = zeta_m v_n~ / budget_m; f* = clamp (J-DOB clamps, R10);      */
/* zeta_m v_n~ = 0 -> f* = f_min (R9).                                     */
/* E = sum_m e_m (user order) + (psi * f_e) * f_e                          */
/* t_free* = max(t_free, max_m (zeta v / f* + O/R)) + phi * (1/f_e)        */
/* ------------------------------------------------------------------ */
static double o_eval_p1(const o_model *m, const o_inst *in, int nt, const int *member, int B_o, double l_o,
                        double fe, const double *f_loc, const double *e_loc, double *fstar, double *tf_out) {
    double inv = 1.0 / fe;
    double phi = o_phi(m, nt, B_o), psi = o_psi(m, nt, B_o);
    double te = phi * inv;
    double u = o_u(m, nt), v = o_v(m, nt);
    double E = 0.0, arr_max = in->t_free;
    for (int i = 0; i < in->M; i++) {
        double e, f;
        if (member[i]) {
            double OR = m->O[nt] / in->R[i];
            double zv = in->zeta[i] * v;
            if (zv == 0.0) {
                f = in->f_min[i];
            } else {
                double budget = (l_o - OR) - te;
                double G = zv / budget;
                f = o_clamp(G, in->f_min[i], in->f_max[i]);
            }
            e = ((in->kappa[i] * u) * f) * f + OR * in->p_u[i];
            double arr = zv / f + OR;
            if (arr > arr_max) arr_max = arr;
        } else {
            f = f_loc[i];
            e = e_loc[i];
        }
        if (fstar) fstar[i] = f;
        E = E + e;
    }
    E = E + (psi * fe) * fe;
    if (tf_out) *tf_out = arr_max + te;
    return E;
}

/* ------------------------------------------------------------------ */
/* J-DOB: Alg. 1 calling Alg. 2, literally.      */
/* mode 0 full; 1 LC only; 2 no edge DVFS (k = 1 at f_e,max);     */
/* 3 binary offloading (n~ in {0, N}).                           */
/* ------------------------------------------------------------------ */
int oracle_jdob(const o_model *m, const o_inst *in, int mode, o_result *r) {
    memset(r, 0, sizeof(*r));
    int st = oracle_check_inst(m, in);
    r->status = st;
    int M = in->M;
    double f_loc[O_MAXM_LARGE], e_loc[O_MAXM_LARGE];
    if (st == O_ST_BADPARAM || st == O_ST_BADMODEL) {
        r->E = r->E_lc = NAN;
        r->t_free_next = in->t_free;
        r->n_tilde = (m->N >= 1 && m->N <= O_MAXN) ? m->N : 0;
        for (int i = 0; i < O_MAXM_LARGE; i++) r->f_user[i] = NAN;
        for (int i = 0; i < O_MAXM_LARGE; i++) r->part[i] = r->n_tilde;
        return st;
    }
    double E_lc = oracle_lc(m, in, f_loc, e_loc);
    r->E_lc = E_lc;
    /* canonical all-local answer (R8, R11, R12) */
    r->E = E_lc;
    r->t_free_next = in->t_free;
    r->f_e = 0.0;
    r->n_tilde = m->N;
    r->j = 0;
    r->mask = 0u;
    for (int i = 0; i < M; i++) {
        r->f_user[i] = f_loc[i];
        r->part[i] = m->N;
    }
    if (st != O_ST_OK || mode == 1) return st;

    long long k_full = o_grid_k(in);
    double E_star = O_INF;
    int best_nt = -1, best_j = 0;
    unsigned best_mask = 0u;
    double best_fe = 0.0, best_tf = in->t_free, best_f[O_MAXM_LARGE];
    static _Thread_local int best_mem[O_MAXM_LARGE], nt_mem[O_MAXM_LARGE];
    int best_any = 0;

    for (int nt = 0; nt <= m->N; nt++) { /* Alg. 1 line 3: traverse partition points */
        if (mode == 3 && nt != 0 && nt != m->N) continue;
        if (nt == m->N) {
            /* R4: n~ = N means local computing: offload set empty, E = E_LC. */
            if (E_lc < E_star) {
                E_star = E_lc;
                best_nt = nt;
                best_j = 0;
                best_mask = 0u;
                best_any = 0;
                best_fe = 0.0;
                best_tf = in->t_free;
                for (int i = 0; i < M; i++) best_f[i] = f_loc[i];
            }
            continue;
        }
        double gamma[O_MAXM_LARGE], th[O_MAXM_LARGE];
        int list[O_MAXM_LARGE];
        oracle_thresholds(m, in, nt, gamma, list, th);

        /* ---- Alg. 2 ---- */
        double E_nt = O_INF;
        int have = 0, nt_j = 0;
        unsigned nt_mask = 0u;
        double nt_fe = 0.0, nt_tf = in->t_free, nt_f[O_MAXM_LARGE];
        int nt_any = 0;
        int ihat = -1; /* -1 encodes "NAN" (R3) */
        for (int i = 0; i < M; i++)
            if (th[i] >= 0.0) {
                ihat = i;
                break;
            }
        int member[O_MAXM_LARGE];
        for (int i = 0; i < M; i++) member[i] = 0;
        if (ihat >= 0)
            for (int i = ihat; i < M; i++) member[list[i]] = 1;
        int B_o = 0;
        double l_o = O_INF;
        for (int i = 0; i < M; i++)
            if (member[i]) {
                B_o++;
                if (in->T[i] < l_o) l_o = in->T[i];
            }
        long long k = (mode == 2) ? 1 : k_full;
        long long j = 0;
        double fe = o_fe(in, j);
        while (fe >= in->fe_min && j < k) { /* sweep edge frequency */
            if (ihat >= 0) {                /* update greedy batching set */
                while (ihat < M && fe < th[ihat]) {
                    member[list[ihat]] = 0;
                    l_o = O_INF;
                    B_o = 0;
                    for (int i = 0; i < M; i++)
                        if (member[i]) {
                            B_o++;
                            if (in->T[i] < l_o) l_o = in->T[i];
                        }
                    ihat++;
                }
            }
            r->n_visit++;
            /* optimal device DVFS under the GPU-occupation guard */
            if (fe >= o_phi(m, nt, B_o) / (l_o - in->t_free)) {
                double fstar[O_MAXM_LARGE], tf;
                double E = o_eval_p1(m, in, nt, member, B_o, l_o, fe, f_loc, e_loc, fstar, &tf);
                r->n_eval++;
                r->n_member += B_o;
                if (E < E_nt) { /* strict improvement */
                    E_nt = E;
                    have = 1;
                    nt_j = (int)j;
                    nt_fe = fe;
                    nt_tf = tf;
                    nt_mask = 0u;
                    nt_any = 0;
                    for (int i = 0; i < M; i++) {
                        if (member[i] && i < 32) nt_mask |= (1u << i);
                        nt_mem[i] = member[i];
                        nt_any |= member[i];
                        nt_f[i] = fstar[i];
                    }
                }
            }
            if (B_o == 0) break;
            j++;
            fe = o_fe(in, j);
        }
        if (have && E_nt < E_star) { /* Alg. 1 strict improvement */
            E_star = E_nt;
            best_nt = nt;
            best_j = nt_j;
            best_mask = nt_mask;
            best_any = nt_any;
            best_fe = nt_fe;
            best_tf = nt_tf;
            for (int i = 0; i < M; i++) {
                best_f[i] = nt_f[i];
                best_mem[i] = nt_mem[i];
            }
        }
    }
    if (best_nt >= 0 && best_any) {
        r->E = E_star;
        r->n_tilde = best_nt;
        r->j = best_j;
        r->mask = best_mask; /* users 0..31 only (M <= 32 instances) */
        r->f_e = best_fe;
        r->t_free_next = best_tf;
        for (int i = 0; i < M; i++) {
            r->f_user[i] = best_f[i];
            r->part[i] = best_mem[i] ? best_nt : m->N;
        }
    }
    /* otherwise the winner is an all-local evaluation: keep the canonical answer (R8). */
    return st;
}

/* ------------------------------------------------------------------ */
/* Brute force (plain definitions, R14).                       */
/* space 0 (general): idx = vec * k + j, vec = sum_m n_m (N+1)^(M-1-m),   */
/*   n_m in {0..N}, n_m = N means local.                                 */
/* space 1 (identical, (P1) exhaustive space P:224): idx = ((n~ 2^M +    */
/*   mask) k + j); n~ = N means all local.                        */
/* Objective: D21 generalised; constraints D6/D7 generalised with ALAP    */
/* batch starts s_n = l_o - S_n / f_e (R14), exact feasibility (R10).     */
/* ------------------------------------------------------------------ */
static int o_space_size(const o_model *m, const o_inst *in, int space, unsigned long long *size) {
    if (in->M > O_MAXM) return O_ST_TOOBIG;
    long long k = o_grid_k(in);
    if (k <= 0) return O_ST_BADPARAM;
    unsigned long long lim = (1ull << 62);
    unsigned long long s = (unsigned long long)k;
    if (space == 0) {
        for (int i = 0; i < in->M; i++) {
            if (s > lim / (unsigned long long)(m->N + 1)) return O_ST_TOOBIG;
            s *= (unsigned long long)(m->N + 1);
        }
    } else {
        if (in->M > 40) return O_ST_TOOBIG;
        unsigned long long f = (unsigned long long)(m->N + 1) << in->M;
        if (s > lim / f) return O_ST_TOOBIG;
        s *= f;
    }
    *size = s;
    return O_ST_OK;
}

unsigned long long oracle_bf_space_size(const o_model *m, const o_inst *in, int space) {
    unsigned long long s = 0;
    if (o_space_size(m, in, space, &s) != O_ST_OK) return 0ull;
    return s;
}

/* Decode a candidate index into a partition vector and a grid index. */
static void o_decode(const o_model *m, const o_inst *in, int space, unsigned long long idx, int *nvec,
                     long long *j) {
    long long k = o_grid_k(in);
    *j = (long long)(idx % (unsigned long long)k);
    unsigned long long t = idx / (unsigned long long)k;
    if (space == 0) {
        for (int i = in->M - 1; i >= 0; i--) {
            nvec[i] = (int)(t % (unsigned long long)(m->N + 1));
            t /= (unsigned long long)(m->N + 1);
        }
    } else {
        unsigned long long mask = t & ((1ull << in->M) - 1ull);
        int nt = (int)(t >> in->M);
        for (int i = 0; i < in->M; i++) nvec[i] = (nt < m->N && ((mask >> i) & 1ull)) ? nt : m->N;
    }
}

/* Evaluate one general configuration (partition vector + f_e).
 * Returns E, or +inf when infeasible (exact checks).  fstar optional. */
static double o_general(const o_model *m, const o_inst *in, const int *nvec, double fe, const double *f_loc,
                        const double *e_loc, double *fstar) {
    int M = in->M, N = m->N;
    int b[O_MAXN + 2];
    double S[O_MAXN + 2], Psi = 0.0;
    /* greedy same-sub-task batching (Fig. 1 caption P:75): b_n = #{m : n_m < n} */
    for (int n = 1; n <= N; n++) {
        b[n] = 0;
        for (int i = 0; i < M; i++)
            if (nvec[i] < n) b[n]++;
    }
    S[N + 1] = 0.0;
    for (int n = N; n >= 1; n--) {
        S[n] = S[n + 1] + (b[n] > 0 ? o_d(m, n, b[n]) * m->A[n] : 0.0);
        Psi = Psi + (b[n] > 0 ? o_c(m, n, b[n]) * m->A[n] : 0.0);
    }
    int any = 0, nmin = N;
    double l_o = O_INF;
    for (int i = 0; i < M; i++)
        if (nvec[i] < N) {
            any = 1;
            if (nvec[i] < nmin) nmin = nvec[i];
            if (in->T[i] < l_o) l_o = in->T[i];
        }
    double inv = 1.0 / fe;
    if (any) {
        /* D6': GPU free before the first batch starts (P:205 generalised) */
        if (!(in->t_free + S[nmin + 1] * inv <= l_o)) return O_INF;
    }
    double E = 0.0;
    for (int i = 0; i < M; i++) {
        double e, f;
        if (nvec[i] < N) {
            int n = nvec[i];
            double OR = m->O[n] / in->R[i];
            double zv = in->zeta[i] * o_v(m, n);
            double budget = (l_o - OR) - S[n + 1] * inv;
            if (zv == 0.0) {
                if (!(budget >= 0.0)) return O_INF;
                f = in->f_min[i];
            } else {
                if (!(budget > 0.0)) return O_INF;
                double G = zv / budget;
                if (G > in->f_max[i]) return O_INF; /* D7' with D13 (exact, R10) */
                f = (G < in->f_min[i]) ? in->f_min[i] : G;
            }
            e = ((in->kappa[i] * o_u(m, n)) * f) * f + OR * in->p_u[i];
        } else {
            f = f_loc[i];
            e = e_loc[i];
        }
        if (fstar) fstar[i] = f;
        E = E + e;
    }
    E = E + (Psi * fe) * fe;
    return E;
}

double oracle_bf_candidate(const o_model *m, const o_inst *in, int space, unsigned long long idx) {
    int st = oracle_check_inst(m, in);
    if (st != O_ST_OK && st != O_ST_REQUIRE) return NAN;
    double f_loc[O_MAXM], e_loc[O_MAXM];
    oracle_lc(m, in, f_loc, e_loc);
    int nvec[O_MAXM];
    long long j;
    o_decode(m, in, space, idx, nvec, &j);
    return o_general(m, in, nvec, o_fe(in, j), f_loc, e_loc, NULL);
}

/* Argmin over [idx_begin, idx_end) with the lowest-index tie-break (strict <). */
int oracle_bf(const o_model *m, const o_inst *in, int space, unsigned long long idx_begin,
              unsigned long long idx_end, double *E_min, long long *idx_min) {
    *E_min = O_INF;
    *idx_min = -1;
    int st = oracle_check_inst(m, in);
    if (st != O_ST_OK && st != O_ST_REQUIRE) return st;
    unsigned long long size;
    int s2 = o_space_size(m, in, space, &size);
    if (s2 != O_ST_OK) return s2;
    if (idx_end > size) idx_end = size;
    double f_loc[O_MAXM], e_loc[O_MAXM];
    oracle_lc(m, in, f_loc, e_loc);
    int nvec[O_MAXM];
    for (unsigned long long idx = idx_begin; idx < idx_end; idx++) {
        long long j;
        o_decode(m, in, space, idx, nvec, &j);
        double E = o_general(m, in, nvec, o_fe(in, j), f_loc, e_loc, NULL);
        if (E < *E_min) {
            *E_min = E;
            *idx_min = (long long)idx;
        }
    }
    return O_ST_OK;
}

/* ------------------------------------------------------------------ */
/* jdob_eval semantics (a11): D20-D22 and their R14/R15 generalisation. */
/* violations: bit0 D6, bit1 any D7, bit2 any D8, bit3 non-positive      */
/* budget, bit4 Require, bit5 f_e outside [f_e,min, f_e,max].            */
/* A constraint lhs <= rhs is violated when lhs > rhs + slack*|rhs|.      */
/* ------------------------------------------------------------------ */
int oracle_eval(const o_model *m, const o_inst *in, const int *nvec, double fe, double slack, double *E_out,
                double *tf_out, double *fstar, unsigned *viol_out) {
    int st = oracle_check_inst(m, in);
    *viol_out = 0u;
    if (st == O_ST_BADPARAM || st == O_ST_BADMODEL) {
        *E_out = NAN;
        *tf_out = NAN;
        return st;
    }
    int M = in->M, N = m->N;
    double f_loc[O_MAXM_LARGE], e_loc[O_MAXM_LARGE];
    oracle_lc(m, in, f_loc, e_loc);
    unsigned viol = 0u;
    double vN = o_v(m, N);
    double Tmin = O_INF;
    for (int i = 0; i < M; i++)
        if (in->T[i] < Tmin) Tmin = in->T[i];
    if (Tmin < in->t_free) viol |= 16u;
    int b[O_MAXN + 2];
    double S[O_MAXN + 2], Psi = 0.0;
    for (int n = 1; n <= N; n++) {
        b[n] = 0;
        for (int i = 0; i < M; i++)
            if (nvec[i] < n) b[n]++;
    }
    S[N + 1] = 0.0;
    for (int n = N; n >= 1; n--) {
        S[n] = S[n + 1] + (b[n] > 0 ? o_d(m, n, b[n]) * m->A[n] : 0.0);
        Psi = Psi + (b[n] > 0 ? o_c(m, n, b[n]) * m->A[n] : 0.0);
    }
    int any = 0, nmin = N;
    double l_o = O_INF;
    for (int i = 0; i < M; i++)
        if (nvec[i] < N) {
            any = 1;
            if (nvec[i] < nmin) nmin = nvec[i];
            if (in->T[i] < l_o) l_o = in->T[i];
        }
    double inv = 1.0 / fe;
    double tol = slack * fabs(l_o);
    double tf = in->t_free;
    if (any) {
        if (!(fe >= in->fe_min && fe <= in->fe_max)) viol |= 32u;
        double start = in->t_free + S[nmin + 1] * inv;
        if (start > l_o + tol) viol |= 1u;
        tf = start;
    }
    double E = 0.0;
    for (int i = 0; i < M; i++) {
        double e, f;
        if (nvec[i] < N) {
            int n = nvec[i];
            double OR = m->O[n] / in->R[i];
            double zv = in->zeta[i] * o_v(m, n);
            double budget = (l_o - OR) - S[n + 1] * inv;
            if (zv == 0.0) {
                if (budget < 0.0) viol |= 8u;
                f = in->f_min[i];
            } else if (budget > 0.0) {
                double G = zv / budget;
                f = o_clamp(G, in->f_min[i], in->f_max[i]);
            } else {
                viol |= 8u;
                f = in->f_max[i];
            }
            e = ((in->kappa[i] * o_u(m, n)) * f) * f + OR * in->p_u[i];
            double arr = zv / f + OR;
            double fin = arr + S[n + 1] * inv;
            if (fin > l_o + tol) viol |= 2u;
            if (fin > tf) tf = fin;
        } else {
            f = f_loc[i];
            e = e_loc[i];
            if ((in->zeta[i] * vN) / f > in->T[i] + slack * fabs(in->T[i])) viol |= 4u;
        }
        if (fstar) fstar[i] = f;
        E = E + e;
    }
    E = E + (Psi * fe) * fe;
    *E_out = E;
    *tf_out = tf;
    *viol_out = viol;
    return st;
}

/* ------------------------------------------------------------------ */
/* Batch drivers (harness: loops over independent instances; optional   */
/* static thread split for the CPU-baseline timing).                      */
/* ------------------------------------------------------------------ */
typedef struct {
    const o_model *models;
    const int *model_id;
    const long long *user_off;
    const double *zeta, *kappa, *f_min, *f_max, *R, *p_u, *T;
    const double *t_free, *fe_min, *fe_max, *rho;
} o_batch;

static void o_make_inst(const o_batch *b, long long i, o_inst *in) {
    long long o = b->user_off[i];
    in->M = (int)(b->user_off[i + 1] - o);
    in->zeta = b->zeta + o;
    in->kappa = b->kappa + o;
    in->f_min = b->f_min + o;
    in->f_max = b->f_max + o;
    in->R = b->R + o;
    in->p_u = b->p_u + o;
    in->T = b->T + o;
    in->t_free = b->t_free[i];
    in->fe_min = b->fe_min[i];
    in->fe_max = b->fe_max[i];
    in->rho = b->rho[i];
}

typedef struct {
    double *E, *E_lc, *t_free_next, *f_e, *f_user;
    int *n_tilde, *j, *status;
    unsigned *mask;
    long long *counts; /* [n_inst*3] n_visit, n_eval, n_member, or NULL */
    int *part;         /* [users] partition point per user, or NULL */
} o_out;

typedef struct {
    const o_batch *b;
    const o_out *out;
    int mode;
    long long i0, i1;
} o_job;

static void *o_solve_range(void *arg) {
    o_job *jb = (o_job *)arg;
    const o_batch *b = jb->b;
    const o_out *out = jb->out;
    for (long long i = jb->i0; i < jb->i1; i++) {
        o_inst in;
        o_make_inst(b, i, &in);
        o_result r;
        const o_model *m = &b->models[b->model_id[i]];
        if (in.M < 1 || in.M > O_MAXM_LARGE) {
            memset(&r, 0, sizeof(r));
            r.status = O_ST_BADPARAM;
            r.E = r.E_lc = NAN;
            r.t_free_next = in.t_free;
            r.n_tilde = m->N;
        } else {
            oracle_jdob(m, &in, jb->mode, &r);
        }
        out->E[i] = r.E;
        out->E_lc[i] = r.E_lc;
        out->t_free_next[i] = r.t_free_next;
        out->f_e[i] = r.f_e;
        out->n_tilde[i] = r.n_tilde;
        out->j[i] = r.j;
        out->status[i] = r.status;
        out->mask[i] = r.mask;
        if (out->f_user && in.M >= 1 && in.M <= O_MAXM_LARGE)
            for (int u = 0; u < in.M; u++) out->f_user[b->user_off[i] + u] = r.f_user[u];
        if (out->part && in.M >= 1 && in.M <= O_MAXM_LARGE)
            for (int u = 0; u < in.M; u++) out->part[b->user_off[i] + u] = r.part[u];
        if (out->counts) {
            out->counts[3 * i + 0] = r.n_visit;
            out->counts[3 * i + 1] = r.n_eval;
            out->counts[3 * i + 2] = r.n_member;
        }
    }
    return NULL;
}

int oracle_solve_batch(const o_batch *b, long long n_inst, int mode, const o_out *out, int n_threads) {
    if (n_threads < 1) n_threads = 1;
    if (n_threads > 256) n_threads = 256;
    if (n_threads == 1 || n_inst < 2) {
        o_job jb = {b, out, mode, 0, n_inst};
        o_solve_range(&jb);
        return 0;
    }
    pthread_t th[256];
    o_job jobs[256];
    for (int t = 0; t < n_threads; t++) {
        jobs[t].b = b;
        jobs[t].out = out;
        jobs[t].mode = mode;
        jobs[t].i0 = n_inst * t / n_threads;
        jobs[t].i1 = n_inst * (t + 1) / n_threads;
        pthread_create(&th[t], NULL, o_solve_range, &jobs[t]);
    }
    for (int t = 0; t < n_threads; t++) pthread_join(th[t], NULL);
    return 0;
}

typedef struct {
    const o_model *m;
    const o_inst *in;
    int space;
    unsigned long long i0, i1;
    double E;
    long long idx;
    int st;
} o_bfjob;

static void *o_bf_range(void *arg) {
    o_bfjob *jb = (o_bfjob *)arg;
    jb->st = oracle_bf(jb->m, jb->in, jb->space, jb->i0, jb->i1, &jb->E, &jb->idx);
    return NULL;
}

/* Multi-threaded BF over [b, e): contiguous ranges, partial argmins merged in index order. */
int oracle_bf_mt(const o_model *m, const o_inst *in, int space, unsigned long long idx_begin,
                 unsigned long long idx_end, int n_threads, double *E_min, long long *idx_min) {
    if (n_threads < 1) n_threads = 1;
    if (n_threads > 256) n_threads = 256;
    pthread_t th[256];
    o_bfjob jobs[256];
    unsigned long long n = idx_end > idx_begin ? idx_end - idx_begin : 0;
    for (int t = 0; t < n_threads; t++) {
        jobs[t].m = m;
        jobs[t].in = in;
        jobs[t].space = space;
        jobs[t].i0 = idx_begin + (unsigned long long)((__uint128_t)n * t / n_threads);
        jobs[t].i1 = idx_begin + (unsigned long long)((__uint128_t)n * (t + 1) / n_threads);
        pthread_create(&th[t], NULL, o_bf_range, &jobs[t]);
    }
    *E_min = O_INF;
    *idx_min = -1;
    int st = O_ST_OK;
    for (int t = 0; t < n_threads; t++) {
        pthread_join(th[t], NULL);
        if (jobs[t].st != O_ST_OK) st = jobs[t].st;
        if (jobs[t].E < *E_min) {
            *E_min = jobs[t].E;
            *idx_min = jobs[t].idx;
        }
    }
    return st;
}

int oracle_eval_batch(const o_batch *b, long long n_inst, const int *partition, const double *fe, double slack,
                      double *E, double *tf, double *f_user, unsigned *viol, int *status) {
    for (long long i = 0; i < n_inst; i++) {
        o_inst in;
        o_make_inst(b, i, &in);
        const o_model *m = &b->models[b->model_id[i]];
        if (in.M < 1 || in.M > O_MAXM_LARGE) {
            E[i] = NAN;
            tf[i] = NAN;
            viol[i] = 0u;
            status[i] = O_ST_BADPARAM;
            continue;
        }
        double fs[O_MAXM_LARGE];
        status[i] = oracle_eval(m, &in, partition + b->user_off[i], fe[i], slack, &E[i], &tf[i], fs, &viol[i]);
        if (f_user)
            for (int u = 0; u < in.M; u++) f_user[b->user_off[i] + u] = fs[u];
    }
    return 0;
}

/* ------------------------------------------------------------------ */
/* Energy-saving statistics (a12, R16): per bucket                     */
/* [0] count OK, [1] sum r, [2] sum r^2, [3] max r, [4] min r,          */
/* [5] sum E_star over M, [6] sum E_LC over M, [7] #offloading (plans    */
/* with f_e* > 0: some user offloads, R18), [8] #status != OK,           */
/* [9..72] histogram of n~* (0..63);  r = 100 (E_LC - E*) / E_LC.        */
/* Default bucket (no bucket array): M - 1 for M <= n_buckets, else the  */
/* instance is not counted.  Summation in instance order.                */
/* ------------------------------------------------------------------ */
#define O_STATS_FIELDS 80
int oracle_stats(long long n_inst, const long long *user_off, const int *bucket, int n_buckets, const double *E,
                 const double *E_lc, const int *n_tilde, const double *f_e, const int *status, double *stats) {
    for (long long x = 0; x < (long long)n_buckets * O_STATS_FIELDS; x++) stats[x] = 0.0;
    for (int bk = 0; bk < n_buckets; bk++) {
        stats[bk * O_STATS_FIELDS + 3] = -O_INF;
        stats[bk * O_STATS_FIELDS + 4] = O_INF;
    }
    for (long long i = 0; i < n_inst; i++) {
        int M = (int)(user_off[i + 1] - user_off[i]);
        int bk = bucket ? bucket[i] : (M >= 1 && M <= n_buckets ? M - 1 : -1);
        if (bk < 0 || bk >= n_buckets) continue;
        double *s = stats + (long long)bk * O_STATS_FIELDS;
        if (status[i] != O_ST_OK) {
            s[8] = s[8] + 1.0;
            continue;
        }
        double r = 100.0 * (E_lc[i] - E[i]) / E_lc[i];
        s[0] = s[0] + 1.0;
        s[1] = s[1] + r;
        s[2] = s[2] + r * r;
        if (r > s[3]) s[3] = r;
        if (r < s[4]) s[4] = r;
        s[5] = s[5] + E[i] / (double)M;
        s[6] = s[6] + E_lc[i] / (double)M;
        if (f_e[i] > 0.0) s[7] = s[7] + 1.0;
        if (n_tilde[i] >= 0 && n_tilde[i] <= 63) s[9 + n_tilde[i]] = s[9 + n_tilde[i]] + 1.0;
    }
    return 0;
}

int oracle_grid_k(const o_inst *in) { return (int)o_grid_k(in); }

/* ------------------------------------------------------------------ */
/* Outer grouping (reading R21).              */
/* "an outer module that groups users by deadline similarity"; */
/* the paper uses the dynamic program for optimal grouping (OG) of its  */
/* reference [shi2022multiuser] whose internals it does not */
/* print; we follow SPEC S:295-303: users sorted by deadline (ascending,*/
/* ties by index), a DP over prefixes where cell i keeps the           */
/* lexicographically best (energy, t_free) of the first i sorted users, */
/* transition j -> i = group {j..i-1} solved by the inner J-DOB with    */
/* t_free = cell j's t_free (a failed Require is costed all-local with  */
/* t_free unchanged, which the inner solver's REQUIRE status returns);  */
/* strict improvement, so ties keep the smallest j.                    */
/* ------------------------------------------------------------------ */
typedef struct {
    double E, t_free_next;
    int status, n_groups;
    int group_of[O_MAXM_LARGE]; /* per user (input index): group number in execution order */
    int part[O_MAXM_LARGE];     /* per user: partition point, N = local */
    double f_user[O_MAXM_LARGE];
    double group_fe[O_MAXM];  /* per group: f_e, 0 = all local */
    int group_start[O_MAXM + 1];
} o_og_result;

static void o_group_inst(const o_inst *in, const int *sorted, int j, int i, double t_free, double *buf, o_inst *g) {
    int n = i - j;
    double *z = buf, *k = buf + 32, *f0 = buf + 64, *f1 = buf + 96, *R = buf + 128, *p = buf + 160, *T = buf + 192;
    for (int q = 0; q < n; q++) {
        int u = sorted[j + q];
        z[q] = in->zeta[u];
        k[q] = in->kappa[u];
        f0[q] = in->f_min[u];
        f1[q] = in->f_max[u];
        R[q] = in->R[u];
        p[q] = in->p_u[u];
        T[q] = in->T[u];
    }
    g->M = n;
    g->zeta = z;
    g->kappa = k;
    g->f_min = f0;
    g->f_max = f1;
    g->R = R;
    g->p_u = p;
    g->T = T;
    g->t_free = t_free;
    g->fe_min = in->fe_min;
    g->fe_max = in->fe_max;
    g->rho = in->rho;
}

int oracle_og(const o_model *m, const o_inst *in, int mode, o_og_result *r) {
    memset(r, 0, sizeof(*r));
    int st = oracle_check_inst(m, in);
    if (st == O_ST_REQUIRE) st = O_ST_OK; /* the DP costs a failed Require per group */
    if (in->M > O_MAXM && st == O_ST_OK) st = O_ST_BADPARAM; /* grouping: M <= 32 */
    r->status = st;
    int M = in->M;
    if (st != O_ST_OK) {
        static _Thread_local o_result lr;
        oracle_jdob(m, in, 1, &lr); /* LC answer (or NaN for malformed input) */
        r->E = lr.E;
        r->t_free_next = in->t_free;
        r->n_groups = 0;
        for (int u = 0; u < M && u < O_MAXM_LARGE; u++) {
            r->part[u] = m->N;
            r->f_user[u] = lr.f_user[u];
        }
        return st;
    }
    /* deadline order, ties by index (insertion sort) */
    int sorted[O_MAXM];
    for (int u = 0; u < M; u++) sorted[u] = u;
    for (int a = 1; a < M; a++) {
        int x = sorted[a], b = a - 1;
        while (b >= 0 && (in->T[x] < in->T[sorted[b]])) {
            sorted[b + 1] = sorted[b];
            b--;
        }
        sorted[b + 1] = x;
    }
    double cE[O_MAXM + 1], cT[O_MAXM + 1];
    int from[O_MAXM + 1];
    cE[0] = 0.0;
    cT[0] = in->t_free;
    from[0] = -1;
    double buf[224];
    for (int i = 1; i <= M; i++) {
        cE[i] = O_INF;
        cT[i] = O_INF;
        from[i] = -1;
        for (int j = 0; j < i; j++) {
            o_inst g;
            o_group_inst(in, sorted, j, i, cT[j], buf, &g);
            o_result gr;
            oracle_jdob(m, &g, mode, &gr);
            double E = cE[j] + gr.E;
            double tf = gr.t_free_next;
            if (E < cE[i] || (E == cE[i] && tf < cT[i])) {
                cE[i] = E;
                cT[i] = tf;
                from[i] = j;
            }
        }
    }
    /* backtrack and re-solve the chosen groups for the schedule */
    int starts[O_MAXM + 1], ng = 0;
    for (int i = M; i > 0; i = from[i]) starts[ng++] = from[i];
    r->E = cE[M];
    r->t_free_next = cT[M];
    r->n_groups = ng;
    for (int gi = 0; gi < ng; gi++) {
        int j = starts[ng - 1 - gi];
        int i = (gi + 1 < ng) ? starts[ng - 2 - gi] : M;
        r->group_start[gi] = j;
        o_inst g;
        o_group_inst(in, sorted, j, i, cT[j], buf, &g);
        o_result gr;
        oracle_jdob(m, &g, mode, &gr);
        r->group_fe[gi] = gr.f_e;
        for (int q = 0; q < i - j; q++) {
            int u = sorted[j + q];
            r->group_of[u] = gi;
            r->part[u] = ((gr.mask >> q) & 1u) ? gr.n_tilde : m->N;
            r->f_user[u] = gr.f_user[q];
        }
    }
    r->group_start[ng] = M;
    return st;
}
