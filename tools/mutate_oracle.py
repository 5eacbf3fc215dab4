#!/usr/bin/env python3
"""Mutation testing of the oracle's pins ('next' item 1).

Each mutant changes one semantic decision of oracle/jdob_oracle.c (a tie rule, a strict or
non-strict comparison, a clamp, an index range, a summation bound).  The tool builds every
mutant into its own shared library, runs the CPU oracle tests against it (JDOB_ORACLE_LIB)
and reports which mutants survive.  A mutant that cannot change any result is listed as
equivalent, with the reason; the goal is 0 non-equivalent survivors.

    python tools/mutate_oracle.py [--jobs 8] [--only NAME ...] [--out FILE]
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import os
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "oracle", "jdob_oracle.c")
sys.path.insert(0, ROOT)
from oracle import CFLAGS  # noqa: E402  (build flags only)

TESTS = ["tests/test_oracle_golden.py", "tests/test_oracle_boundaries.py", "tests/test_oracle_props.py",
         "tests/test_oracle_og.py", "tests/test_oracle_large.py"]

# (name, passage / reading, old text, new text, equivalent-reason or None)
MUTANTS = [
    # --- sort key (Alg. 1 line 5; reading R2) ---
    ("r2_index_only", "R2 tie-break: drop the T key",
     "    if (in->T[a] < in->T[b]) return 1;\n    if (in->T[a] > in->T[b]) return 0;\n", "", None),
    ("r2_T_desc", "R2 tie-break: T descending",
     "    if (in->T[a] < in->T[b]) return 1;\n    if (in->T[a] > in->T[b]) return 0;\n",
     "    if (in->T[a] > in->T[b]) return 1;\n    if (in->T[a] < in->T[b]) return 0;\n", None),
    ("r2_index_desc", "R2 last key: index descending", "    return a < b;\n}", "    return a > b;\n}", None),
    ("gamma_asc", "Alg. 1 line 5: ascending gamma",
     "    if (gamma[a] > gamma[b]) return 1;\n    if (gamma[a] < gamma[b]) return 0;\n",
     "    if (gamma[a] < gamma[b]) return 1;\n    if (gamma[a] > gamma[b]) return 0;\n", None),
    # --- gamma and thresholds (Eq. fth, R1) ---
    ("gamma_no_device", "gamma without the device term (P:241)",
     "gamma[i] = m->O[nt] / in->R[i] + (in->zeta[i] * vn) / in->f_max[i];",
     "gamma[i] = m->O[nt] / in->R[i];", None),
    ("th_own_T", "R1: own deadline instead of the suffix minimum",
     "th[i] = o_phi(m, nt, M - i) / (Lmin - gamma[list[i]]);",
     "th[i] = o_phi(m, nt, M - i) / (in->T[list[i]] - gamma[list[i]]);", None),
    ("th_global_min", "R1: global minimum deadline instead of the suffix minimum",
     "for (int k = i; k < M; k++)\n            if (in->T[list[k]] < Lmin)",
     "for (int k = 0; k < M; k++)\n            if (in->T[list[k]] < Lmin)", None),
    ("th_batch_off_by_one", "Eq. fth: phi(B - i) instead of phi(B - i + 1)",
     "th[i] = o_phi(m, nt, M - i) /", "th[i] = o_phi(m, nt, M - i - 1) /", None),
    # --- Alg. 2 ---
    ("ihat_gt", "Alg. 2 line 2: th > 0 instead of >= 0",
     "if (th[i] >= 0.0) {", "if (th[i] > 0.0) {",
     "th = phi/(L - gamma) with phi > 0 for n~ < N and finite L: th is never +-0"),
    ("member_le", "Alg. 2 line 8: remove while f_e <= th",
     "while (ihat < M && fe < th[ihat]) {", "while (ihat < M && fe <= th[ihat]) {", None),
    ("guard_gt", "Alg. 2 guard strict (P:339)",
     "if (fe >= o_phi(m, nt, B_o) / (l_o - in->t_free)) {", "if (fe > o_phi(m, nt, B_o) / (l_o - in->t_free)) {",
     None),
    ("guard_no_tfree", "Alg. 2 guard without t_free",
     "if (fe >= o_phi(m, nt, B_o) / (l_o - in->t_free)) {", "if (fe >= o_phi(m, nt, B_o) / (l_o)) {", None),
    ("alg2_le", "Alg. 2 strict improvement (P:345)",
     "if (E < E_nt) { /* strict improvement (P:345) */", "if (E <= E_nt) { /* strict improvement (P:345) */", None),
    ("alg1_le", "Alg. 1 strict improvement (P:276)",
     "if (have && E_nt < E_star) {", "if (have && E_nt <= E_star) {", None),
    ("lc_le", "R4: n~ = N compared with <=", "if (E_lc < E_star) {", "if (E_lc <= E_star) {", None),
    ("break_before_eval", "P:348: break before evaluating the empty set",
     "            r->n_visit++;\n", "            r->n_visit++;\n            if (B_o == 0) break;\n", None),
    ("no_break", "P:348: no break on the empty set", "            if (B_o == 0) break; /* P:348 */\n", "", None),
    ("grid_gt", "R7: grid condition f_e > f_e,min",
     "while (o_fe(in, k) >= in->fe_min) {", "while (o_fe(in, k) > in->fe_min) {", None),
    ("sweep_gt", "Alg. 2 line 6: sweep while f_e > f_e,min",
     "while (fe >= in->fe_min && j < k) {", "while (fe > in->fe_min && j < k) {", None),
    # --- D20-D22 ---
    ("no_fmax_clamp", "D20 without the upper clamp", "return (x > fmax) ? fmax : x;", "return x;", None),
    ("no_fmin_clamp", "D20 without the lower clamp", "double x = (G < fmin) ? fmin : G;", "double x = G;", None),
    ("r9_div", "R9: divide even when zeta v = 0", "            if (zv == 0.0) {\n                f = in->f_min[i];\n            } else {\n                double budget = (l_o - OR) - te;",
     "            if (0) {\n                f = in->f_min[i];\n            } else {\n                double budget = (l_o - OR) - te;", None),
    ("d22_no_tfree", "D22: max without t_free", "double E = 0.0, arr_max = in->t_free;", "double E = 0.0, arr_max = 0.0;",
     None),
    ("d22_ge", "D22 running max with >=", "if (arr > arr_max) arr_max = arr;\n        } else {\n            f = f_loc[i];",
     "if (arr >= arr_max) arr_max = arr;\n        } else {\n            f = f_loc[i];", "a max is the same value either way"),
    ("d21_no_upload", "D21 without the upload energy",
     "e = ((in->kappa[i] * u) * f) * f + OR * in->p_u[i];", "e = ((in->kappa[i] * u) * f) * f;", None),
    ("d21_no_edge", "D21 without the edge energy", "    E = E + (psi * fe) * fe;\n    if (tf_out)",
     "    if (tf_out)", None),
    ("budget_no_edge", "Gamma budget without the edge time", "double budget = (l_o - OR) - te;",
     "double budget = (l_o - OR);", None),
    # --- aggregates ---
    ("u_exclusive", "u_n~ sums n < n~", "for (int n = 0; n <= nt; n++) s = s + m->q[n] * m->A[n];",
     "for (int n = 0; n < nt; n++) s = s + m->q[n] * m->A[n];", None),
    ("v_exclusive", "v_n~ sums n < n~", "for (int n = 0; n <= nt; n++) s = s + m->g[n] * m->A[n];",
     "for (int n = 0; n < nt; n++) s = s + m->g[n] * m->A[n];", None),
    ("phi_inclusive", "phi_n~ includes n~", "for (int n = m->N; n >= nt + 1; n--) s = s + o_d(m, n, b) * m->A[n];",
     "for (int n = m->N; n >= nt; n--) s = s + o_d(m, n, b) * m->A[n];", None),
    ("psi_inclusive", "psi_n~ includes n~", "for (int n = m->N; n >= nt + 1; n--) s = s + o_c(m, n, b) * m->A[n];",
     "for (int n = m->N; n >= nt; n--) s = s + o_c(m, n, b) * m->A[n];", None),
    # --- LC and validation (D20 local branch) ---
    ("lc_fmax_T", "LC frequency from f_max instead of T", "double G = (in->zeta[i] * vN) / in->T[i];",
     "double G = (in->zeta[i] * vN) / in->f_max[i];", None),
    ("local_feasible_ge", "P:127 local feasibility strict",
     "if ((in->zeta[i] * vN) / in->f_max[i] > in->T[i]) return O_ST_LOCAL_INFEASIBLE;",
     "if ((in->zeta[i] * vN) / in->f_max[i] >= in->T[i]) return O_ST_LOCAL_INFEASIBLE;", None),
    ("require_le", "Require min T >= t_free (P:259) strict", "if (Tmin < in->t_free) return O_ST_REQUIRE;",
     "if (Tmin <= in->t_free) return O_ST_REQUIRE;", None),
    # --- brute force (R14, R10) ---
    ("bf_d6_lt", "D6' strict", "if (!(in->t_free + S[nmin + 1] * inv <= l_o)) return O_INF;",
     "if (!(in->t_free + S[nmin + 1] * inv < l_o)) return O_INF;", None),
    ("bf_zv0_gt", "D7' with zeta v = 0: budget > 0", "if (!(budget >= 0.0)) return O_INF;",
     "if (!(budget > 0.0)) return O_INF;", None),
    ("bf_budget_ge", "D7' with zeta v > 0: budget >= 0", "                if (!(budget > 0.0)) return O_INF;\n                double G",
     "                if (!(budget >= 0.0)) return O_INF;\n                double G",
     "budget = 0 with zeta v > 0 gives Gamma = +inf > f_max: infeasible either way"),
    ("bf_fmax_ge", "D7'/D13: Gamma >= f_max infeasible", "if (G > in->f_max[i]) return O_INF; /* D7' with D13",
     "if (G >= in->f_max[i]) return O_INF; /* D7' with D13", None),
    ("bf_clamps", "R10: the brute force clamps instead of rejecting",
     "if (G > in->f_max[i]) return O_INF; /* D7' with D13", "if (G > in->f_max[i]) G = in->f_max[i]; /* D7' with D13",
     None),
    ("bf_le", "lowest-index tie-break (S:354-357)", "        if (E < *E_min) {\n            *E_min = E;\n            *idx_min = (long long)idx;",
     "        if (E <= *E_min) {\n            *E_min = E;\n            *idx_min = (long long)idx;", None),
    ("bf_batch_le", "R14 batch count b_n = #{n_m <= n}",
     "            if (nvec[i] < n) b[n]++;\n    }\n    S[N + 1] = 0.0;\n    for (int n = N; n >= 1; n--) {\n        S[n] = S[n + 1] + (b[n] > 0 ? o_d(m, n, b[n]) * m->A[n] : 0.0);\n        Psi = Psi + (b[n] > 0 ? o_c(m, n, b[n]) * m->A[n] : 0.0);\n    }\n    int any = 0, nmin = N;\n    double l_o = O_INF;\n    for (int i = 0; i < M; i++)\n        if (nvec[i] < N) {\n            any = 1;\n            if (nvec[i] < nmin) nmin = nvec[i];\n            if (in->T[i] < l_o) l_o = in->T[i];\n        }\n    double inv = 1.0 / fe;\n    if (any) {",
     "            if (nvec[i] <= n && nvec[i] < N) b[n]++;\n    }\n    S[N + 1] = 0.0;\n    for (int n = N; n >= 1; n--) {\n        S[n] = S[n + 1] + (b[n] > 0 ? o_d(m, n, b[n]) * m->A[n] : 0.0);\n        Psi = Psi + (b[n] > 0 ? o_c(m, n, b[n]) * m->A[n] : 0.0);\n    }\n    int any = 0, nmin = N;\n    double l_o = O_INF;\n    for (int i = 0; i < M; i++)\n        if (nvec[i] < N) {\n            any = 1;\n            if (nvec[i] < nmin) nmin = nvec[i];\n            if (in->T[i] < l_o) l_o = in->T[i];\n        }\n    double inv = 1.0 / fe;\n    if (any) {", None),
    ("bf_start_nmin", "D6' uses S_{n_min} instead of S_{n_min+1}",
     "if (!(in->t_free + S[nmin + 1] * inv <= l_o)) return O_INF;", "if (!(in->t_free + S[nmin] * inv <= l_o)) return O_INF;",
     None),
    # --- eval (a11) ---
    ("eval_d6", "eval D6 bit with >=", "if (start > l_o + tol) viol |= 1u;", "if (start >= l_o + tol) viol |= 1u;", None),
    ("eval_zv0_le", "eval bit 3 at budget = 0 (zeta v = 0)", "if (budget < 0.0) viol |= 8u;", "if (budget <= 0.0) viol |= 8u;",
     None),
    # --- outer grouping (R21) ---
    ("og_no_tf_tie", "R21 cell tie on t_free", "if (E < cE[i] || (E == cE[i] && tf < cT[i])) {", "if (E < cE[i]) {", None),
    ("og_le", "R21 strict improvement", "if (E < cE[i] || (E == cE[i] && tf < cT[i])) {",
     "if (E <= cE[i] || (E == cE[i] && tf < cT[i])) {", None),
    ("og_sort_le", "R21 deadline sort ties by index", "while (b >= 0 && (in->T[x] < in->T[sorted[b]])) {",
     "while (b >= 0 && (in->T[x] <= in->T[sorted[b]])) {", None),
    # --- statistics (a12, R16) ---
    ("stats_r_sign", "R16 reduction sign", "double r = 100.0 * (E_lc[i] - E[i]) / E_lc[i];",
     "double r = 100.0 * (E[i] - E_lc[i]) / E_lc[i];", None),
    ("stats_per_user", "R16 per-user energy", "s[5] = s[5] + E[i] / (double)M;", "s[5] = s[5] + E[i];", None),
]


def build_mutant(name, old, new, tmp):
    src = open(SRC).read()
    n = src.count(old)
    if n != 1:
        return None, f"anchor found {n} times"
    path_c = os.path.join(tmp, f"{name}.c")
    path_so = os.path.join(tmp, f"lib_{name}.so")
    open(path_c, "w").write(src.replace(old, new))
    r = subprocess.run(["gcc", *CFLAGS, "-o", path_so, path_c, "-lm"], capture_output=True, text=True)
    if r.returncode != 0:
        return None, "compile error: " + r.stderr[-300:]
    return path_so, ""


def run_tests(lib):
    env = dict(os.environ, JDOB_ORACLE_LIB=lib)
    t0 = time.time()
    r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-m", "not gpu and not slow", "-p", "no:randomly",
                        *TESTS], cwd=ROOT, env=env, capture_output=True, text=True, timeout=1800)
    first_fail = ""
    for line in r.stdout.splitlines():
        if line.startswith("FAILED") or line.startswith("ERROR"):
            first_fail = line.split(" - ")[0].replace("FAILED ", "").replace("ERROR ", "")
            break
    return r.returncode, first_fail, time.time() - t0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--jobs", type=int, default=os.cpu_count() or 4)
    ap.add_argument("--only", nargs="*")
    ap.add_argument("--out")
    a = ap.parse_args()
    muts = [m for m in MUTANTS if not a.only or m[0] in a.only]
    tmp = tempfile.mkdtemp(prefix="jdob_mut_")
    rows = []

    def job(m):
        name, what, old, new, equiv = m
        lib, err = build_mutant(name, old, new, tmp)
        if lib is None:
            return (name, what, "BUILD-ERROR", err, equiv)
        rc, ff, dt = run_tests(lib)
        status = "killed" if rc != 0 else ("equivalent" if equiv else "SURVIVED")
        return (name, what, status, ff if rc != 0 else (equiv or ""), equiv)

    with cf.ThreadPoolExecutor(max_workers=a.jobs) as ex:
        rows = list(ex.map(job, muts))
    lines = [f"oracle mutation run: {len(rows)} mutants, tests: {' '.join(TESTS)}", ""]
    w = max(len(r[0]) for r in rows)
    for name, what, status, info, _ in rows:
        lines.append(f"{name:<{w}}  {status:<10}  {what}  [{info}]")
    surv = [r for r in rows if r[2] in ("SURVIVED", "BUILD-ERROR")]
    eq = [r for r in rows if r[2] == "equivalent"]
    lines += ["", f"killed {sum(r[2] == 'killed' for r in rows)}, equivalent (declared, survived) {len(eq)}, "
              f"non-equivalent survivors {len(surv)}"]
    txt = "\n".join(lines)
    print(txt)
    if a.out:
        open(a.out, "w").write(txt + "\n")
    return 1 if surv else 0


if __name__ == "__main__":
    sys.exit(main())
