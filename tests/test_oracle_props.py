"""Oracle pins: invariants from the paper and independent brute force on tiny inputs."""
import math

import numpy as np
import pytest

import jdobgen as g
import oracle as O
from tests import indep_bruteforce as IB


@pytest.fixture(scope="module")
def rand_small():
    # M <= 4, N <= 3 (SPEC S:439 sizes), 30 % with t_free > 0
    return g.random_batch(seed=11, n_inst=200, M_lo=1, M_hi=4, N_lo=1, N_hi=3, k_max=12)


@pytest.fixture(scope="module")
def rand_mid():
    return g.random_batch(seed=12, n_inst=400, M_lo=1, M_hi=12, N_lo=1, N_hi=8, k_max=70)


def test_generated_instances_valid(rand_small, rand_mid):
    for b in (rand_small, rand_mid):
        for i in range(b.n_inst):
            assert O.check_inst(b, i) == O.ST_OK


def test_jdob_le_lc(rand_mid):
    # "J-DOB ... consistently consume equal or less energy compared to LC"; exact (R4)
    r = O.solve_batch(rand_mid)
    assert np.all(r["status"] == 0)
    assert np.all(r["E"] <= r["E_lc"])
    assert np.any(r["E"] < r["E_lc"])


def test_thresholds_non_increasing(rand_mid):
    # {f_e^th,i} is non-increasing (from the first non-negative entry); exact in FP64
    for i in range(rand_mid.n_inst):
        N = rand_mid.models[rand_mid.model_id[i]].N
        for nt in range(N):
            gam, lst, th = O.thresholds(rand_mid, i, nt)
            nonneg = np.nonzero(th >= 0)[0]
            if len(nonneg) == 0:
                continue
            t = th[nonneg[0]:]
            assert np.all(t[1:] <= t[:-1])
            # gamma sorted descending
            assert np.all(gam[lst][1:] <= gam[lst][:-1])


def test_plans_feasible_and_consistent(rand_mid):
    # Every returned plan re-verifies through eval (slack 1e-9), and the
    # generalised D21/D22 (R14/R15) reproduce J-DOB's E and t_free* bit-for-bit.
    r = O.solve_batch(rand_mid)
    part = O.partition_from_plan(rand_mid, r)
    fe = np.where(r["mask"] != 0, r["f_e"], rand_mid.fe_max)
    ev = O.eval_batch(rand_mid, part, fe, slack=1e-9)
    assert np.all(ev["violations"] == 0)
    assert np.array_equal(ev["E"], r["E"])
    assert np.array_equal(ev["t_free_next"], r["t_free_next"])
    assert np.array_equal(ev["f_user"], r["f_user"])


def test_dominance_variants(rand_mid):
    # full <= no-edge-DVFS, full <= binary, each <= LC
    full = O.solve_batch(rand_mid, mode=O.MODE_FULL)
    ne = O.solve_batch(rand_mid, mode=O.MODE_NO_EDGE_DVFS)
    bi = O.solve_batch(rand_mid, mode=O.MODE_BINARY)
    lc = O.solve_batch(rand_mid, mode=O.MODE_LC)
    assert np.all(full["E"] <= ne["E"]) and np.all(full["E"] <= bi["E"])
    assert np.all(ne["E"] <= lc["E"]) and np.all(bi["E"] <= lc["E"])
    assert np.array_equal(lc["E"], full["E_lc"])


def test_bf_orderings(rand_small):
    # BF-general <= BF-identical <= J-DOB (slack 1e-12 for ULP boundary cases), and
    # J-DOB == BF-identical at M = 1 (the suffix family is every subset at M = 1).
    for i in range(rand_small.n_inst):
        r = O.jdob(rand_small, i)
        Ei, ii, st = O.bf(rand_small, 1, i=i)
        Eg, ig, st2 = O.bf(rand_small, 0, i=i)
        assert st == 0 and st2 == 0
        assert Eg <= Ei
        assert Ei <= r["E"] * (1 + 1e-12)
        if rand_small.M(i) == 1:
            assert abs(Ei - r["E"]) <= 1e-12 * r["E"]
        # BF-identical index decodes to a candidate whose value is E
        assert O.bf_candidate(rand_small, 1, ii, i=i) == Ei
        assert O.bf_candidate(rand_small, 0, ig, i=i) == Eg


def test_bf_general_reduces_to_identical(rand_small):
    # On identical vectors {n~, N}^M the general evaluation equals the identical one bit-for-bit.
    for i in range(0, rand_small.n_inst, 7):
        M = rand_small.M(i)
        N = rand_small.models[rand_small.model_id[i]].N
        k = O.grid_k(rand_small, i)
        for nt in range(N + 1):
            for mask in range(1 << M):
                for j in (0, k - 1):
                    idx_i = ((nt << M) + mask) * k + j
                    vec = [nt if (nt < N and (mask >> m) & 1) else N for m in range(M)]
                    v = 0
                    for d in vec:
                        v = v * (N + 1) + d
                    idx_g = v * k + j
                    a = O.bf_candidate(rand_small, 1, idx_i, i=i)
                    b = O.bf_candidate(rand_small, 0, idx_g, i=i)
                    assert (a == b) or (math.isinf(a) and math.isinf(b))


def test_bf_vs_independent_bruteforce():
    # Pin both oracle BF spaces to an independent numeric formulation (bisection + ASAP
    # simulation, tests/indep_bruteforce.py).
    b = g.random_batch(seed=21, n_inst=24, M_lo=1, M_hi=3, N_lo=1, N_hi=3, k_max=6, tfree_frac=0.4)
    for i in range(b.n_inst):
        for space in (1, 0):
            Eo, _, st = O.bf(b, space, i=i)
            Ei = IB.brute_force(b, i, space)
            assert st == 0
            assert abs(Eo - Ei) <= 1e-9 * Eo, (i, space, Eo, Ei)


def test_jdob_m1_vs_independent():
    # At M = 1 J-DOB is exact over (n~, subset, grid) -> equals the independent brute force.
    b = g.random_batch(seed=22, n_inst=30, M_lo=1, M_hi=1, N_lo=1, N_hi=5, k_max=30, tfree_frac=0.4)
    for i in range(b.n_inst):
        r = O.jdob(b, i)
        Ei = IB.brute_force(b, i, 1)
        assert abs(r["E"] - Ei) <= 1e-9 * Ei


def _golden_section(fun, a, b, iters=200):
    gr = (math.sqrt(5) - 1) / 2
    c, d = b - gr * (b - a), a + gr * (b - a)
    for _ in range(iters):
        if fun(c) < fun(d):
            b = d
        else:
            a = c
        c, d = b - gr * (b - a), a + gr * (b - a)
    return 0.5 * (a + b)


def test_d20_vs_numeric_minimisation():
    # closed-form f* (D20) matches golden-section minimisation within 0.1 %.
    rng = np.random.default_rng(5)
    n_checked = 0
    for t in range(200):
        b = g.toy_instance("toy-2-m1")
        b.T[0] = rng.uniform(0.12, 0.5)
        b.zeta[0] = rng.uniform(0.5, 1.0)
        b.kappa[0] = rng.uniform(0.5, 2.0) * 1e-27
        nt = int(rng.integers(1, 3))
        fe = float(rng.uniform(0.5e9, 2.1e9))
        m = b.models[0]
        v = sum(m.g[n] * m.A[n] for n in range(1, nt + 1))
        te = sum(m.d[n * 3 + 1] * m.A[n] for n in range(nt + 1, m.N + 1)) / fe
        budget = b.T[0] - m.O[nt] / b.R[0] - te
        if budget <= 0 or b.zeta[0] * v / budget > b.f_max[0]:
            continue
        r = O.eval_config(b, 0, [nt], fe)

        def penal(f):
            lat = b.zeta[0] * v / f + m.O[nt] / b.R[0] + te
            return b.kappa[0] * v * f * f + (1e6 * (lat - b.T[0]) if lat > b.T[0] else 0.0)

        f_num = _golden_section(penal, b.f_min[0], b.f_max[0])
        assert abs(r["f_user"][0] - f_num) <= 1e-3 * f_num
        n_checked += 1
    assert n_checked > 50


def test_grouping_split_examples_sanity():
    # SPEC S:301 (corrected): group {A} then {B} totals 0.03518075 with t_free chaining.
    b = g.toy_instance("toy-2-m1")                       # user A, T = 0.2
    ra = O.jdob(b)
    assert abs(ra["E"] - 0.02248075) < 1e-15
    bb = g.toy_instance("toy-2-m1")
    bb.T[0] = 0.6
    bb.t_free[0] = ra["t_free_next"]
    rb = O.jdob(bb)
    assert abs(rb["E"] - 0.0127) < 1e-12 and rb["f_e"] == 0.6e9
    assert abs(ra["E"] + rb["E"] - 0.03518075) < 1e-12


def test_counts_literal(rand_mid):
    r = O.solve_batch(rand_mid, counts=True)
    c = r["counts"]
    assert np.all(c[:, 1] <= c[:, 0]) and np.all(c[:, 2] >= 0)
    for i in range(0, rand_mid.n_inst, 50):
        rr = O.jdob(rand_mid, i)
        assert (rr["n_visit"], rr["n_eval"], rr["n_member"]) == tuple(c[i])


def test_stats_definition(rand_mid):
    r = O.solve_batch(rand_mid)
    st = O.stats(rand_mid, r, n_buckets=32)
    Ms = np.diff(rand_mid.user_off)
    for bk in range(32):
        sel = (Ms - 1) == bk
        red = 100 * (r["E_lc"][sel] - r["E"][sel]) / r["E_lc"][sel]
        assert st[bk, 0] == sel.sum()
        if sel.sum():
            assert abs(st[bk, 1] - red.sum()) <= 1e-9 * max(1, abs(red.sum()))
            assert st[bk, 3] == red.max() and st[bk, 4] == red.min()
            assert st[bk, 7] == (r["mask"][sel] != 0).sum() == (r["f_e"][sel] > 0).sum()
            assert st[bk, 9:73].sum() == sel.sum()


@pytest.mark.slow
def test_calibrated_regime_sanity():
    # Informational (finding 7): MobileNetV2 identical deadlines reach ~33 % / ~52 % max
    # reduction vs LC at beta = 2.13 / 30.25 (paper 32.8 % / 51.3 %). Unpinned; loose bounds.
    m = g.profiles.mobilenetv2()
    for beta, lo, hi in ((2.13, 25.0, 40.0), (30.25, 45.0, 60.0)):
        best = 0.0
        for M in (1, 2, 4, 8, 16, 24, 32):
            users = dict(zeta=g.profiles.ZETA, kappa=g.profiles.KAPPA, f_min=1.5e9, f_max=2.6e9,
                         R=g.R_TABLE_I, p_u=1.0,
                         T=[float(g.deadline_from_beta(m, g.profiles.ZETA, 2.6e9, beta))] * M)
            b = g.single_instance(m, users)
            r = O.jdob(b)
            best = max(best, 100 * (r["E_lc"] - r["E"]) / r["E_lc"])
        assert lo < best < hi, (beta, best)
