"""Oracle pins for the outer grouping DP (NEXT-1, reading R21: SPEC S:295-303 on top of P:183)."""
import itertools

import numpy as np
import pytest

import jdobgen as g
import oracle as O


def two_users(T):
    b = g.toy_instance("toy-2")
    b.T[:] = T
    return b


def test_split_wins_golden():
    # SPEC S:301 (corrected in SURVEY §4.2): group {A} then {B}: 0.02248075 + 0.0127 = 0.03518075
    r = O.og(two_users([0.2, 0.6]))
    hand_A = 1e6 / 1e8 + 2.5e-29 * 3e8 * (1.29e9) ** 2       # toy-2 M=1 golden
    hand_B = 1e6 / 1e8 + 2.5e-29 * 3e8 * (0.6e9) ** 2        # f_e = 0.6 GHz after t_free = 0.19605
    assert abs(hand_A + hand_B - 0.03518075) < 1e-15
    assert abs(r["E"] - 0.03518075) < 1e-15
    assert r["n_groups"] == 2 and list(r["group_fe"]) == [1.29e9, 0.6e9]
    assert list(r["part"]) == [0, 0]
    # the joint group would cost 0.0642368
    j = O.jdob(two_users([0.2, 0.6]))
    assert abs(j["E"] - 0.0642368) < 1e-12 and r["E"] < j["E"]


def test_joint_wins_golden():
    # deadlines both 0.2 -> joint group 0.0642368 (split would be 0.69748075)
    r = O.og(two_users([0.2, 0.2]))
    assert abs(r["E"] - 0.0642368) < 1e-15 and r["n_groups"] == 1
    a = O.jdob(g.toy_instance("toy-2-m1"))
    bb = g.toy_instance("toy-2-m1")
    bb.t_free[0] = a["t_free_next"]
    b = O.jdob(bb)
    assert b["status"] == O.ST_REQUIRE or b["mask"] == 0
    assert abs(a["E"] + b["E"] - 0.69748075) < 1e-12


@pytest.fixture(scope="module")
def rand():
    return g.random_batch(seed=31, n_inst=120, M_lo=1, M_hi=6, N_lo=1, N_hi=5, k_max=30, tfree_frac=0.3)


def _chain(batch, i, groups, mode=0):
    """Re-evaluate a contiguous partition of the deadline order by chaining t_free (independent of the DP)."""
    M = batch.M(i)
    o0 = int(batch.user_off[i])
    order = sorted(range(M), key=lambda u: (batch.T[o0 + u], u))
    E = 0.0
    tf = float(batch.t_free[i])
    for (a, b) in groups:
        users = [order[q] for q in range(a, b)]
        sub = batch.take([i])
        sub = g.single_instance(batch.models[batch.model_id[i]],
                                {f: [getattr(batch, f)[o0 + u] for u in users] for f in g.Batch.USER_FIELDS},
                                t_free=tf, fe_min=float(batch.fe_min[i]), fe_max=float(batch.fe_max[i]),
                                rho=float(batch.rho[i]))
        r = O.jdob(sub, mode=mode)
        E = E + r["E"]
        tf = r["t_free_next"]
    return E, tf


def test_og_le_single_group_and_lc(rand):
    for i in range(rand.n_inst):
        r = O.og(rand, i)
        j = O.jdob(rand, i)
        assert r["status"] == 0
        assert r["E"] <= j["E"] or j["status"] == O.ST_REQUIRE
        assert r["E"] <= j["E_lc"]


def test_og_schedule_reevaluates_exactly(rand):
    # the returned partition, re-solved group by group with chained t_free, gives the same bits
    for i in range(rand.n_inst):
        r = O.og(rand, i)
        st = list(r["group_start"])
        groups = list(zip(st[:-1], st[1:]))
        E, tf = _chain(rand, i, groups)
        assert E == r["E"] and tf == r["t_free_next"]
        # GPU windows are chained, so every group starts no earlier than the previous group's end


def test_og_vs_all_partitions(rand):
    # the DP returns one contiguous partition of the deadline order: never below the best of all
    # 2^(M-1) partitions, and equal to it when the best partition is reachable greedily (M <= 2)
    for i in range(0, rand.n_inst, 3):
        M = rand.M(i)
        r = O.og(rand, i)
        best = np.inf
        for cuts in itertools.product([0, 1], repeat=M - 1):
            bounds = [0] + [q + 1 for q, c in enumerate(cuts) if c] + [M]
            E, _ = _chain(rand, i, list(zip(bounds[:-1], bounds[1:])))
            best = min(best, E)
        assert r["E"] >= best * (1 - 1e-15)
        if M <= 2:
            assert r["E"] == best


def test_og_plans_feasible(rand):
    # every group's plan is feasible at its chained t_free (eval, slack 1e-9)
    for i in range(rand.n_inst):
        r = O.og(rand, i)
        M = rand.M(i)
        o0 = int(rand.user_off[i])
        order = sorted(range(M), key=lambda u: (rand.T[o0 + u], u))
        tf = float(rand.t_free[i])
        st = list(r["group_start"])
        for gi, (a, b) in enumerate(zip(st[:-1], st[1:])):
            users = [order[q] for q in range(a, b)]
            sub = g.single_instance(rand.models[rand.model_id[i]],
                                    {f: [getattr(rand, f)[o0 + u] for u in users] for f in g.Batch.USER_FIELDS},
                                    t_free=tf, fe_min=float(rand.fe_min[i]), fe_max=float(rand.fe_max[i]),
                                    rho=float(rand.rho[i]))
            part = [int(r["part"][u]) for u in users]
            fe = r["group_fe"][gi] if r["group_fe"][gi] > 0 else float(rand.fe_max[i])
            ev = O.eval_config(sub, 0, part, fe, slack=1e-9)
            assert ev["violations"] & ~16 == 0      # Require may fail for an all-local group only
            if ev["violations"] & 16:
                assert all(p == rand.models[rand.model_id[i]].N for p in part)
            tf = ev["t_free_next"]
        assert tf == r["t_free_next"]


def test_og_more_than_32_users_reports_lc():
    """Grouping is defined for M <= 32 (the per-cell group masks); a valid larger instance is reported
    BADPARAM with its LC answer (f* = the LC frequencies), a locally infeasible one keeps that status."""
    from tests.test_oracle_large import large_instance
    for M in (33, 64):
        b = large_instance(M, seed=M)
        r = O.og(b)
        E_lc, f_loc, _ = O.lc(b)
        assert r["status"] == O.ST_BADPARAM and r["E"] == E_lc and r["n_groups"] == 0
        assert np.array_equal(r["f_user"], f_loc) and (r["part"] == b.models[0].N).all()
        assert r["t_free_next"] == b.t_free[0]
    b = large_instance(40, seed=1)
    b.T[5] = 1e-6
    assert O.og(b)["status"] == O.ST_LOCAL_INFEASIBLE
