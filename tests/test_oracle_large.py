"""Oracle at M > 32 users per instance (SPEC S:442 complexity smoke)."""
import time

import numpy as np
import pytest

import jdobgen as g
import oracle as O


def large_instance(M, seed, beta_lo=0.0, beta_hi=10.0, hetero=False):
    m = g.profiles.mobilenetv2(B_max=max(M, 32))
    rng = np.random.default_rng(seed)
    lat = float(g.min_local_latency(m, np.array([g.profiles.ZETA]), np.array([2.6e9]))[0])
    users = dict(zeta=g.profiles.ZETA, kappa=g.profiles.KAPPA * (rng.uniform(0.5, 2.0, M) if hetero else 1.0),
                 f_min=1.5e9, f_max=2.6e9, R=g.R_TABLE_I * (rng.uniform(0.5, 2.0, M) if hetero else 1.0),
                 p_u=1.0, T=(1.0 + rng.uniform(beta_lo, beta_hi, M)) * lat)
    return g.single_instance(m, users)


@pytest.mark.parametrize("M,hetero", [(33, False), (100, True), (200, False)])
def test_large_m_invariants(M, hetero):
    b = large_instance(M, seed=M, hetero=hetero)
    r = O.jdob(b)
    assert r["status"] == O.ST_OK
    assert r["E"] <= r["E_lc"]
    N = b.models[0].N
    part = r["part"]
    assert set(np.unique(part)) <= {r["n_tilde"], N}
    # the plan re-verifies through eval (D20-D22 generalised, slack 1e-9) with the same bits
    fe = r["f_e"] if r["f_e"] > 0 else float(b.fe_max[0])
    ev = O.eval_config(b, 0, part, fe, slack=1e-9)
    assert ev["violations"] == 0
    assert ev["E"] == r["E"] and ev["t_free_next"] == r["t_free_next"]
    assert np.array_equal(ev["f_user"], r["f_user"])


def test_part_matches_mask_small():
    b = g.random_batch(seed=41, n_inst=100, M_lo=1, M_hi=32, N_lo=1, N_hi=8, k_max=40)
    res = O.solve_batch(b)
    for i in range(b.n_inst):
        o0, N = int(b.user_off[i]), b.models[b.model_id[i]].N
        for u in range(b.M(i)):
            exp = res["n_tilde"][i] if (int(res["mask"][i]) >> u) & 1 else N
            assert res["part"][o0 + u] == exp


def test_complexity_smoke_m1000():
    # M = 1000, N = 19, k ~ 64 completes (oracle: well under a minute)
    b = large_instance(1000, seed=7)
    t0 = time.perf_counter()
    r = O.jdob(b)
    assert time.perf_counter() - t0 < 60
    assert r["status"] == O.ST_OK and r["E"] <= r["E_lc"]
