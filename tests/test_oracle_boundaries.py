"""Oracle pins on the paper's tie and boundary semantics (tests/golden/boundaries.json).

Each instance is constructed so that exactly one tie or boundary rule decides the answer:
the R2 sort tie-break, the strict `<` of Alg. 1 and Alg. 2
(P:345), the non-strict D6 guard and its brute-force form D6', membership at
f_e = f_th, the D20 clamp at f_max (R10), R9 at a zero budget, and the
outer-grouping (E, t_free) tie (R21).  Expected values are hand-derived ('derivation') and
restated as plain arithmetic ('hand_*'), evaluated here without the oracle.
tools/mutate_oracle.py checks that every listed oracle mutant fails at least one of these.
"""
import json
import os

import numpy as np
import pytest

import jdobgen as g
import oracle as O

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "boundaries.json")))
CASES = [k for k in GOLD if not k.startswith("_")]


def hand(expr):
    return eval(expr, {"__builtins__": {}}, {})


def close(a, b, rel=1e-12):
    return abs(a - b) <= rel * max(abs(a), abs(b), 1e-300)


def build(case):
    gd = GOLD[case]
    m = gd["model"]
    N, B = m["N"], m["B_max"]
    d = np.zeros((N + 1) * (B + 1))
    c = np.zeros((N + 1) * (B + 1))
    for n in range(1, N + 1):
        for b in range(1, B + 1):
            d[n * (B + 1) + b] = m["d"][n - 1][b - 1]
            c[n * (B + 1) + b] = m["c"][n - 1][b - 1]
    model = g.Model(case, N, B, np.array(m["A"], float), np.array(m["O"], float), np.array(m["g"], float),
                    np.array(m["q"], float), d, c)
    inst = gd["inst"]
    return g.single_instance(model, gd["users"], t_free=inst["t_free"], fe_min=inst["fe_min"],
                             fe_max=inst["fe_max"], rho=inst["rho"])


@pytest.mark.parametrize("case", CASES)
def test_hand_expressions(case):
    """The stored numbers are the hand derivations (no oracle involved)."""
    for sec in GOLD[case].values():
        if not isinstance(sec, dict):
            continue
        if "hand_E" in sec:
            assert close(hand(sec["hand_E"]), sec["E"]), (case, sec["hand_E"])
        if "hand_tf" in sec:
            assert close(hand(sec["hand_tf"]), sec["t_free_next"]), (case, sec["hand_tf"])
        if "hand" in sec:
            for h, v in zip(sec["hand"], sec["values"]):
                assert close(hand(h), v), (case, h)


@pytest.mark.parametrize("case", [c for c in CASES if "jdob" in GOLD[c]])
def test_jdob(case):
    gd = GOLD[case]["jdob"]
    b = build(case)
    assert O.check_inst(b) == O.ST_OK
    r = O.jdob(b)
    assert r["status"] == O.ST_OK
    assert (r["n_tilde"], r["j"], r["mask"]) == (gd["n_tilde"], gd["j"], gd["mask"])
    assert r["f_e"] == gd["f_e"]
    assert close(r["E"], gd["E"]), (r["E"], gd["E"])
    assert close(r["t_free_next"], gd["t_free_next"])
    assert list(r["f_user"]) == gd["f_user"]                      # bit-exact (the clamps)
    if "counts" in gd:
        cnt = gd["counts"]
        assert (r["n_visit"], r["n_eval"], r["n_member"]) == (cnt["n_visit"], cnt["n_eval"], cnt["n_member"])


@pytest.mark.parametrize("case", [c for c in CASES if "lc" in GOLD[c]])
def test_lc(case):
    E, _, _ = O.lc(build(case))
    assert close(E, GOLD[case]["lc"]["E"])


@pytest.mark.parametrize("case", [c for c in CASES if "thresholds_nt0" in GOLD[c]])
def test_thresholds(case):
    gd = GOLD[case]["thresholds_nt0"]
    gam, lst, th = O.thresholds(build(case), 0, 0)
    assert list(lst) == gd["list"]
    for i, v in enumerate(gd["values"]):
        assert close(th[i], v)


@pytest.mark.parametrize("case,space", [(c, s) for c in CASES for s, key in ((0, "bf_general"), (1, "bf_identical"))
                                        if key in GOLD[c]])
def test_bruteforce(case, space):
    gd = GOLD[case]["bf_general" if space == 0 else "bf_identical"]
    E, idx, st = O.bf(build(case), space)
    assert st == O.ST_OK
    assert idx == gd["idx"]
    assert close(E, gd["E"]) if gd["E"] != 0.0 else E == 0.0
    if "hand_idx" in gd and not gd["hand_idx"].startswith("vector"):
        assert hand(gd["hand_idx"]) == gd["idx"]


@pytest.mark.parametrize("case", [c for c in CASES if "jdob" in GOLD[c]])
def test_plan_through_eval(case):
    """The J-DOB plan re-evaluates (D20-D22) with no violation at slack 0 (the boundaries are
    equalities, which the non-strict constraints admit); bit 3 is never set."""
    gd = GOLD[case]["jdob"]
    b = build(case)
    N = b.models[0].N
    part = [gd["n_tilde"] if (gd["mask"] >> u) & 1 else N for u in range(b.M(0))]
    r = O.eval_config(b, 0, part, gd["f_e"], slack=0.0)
    if case == "r10-gamma-above-fmax":
        # Gamma rounds above f_max: eval reports the clamped plan's D7 finish one ulp-scale late
        assert r["violations"] & ~2 == 0
    else:
        assert r["violations"] == 0, r
    assert close(r["E"], gd["E"])
    assert list(r["f_user"]) == gd["f_user"]


def test_r10_above_precondition():
    """Gamma at the threshold point, in the literal binary64 order of Appendix A, exceeds f_max:
    the instance really exercises the upper clamp of D20."""
    gd = GOLD["r10-gamma-above-fmax"]
    m, u = gd["model"], gd["users"]
    phi = 0.0 + m["d"][1][0] * m["A"][2]
    v1 = 0.0 + 1.0 * m["A"][1]
    OR = m["O"][1] / u["R"]
    gamma = OR + (u["zeta"] * v1) / u["f_max"]
    th = phi / (u["T"][0] - gamma)
    fe = gd["inst"]["fe_max"]
    assert th == fe and gd["inst"]["fe_min"] == fe
    budget = (u["T"][0] - OR) - phi * (1.0 / fe)
    assert (u["zeta"] * v1) / budget > u["f_max"]


@pytest.mark.parametrize("case", [c for c in CASES if "og" in GOLD[c]])
def test_og(case):
    gd = GOLD[case]["og"]
    r = O.og(build(case))
    assert r["status"] == O.ST_OK
    assert r["E"] == gd["E"]
    assert r["t_free_next"] == gd["t_free_next"]
    assert r["n_groups"] == gd["n_groups"]
    assert list(r["group_start"]) == gd["group_start"]
    assert list(r["part"]) == gd["part"]
    assert list(r["group_fe"]) == gd["group_fe"]


def test_stats_of_golden_plans():
    """Statistics (a12, R16: r = 100 (E_LC - E)/E_LC, per-user E/M) of the boundary instances,
    expected values formed from the hand-derived E and E_LC of the golden file."""
    cases = [c for c in CASES if "jdob" in GOLD[c] and "lc" in GOLD[c] and "E" in GOLD[c]["lc"]]
    batch = g.concat([build(c) for c in cases])
    r = O.solve_batch(batch)
    st = O.stats(batch, r, n_buckets=32)
    exp = np.zeros((32, O.STATS_FIELDS))
    exp[:, 3], exp[:, 4] = -np.inf, np.inf
    for c in cases:
        M = len(GOLD[c]["users"]["T"])
        E, El = GOLD[c]["jdob"]["E"], GOLD[c]["lc"]["E"]
        s = exp[M - 1]
        red = 100.0 * (El - E) / El if El != 0.0 else float("nan")
        s[0] += 1
        s[1] += red
        s[2] += red * red
        s[3] = max(s[3], red)
        s[4] = min(s[4], red)
        s[5] += E / M
        s[6] += El / M
        s[7] += GOLD[c]["jdob"]["f_e"] > 0.0          # the plan offloads (R18: f_e = 0 iff all-local)
        s[9 + GOLD[c]["jdob"]["n_tilde"]] += 1
    fin = np.isfinite(exp)
    assert np.array_equal(np.isnan(exp), np.isnan(st))
    ok = fin & np.isfinite(st)
    assert np.allclose(st[ok], exp[ok], rtol=1e-12, atol=0.0)
    assert np.array_equal(np.isinf(exp), np.isinf(st))


def test_mutation_anchors_present():
    """tools/mutate_oracle.py stays applicable: every mutant's anchor occurs exactly once in the
    oracle source (the mutation run itself is profiles/r02_oracle_mutants.txt)."""
    import importlib.util
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    spec = importlib.util.spec_from_file_location("mutate_oracle", os.path.join(root, "tools", "mutate_oracle.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    src = open(mod.SRC).read()
    for name, _, old, new, _ in mod.MUTANTS:
        assert src.count(old) == 1, name
        assert old != new, name
