"""Oracle pins: hand-derived worked examples (tests/golden/toys.json).

Each expected value is recomputed here from its hand derivation (the 'hand'
strings: plain arithmetic on the instance numbers, written from PAPER.md's
equations) and compared with both the stored number and the oracle.
"""
import json
import math
import os

import numpy as np
import pytest

import jdobgen as g
import oracle as O

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "toys.json")))


def hand(expr):
    return eval(expr, {"__builtins__": {}}, {})


def close(a, b, rel=1e-12):
    return abs(a - b) <= rel * max(abs(a), abs(b), 1e-300)


@pytest.mark.parametrize("toy", ["toy-1", "toy-4"])
def test_lc(toy):
    gd = GOLD[toy]["lc"]
    E, f, _ = O.lc(g.toy_instance(toy))
    assert close(hand(gd["hand"]), gd["E"])
    assert close(E, gd["E"])
    assert np.allclose(f, gd["f"], rtol=1e-15)


def test_lc_boundaries():
    # T exactly the minimum local latency -> f = f_max; T huge -> f = f_min
    b = g.toy_instance("toy-1")
    vN = 3e8
    b.T[:] = [vN / 2.6e9, 1e6]
    E, f, e = O.lc(b)
    assert f[0] == 2.6e9 and f[1] == 1.5e9
    assert O.check_inst(b) == O.ST_OK


def test_gamma_toy1():
    gd = GOLD["toy-1"]["gamma"]
    b = g.toy_instance("toy-1")
    for nt, v, h in zip(gd["nt"], gd["values"], gd["hand"]):
        gam, lst, th = O.thresholds(b, 0, nt)
        assert close(gam[0], hand(h)) and close(gam[1], hand(h))
        assert close(gam[0], v, 1e-9)


@pytest.mark.parametrize("toy,key,nt", [("toy-1", "thresholds_nt1", 1), ("toy-2", "thresholds_nt0", 0)])
def test_thresholds(toy, key, nt):
    gd = GOLD[toy][key]
    gam, lst, th = O.thresholds(g.toy_instance(toy), 0, nt)
    assert list(lst) == [0, 1]              # equal gamma: T ascending (R2), T = [0.2, 0.25]
    for i in range(2):
        assert close(th[i], hand(gd["hand"][i]), 1e-12)
        assert close(th[i], gd["values"][i], gd["rel"])
    assert th[0] >= th[1]                  # non-increasing


def test_eval_toy1_examples():
    gd = GOLD["toy-1"]["eval_both_offload_nt1_fe2.1"]
    b = g.toy_instance("toy-1")
    r = O.eval_config(b, 0, gd["nvec"], gd["fe"])
    assert close(r["E"], hand(gd["hand_E"]))
    assert close(r["E"], gd["E"])
    assert close(r["t_free_next"], hand(gd["hand_tf"]))
    assert close(r["t_free_next"], gd["t_free_next"])
    assert r["violations"] == 0
    # empty offload set = LC
    r = O.eval_config(b, 0, [2, 2], 2.1e9)
    assert close(r["E"], 1.35) and r["t_free_next"] == 0.0 and r["violations"] == 0
    # D6 violated with t_free = 0.15
    b.t_free[0] = 0.15
    gd = GOLD["toy-1"]["eval_tfree_0.15_infeasible"]
    r = O.eval_config(b, 0, gd["nvec"], gd["fe"])
    assert r["violations"] & gd["violation_bit"]


@pytest.mark.parametrize("toy", ["toy-1", "toy-2", "toy-2-m1", "toy-2-tfree", "toy-4"])
def test_jdob_golden(toy):
    gd = GOLD[toy]["jdob"]
    r = O.jdob(g.toy_instance(toy))
    assert r["status"] == O.ST_OK
    if "hand_E" in gd:
        assert close(hand(gd["hand_E"]), gd["E"], 1e-12)
    assert close(r["E"], gd["E"], 1e-12)
    assert r["n_tilde"] == gd["n_tilde"] and r["mask"] == gd["mask"] and r["j"] == gd["j"]
    if "f_e" in gd:
        assert r["f_e"] == gd["f_e"]
    if "hand_tf" in gd:
        assert close(hand(gd["hand_tf"]), gd["t_free_next"], 1e-12)
    assert close(r["t_free_next"], gd["t_free_next"], 1e-12)
    if "f_user" in gd:
        assert np.allclose(r["f_user"], gd["f_user"], rtol=1e-15)


def test_toy1_hand_breakdown():
    # SURVEY §0.2 finding 1: user 1 offloading after block 1 at f_e = 0.9 GHz pays
    # 0.225 (device) + 0.004 (upload) + 0.405 (edge) = 0.634 J < 0.675 J locally.
    dev = 1e-27 * 1e8 * 1.5e9 ** 2
    up = 4e5 / 1e8
    edge = 2.5e-27 * 2e8 * 0.9e9 ** 2
    assert close(dev, 0.225) and close(up, 0.004) and close(edge, 0.405)
    assert dev + up + edge < 0.675
    # D6 and D7 at the plan (0.1778 <= 0.25, 0.2485 <= 0.25)
    assert 0.8 * 2e8 / 0.9e9 <= 0.25
    assert 1e8 / 1.5e9 + 4e5 / 1e8 + 0.8 * 2e8 / 0.9e9 <= 0.25


@pytest.mark.parametrize("toy,mode_key", [("toy-2", "jdob_no_edge_dvfs"), ("toy-2-m1", "jdob_no_edge_dvfs")])
def test_no_edge_dvfs_golden(toy, mode_key):
    gd = GOLD[toy][mode_key]
    r = O.jdob(g.toy_instance(toy), mode=O.MODE_NO_EDGE_DVFS)
    assert close(hand(gd["hand_E"]), gd["E"], 1e-12)
    assert close(r["E"], gd["E"], 1e-12)


def test_variants_toy1():
    # toy-1 no-edge 1.35, binary 1.35; toy-2 binary 0.0642368
    b = g.toy_instance("toy-1")
    assert close(O.jdob(b, mode=O.MODE_NO_EDGE_DVFS)["E"], 1.35)
    assert close(O.jdob(b, mode=O.MODE_BINARY)["E"], 1.35)
    assert close(O.jdob(g.toy_instance("toy-2"), mode=O.MODE_BINARY)["E"], 0.0642368)


def test_bf_toy4():
    b = g.toy_instance("toy-4")
    gi = GOLD["toy-4"]["bf_identical"]
    E, idx, st = O.bf(b, 1)
    assert st == 0 and close(E, gi["E"]) and idx == gi["idx"]
    gg = GOLD["toy-4"]["bf_general"]
    E, idx, st = O.bf(b, 0)
    assert close(hand(gg["hand_E"]), gg["E"], 1e-12)
    assert close(E, gg["E"], 1e-12) and idx == gg["idx"]
    k = O.grid_k(b)
    assert k == 3
    assert idx % k == gg["j"]
    vec = idx // k
    assert [vec // 5, vec % 5] == gg["vec"]


@pytest.mark.parametrize("toy", ["toy-1", "toy-2", "toy-2-m1", "toy-2-tfree"])
def test_bf_equals_jdob_on_toys(toy):
    b = g.toy_instance(toy)
    r = O.jdob(b)
    Ei, _, _ = O.bf(b, 1)
    Eg, _, _ = O.bf(b, 0)
    assert close(Ei, r["E"], 1e-12)
    assert Eg <= Ei


def test_rate_and_beta_closed_forms():
    # R = W log2(1 + SNR) with Table I
    assert close(g.rate(10e6, 30.0), 9.967226258835992e7, 1e-12)
    assert close(g.rate(1e7, 0.0), 1e7)
    # beta <-> T pairs of Fig. 4 imply a minimum local latency of ~3.2 ms
    assert abs(10e-3 / (1 + 2.13) - 100e-3 / (1 + 30.25)) < 0.01e-3
    m = g.profiles.mobilenetv2()
    lat = g.min_local_latency(m, np.array([g.profiles.ZETA]), np.array([2.6e9]))[0]
    assert abs(lat - 3.2e-3) < 0.01e-3
    # toy: beta = 0.733333 -> T = 0.2
    T = g.deadline_from_beta(g.profiles.toy1(), 1.0, 2.6e9, 0.7333333333333334)
    assert close(float(T), 0.2, 1e-12)


def test_calibration_closed_forms():
    # d_n(1) = zeta fe_max / (alpha f_max), SPEC S:80 with zeta = 1: 2.1/2.6
    z = 1.0
    d1 = z * 2.1e9 / (1.0 * 2.6e9)
    assert close(d1, 0.8076923076923077, 1e-12)
    # c_n(1) = d1 (kappa/zeta) f_max^3 / (eta fe_max^3): 2.554800e-27 (SURVEY §4.2 corrects S:81)
    c1 = d1 * (1e-27 / z) * 2.6e9 ** 3 / (0.6 * 2.1e9 ** 3)
    assert abs(c1 - 2.5548e-27) < 1e-31


def test_status_codes():
    b = g.toy_instance("toy-1")
    assert O.check_inst(b) == O.ST_OK
    bb = g.toy_instance("toy-1"); bb.T[0] = 0.1          # zeta vN / f_max = 0.1154 > 0.1
    assert O.check_inst(bb) == O.ST_LOCAL_INFEASIBLE
    r = O.jdob(bb)
    assert r["status"] == O.ST_LOCAL_INFEASIBLE and r["mask"] == 0 and r["n_tilde"] == 2
    bb = g.toy_instance("toy-1"); bb.t_free[0] = 0.21    # min T = 0.2 < t_free
    assert O.check_inst(bb) == O.ST_REQUIRE
    r = O.jdob(bb)
    assert r["status"] == O.ST_REQUIRE and close(r["E"], 1.35)
    bb = g.toy_instance("toy-1"); bb.f_min[1] = 3e9      # f_min > f_max
    assert O.check_inst(bb) == O.ST_BADPARAM
    bb = g.toy_instance("toy-1"); bb.R[0] = 0.0
    assert O.check_inst(bb) == O.ST_BADPARAM
    bb = g.toy_instance("toy-1"); bb.models[0].d[1 * 3 + 2] = 0.5   # d_1(2) < d_1(1): non-monotone
    assert O.check_inst(bb) == O.ST_BADMODEL
    bb = g.toy_instance("toy-1"); bb.fe_min[0] = 3e9
    assert O.check_inst(bb) == O.ST_BADPARAM
    r = O.jdob(bb)
    assert r["status"] == O.ST_BADPARAM and math.isnan(r["E"])
