"""GPU parity on the hand-derived tie and boundary instances (tests/golden/boundaries.json).

Each instance is decided by one tie or boundary rule (R2 sort key, strict `<` of Alg. 1/2,
non-strict D6 guard / D6', membership at f_e = f_th, the D20 clamp at f_max, R9 at a zero
budget, the OG (E, t_free) tie).  The CUDA path must reproduce the golden answers and agree
with the oracle bit for bit, in the uniform-users kernel (the instances as written) and in the
general kernel ("hetero twins": a second, never-offloading user with a different R, so the
instance is no longer uniform while the boundary structure is unchanged)."""
import numpy as np
import pytest

import jdobgen as g
import oracle as O
from tests.gpu_util import assert_bits_equal, assert_solve_parity, to_np
from tests.test_gpu_parity import _og_parity, run
from tests.test_oracle_boundaries import CASES, GOLD, build, close

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def J():
    import paper_2504_14611_b200 as J
    return J


JDOB_CASES = [c for c in CASES if "jdob" in GOLD[c]]


def twin(case):
    """The instance plus one user that never offloads (its R is 1e6x smaller: O/R exceeds every
    deadline, so its threshold is negative and it sorts first), with B_max >= M + 1."""
    b = build(case)
    m = b.models[0]
    M1 = b.M(0) + 1
    if m.B_max < M1:  # one more batch column, equal to the last one (d non-decreasing)
        N, B = m.N, m.B_max
        d = np.zeros((N + 1) * (M1 + 1))
        c = np.zeros((N + 1) * (M1 + 1))
        for n in range(1, N + 1):
            for bb in range(1, M1 + 1):
                d[n * (M1 + 1) + bb] = m.d[n * (B + 1) + min(bb, B)]
                c[n * (M1 + 1) + bb] = m.c[n * (B + 1) + min(bb, B)]
        m = g.Model(m.name + "-twin", N, M1, m.A, m.O, m.g, m.q, d, c)
    users = {f: np.concatenate([getattr(b, f), getattr(b, f)[:1]]) for f in g.Batch.USER_FIELDS}
    users["R"][-1] = users["R"][-1] * 1e-6
    users["T"][-1] = float(users["T"].max())
    return g.single_instance(m, users, t_free=float(b.t_free[0]), fe_min=float(b.fe_min[0]),
                             fe_max=float(b.fe_max[0]), rho=float(b.rho[0]))


def check_golden(gpu, i, gd, extra_users=0):
    assert int(gpu["status"][i]) == 0
    assert (int(gpu["n_tilde"][i]), int(gpu["j"][i])) == (gd["n_tilde"], gd["j"])
    assert int(gpu["mask"][i]) == gd["mask"]
    assert float(gpu["f_e"][i]) == gd["f_e"]
    if not extra_users:
        assert close(float(gpu["E"][i]), gd["E"])
        assert close(float(gpu["t_free_next"][i]), gd["t_free_next"])


def test_boundaries_uniform_kernel(J):
    batch = g.concat([build(c) for c in JDOB_CASES])
    _, gpu = run(J, batch)
    orc = O.solve_batch(batch, counts=True)
    assert_solve_parity(gpu, orc, counts=True)
    for i, c in enumerate(JDOB_CASES):
        gd = GOLD[c]["jdob"]
        check_golden(gpu, i, gd)
        o0 = int(batch.user_off[i])
        assert list(gpu["f_user"][o0:o0 + batch.M(i)]) == gd["f_user"]
        if "counts" in gd:
            cnt = gd["counts"]
            assert tuple(gpu["counts"][i]) == (cnt["n_visit"], cnt["n_eval"], cnt["n_member"])


def test_boundaries_general_kernel(J):
    batch = g.concat([twin(c) for c in JDOB_CASES])
    _, gpu = run(J, batch)
    orc = O.solve_batch(batch, counts=True)
    assert_solve_parity(gpu, orc, counts=True)
    for i, c in enumerate(JDOB_CASES):
        gd = GOLD[c]["jdob"]
        # the extra user sorts first and never offloads: the decisions are the golden ones
        check_golden(gpu, i, gd, extra_users=1)
        o0 = int(batch.user_off[i])
        assert list(gpu["f_user"][o0:o0 + len(gd["f_user"])]) == gd["f_user"]


@pytest.mark.parametrize("mode", [1, 2, 3])
def test_boundaries_modes(J, mode):
    batch = g.concat([build(c) for c in JDOB_CASES] + [twin(c) for c in JDOB_CASES])
    _, gpu = run(J, batch, mode=mode)
    assert_solve_parity(gpu, O.solve_batch(batch, mode=mode, counts=True), counts=True)


@pytest.mark.parametrize("case,space", [(c, s) for c in CASES for s, key in ((0, "bf_general"), (1, "bf_identical"))
                                        if key in GOLD[c]])
def test_boundaries_bruteforce(J, case, space):
    gd = GOLD[case]["bf_general" if space == 0 else "bf_identical"]
    for b in (build(case), twin(case)):
        db = J.DeviceBatch(b)
        E, I, S = J.bruteforce(db, space)
        Eo, Io, So = O.bf(b, space)
        assert int(S.item()) == So == 0
        assert_bits_equal(E.cpu().numpy(), np.array([Eo]), f"{case} E")
        assert int(I.item()) == Io
    E, I, _ = J.bruteforce(J.DeviceBatch(build(case)), space)
    assert int(I.item()) == gd["idx"]
    assert close(float(E.item()), gd["E"]) if gd["E"] != 0.0 else float(E.item()) == 0.0


def test_boundaries_eval(J):
    for mk in (build, twin):
        batch = g.concat([mk(c) for c in JDOB_CASES])
        db = J.DeviceBatch(batch)
        res = J.solve_batch(db, partition=True)
        ev = to_np(J.eval_plans(db, plans=res, slack=0.0))
        part = res["partition"].cpu().numpy()
        orc = O.eval_batch(batch, part, res["f_e"].cpu().numpy(), slack=0.0)
        for f in ("E", "t_free_next", "f_user", "status"):
            assert_bits_equal(ev[f], orc[f], f)
        assert_bits_equal(ev["violations"].view(np.uint32), orc["violations"], "violations")
        assert_bits_equal(ev["E"], to_np(res)["E"], "eval E == plan E")


@pytest.mark.parametrize("case", [c for c in CASES if "og" in GOLD[c]])
def test_boundaries_og(J, case):
    b = build(case)
    _og_parity(J, b)
    gd = GOLD[case]["og"]
    res = J.solve_grouped(J.DeviceBatch(b))
    assert float(res["E"][0]) == gd["E"] and float(res["t_free_next"][0]) == gd["t_free_next"]
    assert int(res["n_groups"][0]) == gd["n_groups"]
    assert list(res["partition"].cpu().numpy()) == gd["part"]


def test_boundaries_stats(J):
    batch = g.concat([build(c) for c in JDOB_CASES])
    _, gpu = run(J, batch, stats=True, n_buckets=32)
    st = O.stats(batch, O.solve_batch(batch), n_buckets=32)
    for f in (0, 3, 4, 7, 8):
        assert_bits_equal(gpu["stats"][:, f], st[:, f], f"stats[{f}]")
    assert_bits_equal(gpu["stats"][:, 9:], st[:, 9:], "hist")
    for f in (1, 2, 5, 6):  # fixed-tree sums vs instance-order sums: rel 1e-9, NaN = NaN
        a, b = gpu["stats"][:, f], st[:, f]
        assert np.array_equal(np.isnan(a), np.isnan(b))
        ok = ~np.isnan(a)
        assert np.all(np.abs(a[ok] - b[ok]) <= 1e-9 * np.maximum(np.abs(a[ok]), np.abs(b[ok])))


@pytest.mark.parametrize("case", CASES)
def test_boundaries_fused_verify(J, case):
    """The solver's epilogue verification (row a11) on the boundary instances: the bits of jdob_eval,
    at slack 0 and 1e-9 (the R10 clamp cases sit exactly on D7)."""
    for b in (build(case), twin(case)):
        db = J.DeviceBatch(b)
        for slack in (0.0, 1e-9):
            res = J.solve_batch(db, verify=True, slack=slack)
            ev = to_np(J.eval_plans(db, plans=res, slack=slack))
            assert_bits_equal(res["violations"].cpu().numpy().view(np.uint32), ev["violations"], case)
