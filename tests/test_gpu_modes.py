"""NEXT-2 in one pass (jdob_solve_batch_modes): J-DOB, J-DOB without edge DVFS and binary J-DOB from one
sweep must equal, bit for bit, the separate jdob_solve_batch call of each mode (itself oracle-checked in
test_gpu_parity.py::test_random_modes) -- and the oracle directly on the heterogeneous suite."""
import pytest

import jdobgen as g
import oracle as O
from tests.gpu_util import assert_bits_equal, assert_solve_parity, to_np
from tests.test_gpu_parity import _large_batch, uniformise

pytestmark = pytest.mark.gpu

FIELDS = ("E", "E_lc", "t_free_next", "f_e", "n_tilde", "j", "status", "mask", "f_user", "partition", "stats")


@pytest.fixture(scope="module")
def J():
    import paper_2504_14611_b200 as J
    return J


def check(J, b, oracle=False, n_buckets=None):
    db = J.DeviceBatch(b)
    kw = dict(stats=n_buckets is not None, n_buckets=n_buckets, partition=True)
    multi = {m: to_np(r) for m, r in J.solve_batch_modes(db, **kw).items()}
    for mode in (J.MODE_FULL, J.MODE_NO_EDGE_DVFS, J.MODE_BINARY):
        one = to_np(J.solve_batch(db, mode=mode, **kw))
        for f in FIELDS:
            if f in one:
                assert_bits_equal(multi[mode][f], one[f], f"mode {mode} {f}")
        if oracle:
            assert_solve_parity(multi[mode], O.solve_batch(b, mode=mode))
    return multi


@pytest.mark.parametrize("seed,M_hi,N_hi,k_max", [(191, 8, 6, 40), (192, 32, 19, 120)])
def test_modes_random(J, seed, M_hi, N_hi, k_max):
    b = g.random_batch(seed=seed, n_inst=1500, M_lo=1, M_hi=M_hi, N_lo=1, N_hi=N_hi, k_max=k_max)
    check(J, b, oracle=True)


def test_modes_uniform_and_configs(J):
    check(J, uniformise(g.random_batch(seed=193, n_inst=1500, M_lo=1, M_hi=20, N_lo=1, N_hi=12, k_max=64), 193))
    c3 = g.config_batch("c3", n_inst=20000)
    check(J, c3, n_buckets=3)
    c2 = g.config_batch("c2", n_inst=20000)
    check(J, c2, n_buckets=7)


def test_modes_zero_energy_ties(J):
    """Every configuration costs E_LC = 0: each mode's answer is its (E, n~, j) tie rule against its own
    first all-local evaluation, through the literal re-sweep."""
    b = g.random_batch(seed=194, n_inst=800, M_lo=1, M_hi=32, N_lo=1, N_hi=12, k_max=50)
    b.kappa[:] = 0.0
    b.p_u[:] = 0.0
    for m in b.models:
        m.c[:] = 0.0
    check(J, b, oracle=True)


def test_modes_large_m_and_edge_cases(J):
    check(J, _large_batch([40, 33, 70], 195, hetero=True, tfree=True))
    b = g.random_batch(seed=196, n_inst=300, M_lo=1, M_hi=12, N_lo=1, N_hi=8, k_max=30)
    b.T[b.user_off[3]] = -1.0          # BADPARAM
    b.t_free[5] = 10.0 * b.T[b.user_off[5]:b.user_off[6]].max()   # REQUIRE
    check(J, b, oracle=True)
