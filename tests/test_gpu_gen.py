"""T9: the device generator of the C5 workload (jdob_generate_c5_*, csrc/gen.cu) writes
the same arrays as the host generator jdobgen.config_c5, bit for bit, for any instance range; and the
C5 Monte Carlo run from device-generated instances (no input H2D) matches the oracle on a prefix."""
import numpy as np
import pytest

import jdobgen as g
import oracle as O
from tests.gpu_util import assert_bits_equal, to_np

pytestmark = pytest.mark.gpu

FIELDS = ("model_id", "user_off", "zeta", "kappa", "f_min", "f_max", "R", "p_u", "T", "t_free", "fe_min", "fe_max",
          "rho", "bucket")


@pytest.fixture(scope="module")
def J():
    import paper_2504_14611_b200 as J
    return J


@pytest.mark.parametrize("begin,n,hetero", [(0, 50_000, False), (123_457, 20_000, False), (9_000_000, 7_000, True)])
def test_device_generator_bit_identical(J, begin, n, hetero):
    host = g.config_c5(n_inst=n, inst_begin=begin, hetero=hetero)
    models, params = g.c5_device_inputs(inst_begin=begin, hetero=hetero)
    db = J.DeviceBatch.generate_c5(models, params, n)
    assert db.n_users == host.n_users
    for f in FIELDS:
        assert_bits_equal(db.t[f].cpu().numpy(), np.asarray(getattr(host, f)), f)


def test_c5_device_generated_prefix_vs_oracle(J):
    """10^7 instances generated on the device and solved there; the first 10^6 are regenerated on the
    host and solved by the oracle: every decision and energy equal bit for bit (the statistics of the
    whole run come from the same device arrays)."""
    n, pre = 10_000_000, 1_000_000
    models, params = g.c5_device_inputs()
    db = J.DeviceBatch.generate_c5(models, params, n)
    res = J.solve_batch(db, f_user=False)
    st = J.stats(db, res, n_buckets=480)
    gpu = to_np({k: v[:pre] for k, v in res.items() if k in ("E", "E_lc", "t_free_next", "f_e", "n_tilde", "j",
                                                               "status", "mask")})
    host = g.config_c5(n_inst=pre)
    orc = O.solve_batch(host, threads=16)
    for f in ("E", "E_lc", "t_free_next", "f_e", "n_tilde", "j", "status"):
        assert_bits_equal(gpu[f], orc[f], f)
    assert np.array_equal(gpu["mask"], orc["mask"])
    assert float(st[:, 0].sum().item()) + float(st[:, 8].sum().item()) == n
