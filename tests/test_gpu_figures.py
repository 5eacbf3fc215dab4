"""NEXT-3 parity: the instances behind the Fig. 4/5-style sweeps (experiments/figures.py) solved on the
GPU equal the oracle bit for bit -- every method of Fig. 4 (LC, J-DOB, no edge DVFS, binary)
on all 64 identical-deadline instances, and the outer grouping DP with each inner method on a sample
of the Fig. 5 trials."""
import os
import sys

import numpy as np
import pytest

import oracle as O
from tests.gpu_util import assert_bits_equal, to_np

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "experiments"))
import figures as F  # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def J():
    import paper_2504_14611_b200 as J
    return J


def test_fig4_instances_vs_oracle(J):
    for beta, T, Ms, b in F.fig4_batches():
        db = J.DeviceBatch(b)
        multi = {m: to_np(r) for m, r in J.solve_batch_modes(db, f_user=False).items()}  # the sweep's call
        for name, mode in F.METHODS:
            gpu = to_np(J.solve_batch(db, mode=mode, f_user=False))
            orc = O.solve_batch(b, mode=mode)
            for f in ("E", "E_lc", "t_free_next", "f_e", "n_tilde", "j", "status"):
                assert_bits_equal(gpu[f], orc[f], f"fig4 beta={beta} {name} {f}")
                if mode != J.MODE_LC:
                    assert_bits_equal(multi[mode][f], orc[f], f"fig4 one-pass beta={beta} {name} {f}")
            if mode == J.MODE_LC:
                assert_bits_equal(multi[J.MODE_FULL]["E_lc"], orc["E"], f"fig4 one-pass LC beta={beta}")


def test_fig5_grouped_instances_vs_oracle(J):
    for M, lo, hi, b in F.fig5_batches(trials=4):
        db = J.DeviceBatch(b)
        for name, mode in F.METHODS:
            gpu = to_np(J.solve_grouped(db, mode=mode, f_user=False))
            orc = O.og_batch(b, mode=mode)
            assert_bits_equal(gpu["E"], orc["E"], f"fig5 M={M} [{lo},{hi}] {name} E")
            assert_bits_equal(gpu["n_groups"], orc["n_groups"], f"fig5 M={M} [{lo},{hi}] {name} groups")
