"""Helpers for the GPU parity tests (compare CUDA results with the oracle)."""
import numpy as np


def to_np(res):
    out = {}
    for k, v in res.items():
        if v is None:
            continue
        a = v.detach().cpu().numpy()
        if k == "mask":
            a = a.view(np.uint32)
        out[k] = a
    return out


def assert_bits_equal(a, b, name):
    a = np.asarray(a)
    b = np.asarray(b)
    assert a.shape == b.shape, (name, a.shape, b.shape)
    if a.dtype.kind == "f":
        ai = a.view(np.int64)
        bi = b.view(np.int64)
        bad = np.nonzero((ai != bi) & ~(np.isnan(a) & np.isnan(b)))[0]
    else:
        bad = np.nonzero(a != b)[0]
    assert len(bad) == 0, f"{name}: {len(bad)} mismatches, first at {bad[:5]}: gpu={a[bad[:5]]} oracle={b[bad[:5]]}"


SOLVE_FIELDS = ("E", "E_lc", "t_free_next", "f_e", "n_tilde", "j", "status", "mask")


def assert_solve_parity(gpu, orc, fields=SOLVE_FIELDS, f_user=True, counts=False):
    """Decisions bit-exact; energies/times identical under the arithmetic contract
    (the north_star tolerance is relative 1e-9; the contract makes them bit-equal)."""
    for f in fields:
        assert_bits_equal(gpu[f], orc[f], f)
    if f_user:
        ok = orc["status"] <= 2
        # f_user of malformed instances is NaN on both sides (not written for M out of range)
        assert_bits_equal(gpu["f_user"], orc["f_user"], "f_user") if ok.all() else None
    if counts:
        assert_bits_equal(gpu["counts"], orc["counts"], "counts")


def rel_close(a, b, rel):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return np.all(np.abs(a - b) <= rel * np.maximum(np.abs(a), np.abs(b)) + 0.0)
