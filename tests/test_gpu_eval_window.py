"""K3's shared-memory windows (eval.cu): every way a tile's users can reach the kernel gives the
oracle's bits -- tiles whose users need several windows (M up to 32), instances that read no users
(empty, more than 32 users) mixed into the tiles, and user arrays whose base is not
16-byte aligned (the plain-load path instead of the bulk copies)."""
import copy

import numpy as np
import pytest

import jdobgen as g
import oracle as O
from tests.gpu_util import assert_bits_equal, to_np

pytestmark = pytest.mark.gpu

FIELDS = ("E", "t_free_next", "f_user", "status")


@pytest.fixture(scope="module")
def J():
    import paper_2504_14611_b200 as J
    return J


def mixed_batch(seed=150, n=1500):
    """Random instances (M up to 32) with malformed ones mixed in: empty instances (two equal
    offsets; a neighbour then owns the users) and instances with 33+ users."""
    b = g.random_batch(seed=seed, n_inst=n, M_hi=32, N_hi=8, k_max=40)
    rng = np.random.default_rng(seed)
    off = b.user_off.copy()
    for i in rng.choice(np.arange(1, n - 2), 12, replace=False):
        off[i] = off[i - 1]           # instance i - 1 empty, instance i takes its users
    for i in rng.choice(np.arange(2, n - 3), 6, replace=False):
        off[i] = off[i + 1]           # instance i empty; i - 1 has M(i-1) + M(i) users (often > 32)
    b.user_off = np.maximum.accumulate(off)
    return b


def general_vectors(b, seed):
    rng = np.random.default_rng(seed)
    part = np.zeros(b.n_users, np.int32)
    for i in range(b.n_inst):
        o0, o1 = int(b.user_off[i]), int(b.user_off[i + 1])
        mid = int(b.model_id[i])
        N = b.models[mid].N if 0 <= mid < len(b.models) else 1
        part[o0:o1] = rng.integers(0, N + 1, o1 - o0)
    fe = np.array([b.fe_max[i] - rng.integers(0, 5) * b.rho[i] for i in range(b.n_inst)])
    return part, fe


def unaligned(J, db):
    """The same batch with every user array moved to a base 8 bytes past a 16-byte boundary."""
    import torch
    d2 = copy.copy(db)
    d2.t = dict(db.t)
    keep = {}
    ptrs = {}
    for f in J.DeviceBatch.USER:
        t = db.t[f]
        pad = torch.empty(t.numel() + 1, dtype=t.dtype, device=t.device)
        pad[1:] = t
        keep[f] = pad
        ptrs[f] = pad.data_ptr() + 8
        assert ptrs[f] % 16 == 8
    d2._keep_unaligned = keep
    fields = {"model_id": db.t["model_id"].data_ptr(), "user_off": db.t["user_off"].data_ptr()}
    fields.update(ptrs)
    for f in J.DeviceBatch.INST:
        fields[f] = db.t[f].data_ptr()
    fields["bucket"] = None if db.t["bucket"] is None else db.t["bucket"].data_ptr()
    d2.jbatch = type(db.jbatch)(db.n_inst, db.n_models, *[fields[f] for f in ("model_id", "user_off") +
                                                          J.DeviceBatch.USER + J.DeviceBatch.INST + ("bucket",)])
    return d2


@pytest.mark.parametrize("seed", [150, 151])
def test_eval_windows_general_vectors(J, seed):
    import torch
    b = mixed_batch(seed)
    part, fe = general_vectors(b, seed)
    orc = O.eval_batch(b, part, fe, slack=1e-9)
    st = orc["status"]
    assert (st == 3).sum() >= 15  # malformed instances are present (BADPARAM)
    db = J.DeviceBatch(b)
    for view in (db, unaligned(J, db)):
        ev = to_np(J.eval_plans(view, torch.from_numpy(part), torch.from_numpy(fe), slack=1e-9))
        for f in FIELDS:
            if f == "f_user":   # users of malformed instances carry no result
                ok = np.repeat(st == 0, np.diff(b.user_off))
                assert_bits_equal(ev[f][ok], orc[f][ok], f)
            else:
                assert_bits_equal(ev[f], orc[f], f)
        assert_bits_equal(ev["violations"].view(np.uint32), orc["violations"], "violations")


def test_eval_windows_plans(J):
    """Plan form (the bench step's call) on a random batch with M up to 32 (several windows per tile),
    aligned and unaligned, against the oracle's eval of the mask-derived partition."""
    b = g.random_batch(seed=152, n_inst=2500, M_hi=32, N_hi=10, k_max=64)
    db = J.DeviceBatch(b)
    res = J.solve_batch(db, partition=True)
    part = J.plan_partition(db, res).cpu().numpy()
    orc = O.eval_batch(b, part, res["f_e"].cpu().numpy(), slack=1e-9)
    for view in (db, unaligned(J, db)):
        ev = to_np(J.eval_plans(view, plans=res, slack=1e-9))
        for f in FIELDS:
            assert_bits_equal(ev[f], orc[f], f)
        assert_bits_equal(ev["violations"].view(np.uint32), orc["violations"], "violations")
