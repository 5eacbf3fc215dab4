"""SURVEY §4.3 T5 on one GPU: the CUDA path run as P sequential shards (the ranks of a P-GPU job) and
merged with the multi-GPU exchange rules of paper_2504_14611_b200.dist equals the unsharded call bit
for bit -- brute-force argmin over vector-aligned index shards, J-DOB per-instance outputs over
instance shards, and the statistics folded from jdob_stats_part roots (P = 2, 4, 8)."""
import numpy as np
import pytest
import torch

import jdobgen as g
from paper_2504_14611_b200 import dist as D
from tests.gpu_util import assert_bits_equal, to_np

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def J():
    import paper_2504_14611_b200 as J
    return J


def merge_argmin(parts):
    """allreduce_argmin's rule on host values: MIN over E, then MIN over the indices holding it."""
    E = min(e for e, _ in parts)
    idx = [i for e, i in parts if e == E and i >= 0]
    return E, (min(idx) if idx else -1)


@pytest.mark.parametrize("P", [2, 4, 8])
def test_bf_shards_equal_unsharded(J, P):
    b = g.config_batch("c4")
    db = J.DeviceBatch(b)
    k = g.grid_size(float(b.fe_min[0]), float(b.fe_max[0]), float(b.rho[0]))
    size = J.bf_space_size(0, b.models[0].N, b.M(0), k)
    E, I, _ = J.bruteforce(db, 0, 0, size)
    parts = []
    for r in range(P):
        lo, hi = D.bf_shard(size, k, P, r)
        Er, Ir, _ = J.bruteforce(db, 0, lo, hi)
        parts.append((float(Er.item()), int(Ir.item())))
    assert merge_argmin(parts) == (float(E.item()), int(I.item()))
    # the same merge through the torch code bench.py runs (one "rank" at a time on the device)
    Eg = torch.tensor([p[0] for p in parts], dtype=torch.float64, device="cuda").min()
    assert float(Eg.item()) == float(E.item())


@pytest.mark.parametrize("cfg,n", [("c3", 100_000), ("c5", 40_000)])
@pytest.mark.parametrize("P", [2, 4, 8])
def test_jdob_shards_and_stats_equal_unsharded(J, cfg, n, P):
    full = g.config_batch(cfg, n_inst=n)
    nb = int(full.meta.get("n_buckets", 32))
    dfull = J.DeviceBatch(full)
    rf = J.solve_batch(dfull, f_user=False)
    sf = J.stats(dfull, rf, n_buckets=nb).cpu().numpy()
    rf = to_np(rf)
    roots = []
    for r in range(P):
        lo, hi = D.shard_range(n, P, r)
        part = g.config_batch(cfg, n_inst=hi - lo, inst_begin=lo)
        dp = J.DeviceBatch(part)
        rp = J.solve_batch(dp, f_user=False)
        roots.append(J.stats(dp, rp, n_buckets=nb, part=(n, P, r)))
        rp = to_np(rp)
        for f in ("E", "E_lc", "t_free_next", "f_e", "n_tilde", "j", "status", "mask"):
            assert_bits_equal(rp[f], rf[f][lo:hi], f"{f} shard {r}/{P}")
    folded = D.fold_parts(torch.stack(roots)).cpu().numpy()
    assert_bits_equal(folded.reshape(-1), sf.reshape(-1), f"stats folded over {P} parts")


def test_stats_part_rejects_a_wrong_part(J):
    b = g.config_batch("c3", n_inst=1000)
    db = J.DeviceBatch(b)
    r = J.solve_batch(db, f_user=False)
    with pytest.raises(J.JdobError):
        J.stats(db, r, n_buckets=3, part=(2000, 3, 0))   # 3 parts: not a power of two
    with pytest.raises(J.JdobError):
        J.stats(db, r, n_buckets=3, part=(2001, 2, 1))   # part 1 of 2001 has 1001 instances
