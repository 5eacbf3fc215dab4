"""Multi-process (world size 2, gloo, CPU) tests of the sharding and exchange logic.

Each rank computes its shard with the oracle (the CUDA kernels need a GPU; the
host-side sharding/merge code is the same), then merges through
paper_2504_14611_b200.dist exactly as bench.py does over NCCL."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import jdobgen as g
import oracle as O
from paper_2504_14611_b200 import dist as D


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, fn, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        q.put((rank, fn(rank, world)))
    finally:
        dist.destroy_process_group()


def run_world(fn, world=2):
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_worker, args=(r, world, port, fn, q)) for r in range(world)]
    for p in ps:
        p.start()
    out = dict(q.get(timeout=300) for _ in range(world))
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    return out


def _bf_shard_fn(rank, world):
    b = g.toy_instance("toy-4")
    size = O.bf_space_size(b, 0)
    k = O.grid_k(b)
    lo, hi = D.bf_shard(size, k, world, rank)
    E, idx, _ = O.bf(b, 0, lo, hi)
    Et = torch.tensor([E], dtype=torch.float64)
    It = torch.tensor([idx], dtype=torch.int64)
    Eg, Ig = D.allreduce_argmin(Et, It, dist)
    return float(Eg.item()), int(Ig.item()), lo, hi


def test_bf_sharded_argmin_equals_sequential():
    out = run_world(_bf_shard_fn)
    b = g.toy_instance("toy-4")
    E, idx, _ = O.bf(b, 0)
    size = O.bf_space_size(b, 0)
    assert out[0][2] == 0 and out[1][3] == size and out[0][3] == out[1][2]
    for r in (0, 1):
        assert out[r][0] == E and out[r][1] == idx


def _bf_tie_fn(rank, world):
    # equal E on both ranks: the lower index must win; a rank with no feasible candidate never wins
    E = torch.tensor([1.5], dtype=torch.float64)
    I = torch.tensor([100 if rank == 1 else 7], dtype=torch.int64)
    a = D.allreduce_argmin(E, I, dist)
    E2 = torch.tensor([float("inf") if rank == 0 else 2.0], dtype=torch.float64)
    I2 = torch.tensor([-1 if rank == 0 else 55], dtype=torch.int64)
    b = D.allreduce_argmin(E2, I2, dist)
    return float(a[0]), int(a[1]), float(b[0]), int(b[1])


def test_bf_tie_break_and_empty_rank():
    out = run_world(_bf_tie_fn)
    for r in (0, 1):
        assert out[r] == (1.5, 7, 2.0, 55)


def _stats_fn(rank, world):
    b = g.config_batch("c3", n_inst=3000)
    lo, hi = D.shard_range(b.n_inst, world, rank)
    sub = b.subset(lo, hi)
    res = O.solve_batch(sub)
    st = torch.from_numpy(O.stats(sub, res, n_buckets=3))
    red = D.allreduce_stats(st, dist)
    return red.numpy()


def test_stats_sharded_equals_full():
    out = run_world(_stats_fn)
    b = g.config_batch("c3", n_inst=3000)
    full = O.stats(b, O.solve_batch(b), n_buckets=3)
    for r in (0, 1):
        st = out[r]
        for f in (0, 3, 4, 7, 8):
            assert np.array_equal(st[:, f], full[:, f])
        assert np.array_equal(st[:, 9:], full[:, 9:])
        for f in (1, 2, 5, 6):
            assert np.allclose(st[:, f], full[:, f], rtol=1e-12, atol=0)


def test_shard_ranges_cover():
    for n in (0, 1, 7, 1000):
        for w in (1, 2, 3, 8):
            rs = [D.shard_range(n, w, r) for r in range(w)]
            assert rs[0][0] == 0 and rs[-1][1] == n
            assert all(rs[i][1] == rs[i + 1][0] for i in range(w - 1))
    size, k = 12 ** 8 * 64, 64
    rs = [D.bf_shard(size, k, 8, r) for r in range(8)]
    assert rs[0][0] == 0 and rs[-1][1] == size and all(a % k == 0 for a, _ in rs)


def _fold_fn(rank, world):
    # per-rank roots (random, with the max/min fields) folded over gloo: every rank gets the pairwise fold
    rng = np.random.default_rng(100 + rank)
    st = torch.from_numpy(rng.random((3, 80)) * 10.0 ** rng.integers(-3, 4, (3, 80)))
    return D.fold_stats(st, dist).numpy(), st.numpy()


def test_fold_stats_is_the_pairwise_tree():
    out = run_world(_fold_fn)
    roots = np.stack([out[0][1], out[1][1]])
    want = roots[0] + roots[1]
    want[:, 3] = np.maximum(roots[0][:, 3], roots[1][:, 3])
    want[:, 4] = np.minimum(roots[0][:, 4], roots[1][:, 4])
    for r in (0, 1):
        assert np.array_equal(out[r][0], want)
    # four parts: ((p0 + p1) + (p2 + p3)), field by field
    rng = np.random.default_rng(5)
    p = rng.random((4, 2, 80))
    f = D.fold_parts(torch.from_numpy(p)).numpy()
    s = (p[0] + p[1]) + (p[2] + p[3])
    assert np.array_equal(f[:, 5], s[:, 5])
    assert np.array_equal(f[:, 3], p[:, :, 3].max(0)) and np.array_equal(f[:, 4], p[:, :, 4].min(0))
