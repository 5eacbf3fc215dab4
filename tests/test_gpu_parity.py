"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle, element by element.

Bar (BASELINE.json north_star): decisions and partition indices bit-exact; energies
within relative 1e-9 -- the arithmetic contract makes them bit-identical, which is
what these tests assert."""
import numpy as np
import pytest

import jdobgen as g
import oracle as O
from tests.gpu_util import assert_bits_equal, assert_solve_parity, rel_close, to_np

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def J():
    import paper_2504_14611_b200 as J
    return J


PRODUCT_FIELDS = ("E", "E_lc", "t_free_next", "f_e", "n_tilde", "j", "status", "mask", "f_user")


def run(J, batch, mode=0, counts=True, stats=False, n_buckets=None):
    """Solve on the GPU.  With counts, the literal (unpruned) sweep runs; the pruned product path
    (no counters) and its executed-work variant run as well and must give the same bits."""
    db = J.DeviceBatch(batch)
    res = J.solve_batch(db, mode=mode, counts=counts, stats=stats, n_buckets=n_buckets)
    import torch
    torch.cuda.synchronize()
    out = to_np(res)
    if counts:
        for kw in (dict(), dict(work=True)):
            alt = to_np(J.solve_batch(db, mode=mode, stats=stats, n_buckets=n_buckets, **kw))
            for f in PRODUCT_FIELDS + (("stats",) if stats else ()):
                assert_bits_equal(alt[f], out[f], f"pruned vs literal {f} {kw}")
            if kw:
                check_work(batch, alt["work"], out["counts"], mode)
    return db, out


def check_work(batch, work, counts, mode):
    """Executed work of the pruned sweep: at most the literal work (twice in the rare E = E_LC re-sweep)."""
    N = np.array([batch.models[m].N for m in batch.model_id])
    assert (work[:, 0] <= 2 * N).all()
    assert (work[:, 1:] <= 2 * counts).all()
    assert (work >= 0).all()


@pytest.mark.parametrize("toy", ["toy-1", "toy-2", "toy-2-m1", "toy-2-tfree", "toy-4"])
def test_toys(J, toy):
    b = g.toy_instance(toy)
    _, gpu = run(J, b)
    orc = O.solve_batch(b, counts=True)
    assert_solve_parity(gpu, orc, counts=True)


@pytest.mark.parametrize("seed,M_hi,N_hi,k_max", [(101, 4, 3, 12), (102, 12, 8, 70), (103, 32, 12, 70),
                                                 (104, 32, 5, 200), (105, 20, 19, 64)])
def test_random_full(J, seed, M_hi, N_hi, k_max):
    b = g.random_batch(seed=seed, n_inst=1500, M_lo=1, M_hi=M_hi, N_lo=1, N_hi=N_hi, k_max=k_max)
    _, gpu = run(J, b)
    orc = O.solve_batch(b, counts=True)
    assert_solve_parity(gpu, orc, counts=True)


def uniformise(b, seed=0):
    """Copy user 0's device parameters to every user of each instance (only T differs),
    keeping every user locally feasible: the kernel's uniform-users path."""
    rng = np.random.default_rng(seed)
    for i in range(b.n_inst):
        o0, o1 = int(b.user_off[i]), int(b.user_off[i + 1])
        for f in ("zeta", "kappa", "f_min", "f_max", "R", "p_u"):
            getattr(b, f)[o0:o1] = getattr(b, f)[o0]
        lat = float(g.min_local_latency(b.models[b.model_id[i]], np.array([b.zeta[o0]]), np.array([b.f_max[o0]]))[0])
        beta = rng.uniform(0, 10, o1 - o0)
        if rng.uniform() < 0.3:
            beta[:] = beta[0]
        b.T[o0:o1] = (1.0 + beta) * lat
        if b.t_free[i] > b.T[o0:o1].min():
            b.t_free[i] = 0.5 * b.T[o0:o1].min()
    return b


@pytest.mark.parametrize("seed,M_hi,N_hi,k_max", [(161, 8, 6, 40), (162, 32, 19, 200)])
def test_random_uniform_users(J, seed, M_hi, N_hi, k_max):
    b = uniformise(g.random_batch(seed=seed, n_inst=1500, M_lo=1, M_hi=M_hi, N_lo=1, N_hi=N_hi, k_max=k_max), seed)
    _, gpu = run(J, b)
    orc = O.solve_batch(b, counts=True)
    assert_solve_parity(gpu, orc, counts=True)


@pytest.mark.parametrize("M_lo,M_hi", [(17, 32), (32, 32)])
def test_uniform_differing_deadlines_wide(J, M_lo, M_hi):
    """The differing-deadline kernel's RD prefix/suffix sums and bounds up to M = 32 (no lane M there),
    deadlines at every scale: pruned, executed-work and literal runs agree and match the oracle."""
    b = uniformise(g.random_batch(seed=172 + M_lo, n_inst=600, M_lo=M_lo, M_hi=M_hi, N_lo=2, N_hi=14,
                                  k_max=64), 172)
    rng = np.random.default_rng(M_lo)
    for i in range(b.n_inst):
        o0, o1 = int(b.user_off[i]), int(b.user_off[i + 1])
        lat = b.T[o0:o1].min()
        if i % 3 == 0:
            b.T[o0:o1] = lat * (1.0 + rng.uniform(0.0, 0.5, o1 - o0))
        elif i % 3 == 1:
            b.T[o0:o1] = lat * (1.0 + rng.uniform(5.0, 30.0, o1 - o0))
    _, gpu = run(J, b)
    assert_solve_parity(gpu, O.solve_batch(b, counts=True, threads=8), counts=True)


def test_uniform_differing_deadlines_tight_bound(J):
    """The differing-deadline kernel's batch-coupled n~ bound: uniform users with tight
    and loose deadlines (LC wins often, so most n~ are skipped by the bound against E_LC), a user whose
    deadline equals t_free (L_p = t_free: no f_e passes the guard for that set start) and small t_free
    gaps; the pruned product path, its executed-work run and the literal counters agree bit for bit,
    and all match the oracle."""
    b = uniformise(g.random_batch(seed=171, n_inst=2000, M_lo=2, M_hi=16, N_lo=2, N_hi=12, k_max=64), 171)
    rng = np.random.default_rng(171)
    for i in range(b.n_inst):
        o0, o1 = int(b.user_off[i]), int(b.user_off[i + 1])
        lat = b.T[o0:o1].min()
        r = rng.uniform()
        if r < 0.3:    # tight: beta in [0, 0.6]
            b.T[o0:o1] = lat * (1.0 + rng.uniform(0.0, 0.6, o1 - o0))
        if r > 0.8:    # one user's deadline equals t_free (> 0)
            b.t_free[i] = 0.25 * b.T[o0:o1].min()
            b.T[o0 + int(rng.integers(0, o1 - o0))] = b.t_free[i]
    b.T[b.user_off[0]:b.user_off[1]] = np.linspace(1.0, 2.0, b.M(0)) * b.T[b.user_off[0]]  # differing
    _, gpu = run(J, b)
    orc = O.solve_batch(b, counts=True)
    assert_solve_parity(gpu, orc, counts=True)
    assert (gpu["n_tilde"] == np.array([b.models[m].N for m in b.model_id])).mean() > 0.05  # LC wins often


@pytest.mark.parametrize("uniform", [False, True])
def test_grid_length_cache(J, uniform):
    """K1 caches k per warp keyed by (f_e,min, f_e,max, rho): instances that share f_e,max and rho but
    not f_e,min (different k), interleaved so that every warp meets several grids in turn, and runs
    of equal grids (cache hits).  C2-sized batch so the persistent warps take many instances each."""
    b = g.config_batch("c2", n_inst=40000)
    if not uniform:  # user 0 of every instance gets its own kappa: the general kernel
        b.kappa[b.user_off[:-1]] *= 1.5
    rng = np.random.default_rng(11)
    choices = np.array([0.2e9, 0.2e9, 0.5e9, 1.3e9, 2.05e9])      # k = 64, 64, 54, 27, 2 at rho = 30 MHz
    b.fe_min = choices[rng.integers(0, len(choices), b.n_inst)]
    b.fe_min[: b.n_inst // 4] = 0.5e9                                # a long run of one grid
    _, gpu = run(J, b, counts=False)
    orc = O.solve_batch(b)
    assert_solve_parity(gpu, orc, counts=False)


@pytest.mark.parametrize("uniform", [False, True])
def test_deep_models_and_long_grids(J, uniform):
    """N > 32 (two n~ bounds per lane, two-word candidate ballots), grids longer than the 1/f_e cache
    (k up to 300 > 192), M up to 32: literal, pruned and executed-work sweeps against the oracle."""
    b = g.random_batch(seed=300, n_inst=300, M_lo=1, M_hi=32, N_lo=33, N_hi=63, k_max=300)
    if uniform:
        b = uniformise(b, 300)
    _, gpu = run(J, b)
    orc = O.solve_batch(b, counts=True)
    assert_solve_parity(gpu, orc, counts=True)


@pytest.mark.parametrize("uniform", [False, True])
def test_zero_energy_ties(J, uniform):
    """kappa = p_u = 0 and c = 0: every configuration costs exactly E_LC = 0, so the answer is decided
    by the (E, n~, j) tie rule against the first all-local evaluation (R8).  The pruned sweep skips
    every n~ after the first (lb = 0 >= best = 0) and must fall back to the literal re-sweep."""
    b = g.random_batch(seed=181, n_inst=800, M_lo=1, M_hi=32, N_lo=1, N_hi=12, k_max=50)
    if uniform:
        b = uniformise(b, 181)
    b.kappa[:] = 0.0
    b.p_u[:] = 0.0
    for m in b.models:
        m.c[:] = 0.0
    _, gpu = run(J, b)
    orc = O.solve_batch(b, counts=True)
    assert_solve_parity(gpu, orc, counts=True)
    assert (orc["E"][orc["status"] == 0] == 0.0).all()


@pytest.mark.parametrize("mode", [1, 2, 3])
def test_random_modes(J, mode):
    b = g.random_batch(seed=110 + mode, n_inst=800, M_lo=1, M_hi=16, N_lo=1, N_hi=8, k_max=64)
    _, gpu = run(J, b, mode=mode)
    orc = O.solve_batch(b, mode=mode, counts=True)
    assert_solve_parity(gpu, orc, counts=True)


def test_edge_cases(J):
    """Degenerate inputs: statuses, M = 1 and M = 32, k = 1, equal-gamma ties, Require equality."""
    parts = []
    b = g.toy_instance("toy-1"); b.T[0] = 0.1; parts.append(b)                # LOCAL_INFEASIBLE
    b = g.toy_instance("toy-1"); b.t_free[0] = 0.21; parts.append(b)           # REQUIRE
    b = g.toy_instance("toy-1"); b.t_free[0] = 0.2; parts.append(b)            # Require with equality (allowed)
    b = g.toy_instance("toy-1"); b.f_min[1] = 3e9; parts.append(b)             # BADPARAM
    b = g.toy_instance("toy-1"); b.R[0] = np.nan; parts.append(b)              # BADPARAM (non-finite)
    b = g.toy_instance("toy-1"); b.models[0].d[1 * 3 + 2] = 0.5; parts.append(b)  # BADMODEL
    b = g.toy_instance("toy-1"); b.fe_min[0] = b.fe_max[0]; parts.append(b)    # k = 1
    b = g.toy_instance("toy-1"); b.rho[0] = 1.0; parts.append(b)               # k > JDOB_MAX_K -> BADPARAM
    b = g.toy_instance("toy-2"); b.T[:] = 0.2; parts.append(b)                 # exact gamma and T ties
    b = g.toy_instance("toy-2"); b.zeta[:] = 0.0; parts.append(b)              # zeta = 0 (R9)
    for b in parts:
        _, gpu = run(J, b)
        orc = O.solve_batch(b, counts=True)
        assert_solve_parity(gpu, orc, counts=True, f_user=orc["status"][0] <= 2)
    # M = 32 homogeneous users (all-equal gamma) on the C5 MobileNetV2 profile
    m = g.profiles.mobilenetv2()
    users = dict(zeta=g.profiles.ZETA, kappa=g.profiles.KAPPA, f_min=1.5e9, f_max=2.6e9, R=g.R_TABLE_I, p_u=1.0,
                 T=[float(g.deadline_from_beta(m, g.profiles.ZETA, 2.6e9, 2.13))] * 32)
    b = g.single_instance(m, users)
    _, gpu = run(J, b)
    assert_solve_parity(gpu, O.solve_batch(b, counts=True), counts=True)


def test_empty_batch(J):
    b = g.random_batch(seed=1, n_inst=3).subset(0, 0)
    db = J.DeviceBatch(b)
    res = J.solve_batch(db)
    assert res["E"].numel() == 0


@pytest.mark.parametrize("cfg,n", [("c2", 1 << 20), ("c3", 100_000), ("c5", 1_000_000)])
def test_configs_full_size_sampled(J, cfg, n):
    """BASELINE configs at full size in the bench launch configuration; oracle on a sample."""
    b = g.config_batch(cfg, n_inst=n)
    db, gpu = run(J, b, counts=True, stats=True, n_buckets=b.meta["n_buckets"])
    rng = np.random.default_rng(7)
    idx = np.unique(np.concatenate([rng.choice(b.n_inst, 1500, replace=False), [0, b.n_inst - 1]]))
    sub = b.take(idx)
    orc = O.solve_batch(sub, counts=True, threads=8)
    o0 = b.user_off[idx]
    uidx = np.concatenate([np.arange(b.user_off[i], b.user_off[i + 1]) for i in idx])
    for f in ("E", "E_lc", "t_free_next", "f_e", "n_tilde", "j", "status", "mask"):
        assert_bits_equal(gpu[f][idx], orc[f], f)
    assert_bits_equal(gpu["f_user"][uidx], orc["f_user"], "f_user")
    assert_bits_equal(gpu["counts"][idx], orc["counts"], "counts")
    # invariants at full size
    assert np.all(gpu["status"] == 0)
    assert np.all(gpu["E"] <= gpu["E_lc"])
    # statistics: oracle definition over the GPU's per-instance outputs
    st_o = O.stats(b, dict(gpu, mask=gpu["mask"]), n_buckets=b.meta["n_buckets"])
    st_g = gpu["stats"]
    for f in (0, 3, 4, 7, 8):
        assert_bits_equal(st_g[:, f], st_o[:, f], f"stats[{f}]")
    assert_bits_equal(st_g[:, 9:73], st_o[:, 9:73], "stats hist")
    for f in (1, 2, 5, 6):
        assert rel_close(st_g[:, f], st_o[:, f], 1e-9), f


def test_c2_full_batch_vs_oracle(J):
    """The bench workload C2 at its full size (2^20 instances: the equal-deadline kernel) against the
    oracle on every instance (the bench's cpu_baseline leg does the same at run time)."""
    b = g.config_batch("c2", n_inst=1 << 20)
    gpu = to_np(J.solve_batch(J.DeviceBatch(b)))
    assert_solve_parity(gpu, O.solve_batch(b, threads=16))


def test_c3_full_batch_vs_oracle(J):
    """BASELINE config C3 at its full size (10^5 instances, M 4..20, differing deadlines: the
    differing-deadline kernel with the batch-coupled bound) against the oracle on every instance."""
    b = g.config_batch("c3", n_inst=100_000)
    db = J.DeviceBatch(b)
    gpu = to_np(J.solve_batch(db, partition=True))
    orc = O.solve_batch(b, threads=16)
    assert_solve_parity(gpu, orc)
    assert_bits_equal(gpu["partition"], O.partition_from_plan(b, orc), "partition vs the oracle plan")


def test_stats_small_exact(J):
    b = g.random_batch(seed=120, n_inst=3000, M_hi=32, N_hi=6, k_max=40)
    _, gpu = run(J, b, stats=True, n_buckets=32)
    orc = O.solve_batch(b)
    st = O.stats(b, orc, n_buckets=32)
    for f in (0, 3, 4, 7, 8):
        assert_bits_equal(gpu["stats"][:, f], st[:, f], f"stats[{f}]")
    assert_bits_equal(gpu["stats"][:, 9:], st[:, 9:], "hist")
    for f in (1, 2, 5, 6):
        assert rel_close(gpu["stats"][:, f], st[:, f], 1e-9)


def test_stats_entry_point_same_bits(J):
    # jdob_stats as a call of its own: the same fixed tree, so the same bits as the solve's stats output
    b = g.random_batch(seed=121, n_inst=5000, M_hi=32, N_hi=6, k_max=40)
    db = J.DeviceBatch(b)
    res = J.solve_batch(db, stats=True, n_buckets=32)
    sep = J.stats(db, res, n_buckets=32)
    assert_bits_equal(sep.cpu().numpy().reshape(-1), res["stats"].cpu().numpy().reshape(-1), "jdob_stats")
    st = O.stats(b, O.solve_batch(b), n_buckets=32)
    for f in (0, 3, 4, 7, 8):
        assert_bits_equal(sep.cpu().numpy()[:, f], st[:, f], f"stats[{f}]")


def test_determinism(J):
    b = g.config_batch("c3", n_inst=20000)
    db = J.DeviceBatch(b)
    r1 = to_np(J.solve_batch(db, counts=True, stats=True, n_buckets=3))
    r2 = to_np(J.solve_batch(db, counts=True, stats=True, n_buckets=3))
    for k in r1:
        assert_bits_equal(r1[k].reshape(-1), r2[k].reshape(-1), k)


def test_eval_parity_and_plan_feasibility(J):
    import torch
    b = g.random_batch(seed=130, n_inst=2000, M_hi=24, N_hi=10, k_max=64)
    db = J.DeviceBatch(b)
    res = J.solve_batch(db, partition=True)
    part = J.plan_partition(db, res)
    fe = res["f_e"]
    assert_bits_equal(part.cpu().numpy(), O.partition_from_plan(b, to_np(res)), "partition vs mask-derived")
    ev = to_np(J.eval_plans(db, part, fe, slack=1e-9))
    ev2 = to_np(J.eval_plans(db, plans=res, slack=1e-9))
    for f in ev:
        assert_bits_equal(ev[f], ev2[f], "plan-form eval " + f)
    rn = to_np(res)
    assert np.all(ev["violations"] == 0)
    assert_bits_equal(ev["E"], rn["E"], "eval E == plan E")
    assert_bits_equal(ev["t_free_next"], rn["t_free_next"], "eval t_free == D22")
    orc = O.eval_batch(b, part.cpu().numpy(), fe.cpu().numpy(), slack=1e-9)
    for f in ("E", "t_free_next", "f_user", "status"):
        assert_bits_equal(ev[f], orc[f], f)
    assert_bits_equal(ev["violations"].view(np.uint32), orc["violations"], "violations")


def test_eval_general_vectors(J):
    import torch
    b = g.random_batch(seed=131, n_inst=1500, M_hi=12, N_hi=8, k_max=30)
    rng = np.random.default_rng(3)
    part = np.concatenate([rng.integers(0, b.models[b.model_id[i]].N + 1, b.M(i)) for i in range(b.n_inst)])
    fe = np.array([b.fe_max[i] - rng.integers(0, 5) * b.rho[i] for i in range(b.n_inst)])
    db = J.DeviceBatch(b)
    ev = to_np(J.eval_plans(db, torch.from_numpy(part.astype(np.int32)), torch.from_numpy(fe), slack=1e-9))
    orc = O.eval_batch(b, part, fe, slack=1e-9)
    for f in ("E", "t_free_next", "f_user", "status"):
        assert_bits_equal(ev[f], orc[f], f)
    assert_bits_equal(ev["violations"].view(np.uint32), orc["violations"], "violations")


def test_host_api_matches_device(J):
    b = g.random_batch(seed=140, n_inst=1000, M_hi=16, N_hi=8, k_max=50)
    _, gpu = run(J, b, counts=False)
    hb = J.HostBuffers(b, f_user=True)
    h2d, d2h = J.solve_batch_host(hb)
    assert h2d > 0 and d2h > 0
    host = {k: v.numpy() for k, v in hb.out.items() if v is not None}
    host["mask"] = host["mask"].view(np.uint32)
    for f in ("E", "E_lc", "t_free_next", "f_e", "n_tilde", "j", "status", "mask", "f_user"):
        assert_bits_equal(host[f], gpu[f], f)


def test_host_api_rejects_bad_offsets_and_releases_pool(J):
    """a decreasing host user_off is rejected (EINVAL) before any copy of the bad chunk;
    the private pool can be trimmed and the next call works."""
    b = g.random_batch(seed=142, n_inst=300, M_hi=8, N_hi=5, k_max=20)
    hb = J.HostBuffers(b)
    uo = hb.t["user_off"]
    keep = uo.clone()
    uo[150] = uo[151] + 5                                  # user_off[150] > user_off[151]
    with pytest.raises(J.JdobError, match="user_off"):
        J.solve_batch_host(hb)
    uo.copy_(keep)
    uo[0] = -1
    with pytest.raises(J.JdobError, match="user_off"):
        J.solve_batch_host(hb)
    uo.copy_(keep)
    J.release_pool()
    J.solve_batch_host(hb)
    orc = O.solve_batch(b)
    assert_bits_equal(hb.out["E"].numpy(), orc["E"], "E after release")


def test_host_api_large_m_and_partition(J):
    """Host API on a batch mixing M <= 32 and M > 32 (block path), per-user partition copied back."""
    small = g.random_batch(seed=141, n_inst=200, M_lo=1, M_hi=32, N_lo=1, N_hi=8, k_max=40)
    mix = g.concat([small, _large_batch([40, 90, 33], seed=5)])
    db = J.DeviceBatch(mix)
    dev = to_np(J.solve_batch(db, partition=True))
    hb = J.HostBuffers(mix, f_user=True, partition=True)
    J.solve_batch_host(hb)
    host = {k: v.numpy() for k, v in hb.out.items() if v is not None}
    host["mask"] = host["mask"].view(np.uint32)
    for f in ("E", "E_lc", "t_free_next", "f_e", "n_tilde", "j", "status", "mask", "f_user", "partition"):
        assert_bits_equal(host[f], dev[f], f)
    orc = O.solve_batch(mix)
    assert_bits_equal(host["partition"], orc["part"], "partition vs oracle")


def test_host_api_chunked_pipeline(J):
    # > 131072 instances: several copy/compute pipeline chunks on two internal streams
    b = g.config_batch("c3", n_inst=300_000)
    _, gpu = run(J, b, counts=True, stats=True, n_buckets=3)
    hb = J.HostBuffers(b, f_user=True, stats=True, n_buckets=3)
    h2d, d2h = J.solve_batch_host(hb)
    assert h2d >= b.nbytes()
    host = {k: v.numpy() for k, v in hb.out.items() if v is not None}
    host["mask"] = host["mask"].view(np.uint32)
    for f in ("E", "E_lc", "t_free_next", "f_e", "n_tilde", "j", "status", "mask", "f_user"):
        assert_bits_equal(host[f], gpu[f], f)
    assert_bits_equal(host["stats"].reshape(3, -1), gpu["stats"], "stats")


@pytest.mark.parametrize("cfg,n", [("c2", 300_000), ("c3", 50_000), ("c5", 40_000)])
def test_shared_host_api_equals_full(J, cfg, n):
    """jdob_solve_shared_host (users' device parameters once per instance, expanded on the device)
    returns the bits of jdob_solve_batch_host on the per-user arrays, with fewer bytes copied in."""
    b = g.config_batch(cfg, n_inst=n)
    nb = int(b.meta.get("n_buckets", 32))
    full = J.HostBuffers(b, f_user=True, stats=True, n_buckets=nb)
    h_full, _ = J.solve_batch_host(full)
    sh = J.HostBuffers(b, f_user=True, stats=True, n_buckets=nb, shared=True)
    h_sh, _ = J.solve_batch_host(sh)
    assert h_sh < h_full
    for f in ("E", "E_lc", "t_free_next", "f_e", "n_tilde", "j", "status", "mask", "f_user", "stats"):
        assert_bits_equal(sh.out[f].numpy().reshape(-1), full.out[f].numpy().reshape(-1), f)
    het = g.random_batch(seed=143, n_inst=50, M_lo=2, M_hi=8, N_hi=5, k_max=20, equal_gamma_frac=0.0)
    with pytest.raises(ValueError):
        J.HostBuffers(het, shared=True)


# ------------------------------- brute force -------------------------------------
@pytest.mark.parametrize("toy", ["toy-1", "toy-2", "toy-2-m1", "toy-2-tfree", "toy-4"])
@pytest.mark.parametrize("space", [0, 1])
def test_bf_toys(J, toy, space):
    b = g.toy_instance(toy)
    db = J.DeviceBatch(b)
    E, I, S = J.bruteforce(db, space)
    Eo, Io, So = O.bf(b, space)
    assert int(S.item()) == So == 0
    assert_bits_equal(E.cpu().numpy(), np.array([Eo]), "E")
    assert int(I.item()) == Io


def test_bf_random_full_and_ranges(J):
    b = g.random_batch(seed=150, n_inst=60, M_lo=1, M_hi=5, N_lo=1, N_hi=4, k_max=20, tfree_frac=0.4)
    rng = np.random.default_rng(0)
    for i in range(b.n_inst):
        bi = b.subset(i, i + 1)
        db = J.DeviceBatch(bi)
        for space in (0, 1):
            size = O.bf_space_size(bi, space)
            ranges = [(0, size)]
            for _ in range(2):
                lo = int(rng.integers(0, size))
                hi = int(rng.integers(lo, size + 1))
                ranges.append((lo, hi))
            for lo, hi in ranges:
                E, I, S = J.bruteforce(db, space, lo, hi)
                Eo, Io, So = O.bf(bi, space, lo, hi)
                assert int(S.item()) == So
                assert_bits_equal(E.cpu().numpy(), np.array([Eo]), f"E {i} {space} {lo} {hi}")
                assert int(I.item()) == Io


@pytest.mark.parametrize("N_lo,N_hi", [(1, 3), (9, 15), (16, 17)])
def test_bf_m8_constant_layout(J, N_lo, N_hi):
    """M = 8: N <= 15 takes the constant-layout kernel (rows padded to 16), N = 16, 17 the generic M = 8
    kernel; random models, t_free > 0 on some, oracle-checked on sub-ranges (the spaces reach 18^8 * k)
    and in full where small, both index spaces."""
    b = g.random_batch(seed=160 + N_lo, n_inst=6, M_lo=8, M_hi=8, N_lo=N_lo, N_hi=N_hi, k_max=6, tfree_frac=0.5)
    rng = np.random.default_rng(N_lo)
    for i in range(b.n_inst):
        bi = b.subset(i, i + 1)
        db = J.DeviceBatch(bi)
        for space in (0, 1):
            size = O.bf_space_size(bi, space)
            ranges = [(0, min(size, 400_000))]
            for _ in range(2):
                lo = int(rng.integers(0, max(1, size - 300_000)))
                ranges.append((lo, min(size, lo + int(rng.integers(1, 300_000)))))
            for lo, hi in ranges:
                E, I, S = J.bruteforce(db, space, lo, hi)
                Eo, Io, So = O.bf(bi, space, lo, hi, threads=8)
                assert int(S.item()) == So
                assert_bits_equal(E.cpu().numpy(), np.array([Eo]), f"E {i} {space} {lo} {hi}")
                assert int(I.item()) == Io


def test_bf_tight_deadlines(J):
    """Deadlines just above the local minimum (beta in [0, 0.6]) and t_free > 0: most candidates are
    infeasible and the optimum sits near the feasibility boundary, where the exact vector bounds
    (deadline-driven offloader terms, the D7'-implied f_e bound, the edge-only j skip) are tightest.
    M = 7 and 8 (the M = 8 instantiation is the C4 path), both spaces, full and partial ranges."""
    b = g.random_batch(seed=152, n_inst=24, M_lo=7, M_hi=8, N_lo=1, N_hi=2, k_max=12, tfree_frac=0.5)
    rng = np.random.default_rng(2)
    for i in range(b.n_inst):
        o0, o1 = int(b.user_off[i]), int(b.user_off[i + 1])
        lat = g.min_local_latency(b.models[b.model_id[i]], b.zeta[o0:o1], b.f_max[o0:o1])
        b.T[o0:o1] = (1.0 + rng.uniform(0.0, 0.6, o1 - o0)) * lat
        if b.t_free[i] > 0:
            b.t_free[i] = rng.uniform(0.0, 0.5) * b.T[o0:o1].min()
    for i in range(b.n_inst):
        bi = b.subset(i, i + 1)
        db = J.DeviceBatch(bi)
        for space in (0, 1):
            size = O.bf_space_size(bi, space)
            lo = int(rng.integers(0, size))
            for r0, r1 in ((0, size), (lo, size), (0, max(lo, 1))):
                E, I, S = J.bruteforce(db, space, r0, r1)
                Eo, Io, So = O.bf(bi, space, r0, r1)
                assert int(S.item()) == So
                assert_bits_equal(E.cpu().numpy(), np.array([Eo]), f"E {i} {space} {r0} {r1}")
                assert int(I.item()) == Io


def test_bf_random_scales_full_space(J):
    """K2's exact vector bounds and margins over many random instances: M 2..8, N 1..4, heterogeneous
    users, deadlines at every scale (beta in [0, 0.3] .. [5, 30]) and t_free > 0, each whole general space
    against the literal oracle."""
    rng = np.random.default_rng(77)
    b = g.random_batch(seed=177, n_inst=150, M_lo=2, M_hi=8, N_lo=1, N_hi=4, k_max=20, tfree_frac=0.4)
    scales = ((0.0, 0.3), (0.0, 1.0), (1.0, 5.0), (5.0, 30.0))
    n_off = 0
    for i in range(b.n_inst):
        o0, o1 = int(b.user_off[i]), int(b.user_off[i + 1])
        lat = g.min_local_latency(b.models[b.model_id[i]], b.zeta[o0:o1], b.f_max[o0:o1])
        lo, hi = scales[i % len(scales)]
        b.T[o0:o1] = (1.0 + rng.uniform(lo, hi, o1 - o0)) * lat
        b.t_free[i] = rng.uniform(0.0, 0.5) * b.T[o0:o1].min() if rng.uniform() < 0.4 else 0.0
    for i in range(b.n_inst):
        bi = b.subset(i, i + 1)
        size = O.bf_space_size(bi, 0)
        if size > 3_000_000:
            continue
        E, I, S = J.bruteforce(J.DeviceBatch(bi), 0, 0, size)
        Eo, Io, So = O.bf(bi, 0, 0, size)
        assert int(S.item()) == So
        assert_bits_equal(E.cpu().numpy(), np.array([Eo]), f"E {i}")
        assert int(I.item()) == Io
        n_off += int(Io >= 0)
    assert n_off >= 50


def test_bf_zero_energy_ties(J):
    """kappa = p_u = c = 0: every feasible candidate has E = 0, so the answer is the lowest feasible
    index -- the vector bound (LB = 0 >= best = 0) must never drop a lower-index tie."""
    b = g.random_batch(seed=151, n_inst=30, M_lo=1, M_hi=6, N_lo=1, N_hi=5, k_max=24, tfree_frac=0.4)
    b.kappa[:] = 0.0
    b.p_u[:] = 0.0
    for m in b.models:
        m.c[:] = 0.0
    rng = np.random.default_rng(1)
    for i in range(b.n_inst):
        bi = b.subset(i, i + 1)
        db = J.DeviceBatch(bi)
        for space in (0, 1):
            size = O.bf_space_size(bi, space)
            lo = int(rng.integers(0, max(size // 2, 1)))
            for a, c in ((0, size), (lo, size)):
                E, I, S = J.bruteforce(db, space, a, c)
                Eo, Io, So = O.bf(bi, space, a, c)
                assert int(S.item()) == So
                assert_bits_equal(E.cpu().numpy(), np.array([Eo]), f"E {i} {space} {a}")
                assert int(I.item()) == Io


def test_bf_larger_M(J):
    # M in 9..16 and 17..32 exercise the other kernel specialisations (small N keeps spaces small)
    for seed, M_lo, M_hi, N_hi in ((151, 9, 12, 1), (152, 17, 20, 1)):
        b = g.random_batch(seed=seed, n_inst=4, M_lo=M_lo, M_hi=M_hi, N_lo=1, N_hi=N_hi, k_max=4)
        for i in range(b.n_inst):
            bi = b.subset(i, i + 1)
            db = J.DeviceBatch(bi)
            size = O.bf_space_size(bi, 0)
            hi = min(size, 3_000_000)
            for space, end in ((0, hi), (1, None)):
                E, I, S = J.bruteforce(db, space, 0, end if end is not None else O.bf_space_size(bi, 1))
                Eo, Io, So = O.bf(bi, space, 0, end if end is not None else O.bf_space_size(bi, 1), threads=8)
                assert_bits_equal(E.cpu().numpy(), np.array([Eo]), "E")
                assert int(I.item()) == Io


def test_bf_c4_full(J):
    """C4 at full size (2.75e10 candidates) in the bench launch configuration: the winner
    re-evaluated by the oracle, sampled sub-ranges equal, BF-general <= BF-identical <= J-DOB."""
    b = g.config_batch("c4")
    db = J.DeviceBatch(b)
    size = O.bf_space_size(b, 0)
    E, I, S = J.bruteforce(db, 0, 0, size)
    E, I = float(E.item()), int(I.item())
    assert int(S.item()) == 0 and I >= 0
    assert O.bf_candidate(b, 0, I) == E
    Ei, Ii, _ = O.bf(b, 1)
    Eg, Ig, Sg = J.bruteforce(db, 1)
    assert float(Eg.item()) == Ei and int(Ig.item()) == Ii
    r = O.jdob(b)
    assert E <= Ei <= r["E"] * (1 + 1e-12)
    rng = np.random.default_rng(4)
    for _ in range(6):
        lo = int(rng.integers(0, size - 3_000_000))
        hi = lo + int(rng.integers(1, 3_000_000))
        Eg, Ig, _ = J.bruteforce(db, 0, lo, hi)
        Eo, Io, _ = O.bf(b, 0, lo, hi, threads=8)
        assert_bits_equal(Eg.cpu().numpy(), np.array([Eo]), "E range")
        assert int(Ig.item()) == Io
    # the range containing the winner
    lo, hi = max(0, I - 1_000_000), min(size, I + 1_000_000)
    Eo, Io, _ = O.bf(b, 0, lo, hi, threads=8)
    assert Eo == E and Io == I


# ------------------------------- outer grouping (NEXT-1) --------------------------
def _og_parity(J, b, mode=0):
    db = J.DeviceBatch(b)
    res = J.solve_grouped(db, mode=mode)
    import torch
    torch.cuda.synchronize()
    gpu = {k: v.cpu().numpy() for k, v in res.items() if v is not None}
    orc = O.og_batch(b, mode=mode)
    for f in ("E", "t_free_next", "status", "n_groups", "group_of", "part", "f_user"):
        gf = "partition" if f == "part" else f
        assert_bits_equal(gpu[gf].reshape(-1), orc[f].reshape(-1), "og " + f)
    assert_bits_equal(gpu["group_fe"], orc["group_fe"], "og group_fe")


def test_og_toys(J):
    for T in ([0.2, 0.6], [0.2, 0.2], [0.6, 0.2]):
        b = g.toy_instance("toy-2")
        b.T[:] = T
        _og_parity(J, b)


@pytest.mark.parametrize("seed,M_hi,N_hi", [(171, 6, 5), (172, 16, 8)])
def test_og_random(J, seed, M_hi, N_hi):
    b = g.random_batch(seed=seed, n_inst=300, M_lo=1, M_hi=M_hi, N_lo=1, N_hi=N_hi, k_max=40, tfree_frac=0.4)
    _og_parity(J, b)


def test_og_c3_sample(J):
    # the paper's different-deadline setting: OG + J-DOB on C3-like instances
    b = g.config_batch("c3", n_inst=400)
    _og_parity(J, b)
    b = g.config_batch("c3", n_inst=200)
    _og_parity(J, b, mode=2)


def test_og_statuses(J):
    parts = []
    b = g.toy_instance("toy-1"); b.T[0] = 0.1; parts.append(b)        # LOCAL_INFEASIBLE
    b = g.toy_instance("toy-1"); b.t_free[0] = 0.21; parts.append(b)   # Require fails for the first group
    b = g.toy_instance("toy-1"); b.f_min[1] = 3e9; parts.append(b)     # BADPARAM
    for b in parts:
        _og_parity(J, b)


# ------------------------------- M > 32 (NEXT-4) -----------------------------------
def _large_batch(Ms, seed, hetero=False, tfree=False):
    from tests.test_oracle_large import large_instance
    b = g.concat([large_instance(M, seed + q, hetero=hetero) for q, M in enumerate(Ms)])
    if tfree:
        for i in range(b.n_inst):
            b.t_free[i] = 0.5 * b.T[b.user_off[i]:b.user_off[i + 1]].min()
    return b


def _large_parity(J, b, mode=0):
    db = J.DeviceBatch(b)
    res = J.solve_batch(db, mode=mode, counts=True, partition=True)
    import torch
    torch.cuda.synchronize()
    gpu = to_np(res)
    orc = O.solve_batch(b, mode=mode, counts=True)
    for f in ("E", "E_lc", "t_free_next", "f_e", "n_tilde", "j", "status", "counts", "f_user"):
        assert_bits_equal(gpu[f].reshape(-1), orc[f].reshape(-1), "large " + f)
    assert_bits_equal(gpu["partition"], orc["part"], "large partition")
    prod = to_np(J.solve_batch(db, mode=mode, partition=True))
    for f in PRODUCT_FIELDS + ("partition",):
        assert_bits_equal(prod[f], gpu[f], "large pruned " + f)


@pytest.mark.parametrize("hetero,tfree", [(False, False), (True, True)])
def test_large_m_parity(J, hetero, tfree):
    _large_parity(J, _large_batch([33, 48, 64, 100, 257], seed=3, hetero=hetero, tfree=tfree))


def test_large_m_mixed_batch_and_modes(J):
    # M <= 32 (warp path) and M > 32 (block path) in one batch
    small = g.random_batch(seed=191, n_inst=40, M_lo=1, M_hi=32, N_lo=1, N_hi=8, k_max=40)
    mix = g.concat([small, _large_batch([40, 77], seed=9)])
    for mode in (0, 2, 3):
        _large_parity(J, mix, mode=mode)
    # statuses on the block path: local infeasibility and Require
    bb = _large_batch([50, 60], seed=11)
    bb.T[3] = 1e-6
    bb.t_free[1] = 10.0
    _large_parity(J, bb)


def test_large_m_complexity_smoke(J):
    # M = 1000, N = 19, k ~ 64 well under 10 s, bit-exact vs the oracle
    import time
    import torch
    b = _large_batch([1000], seed=7)
    db = J.DeviceBatch(b)
    J.solve_batch(db)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = J.solve_batch(db, partition=True)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    assert dt < 10.0
    orc = O.solve_batch(b)
    gpu = to_np(res)
    for f in ("E", "n_tilde", "j", "t_free_next"):
        assert_bits_equal(gpu[f], orc[f], f)
    assert_bits_equal(gpu["partition"], orc["part"], "partition")


def test_og_more_than_32_users(J):
    """OG on a batch mixing M <= 32 with 32 < M <= B_max (reported BADPARAM with the LC answer, as the
    oracle does), plus a malformed and a locally infeasible large instance."""
    small = g.random_batch(seed=173, n_inst=50, M_lo=1, M_hi=12, N_lo=1, N_hi=6, k_max=30, tfree_frac=0.4)
    big = _large_batch([33, 48, 64, 40, 41], seed=21)
    big.R[int(big.user_off[3]) + 2] = np.nan          # malformed user -> BADPARAM, NaN answer
    big.T[int(big.user_off[4]) + 7] = 1e-6            # locally infeasible -> LOCAL_INFEASIBLE, LC answer
    _og_parity(J, g.concat([small, big]))


def _c4_oracle_chunks():
    import json
    import os
    p = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles",
                     "r02_c4_oracle_full.ckpt.jsonl")
    if not os.path.exists(p):
        return None
    return [json.loads(line) for line in open(p)]


def test_bf_c4_full_space_vs_oracle(J):
    """The whole C4 general space (2.75e10 candidates) against the oracle's literal scan of every
    candidate (profiles/r02_c4_oracle_full.*, written by tools/c4_oracle_full.py, which calls only
    oracle/): the argmin of each of the 256 vector-aligned chunks is equal, bits and index, and so is
    the argmin over the whole space."""
    chunks = _c4_oracle_chunks()
    if chunks is None or len(chunks) < 256:
        pytest.skip("full-space oracle record not committed")
    b = g.config_batch("c4")
    db = J.DeviceBatch(b)
    size = O.bf_space_size(b, 0)
    best = (float("inf"), -1)
    for c in sorted(chunks, key=lambda r: r["chunk"]):
        E, I, S = J.bruteforce(db, 0, c["lo"], c["hi"])
        Eo = float.fromhex(c["E"])
        assert (float(E.item()), int(I.item())) == (Eo, c["idx"]), c["chunk"]
        if Eo < best[0]:
            best = (Eo, c["idx"])
    E, I, _ = J.bruteforce(db, 0, 0, size)
    assert (float(E.item()), int(I.item())) == best


def test_bf_work_counters(J):
    """The counting instantiation of K2 returns the same argmin; its counters are consistent: every
    vector of the range is visited once, each pruning stage passes a subset of the previous one, and
    the evaluated candidates are at most the range's."""
    b = g.config_batch("c4")
    db = J.DeviceBatch(b)
    k = 64
    for lo, hi in ((0, 12 ** 8 * k), (12 ** 7 * k + 5, 3 * 12 ** 7 * k - 7)):
        E, I, S = J.bruteforce(db, 0, lo, hi)
        Ew, Iw, Sw, W = J.bruteforce(db, 0, lo, hi, work=True)
        assert (float(Ew.item()), int(Iw.item())) == (float(E.item()), int(I.item()))
        w = W.cpu().numpy()
        nvec = (hi + k - 1) // k - lo // k
        assert w[0] == nvec
        assert w[0] >= w[1] >= w[2] >= w[3] >= 0
        assert w[4] + w[6] <= hi - lo
        assert w[8] <= 8 * w[4] and w[5] <= w[8]
    # identical space and a small instance: the scan without pruning opportunities counts everything
    t = g.toy_instance("toy-4")
    dt = J.DeviceBatch(t)
    for space in (0, 1):
        E, I, S, W = J.bruteforce(dt, space, work=True)
        Eo, Io, So = O.bf(t, space)
        assert (float(E.item()), int(I.item())) == (Eo, Io)
        assert int(W[0].item()) == O.bf_space_size(t, space) // O.grid_k(t)


def _verify_batches():
    yield "random-t_free", g.random_batch(seed=160, n_inst=3000, M_hi=32, N_hi=12, k_max=80, tfree_frac=0.5)
    yield "random-small", g.random_batch(seed=161, n_inst=3000, M_hi=6, N_hi=4, k_max=20, identical_T_frac=0.7)
    yield "c2", g.config_batch("c2", n_inst=20000)
    yield "c3", g.config_batch("c3", n_inst=20000)
    yield "c5", g.config_batch("c5", n_inst=20000)


@pytest.mark.parametrize("slack", [0.0, 1e-9])
@pytest.mark.parametrize("mode", [0, 1, 2, 3])
def test_fused_verify_equals_eval(J, mode, slack):
    """Row a11 in the solver's epilogue: the violation bits of every plan equal jdob_eval's for the
    (n_tilde, mask, f_e) outputs at the same slack; the other outputs are unchanged."""
    for name, b in _verify_batches():
        db = J.DeviceBatch(b)
        plain = to_np(J.solve_batch(db, mode=mode))
        res = J.solve_batch(db, mode=mode, verify=True, slack=slack)
        ev = to_np(J.eval_plans(db, plans=res, slack=slack))
        out = to_np(res)
        for f in PRODUCT_FIELDS:
            assert_bits_equal(out[f], plain[f], f"{name} {f}")
        assert_bits_equal(out["violations"].view(np.uint32), ev["violations"], f"{name} violations")
