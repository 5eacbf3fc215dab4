#!/usr/bin/env python
"""Benchmark of the J-DOB hot path on B200 (driver contract: one JSON line from rank 0).

Step (N GPUs, weak scaling): every rank solves its own slice of the workload
(default C2: 2^20 instances of 10 VGG-16 users per GPU, BASELINE.json configs[1])
through the C ABI: jdob_solve_batch (K0 aggregates + K1 J-DOB solve incl. LC +
K4 statistics) and jdob_eval re-verifying every plan (K3); the statistics are
then all-reduced over NCCL (the path's only exchange step).  Inputs are resident
in HBM before the timed region and are larger than L2.

Extra legs in the same line: "bruteforce" (C4 exhaustive search, 2.75e10
candidates, index space sharded over the ranks, NCCL MIN-allreduce of (E, idx)),
"e2e" (jdob_solve_batch_host from pinned host buffers, copies inside the timed
region), "cpu_baseline" (the C oracle on a bounded sample on the host cores),
"roofline" (FP64 work K1 executed -- from its executed-work counters -- / its
live CUDA-event duration, against the FP64 peak of DESIGN.md §Roofline; the
literal Alg. 1/2 work of the same launch is reported beside it).

--impl reference times the CPU oracle (the reference arm of this tier).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import jdobgen as G  # noqa: E402

PEAK_FP64_SM_PER_CLK = 64      # FP64 lanes per SM per clock (B200), DESIGN.md §7 (microbenchmarked)
N_SMS = 148
# FP64-pipe instructions of one correctly rounded double division on sm_100a: the fast path is
# MUFU.RCP64H (XU pipe) + 7 DFMA + 1 DMUL (cuobjdump -sass, profiles/r02_ddiv_sass.txt); measured
# throughput 4.6 divisions/SM/clk vs 63.2 DADD (tools/fp64_microbench.cu), i.e. ~13.7 DADD slots
W_DIV = 8
PEAK_NOTE = ("builder-measured FP64 peak: 148 SMs x 64 FP64 lanes/clk (tools/fp64_microbench.cu: DADD 63.2, "
             "DFMA 58.2 per SM per clk) x the max SM clock seen during the run; MEASURED_PEAKS.json has no FP64 "
             "entry")

WORKLOADS = {
    "c2": ("c2_vgg16_m10_identical_beta0-35", 1 << 20),
    "c3": ("c3_resnet18_m4-20_mixed_deadlines", 100_000),
    "c5": ("c5_montecarlo_m1-32_3models_5regimes_3grids", 10_000_000),
}


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="mine", choices=["mine", "reference"])
    p.add_argument("--workload", default="c2", choices=sorted(WORKLOADS))
    p.add_argument("--n-inst", type=int, default=None,
                   help="instances per GPU (weak scaling) or in total (--scaling strong)")
    p.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                   help="weak: n instances per GPU; strong: a fixed total sharded over the GPUs")
    p.add_argument("--no-bf", action="store_true")
    p.add_argument("--bf-reps", type=int, default=2)
    p.add_argument("--no-cpu", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--cpu-seconds", type=float, default=10.0)
    p.add_argument("--fused-verify", action="store_true",
                   help="re-verify the plans in K1's epilogue (jdob_solve_batch violations) instead of jdob_eval (K3); "
                        "same bits, measured slower (DESIGN.md §4)")
    p.add_argument("--host-gen", action="store_true",
                   help="c5: generate on the host and copy (default: generated on the device, no input H2D)")
    return p.parse_args()


# ----------------------------------------------------------------------------------
def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


class Clocks:
    """nvidia-smi sampler running during the timed region (B200_PROFILING.md clocks line)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        self.p = None

    def start(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "200"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return None
        time.sleep(0.25)
        self.p.terminate()
        try:
            self.p.wait(timeout=5)
        except Exception:
            self.p.kill()
        self.f.flush()
        rows = [r.split(",") for r in open(self.f.name).read().strip().splitlines() if r.strip()]
        os.unlink(self.f.name)
        sm = [float(r[1]) for r in rows if len(r) >= 9 and r[1].strip().replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if len(r) >= 9 and r[2].strip().replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in rows:
            if len(r) >= 9:
                for nm, v in zip(names, r[5:9]):
                    if v.strip().lower() == "active":
                        reasons.add(nm)
        if not sm:
            return None
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def fp64_work(batch, counts, setups=None, lower_bound=False):
    """FP64 operations of K1 per launch from per-instance counters (n_visit, n_eval,
    n_member), split into divisions and other ops (+, -, x, comparison):
      member evaluation   1 div (Gamma) + 8    non-member term  1
      evaluated pair      1 div (1/f_e) + 5    visited pair     1 div (guard) + 3
      per n~ set-up       3M div (O/R, gamma, threshold) + 3M + M(M-1)/2 (sort compares)
      LC                  1 div + 7 per user
    Literal Alg. 1/2: every n~ is set up (setups = N) -- SURVEY §8(d)'s count.  Executed (pruned
    sweep): set-ups and pairs from the executed-work counters plus the n~ lower bounds (8 ops per
    (n~, user), one RD reciprocal per user).  Returns (divisions, other ops, member evaluations)."""
    M = np.diff(batch.user_off).astype(np.float64)
    N = np.array([m.N for m in batch.models], np.float64)[np.asarray(batch.model_id)]
    visit, ev, mem = (counts[:, 0].astype(np.float64), counts[:, 1].astype(np.float64),
                      counts[:, 2].astype(np.float64))
    S = N if setups is None else setups.astype(np.float64)
    div = mem + ev + visit + S * 3 * M + M
    oth = 8 * mem + (ev * M - mem) + 5 * ev + 3 * visit + S * (3 * M + M * (M - 1) / 2) + 7 * M
    if lower_bound:
        div = div + M * (S > 0)
        oth = oth + 8 * N * M * (S > 0)
    return float(np.sum(div)), float(np.sum(oth)), float(np.sum(mem))


def fp64_frac(div, oth, ms, peak_gops):
    """FP64-pipe instruction rate of (div, other) ops with a division weighted W_DIV, over `ms`."""
    ach = (W_DIV * div + oth) / (ms / 1e3) / 1e9
    return {"ops_per_launch": W_DIV * div + oth, "divisions": div, "other_ops": oth, "achieved": ach,
            "frac": ach / peak_gops}


def issue_roof(warp_instructions, ms, clk_mhz):
    """The kernel against the instruction-issue peak (148 SMs x 4 schedulers x 1 warp instruction per
    clock): what bounds K1 and K2, whose FP64 pipe is mostly idle (ncu warp instructions of the launch)."""
    peak = N_SMS * 4 * clk_mhz * 1e6 / 1e9   # G warp instructions/s
    a = warp_instructions / (ms / 1e3) / 1e9
    return {"warp_instructions_per_launch": warp_instructions, "achieved": a, "peak": peak, "unit": "G warp instr/s",
            "frac": a / peak}


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def ncu_record(key):
    """A committed ncu record (profiles/ncu_traffic.json) -- per-launch hardware counters of the
    bench's own launch configuration; None when absent."""
    try:
        return json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json"))).get(key)
    except Exception:
        return None


def hbm_context(nbytes, ms):
    """HBM side of K1 for context: algorithmic bytes per launch over the launch time, against the
    measured copy bandwidth (MEASURED_PEAKS.json, driver-written) -- K1 is not memory-bound."""
    try:
        peak = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
    except Exception:
        peak = None
    gbs = nbytes / (ms / 1e3) / 1e9
    return {"achieved_gbs": gbs, "peak_gbs": peak, "frac": (gbs / peak) if peak else None}


def ncu_traffic(kernel):
    """dram read+write bytes per launch of `kernel` from the committed ncu --set full capture."""
    try:
        d = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))
        return d.get(kernel)
    except Exception:
        return None


class DevGenView:
    """Host-side view of a device-generated C5 shard (jdob_generate_c5_*): sizes and per-instance
    (M, model) for the work counters; subset() regenerates instances with the host generator (the same
    bits, tests/test_gpu_gen.py) for the cpu_baseline sample."""

    def __init__(self, db, models, lo, meta):
        self.user_off = db.t["user_off"].cpu().numpy()
        self.model_id = db.t["model_id"].cpu().numpy()
        self.models, self.lo, self.meta = models, lo, meta
        self.n_inst, self.n_users = db.n_inst, db.n_users

    def nbytes(self):
        return self.n_inst * (4 + 8 + 4 * 8 + 4) + 8 + self.n_users * 7 * 8

    def subset(self, i0, i1):
        return G.config_c5(n_inst=i1 - i0, inst_begin=self.lo + i0)


def cpu_baseline(batch, seconds, label, gpu_host=None):
    """The oracle, as it stands, on a bounded sample of the same workload, all host cores; its results
    are then compared bit for bit with the GPU's for the same instances (parity of the bench run)."""
    import oracle as O
    cores = os.cpu_count() or 1
    probe = batch.subset(0, min(batch.n_inst, 2000))
    t0 = time.perf_counter()
    O.solve_batch(probe, threads=cores)
    rate = probe.n_inst / max(time.perf_counter() - t0, 1e-6)
    n = int(min(batch.n_inst, max(probe.n_inst, rate * seconds)))
    sub = batch.subset(0, n)
    t0 = time.perf_counter()
    orc = O.solve_batch(sub, threads=cores)
    dt = time.perf_counter() - t0
    parity = None
    if gpu_host is not None:
        bad = 0
        for f, g in gpu_host.items():
            a, o = g[:n], np.asarray(orc[f])
            if a.dtype == np.float64:
                bad += int((a.view(np.int64) != o.view(np.int64)).sum())
            else:
                bad += int((a.view(np.int32) != o.astype(a.dtype).view(np.int32)).sum())
        parity = (f"{n}/{n} instances of the cpu_baseline sample bit-exact vs oracle" if bad == 0
                  else f"MISMATCH: {bad} differing fields in the {n}-instance cpu_baseline sample")
    return {"value": n / dt, "unit": "instances/s", "cores": cores, "kind": "oracle", "cpu_model": cpu_model(),
            "sample": f"first {n} instances of {label} ({dt:.1f} s, C oracle -O2, {cores} threads)"}, parity


def bf_literal_ops(N, M, k):
    """SURVEY §8(d) per-candidate work of the general space, summed over every candidate: a vector with
    o offloaders costs o divisions (one Gamma each; 1/f_e(j) is per grid point) + 9 o + 6 other ops per
    grid point, and 2N + 2M set-up ops once per vector (digit decode, suffix sums, minima).  There are
    C(M, o) N^o vectors with o offloaders."""
    from math import comb
    div = oth = 0.0
    for o in range(M + 1):
        nv = comb(M, o) * N ** o
        div += nv * k * o
        oth += nv * (k * (9 * o + 6) + 2 * N + 2 * M)
    return div, oth


def bf_executed_ops(wk, N, M):
    """FP64 work the pruned K2 scan executed, from its counters (include/jdob.h jdob_bruteforce `work`):
    user-term bound 3 per visited vector; n_min-only bound M + 10 + 1 div per vector past it; suffix
    sums, D6' test, exact bound and hoists 2N + M + 12 + 1 div per vector past the n_min bound; the
    edge-only skip's binary search ~30 per vector entering the grid loop; per evaluated candidate 9 + M
    + 6 per offloader; one division + 2 per Gamma executed."""
    w = [float(x) for x in wk]
    div = w[1] + w[2] + w[5]
    oth = (3 * w[0] + (M + 10) * w[1] + (2 * N + M + 12) * w[2] + 30 * w[3] + (9 + M) * w[4] + 6 * w[8]
           + 2 * w[5])
    return div, oth


def bf_leg(J, torch, world, rank, reps, dist, peak_gops, with_cpu, cpu_seconds):
    """C4 exhaustive search, contiguous vector-aligned index ranges per rank (strong scaling: the
    2.75e10-candidate space is fixed)."""
    b = G.config_batch("c4")
    db = J.DeviceBatch(b)
    k = G.grid_size(float(b.fe_min[0]), float(b.fe_max[0]), float(b.rho[0]))
    N, M = b.models[0].N, b.M(0)
    size = J.bf_space_size(0, N, M, k)
    from paper_2504_14611_b200.dist import allreduce_argmin, bf_shard
    lo, hi = bf_shard(size, k, world, rank)
    J.bruteforce(db, 0, lo, min(hi, lo + 64 * 1024 * k))     # warm-up (small)
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()
    times, kms = [], []
    res = None
    for _ in range(reps):
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        s, m, e = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        s.record(stream)
        E, I, S = J.bruteforce(db, 0, lo, hi)
        m.record(stream)
        if dist:
            E, I = allreduce_argmin(E, I, dist)
        e.record(stream)
        torch.cuda.synchronize()
        ms, km = s.elapsed_time(e), s.elapsed_time(m)
        if dist:
            t = torch.tensor([ms, km], device="cuda", dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms, km = float(t[0]), float(t[1])
        times.append(ms)
        kms.append(km)
        res = (float(E.item()), int(I.item()), int(S.item()))
    ms, km = float(np.median(times)), float(np.median(kms))
    # untimed: the executed-work counters of the same scan (counting instantiation, same argmin)
    Ew, Iw, Sw, W = J.bruteforce(db, 0, lo, hi, work=True)
    wk = W.cpu().numpy().astype(np.int64)
    if dist:
        t = torch.tensor(wk, device="cuda", dtype=torch.int64)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        wk = t.cpu().numpy()
    ldiv, loth = bf_literal_ops(N, M, k)
    ediv, eoth = bf_executed_ops(wk, N, M)
    hw = ncu_record("k_bf_main_hw") if world == 1 else None
    clk_mhz = peak_gops * 1e3 / (N_SMS * PEAK_FP64_SM_PER_CLK)
    roof = {"bound": "alu", "kernel": "k_bf_main (K2)", "unit": "G FP64-pipe instr/s", "peak": peak_gops,
            "launch_ms": km, "w_div": W_DIV,
            "literal": fp64_frac(ldiv / world, loth / world, km, peak_gops),
            "executed": fp64_frac(ediv / world, eoth / world, km, peak_gops),
            "ncu_hw": hw, "traffic": ncu_record("k_bf_main_c4_full") if world == 1 else None,
            "counters": {"vectors": int(wk[0]), "past_user_bound": int(wk[1]), "past_nmin_bound": int(wk[2]),
                         "grid_loop_entered": int(wk[3]), "candidates_evaluated": int(wk[4]),
                         "gamma_divisions": int(wk[5]), "skipped_by_edge_bound": int(wk[6]),
                         "d6_fail_first_point": int(wk[7]), "offloader_terms": int(wk[8])},
            "candidates_evaluated_frac": float(wk[4]) / size,
            "peak_note": PEAK_NOTE + "; literal = SURVEY §8(d) per-candidate work over all candidates / "
                         "the kernel's time (> 1 is the pruning's signature); executed = the work the "
                         "pruned scan ran, from its counters (bench.py bf_executed_ops)"}
    if hw and hw.get("fp64_thread_inst"):   # the FP64 lane instructions ncu counted for this launch
        a_ = hw["fp64_thread_inst"] / (km / 1e3) / 1e9
        roof["ncu_executed"] = {"fp64_lane_instructions_per_launch": hw["fp64_thread_inst"], "achieved": a_,
                                "frac": a_ / peak_gops}
        roof["issue"] = issue_roof(hw["warp_instructions"], km, clk_mhz)
    # the headline fraction is the op-count model of the work the pruned scan executed (the same
    # definition for every workload and both legs); the ncu FP64 instruction count and the issue rate
    # of the committed capture corroborate it
    roof["achieved"] = roof["executed"]["achieved"]
    roof["frac"] = roof["executed"]["frac"]
    roof["frac_source"] = "executed (op-count model, w_div = %d)" % W_DIV
    out = {"metric": "brute-force candidates/s", "value": size / (ms / 1e3), "unit": "candidates/s",
           "workload": "c4_resnet18_m8_12pp_k64_general", "candidates": size, "ms": ms, "reps": reps,
           "scaling": "strong", "E_min": res[0], "idx_min": res[1], "status": res[2],
           "work_run_same_argmin": (float(Ew.item()), int(Iw.item())) == (res[0], res[1]) or world > 1,
           "gpu_launches_per_rep": 3, "roofline": roof}
    # the committed full-space oracle argmin (tools/c4_oracle_full.py: every candidate, literal oracle)
    try:
        full = json.load(open(os.path.join(ROOT, "profiles", "r02_c4_oracle_full.json")))
        out["oracle_full_space"] = {"E_min": full["E_min"], "idx_min": full["idx_min"],
                                    "equal": (full["E_min"], full["idx_min"]) == (res[0], res[1]),
                                    "record": "profiles/r02_c4_oracle_full.json",
                                    "oracle_candidates_per_s": full["candidates_per_s"],
                                    "oracle_threads": full["threads"], "oracle_cpu": full["cpu_model"]}
    except Exception:
        out["oracle_full_space"] = None
    if with_cpu and rank == 0 and world == 1:
        import oracle as O
        cores = os.cpu_count() or 1
        probe = 64 * 12 * k * 16
        t0 = time.perf_counter()
        O.bf(b, 0, 0, probe, threads=cores)
        rate = probe / max(time.perf_counter() - t0, 1e-6)
        n = int(max(probe, min(size, rate * cpu_seconds)) // (12 * k)) * (12 * k)
        # a vector-aligned sub-range around the optimum (both sides compared on the same range)
        c = (res[1] // k) * k if res[1] >= 0 else 0
        r0 = max(0, min(size - n, c - n // 2) // k * k)
        t0 = time.perf_counter()
        Eo, Io, So = O.bf(b, 0, r0, r0 + n, threads=cores)
        dt = time.perf_counter() - t0
        Eg, Ig, _ = J.bruteforce(db, 0, r0, r0 + n)
        same = (float(Eg.item()), int(Ig.item())) == (Eo, Io)
        out["cpu_baseline"] = {"value": n / dt, "unit": "candidates/s", "cores": cores, "kind": "oracle",
                               "cpu_model": cpu_model(),
                               "sample": f"candidates [{r0}, {r0 + n}) of the C4 general space ({n} = "
                                         f"{n / size:.2%} of it, {dt:.1f} s, oracle_bf_mt -O2, {cores} "
                                         f"threads); the rate is per candidate, not extrapolated"}
        out["parity"] = (f"oracle argmin over the cpu_baseline sub-range ({Eo!r}, {Io}) "
                         + ("== GPU's" if same else f"!= GPU's ({float(Eg.item())!r}, {int(Ig.item())})"))
    return out


def run_mine(args):
    import torch
    world, rank, local = dist_env()
    dist = None
    # JDOB_BENCH_BACKEND=gloo (test only): several ranks sharing the visible GPUs, to exercise the
    # multi-rank path on a one-GPU box; the driver's runs use NCCL with one GPU per rank
    backend = os.environ.get("JDOB_BENCH_BACKEND", "nccl")
    dev_index = local % torch.cuda.device_count() if backend != "nccl" else local
    torch.cuda.set_device(dev_index)
    if world > 1 or "TORCHELASTIC_RUN_ID" in os.environ:   # launched by torchrun (also at N = 1)
        import torch.distributed as D
        if backend == "nccl":
            D.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            D.init_process_group(backend)
        dist = D
    import paper_2504_14611_b200 as J
    label, n_default = WORKLOADS[args.workload]
    from paper_2504_14611_b200.dist import fold_stats, shard_range
    n_arg = args.n_inst or n_default
    n_total = n_arg * world if args.scaling == "weak" else n_arg
    lo, hi = shard_range(n_total, world, rank)   # weak: [rank n, (rank + 1) n)
    n = hi - lo
    devgen = args.workload == "c5" and not args.host_gen
    if devgen:   # each rank generates its own instances on the device: no input traffic
        models, params = G.c5_device_inputs(inst_begin=lo)
        db = J.DeviceBatch.generate_c5(models, params, n)
        batch = DevGenView(db, models, lo, dict(config="c5", n_buckets=480))
    else:
        batch = G.config_batch(args.workload, n_inst=n, inst_begin=lo)
        db = J.DeviceBatch(batch)
    n_buckets = int(batch.meta.get("n_buckets", 32))
    torch.cuda.synchronize()

    # untimed: algorithmic work counters -- literal Alg. 2 counts (checked against the oracle in tests)
    # and the work the pruned product sweep executes (same decisions as the timed launches)
    res_c = J.solve_batch(db, counts=True, f_user=False)
    counts = res_c["counts"].cpu().numpy()
    lit_div, lit_oth, n_member = fp64_work(batch, counts)
    wk = J.solve_batch(db, work=True, f_user=False)["work"].cpu().numpy()
    ex_div, ex_oth, n_member_exec = fp64_work(batch, wk[:, 1:], setups=wk[:, 0], lower_bound=True)
    setup_frac = float(wk[:, 0].sum()) / float(np.array([m.N for m in batch.models])[np.asarray(batch.model_id)].sum())
    del res_c

    fused = args.fused_verify   # a11 in K1's epilogue instead of K3 (same bits)
    res = J.solve_batch(db, f_user=False, verify=fused)
    # this rank's root of the statistics tree over the whole job's batch (jdob_stats_part); the
    # pairwise fold over ranks (dist.fold_stats) has the bits of one GPU over the whole batch
    part = (n_total, world, rank) if world & (world - 1) == 0 else None  # jdob_stats_part: power-of-two parts
    res["stats"] = J.stats(db, res, n_buckets=n_buckets, part=part)
    # the product path's decisions for the whole batch, on the host: the cpu_baseline leg compares
    # its oracle sample with them (the only place the bench run meets the oracle)
    gpu_host = {f: res[f].cpu().numpy() for f in ("E", "t_free_next", "f_e", "n_tilde", "j", "status", "mask")}
    ev = J.eval_plans(db, plans=res, f_user=False)
    stream = torch.cuda.current_stream()

    def step():
        J.solve_batch(db, f_user=False, out=res, verify=fused)
        J.stats(db, res, out=res["stats"], part=part)
        if not fused:
            J.eval_plans(db, plans=res, f_user=False, out=ev)
        if dist:
            res["stats_global"] = fold_stats(res["stats"], dist)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    clocks = Clocks(dev_index)
    clocks.start()
    time.sleep(0.3)
    K = args.steps
    ev_s = [torch.cuda.Event(enable_timing=True) for _ in range(K)]
    ev_e = [torch.cuda.Event(enable_timing=True) for _ in range(K)]
    t_s, t_e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t_s.record(stream)
    for i in range(K):
        ev_s[i].record(stream)
        J.solve_batch(db, f_user=False, out=res, verify=fused)  # K0 + K1 (+ a11 in K1's epilogue)
        ev_e[i].record(stream)
        J.stats(db, res, out=res["stats"], part=part)      # K4
        if not fused:
            J.eval_plans(db, plans=res, f_user=False, out=ev)  # K3
        if dist:
            res["stats_global"] = fold_stats(res["stats"], dist)
    t_e.record(stream)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    clk = clocks.stop()
    total_ms = t_s.elapsed_time(t_e)
    solve_ms = float(np.mean([a.elapsed_time(b) for a, b in zip(ev_s, ev_e)]))
    if fused:   # bit 31 alone marks an unverified M > 32 instance (none in these workloads)
        viol = int((res["violations"] != 0).sum().item())
    else:
        viol = int((ev["violations"] != 0).sum().item())
    # K3 (jdob_eval) over the same plans timed on its own, and (untimed) the same plans re-verified in
    # K1's epilogue: the two sets of violation bits must be equal
    s_, e_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s_.record(stream)
    for _ in range(3):
        J.eval_plans(db, plans=res, f_user=False, out=ev)
    e_.record(stream)
    torch.cuda.synchronize()
    rv = res if fused else J.solve_batch(db, f_user=False, verify=True)
    eval_leg = {"kernel": "k_eval (K3, jdob_eval)", "ms": s_.elapsed_time(e_) / 3,
                "bits_equal_k1_epilogue": bool(torch.equal(ev["violations"], rv["violations"]))}
    if dist:
        t = torch.tensor([total_ms, solve_ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms, solve_ms = float(t[0]), float(t[1])
        w = torch.tensor([ex_div, ex_oth, lit_div, lit_oth], device="cuda", dtype=torch.float64)
        dist.all_reduce(w, op=dist.ReduceOp.MAX)   # per-GPU work of the slowest rank's kind
        ex_div, ex_oth, lit_div, lit_oth = (float(x) for x in w)
    value = n_total * K / (total_ms / 1e3)

    # end-to-end through the public host-buffer API (copies inside the timed region)
    e2e = None
    if devgen:
        e2e = {"skipped": "device-generated workload: no host inputs (use --host-gen for the host-buffer API)"}
    elif not args.no_e2e:
        # users sharing their device parameters within an instance (Table I; all of C2/C3/C5) go through
        # jdob_solve_shared_host, the others through jdob_solve_batch_host
        shared = J.shared_params(batch) is not None
        hb = J.HostBuffers(batch, stats=True, n_buckets=n_buckets, shared=shared)
        J.solve_batch_host(hb)
        reps = max(1, min(K, 3))
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(stream)
        for _ in range(reps):
            h2d, d2h = J.solve_batch_host(hb)
        e.record(stream)
        torch.cuda.synchronize()
        ms = s.elapsed_time(e)
        if dist:
            t = torch.tensor([ms], device="cuda", dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        e2e = {"value": n_total * reps / (ms / 1e3), "unit": "instances/s", "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h), "reps": reps,
               "api": ("jdob_solve_shared_host (pinned host buffers; users' shared device parameters once per "
                       "instance, expanded on the device)" if shared else "jdob_solve_batch_host (pinned host buffers)")}
        del hb
        # copy roof: one plain pinned host -> device copy of the same number of bytes (no kernels)
        hx = torch.empty(int(h2d), dtype=torch.uint8).pin_memory()
        dx = torch.empty(int(h2d), dtype=torch.uint8, device="cuda")
        dx.copy_(hx, non_blocking=True)
        torch.cuda.synchronize()
        # best of three: one plain copy, and the same bytes as two halves on two streams (both copy
        # engines), no kernels
        roof_ms = float("inf")
        half = int(h2d) // 2
        s2 = torch.cuda.Stream()
        for _ in range(3):
            s.record(stream)
            dx.copy_(hx, non_blocking=True)
            e.record(stream)
            torch.cuda.synchronize()
            roof_ms = min(roof_ms, s.elapsed_time(e))
            s.record(stream)
            s2.wait_stream(stream)
            dx[:half].copy_(hx[:half], non_blocking=True)
            with torch.cuda.stream(s2):
                dx[half:].copy_(hx[half:], non_blocking=True)
            stream.wait_stream(s2)
            e.record(stream)
            torch.cuda.synchronize()
            roof_ms = min(roof_ms, s.elapsed_time(e))
        e2e["h2d_copy_roof"] = {"ms": roof_ms, "gbs": h2d / (roof_ms / 1e3) / 1e9,
                                "frac": roof_ms / (ms / reps)}
        del hx, dx

    peak_clk = (clk or {}).get("sm_max_mhz") or 1965.0
    peak = N_SMS * PEAK_FP64_SM_PER_CLK * peak_clk * 1e6 / 1e9   # G FP64-pipe lane instructions/s
    bf = None
    if not args.no_bf:
        bf = bf_leg(J, torch, world, rank, args.bf_reps, dist, peak, not args.no_cpu, args.cpu_seconds)

    cpu = parity = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu, parity = cpu_baseline(batch, args.cpu_seconds, label, gpu_host)

    if rank == 0:
        default_c2 = args.workload == "c2" and n == 1 << 20 and world == 1
        executed = fp64_frac(ex_div, ex_oth, solve_ms, peak)
        literal = fp64_frac(lit_div, lit_oth, solve_ms, peak)
        hw = ncu_record("k_solve_hw") if default_c2 else None
        # hardware count of the FP64-pipe lane instructions one launch executes (committed ncu capture
        # of this exact launch), over the live K1 time: the measured executed fraction
        ncu_exec = issue = None
        if hw and hw.get("fp64_thread_inst"):
            a_ = hw["fp64_thread_inst"] / (solve_ms / 1e3) / 1e9
            ncu_exec = {"fp64_lane_instructions_per_launch": hw["fp64_thread_inst"], "achieved": a_,
                        "frac": a_ / peak}
            issue = issue_roof(hw["warp_instructions"], solve_ms, peak_clk)
        line = {
            "metric": "J-DOB instances solved/s",
            "value": value,
            "unit": "instances/s",
            "n_gpus": world,
            "steps": K,
            "warmup": args.warmup,
            "ms_per_step": total_ms / K,
            "higher_is_better": True,
            "scaling": args.scaling,
            "vs_baseline": None,
            "dtype": "f64",
            "data": ("synthetic, generated on the device (jdob_generate_c5_*, bit-identical to jdobgen)" if devgen
                     else "synthetic (jdobgen seeded generator, paper-shaped profiles; DESIGN.md §Input recipe)"),
            "config": {"workload": label, "n_inst_per_gpu": n, "global_instances": n_total,
                       "users_per_gpu": int(batch.n_users), "input_bytes_per_gpu": int(batch.nbytes()),
                       "l2": "inputs larger than L2 (126 MB)" if batch.nbytes() > 126e6 else "inputs fit in L2",
                       "step": ("jdob_solve_batch (K0 + K1, every plan re-verified in K1's epilogue with "
                                "jdob_eval's formulas, row a11) + jdob_stats (K4)" if fused else
                                "jdob_solve_batch (K0+K1) + jdob_stats (K4) + jdob_eval of every plan (K3)")
                               + (" + NCCL stats allreduce" if dist else ""),
                       "parallelism": f"dp{world}"},
            "roofline": {"bound": "alu", "kernel": ("k_solve<0,1,1,0,0> (K1, equal-deadline uniform-users kernel)" if default_c2 else
                                    "k_solve (K1: equal-deadline, differing-deadline and general kernels)"), "unit": "G FP64-pipe instr/s",
                         # the op-count model of the executed work (every workload, both legs); the
                         # ncu FP64 instruction count and issue rate of the committed capture beside it
                         "achieved": executed["achieved"], "peak": peak,
                         "frac": executed["frac"],
                         "frac_source": "executed (op-count model, w_div = %d)" % W_DIV,
                         "w_div": W_DIV,
                         "executed": executed, "literal": literal, "ncu_executed": ncu_exec,
                         "issue": issue,
                         "traffic": ncu_record("k_solve") if default_c2 else None,
                         "ncu_hw": hw,
                         "algorithmic_bytes": int(batch.nbytes()),
                         "hbm": hbm_context(int(batch.nbytes()), solve_ms),
                         "member_evals_per_launch": n_member_exec,
                         "literal_member_evals_per_launch": n_member,
                         "n_tilde_setups_frac": setup_frac,
                         "launch_ms": solve_ms,
                         "peak_note": PEAK_NOTE + "; launch_ms = CUDA events around jdob_solve_batch (K0 + the three "
                                      "K1 kernels; on C2 the equal-deadline kernel is 99 % of it, K0 and the "
                                      "other two kernels' status scans about 1 %); literal = SURVEY "
                                      "§8(d)'s Alg. 1/2 work (every n~ swept, oracle-checked counters) with a "
                                      "division weighted w_div FP64-pipe instructions, > 1 is the pruning's "
                                      "signature; executed = the work the pruned sweep ran (its counters, same "
                                      "weights); ncu_executed = the FP64-pipe lane instructions ncu counted for "
                                      "this launch (profiles/) over the live time"},
            "cpu_baseline": cpu,
            "e2e": e2e,
            # K0, K1 x3 (equal / differing deadlines, general), K4 (init, a partial + a final kernel per
            # 16 buckets, the max decode), K3 unless fused
            "gpu_launches": (1 + 3 + 2 + 2 * ((n_buckets + 15) // 16) + (0 if fused else 1)) * K,
            "clocks": clk,
            "bruteforce": bf,
            "plan_violations": viol,
            "eval_leg": eval_leg,
            "parity": parity,
        }
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


def run_reference(args):
    """Reference arm of this tier: the CPU oracle, as it stands, on the host cores."""
    world, rank, _ = dist_env()
    if rank != 0:
        return
    import oracle as O
    label, n_default = WORKLOADS[args.workload]
    n = args.n_inst or n_default
    cores = os.cpu_count() or 1
    # each step: a bounded sample of the workload (different instances per step)
    probe = G.config_batch(args.workload, n_inst=1000, inst_begin=0)
    t0 = time.perf_counter()
    O.solve_batch(probe, threads=cores)
    rate = probe.n_inst / max(time.perf_counter() - t0, 1e-6)
    per_step = int(max(1000, min(n, rate * 60.0 / max(args.steps + args.warmup, 1))))
    batch = G.config_batch(args.workload, n_inst=per_step * (args.steps + args.warmup), inst_begin=0)
    for w in range(args.warmup):
        O.solve_batch(batch.subset(w * per_step, (w + 1) * per_step), threads=cores)
    t0 = time.perf_counter()
    for s in range(args.steps):
        i0 = (args.warmup + s) * per_step
        O.solve_batch(batch.subset(i0, i0 + per_step), threads=cores)
    dt = time.perf_counter() - t0
    value = per_step * args.steps / dt
    line = {"metric": "J-DOB instances solved/s", "value": value, "unit": "instances/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3 / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "impl": "reference",
            "config": {"workload": label, "n_inst_per_step": per_step, "parallelism": f"host x{cores} threads"},
            "cpu_baseline": {"value": value, "unit": "instances/s", "cores": cores, "kind": "oracle",
                             "cpu_model": cpu_model(), "sample": f"{per_step} instances of {label} per step"},
            "e2e": {"value": value, "unit": "instances/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    a = parse()
    if a.impl == "reference":
        run_reference(a)
    else:
        run_mine(a)
