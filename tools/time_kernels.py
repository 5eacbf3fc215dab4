"""Quick kernel timing for optimisation experiments (JDOB_LIB selects a library build)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import jdobgen as G  # noqa: E402
import paper_2504_14611_b200 as J  # noqa: E402


def t_solve(cfg, n, mode=None):
    mode = J.MODE_FULL if mode is None else mode
    b = G.config_batch(cfg, n_inst=n)
    db = J.DeviceBatch(b)
    res = J.solve_batch(db, f_user=False, mode=mode)
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        J.solve_batch(db, f_user=False, out=res, mode=mode)
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    ms = float(np.median(ts))
    return {"cfg": cfg + ("" if mode == J.MODE_FULL else "_mode%d" % mode), "n": n, "ms": ms, "inst_per_s": n / ms * 1e3, "E_sum": float(res["E"].sum().item())}


def t_stats(cfg, n):
    """solve with the bucketed statistics (K4) minus solve without: K4's share of a step."""
    b = G.config_batch(cfg, n_inst=n)
    db = J.DeviceBatch(b)
    out = {}
    for st in (False, True):
        kw = dict(stats=True, n_buckets=int(b.meta.get("n_buckets", 32))) if st else {}
        res = J.solve_batch(db, f_user=False, **kw)
        torch.cuda.synchronize()
        ts = []
        for _ in range(7):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            J.solve_batch(db, f_user=False, out=res, **kw)
            e.record()
            torch.cuda.synchronize()
            ts.append(s.elapsed_time(e))
        out[st] = float(np.median(ts))
    return {"cfg": cfg + "_stats", "n": n, "ms": out[True] - out[False], "solve_ms": out[False]}


def t_e2e(cfg, n, shared=False):
    """jdob_solve_batch_host (jdob_solve_shared_host) from pinned host buffers (copies inside), median of 5."""
    b = G.config_batch(cfg, n_inst=n)
    hb = J.HostBuffers(b, stats=True, n_buckets=int(b.meta.get("n_buckets", 32)), shared=shared)
    J.solve_batch_host(hb)
    ts = []
    for _ in range(5):
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        J.solve_batch_host(hb)
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    ms = float(np.median(ts))
    return {"cfg": cfg + ("_e2e_shared" if shared else "_e2e"), "n": n, "ms": ms, "inst_per_s": n / ms * 1e3}


def t_eval(cfg, n):
    b = G.config_batch(cfg, n_inst=n)
    db = J.DeviceBatch(b)
    res = J.solve_batch(db, f_user=False)
    ev = J.eval_plans(db, plans=res, f_user=False)
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        J.eval_plans(db, plans=res, f_user=False, out=ev)
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    ms = float(np.median(ts))
    return {"cfg": cfg + "_eval", "n": n, "ms": ms, "inst_per_s": n / ms * 1e3}


def t_modes(cfg, n):
    """jdob_solve_batch_modes (J-DOB + its two variants in one pass) against the three separate calls."""
    b = G.config_batch(cfg, n_inst=n)
    db = J.DeviceBatch(b)
    J.solve_batch_modes(db, f_user=False)
    torch.cuda.synchronize()
    out = {}
    for name, fn in (("one_pass", lambda: J.solve_batch_modes(db, f_user=False)),
                     ("three_calls", lambda: [J.solve_batch(db, mode=m, f_user=False) for m in (0, 2, 3)])):
        fn()
        torch.cuda.synchronize()
        ts = []
        for _ in range(5):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            fn()
            e.record()
            torch.cuda.synchronize()
            ts.append(s.elapsed_time(e))
        out[name] = float(np.median(ts))
    return {"cfg": cfg + "_modes", "n": n, "ms_one_pass": out["one_pass"], "ms_three_calls": out["three_calls"]}


def t_bf(frac):
    b = G.config_batch("c4")
    db = J.DeviceBatch(b)
    size = J.bf_space_size(0, b.models[0].N, b.M(0), 64)
    hi = int(size * frac) // 64 * 64
    J.bruteforce(db, 0, 0, hi // 16)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    E, I, S = J.bruteforce(db, 0, 0, hi)
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e)
    return {"cfg": "c4bf", "cand": hi, "ms": ms, "cand_per_s": hi / ms * 1e3, "E": float(E.item()), "I": int(I.item())}


def t_grouped(cfg, n):
    b = G.config_batch(cfg, n_inst=n)
    db = J.DeviceBatch(b)
    J.solve_grouped(db, f_user=False)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    r = J.solve_grouped(db, f_user=False)
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e)
    return {"cfg": cfg + "_grouped", "n": n, "ms": ms, "inst_per_s": n / ms * 1e3,
            "mean_groups": float(r["n_groups"].float().mean().item())}


if __name__ == "__main__":
    lib = os.environ.get("JDOB_LIB", "default")
    which = sys.argv[1:] or ["c2", "c3", "c5", "bf"]
    todo = {"c2": lambda: t_solve("c2", 1 << 20), "c3": lambda: t_solve("c3", 100_000),
            "c5": lambda: t_solve("c5", 1_000_000), "bf": lambda: t_bf(0.25),
            "og": lambda: t_grouped("c3", 100_000), "eval": lambda: t_eval("c2", 1 << 20),
            "stats": lambda: t_stats("c2", 1 << 20), "modes2": lambda: t_modes("c2", 1 << 20),
            "modes3": lambda: t_modes("c3", 100_000), "e2e": lambda: t_e2e("c2", 1 << 20), "e2es": lambda: t_e2e("c2", 1 << 20, True), "c2lc": lambda: t_solve("c2", 1 << 20, J.MODE_LC),
            "c2noedge": lambda: t_solve("c2", 1 << 20, J.MODE_NO_EDGE_DVFS), "stats5": lambda: t_stats("c5", 1_000_000)}
    for r in (todo[w]() for w in which):
        r["lib"] = os.path.basename(lib)
        print(json.dumps(r), flush=True)
