"""Figure-style sweeps of the paper's experiments on the GPU path.

Fig. 4: identical deadlines, beta = 2.13 (T = 10 ms) and beta = 30.25 (T = 100 ms),
average energy per user vs. the number of users M, for LC, J-DOB, J-DOB without edge DVFS
and J-DOB binary (IP-SSA is out of scope).
Fig. 5: different deadlines, M = 10 and 20, beta ~ U over [4.5, 5.5], [2, 8],
[0, 10] i.i.d. per user, the outer grouping DP with each inner method,
mean over random trials (50 in the paper; `--trials` here).

Workload: the synthetic MobileNetV2 per-block profile and Table I users of jdobgen.
The paper's absolute numbers depend on unpublished RTX 3090 profiles, so only the trends and the
order of magnitude of the maximum reductions (paper: 32.8 %, 51.3 %, 45.27 %, 44.74 %) are
comparable; nothing here is a parity pin.

usage: python experiments/figures.py [--trials 50] [--out results]
"""
from __future__ import annotations

import argparse
import csv
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import jdobgen as G  # noqa: E402

METHODS = (("LC", 1), ("J-DOB", 0), ("J-DOB w/o edge DVFS", 2), ("J-DOB binary", 3))


def users_batch(model, T_lists, seed_tag=""):
    """One instance per deadline list, Table I users."""
    z, k = G.profiles.ZETA, G.profiles.KAPPA
    Ms = [len(T) for T in T_lists]
    n_users = sum(Ms)
    cols = dict(zeta=np.full(n_users, z), kappa=np.full(n_users, k), f_min=np.full(n_users, 1.5e9),
                f_max=np.full(n_users, 2.6e9), R=np.full(n_users, G.R_TABLE_I), p_u=np.full(n_users, 1.0),
                T=np.concatenate([np.asarray(T, float) for T in T_lists]))
    n = len(T_lists)
    inst = dict(t_free=np.zeros(n), fe_min=np.full(n, 0.2e9), fe_max=np.full(n, 2.1e9), rho=np.full(n, 0.03e9))
    return G._batch_from_lists([model], np.zeros(n, np.int32), Ms, cols, inst)


def fig4_batches():
    """(beta, T, Ms, batch): one instance per M = 1..32 at the identical deadline of beta."""
    m = G.profiles.mobilenetv2()
    out = []
    for beta in (2.13, 30.25):
        T = float(G.deadline_from_beta(m, G.profiles.ZETA, 2.6e9, beta))
        Ms = list(range(1, 33))
        out.append((beta, T, Ms, users_batch(m, [[T] * M for M in Ms])))
    return out


def fig5_batches(trials, seed=55):
    """(M, lo, hi, batch): `trials` instances of M users with beta ~ U[lo, hi] i.i.d.."""
    m = G.profiles.mobilenetv2()
    lat = float(G.min_local_latency(m, np.array([G.profiles.ZETA]), np.array([2.6e9]))[0])
    out = []
    for M in (10, 20):
        for (lo, hi) in ((4.5, 5.5), (2.0, 8.0), (0.0, 10.0)):
            ids = np.arange(trials)
            beta = G.uniform(G.draw(seed, np.repeat(ids, M), np.tile(np.arange(M), trials), G.F_BETA_USER), lo, hi)
            T = (1.0 + beta) * lat
            out.append((M, lo, hi, users_batch(m, [list(T[t * M:(t + 1) * M]) for t in range(trials)])))
    return out


def fig4(J, out_dir):
    import torch
    rows = []
    for beta, T, Ms, b in fig4_batches():
        db = J.DeviceBatch(b)
        # J-DOB and its two variants from one pass (jdob_solve_batch_modes); LC is every result's E_lc
        multi = J.solve_batch_modes(db, f_user=False)
        torch.cuda.synchronize()
        res = {}
        for name, mode in METHODS:
            r = multi[J.MODE_FULL] if mode == J.MODE_LC else multi[mode]
            res[name] = (r["E_lc"] if mode == J.MODE_LC else r["E"]).cpu().numpy() / np.array(Ms)
        for q, M in enumerate(Ms):
            row = dict(beta=beta, T_ms=T * 1e3, M=M)
            for name, _ in METHODS:
                row[name] = res[name][q]
            row["reduction_%"] = 100 * (1 - res["J-DOB"][q] / res["LC"][q])
            rows.append(row)
    with open(os.path.join(out_dir, "fig4.csv"), "w", newline="") as f:
        w = csv.DictWriter(f, fieldnames=list(rows[0].keys()))
        w.writeheader()
        w.writerows(rows)
    return rows


def fig5(J, out_dir, trials, seed=55):
    import torch
    rows = []
    for M, lo, hi, b in fig5_batches(trials, seed):
        db = J.DeviceBatch(b)
        row = dict(M=M, beta_lo=lo, beta_hi=hi, trials=trials)
        for name, mode in METHODS:
            r = J.solve_grouped(db, mode=mode, f_user=False)
            torch.cuda.synchronize()
            row[name] = float(r["E"].cpu().numpy().mean() / M)
            if name == "J-DOB":
                row["mean_groups"] = float(r["n_groups"].cpu().numpy().mean())
        row["reduction_%"] = 100 * (1 - row["J-DOB"] / row["LC"])
        rows.append(row)
    with open(os.path.join(out_dir, "fig5.csv"), "w", newline="") as f:
        w = csv.DictWriter(f, fieldnames=list(rows[0].keys()))
        w.writeheader()
        w.writerows(rows)
    return rows


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--trials", type=int, default=50)
    ap.add_argument("--out", default=os.path.join(ROOT, "results"))
    a = ap.parse_args()
    os.makedirs(a.out, exist_ok=True)
    import paper_2504_14611_b200 as J
    r4 = fig4(J, a.out)
    r5 = fig5(J, a.out, a.trials)
    summ = {
        "fig4_max_reduction_%": {str(beta): max(r["reduction_%"] for r in r4 if r["beta"] == beta)
                                 for beta in (2.13, 30.25)},
        "fig4_paper_%": {"2.13": 32.8, "30.25": 51.3},
        "fig5_max_reduction_%": {str(M): max(r["reduction_%"] for r in r5 if r["M"] == M) for M in (10, 20)},
        "fig5_paper_%": {"10": 45.27, "20": 44.74},
        "dominance_ok": all(r["J-DOB"] <= min(r["LC"], r["J-DOB w/o edge DVFS"], r["J-DOB binary"]) * (1 + 1e-12)
                            for r in r4 + r5),
        "trials": a.trials,
    }
    with open(os.path.join(a.out, "figures_summary.json"), "w") as f:
        json.dump(summ, f, indent=1)
    print(json.dumps(summ))


if __name__ == "__main__":
    main()
