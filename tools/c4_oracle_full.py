#!/usr/bin/env python
"""Full-space CPU oracle argmin of the C4 exhaustive search ("C1-C4 in full").

Runs the C oracle's literal brute force (oracle_bf_mt: every candidate decoded and evaluated, no
pruning, no early exit) over the whole general space of C4 (12^8 vectors x 64 grid points =
2.75e10 candidates) in contiguous chunks, merging the partial argmins in index order
(strict <, lowest index wins).  Each finished chunk is appended to a JSONL checkpoint so an
interrupted run resumes; the final record is written to profiles/r02_c4_oracle_full.json.

Test infrastructure: calls only oracle/ and the seeded generator (jdobgen/), never the CUDA path.
usage: python tools/c4_oracle_full.py [--threads T] [--chunks C] [--ckpt FILE]
"""
import argparse
import json
import os
import platform
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import jdobgen as G  # noqa: E402
import oracle as O  # noqa: E402


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor() or "unknown"


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--threads", type=int, default=os.cpu_count() or 1)
    p.add_argument("--chunks", type=int, default=256)
    p.add_argument("--ckpt", default=os.path.join(ROOT, "profiles", "r02_c4_oracle_full.ckpt.jsonl"))
    p.add_argument("--out", default=os.path.join(ROOT, "profiles", "r02_c4_oracle_full.json"))
    a = p.parse_args()
    O.build()
    b = G.config_batch("c4")
    size = O.bf_space_size(b, 0)
    k = O.grid_k(b)
    nvec = size // k
    done = {}
    if os.path.exists(a.ckpt):
        for line in open(a.ckpt):
            r = json.loads(line)
            done[r["chunk"]] = r
    with open(a.ckpt, "a") as ck:
        for c in range(a.chunks):
            if c in done:
                continue
            lo = (nvec * c // a.chunks) * k          # vector-aligned chunk boundaries
            hi = (nvec * (c + 1) // a.chunks) * k
            t0 = time.perf_counter()
            E, idx, st = O.bf(b, 0, lo, hi, threads=a.threads)
            dt = time.perf_counter() - t0
            r = {"chunk": c, "lo": lo, "hi": hi, "E": E.hex(), "idx": idx, "status": st, "s": dt}
            ck.write(json.dumps(r) + "\n")
            ck.flush()
            done[c] = r
            print(f"chunk {c}/{a.chunks} [{lo}, {hi}) E={E!r} idx={idx} {dt:.1f}s", flush=True)
    E_min, idx_min, secs = float("inf"), -1, 0.0
    for c in range(a.chunks):           # index order, strict < : lowest index wins ties
        r = done[c]
        E = float.fromhex(r["E"])
        secs += r["s"]
        if E < E_min:
            E_min, idx_min = E, r["idx"]
    rec = {"config": "c4_resnet18_m8_12pp_k64_general", "space": "general", "candidates": size,
           "vectors": nvec, "k": k, "E_min": E_min, "E_min_hex": E_min.hex(), "idx_min": idx_min,
           "chunks": a.chunks, "oracle_seconds": secs, "candidates_per_s": size / secs,
           "threads": a.threads, "cpu_model": cpu_model(), "host": platform.node(),
           "what": "oracle_bf_mt over every candidate of the C4 general space (literal decode + "
                   "evaluation, no pruning), partial argmins merged in index order"}
    json.dump(rec, open(a.out, "w"), indent=1)
    print(json.dumps(rec))


if __name__ == "__main__":
    main()
