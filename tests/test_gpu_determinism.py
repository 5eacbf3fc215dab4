"""results independent of the launch grid.  The persistent grids of K1 and K2 are
divided by JDOB_GRID_DIV in a subprocess (a test hook, read once per process); the J-DOB outputs, the
statistics and the brute-force argmin must equal the default grid's bit for bit."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import sys, json, numpy as np
sys.path.insert(0, %r)
import jdobgen as g, paper_2504_14611_b200 as J
out = {}
for cfg, n in (("c3", 30000), ("c5", 20000)):
    b = g.config_batch(cfg, n_inst=n)
    db = J.DeviceBatch(b)
    r = J.solve_batch(db, f_user=True, stats=True, n_buckets=int(b.meta["n_buckets"]))
    for f in ("E", "t_free_next", "f_e", "n_tilde", "j", "status", "mask", "f_user", "stats"):
        out[cfg + f] = r[f].cpu().numpy().reshape(-1).view(np.uint8).tobytes().hex()
c4 = J.DeviceBatch(g.config_batch("c4"))
E, I, S = J.bruteforce(c4, 0, 0, 12 ** 7 * 64)
out["bf"] = [float(E.item()), int(I.item())]
print(json.dumps(out))
""" % ROOT


def run(div):
    env = dict(os.environ)
    if div > 1:
        env["JDOB_GRID_DIV"] = str(div)
    else:
        env.pop("JDOB_GRID_DIV", None)
    r = subprocess.run([sys.executable, "-c", SCRIPT], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    return json.loads(r.stdout.strip().splitlines()[-1])


def test_results_independent_of_grid_size():
    base = run(1)
    for div in (3, 16):
        other = run(div)
        assert other.keys() == base.keys()
        for k in base:
            assert other[k] == base[k], (div, k)
