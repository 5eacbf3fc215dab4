"""Small end-to-end run of every kernel for compute-sanitizer (memcheck / racecheck / synccheck / initcheck)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import jdobgen as G  # noqa: E402
import paper_2504_14611_b200 as J  # noqa: E402

b = G.random_batch(seed=5, n_inst=64, M_lo=1, M_hi=32, N_lo=1, N_hi=12, k_max=70, tfree_frac=0.4)
db = J.DeviceBatch(b)
res = J.solve_batch(db, counts=True, stats=True, n_buckets=32, partition=True)
J.solve_batch(db, stats=True, n_buckets=32)          # pruned product path
J.solve_batch(db, work=True, partition=True)         # executed-work counters
J.eval_plans(db, plans=res)
J.eval_plans(db, J.plan_partition(db, res), res["f_e"])
J.solve_grouped(J.DeviceBatch(b.subset(0, 16)))
c = G.config_batch("c3", n_inst=64)
J.solve_batch(J.DeviceBatch(c), stats=True, n_buckets=3)
t = G.toy_instance("toy-4")
dt = J.DeviceBatch(t)
J.bruteforce(dt, 0)
J.bruteforce(dt, 1)
small = G.random_batch(seed=9, n_inst=1, M_lo=9, M_hi=9, N_lo=1, N_hi=1, k_max=3)
J.bruteforce(J.DeviceBatch(small), 0)
J.solve_batch(J.DeviceBatch(c), work=True)
big = G.concat([G.random_batch(seed=3, n_inst=8, M_lo=1, M_hi=32, N_lo=1, N_hi=8, k_max=40)])
from tests.test_oracle_large import large_instance  # noqa: E402
lb = G.concat([large_instance(40, 1), large_instance(70, 2, hetero=True)])
J.solve_batch(J.DeviceBatch(lb), partition=True)
J.solve_batch(J.DeviceBatch(lb), counts=True, partition=True)
r5 = G.random_batch(seed=21, n_inst=1, M_lo=5, M_hi=5, N_lo=3, N_hi=3, k_max=20)
J.bruteforce(J.DeviceBatch(r5), 0)
J.solve_batch(db, verify=True, slack=1e-9)           # row a11 in K1's epilogue
J.bruteforce(J.DeviceBatch(r5), 0, work=True)        # K2 counting instantiation
dc = J.DeviceBatch(c)
rc = J.solve_batch(dc)
for P in (1, 2, 4):                                  # statistics subtrees (jdob_stats_part)
    for r in range(P):
        lo, hi = r * 64 // P, (r + 1) * 64 // P
        part = J.DeviceBatch(G.config_batch("c3", n_inst=hi - lo, inst_begin=lo))
        J.stats(part, J.solve_batch(part), n_buckets=3, part=(64, P, r))
models, params = G.c5_device_inputs(inst_begin=1000)  # K6 device generator
g5 = J.DeviceBatch.generate_c5(models, params, 3000)
J.solve_batch(g5, stats=True, n_buckets=480)
hb = J.HostBuffers(c, stats=True, n_buckets=3)
J.solve_batch_host(hb)
c2 = G.config_batch("c2", n_inst=300)                # equal-deadline uniform kernel, K3 windows
d2 = J.DeviceBatch(c2)
r2 = J.solve_batch(d2, stats=True, n_buckets=7)
J.eval_plans(d2, plans=r2, f_user=False)
J.solve_batch_host(J.HostBuffers(c2, stats=True, n_buckets=7, shared=True))
torch.cuda.synchronize()
print("sanitize run ok")
