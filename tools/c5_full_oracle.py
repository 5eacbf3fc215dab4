"""The whole C5 bench workload against the oracle: 10^7 instances generated on the device and solved
there (the bench's launch configuration), every instance regenerated on the host in chunks of 10^6 and
solved by the 16-thread oracle; every decision and energy compared bit for bit.  Writes a JSON summary
(profiles/r02_c5_1e7_oracle.json when run by the profiling pass).

usage: python tools/c5_full_oracle.py OUT.json [n_inst]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import jdobgen as G  # noqa: E402
import oracle as O  # noqa: E402
import paper_2504_14611_b200 as J  # noqa: E402

FIELDS = ("E", "E_lc", "t_free_next", "f_e", "n_tilde", "j", "status", "mask")

out_path = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 10_000_000
chunk = 1_000_000
models, params = G.c5_device_inputs()
db = J.DeviceBatch.generate_c5(models, params, n)
res = J.solve_batch(db, f_user=False)
torch.cuda.synchronize()
gpu = {k: res[k].cpu().numpy() for k in FIELDS}
gpu["mask"] = gpu["mask"].view(np.uint32)
mism = {f: 0 for f in FIELDS}
t0 = time.time()
for c0 in range(0, n, chunk):
    host = G.config_c5(n_inst=min(chunk, n - c0), inst_begin=c0)
    orc = O.solve_batch(host, threads=16)
    for f in FIELDS:
        a = gpu[f][c0:c0 + host.n_inst]
        b = np.asarray(orc[f])
        if a.dtype.kind == "f":
            bad = (a.view(np.int64) != b.view(np.int64)) & ~(np.isnan(a) & np.isnan(b))
        else:
            bad = a != b.astype(a.dtype)
        mism[f] += int(bad.sum())
summary = {"workload": "c5_montecarlo_m1-32_3models_5regimes_3grids", "instances": n,
           "gpu": "device-generated (jdob_generate_c5_*), jdob_solve_batch in the bench's configuration",
           "oracle": "host-generated (jdobgen.config_c5), oracle.solve_batch, 16 threads, chunks of 10^6",
           "oracle_seconds": round(time.time() - t0, 1), "mismatches": mism,
           "all_equal": all(v == 0 for v in mism.values())}
json.dump(summary, open(out_path, "w"), indent=1)
print(json.dumps(summary))
