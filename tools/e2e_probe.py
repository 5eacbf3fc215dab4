"""Where the end-to-end time goes: the host API (shared-parameter form) in FULL and in LC mode (the
LC solve is short, so that run is the copy pipeline), against the device-resident solve alone and a
plain pinned copy of the same input bytes."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import jdobgen as G  # noqa: E402
import paper_2504_14611_b200 as J  # noqa: E402


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    return float(np.median(ts))


b = G.config_batch("c2", n_inst=1 << 20)
for shared in (True, False):
    hb = J.HostBuffers(b, stats=True, n_buckets=7, shared=shared)
    h2d = {}

    def run(mode):
        h2d["b"] = J.solve_batch_host(hb, mode=mode)[0]
    full = timed(lambda: run(J.MODE_FULL))
    lc = timed(lambda: run(J.MODE_LC))
    nb = h2d["b"]
    hx = torch.empty(int(nb), dtype=torch.uint8).pin_memory()
    dx = torch.empty(int(nb), dtype=torch.uint8, device="cuda")
    cp = timed(lambda: dx.copy_(hx, non_blocking=True))
    print({"shared": shared, "h2d_MB": nb / 1e6, "host_full_ms": full, "host_lc_ms": lc, "plain_copy_ms": cp})
db = J.DeviceBatch(b)
r = J.solve_batch(db, f_user=False)
print({"device_solve_ms": timed(lambda: J.solve_batch(db, f_user=False, out=r)),
       "device_lc_ms": timed(lambda: J.solve_batch(db, f_user=False, out=r, mode=J.MODE_LC))})
