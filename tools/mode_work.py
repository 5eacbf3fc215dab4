import os, sys, json
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import jdobgen as G, paper_2504_14611_b200 as J
b = G.config_batch("c2", n_inst=1 << 20)
db = J.DeviceBatch(b)
for mode in (0, 2, 3):
    r = J.solve_batch(db, mode=mode, f_user=False, work=True)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(); J.solve_batch(db, mode=mode, f_user=False); e.record(); torch.cuda.synchronize()
    wk = r["work"].cpu().numpy()
    print(json.dumps({"mode": mode, "ms": s.elapsed_time(e), "setups": float(wk[:, 0].mean()), "visit": float(wk[:, 1].mean()),
                      "lc_frac": float((r["n_tilde"].cpu().numpy() == 16).mean())}))
