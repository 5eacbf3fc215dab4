import os, sys, json
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import jdobgen as G, paper_2504_14611_b200 as J
for cfg, n in (("c2", 1 << 20), ("c3", 100000), ("c5", 1000000)):
    b = G.config_batch(cfg, n_inst=n)
    db = J.DeviceBatch(b)
    r = J.solve_batch(db, work=True, f_user=False)
    wk = r["work"].cpu().numpy(); nt = r["n_tilde"].cpu().numpy()
    Ns = np.array([m.N for m in b.models])[b.model_id]
    lc = nt == Ns
    out = {"cfg": cfg, "lib": os.path.basename(os.environ.get("JDOB_LIB", "default")),
           "setups_mean": float(wk[:, 0].mean()), "lc_win_frac": float(lc.mean()),
           "setups_mean_lc": float(wk[lc, 0].mean()) if lc.any() else None,
           "setups_mean_off": float(wk[~lc, 0].mean()) if (~lc).any() else None,
           "setup_hist": np.bincount(wk[:, 0].astype(int), minlength=8)[:12].tolist(),
           "nt_hist": np.bincount(nt, minlength=17)[:40].tolist(),
           "visit_mean": float(wk[:, 1].mean()), "eval_mean": float(wk[:, 2].mean()), "member_mean": float(wk[:, 3].mean())}
    print(json.dumps(out), flush=True)
