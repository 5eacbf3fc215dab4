"""Write profiles/ncu_traffic.json from an ncu --set full capture (tools/profile_r02f.sh): per-launch DRAM
traffic and the hardware counters bench.py reports beside its roofline (committed, so the bench line is
reproducible from profiles/).  usage: python tools/ncu_records.py gpurun_out/r02f"""
import csv
import io
import json
import os
import subprocess
import sys

O = sys.argv[1]
CAP = os.path.basename(O.rstrip("/"))


def raw(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(txt)))
    return dict(zip(r[0], r[2])), dict(zip(r[0], r[1]))


SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-6, "us": 1e-3, "ms": 1.0, "s": 1e3}


def num(d, k):
    return float(d[k].replace(",", ""))


def hw(d, u):
    stalls = {}
    for k, v in d.items():
        if k.startswith("smsp__average_warps_issue_stalled") and k.endswith("per_issue_active.ratio"):
            try:
                stalls[k[34:-23]] = float(v.replace(",", ""))
            except ValueError:
                pass
    top = ", ".join(f"{k}={v:.2f}" for k, v in sorted(stalls.items(), key=lambda x: -x[1])[:7])
    return {"ncu_ms": round(num(d, "gpu__time_duration.sum") * SCALE[u["gpu__time_duration.sum"]], 4),
            "issue_active": round(num(d, "smsp__issue_active.avg.pct_of_peak_sustained_active") / 100, 3),
            "fp64_pipe_active": round(num(d, "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active") / 100, 3),
            "warps_active": round(num(d, "sm__warps_active.avg.pct_of_peak_sustained_active") / 100, 3),
            "warp_instructions": int(num(d, "smsp__inst_executed.sum")),
            "fp64_thread_inst": int(num(d, "smsp__sass_thread_inst_executed_op_fp64_pred_on.sum")),
            "shared_bank_conflicts": int(num(d, "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum")),
            "top_stalls": top}


def traffic(d, u):
    return int(sum(num(d, k) * SCALE[u[k]] for k in ("dram__bytes_read.sum", "dram__bytes_write.sum")))


out = {"_about": f"Per-launch hardware counters of the bench's own launch configurations from the committed ncu "
                 f"--set full captures (capture {CAP}, profiles/r02_ncu_full_summary.txt): k_solve = K1 "
                 f"equal-deadline uniform-users kernel k_solve<0,1,1,0,0> on C2 (2^20 instances, bench default); "
                 f"k_solve_c3/_c5 = the differing-deadline kernel k_solve<0,1,1,0,1> on C3 / C5 (10^6); "
                 f"k_bf_main = K2 k_bf_main<8,1,0,1,1> over the full C4 space; k_eval = K3 on the C2 plans. "
                 f"traffic = dram__bytes_read.sum + dram__bytes_write.sum; fp64_thread_inst = "
                 f"smsp__sass_thread_inst_executed_op_fp64_pred_on.sum (FP64 lane instructions)."}
for key, rep, tkey in (("k_solve", "prof_solve", "k_solve"), ("k_solve_c3", "prof_solve_c3", None),
                       ("k_solve_c5_1e6", "prof_solve_c5", None), ("k_bf_main", "prof_bf", "k_bf_main_c4_full"),
                       ("k_eval", "prof_eval", "k_eval")):
    d, u = raw(os.path.join(O, rep + ".ncu-rep"))
    out[key + "_hw"] = hw(d, u)
    if tkey:
        out[tkey] = traffic(d, u)
json.dump(out, open("profiles/ncu_traffic.json", "w"), indent=1)
print(json.dumps(out, indent=1)[:3000])
