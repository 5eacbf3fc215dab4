"""One-screen summary of an ncu report (key SOL, pipe, occupancy and stall metrics)."""
import csv
import io
import subprocess
import sys

WANT = ["gpu__time_duration.sum", "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "smsp__thread_inst_executed_per_inst_executed.ratio",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "smsp__sass_thread_inst_executed_op_dadd_pred_on.sum", "smsp__sass_thread_inst_executed_op_dmul_pred_on.sum",
        "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum", "smsp__sass_thread_inst_executed_op_fp64_pred_on.sum",
        "sm__sass_thread_inst_executed_op_fp64_pred_on.sum", "smsp__inst_executed_pipe_fp64.sum",
        "sm__inst_executed_pipe_fp64.sum"]
for rep in sys.argv[1:]:
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(txt)))
    h, u = r[0], r[1]
    print("==", rep)
    for row in r[2:]:
        kn = row[h.index("Kernel Name")] if "Kernel Name" in h else ""
        print("  kernel:", kn[:80])
        for w in WANT:
            if w in h:
                i = h.index(w)
                print(f"  {w:70s} {u[i]:10s} {row[i]}")
        st = []
        for i, name in enumerate(h):
            if name.startswith("smsp__average_warps_issue_stalled") and name.endswith("per_issue_active.ratio"):
                try:
                    st.append((float(row[i]), name[34:-23]))
                except ValueError:
                    pass
        print("  stalls/issue:", ", ".join(f"{n}={v:.2f}" for v, n in sorted(st, reverse=True)[:7]))
