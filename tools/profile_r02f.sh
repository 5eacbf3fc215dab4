#!/bin/bash
# Round-2 final profiling pass (one B200 under gpurun), after the K1 kernel split and the staged K3:
# launch list of the bench step, ncu --set full (+ FP64 instruction counters) of K1 (equal-deadline
# kernel on C2, differing-deadline kernel on C3 and C5), K2 (full C4), K3, K4, (no compute-sanitizer:
# closed on the pool).  Outputs in $OUT (default gpurun_out/r02f).  The bench lines are a second pass
# (tools/bench_r02f.sh) once profiles/ncu_traffic.json holds this capture's counters.
set -x
OUT=${OUT:-gpurun_out/r02f}
mkdir -p $OUT
X="--metrics smsp__sass_thread_inst_executed_op_fp64_pred_on.sum,smsp__inst_executed_pipe_fp64.sum"
python __graft_entry__.py > $OUT/build.log 2>&1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/gpu.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
    python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --bf-reps 1 > $OUT/launches_bench.log 2>&1
timeout 900 ncu --set full $X --clock-control none --import-source on --kernel-name-base mangled \
    -k regex:k_solveILb0ELb1ELb1ELb0ELb0E -c 1 -o $OUT/prof_solve -f \
    python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-bf > $OUT/prof_solve.log 2>&1
timeout 900 ncu --set full $X --clock-control none --import-source on --kernel-name-base mangled \
    -k regex:k_solveILb0ELb1ELb1ELb0ELb1E -c 1 -o $OUT/prof_solve_c3 -f \
    python bench.py --workload c3 --steps 1 --warmup 1 --no-e2e --no-cpu --no-bf > $OUT/prof_solve_c3.log 2>&1
timeout 900 ncu --set full $X --clock-control none --import-source on --kernel-name-base mangled \
    -k regex:k_solveILb0ELb1ELb1ELb0ELb1E -c 1 -o $OUT/prof_solve_c5 -f \
    python bench.py --workload c5 --n-inst 1000000 --steps 1 --warmup 1 --no-e2e --no-cpu --no-bf > $OUT/prof_solve_c5.log 2>&1
timeout 900 ncu --set full $X --clock-control none --import-source on --kernel-name-base mangled \
    -k regex:k_bf_mainILi8ELb1ELb0E -c 1 -o $OUT/prof_bf -f \
    python tools/profile_bf.py 1.0 > $OUT/prof_bf.log 2>&1
timeout 600 ncu --set full $X --clock-control none --import-source on -k regex:k_eval -c 1 -o $OUT/prof_eval -f \
    python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu --no-bf > $OUT/prof_eval.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_stats_partial -c 1 -o $OUT/prof_stats -f \
    python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu --no-bf > $OUT/prof_stats.log 2>&1
# (compute-sanitizer is closed on the GPU pool since this pass was written: profiles/r02_compute_sanitizer.txt
# is the earlier r02s capture)
ls -la $OUT
