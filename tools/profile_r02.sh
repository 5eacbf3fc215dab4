#!/bin/bash
# Round-2 profiling pass (one B200 under gpurun): bench lines, launch list, ncu --set full of the
# product kernels with the FP64 instruction counters.  Outputs in $OUT (default gpurun_out/r02p).
set -x
OUT=${OUT:-gpurun_out/r02p}
mkdir -p $OUT
X="--metrics smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_fp64_pred_on.sum,sm__sass_thread_inst_executed_op_fp64_pred_on.sum,smsp__inst_executed_pipe_fp64.sum,sm__inst_executed_pipe_fp64.sum"
python __graft_entry__.py > $OUT/build.log 2>&1
[ -z "$NOBENCH" ] && python bench.py > $OUT/bench_default.jsonl 2> $OUT/bench_default.err
[ -n "$C5" ] && python bench.py --workload c5 --no-bf > $OUT/bench_c5.jsonl 2> $OUT/bench_c5.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
    python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --bf-reps 1 > $OUT/launches_bench.log 2>&1
timeout 900 ncu --set full $X --clock-control none --import-source on --kernel-name-base mangled \
    -k regex:k_solveILb0ELb1ELb1E -c 1 -o $OUT/prof_solve -f \
    python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-bf > $OUT/prof_solve.log 2>&1
timeout 900 ncu --set full $X --clock-control none --import-source on --kernel-name-base mangled \
    -k regex:k_bf_mainILi8ELb1ELb0E -c 1 -o $OUT/prof_bf -f \
    python tools/profile_bf.py 1.0 > $OUT/prof_bf.log 2>&1
[ -n "$EVAL" ] && timeout 600 ncu --set full $X --clock-control none --import-source on -k regex:k_eval -c 1 -o $OUT/prof_eval -f \
    python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu --no-bf > $OUT/prof_eval.log 2>&1
ls -la $OUT
