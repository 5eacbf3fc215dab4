#!/bin/bash
# Profiling pass (run under gpurun on one B200): FP64 microbenchmark, the default bench line,
# ncu launch list of the bench step, ncu --set full of the top kernels.  Outputs land in $OUT.
set -x
OUT=${OUT:-gpurun_out}
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/gpu.txt
nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false -o /tmp/fp64mb tools/fp64_microbench.cu && /tmp/fp64mb > $OUT/fp64_microbench.jsonl
python __graft_entry__.py
python bench.py > $OUT/bench_default.jsonl 2> $OUT/bench_default.err
python bench.py --workload c5 --no-bf --no-cpu > $OUT/bench_c5.jsonl 2> $OUT/bench_c5.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
    python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --bf-reps 1 > $OUT/launches_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled \
    -k regex:k_solveILb0ELb1ELb1E -c 1 -o $OUT/prof_solve -f \
    python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-bf > $OUT/prof_solve.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled \
    -k regex:k_solveILb0ELb1ELb1E -c 1 -o $OUT/prof_solve_c5 -f \
    python bench.py --workload c5 --steps 1 --warmup 1 --no-e2e --no-cpu --no-bf > $OUT/prof_solve_c5.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_bf_main -c 1 -o $OUT/prof_bf -f \
    python tools/profile_bf.py 1.0 > $OUT/prof_bf.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_eval -c 1 -o $OUT/prof_eval -f \
    python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu --no-bf > $OUT/prof_eval.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_stats_partial -c 1 -o $OUT/prof_stats -f \
    python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu --no-bf > $OUT/prof_stats.log 2>&1
for tool in memcheck racecheck synccheck; do
    timeout 900 compute-sanitizer --tool $tool python tools/sanitize_run.py > $OUT/sanitize_$tool.txt 2>&1
done
timeout 900 compute-sanitizer --tool initcheck python tools/sanitize_run.py > $OUT/sanitize_initcheck.txt 2>&1
ls -la $OUT
