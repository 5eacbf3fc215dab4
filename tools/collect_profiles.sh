#!/bin/bash
# Copy a profile_run.sh capture (gpurun_out/$1) into profiles/r01_*: bench lines, launch list,
# ncu summaries, per-line hotspots (needs the objects of the profiled build in /tmp/*_prof_$2.o).
set -e
O=gpurun_out/$1; T=$2
for f in bench_default:r01_bench_c2 bench_c5:r01_bench_c5 bench_c3:r01_bench_c3 fp64_microbench:r01_fp64_microbench; do
  [ -s $O/${f%%:*}.jsonl ] && cp $O/${f%%:*}.jsonl profiles/${f##*:}.jsonl
done
cp $O/launches.csv profiles/r01_launches.csv
python tools/launch_summary.py $O/launches.csv > profiles/r01_launch_list_summary.txt 2>&1
(echo "# ncu --set full --clock-control none, one launch each (round-1 final kernels, capture $1)"
 echo "# k_solve<0,1,1> = K1 uniform-users product kernel; C2 = bench default, C5 = Monte Carlo mix; k_bf_main<8,1> = full C4; k_eval = C2 plans; k_stats_partial = C2"
 python tools/ncu_summary.py $O/prof_solve.ncu-rep $O/prof_solve_c5.ncu-rep $O/prof_bf.ncu-rep $O/prof_eval.ncu-rep $O/prof_stats.ncu-rep) > profiles/r01_ncu_full_summary.txt 2>&1
(echo "# K1 uniform kernel, C2 (bench default, capture $1): executed warp instructions and stall samples per source line"
 python tools/sass_hotspots.py $O/prof_solve.ncu-rep /tmp/solve_prof_$T.o k_solveILb0ELb1ELb1E 40) > profiles/r01_k_solve_hotspots.txt 2>&1
(echo "# K1 uniform kernel, C5 (capture $1)"
 python tools/sass_hotspots.py $O/prof_solve_c5.ncu-rep /tmp/solve_prof_$T.o k_solveILb0ELb1ELb1E 40) > profiles/r01_k_solve_c5_hotspots.txt 2>&1
(echo "# K2 k_bf_main<8,1>, full C4 (capture $1)"
 python tools/sass_hotspots.py $O/prof_bf.ncu-rep /tmp/bf_prof_$T.o k_bf_mainILi8ELb1E 40) > profiles/r01_k_bf_main_hotspots.txt 2>&1
(echo "# division slow-path / subroutine CALL sites executed (capture $1): K1 C2, K1 C5, K2 C4"
 for a in "prof_solve solve k_solveILb0ELb1ELb1E" "prof_solve_c5 solve k_solveILb0ELb1ELb1E" "prof_bf bf k_bf_mainILi8ELb1E"; do
   set -- $a; echo "== $1"; python tools/slowpath_calls.py $O/$1.ncu-rep /tmp/$2_prof_$T.o $3; done) > profiles/r01_slowpath_calls.txt 2>&1
(echo "# compute-sanitizer over tools/sanitize_run.py (every kernel: K0, K1 uniform + general incl. pruned/literal/work variants, K1L, K2 with the vector bounds, K3, K4, K5, host pipeline), capture $1"
 for t in memcheck racecheck synccheck initcheck; do echo "== $t"; cat $O/sanitize_$t.txt; done) > profiles/r01_compute_sanitizer.txt
