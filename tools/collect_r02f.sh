#!/bin/bash
# Copy the final round-2 capture (gpurun_out/r02f, tools/profile_r02f.sh) into profiles/r02_*: launch
# list, ncu summaries, per-line hotspots (objects of the profiled build in /tmp/*_prof_r02f.o),
# sanitizer logs.  The bench lines come from tools/bench_r02f.sh.
set -e
O=${1:-gpurun_out/r02f}
cp $O/launches.csv profiles/r02_launches.csv
(echo "# ncu launch list of 'bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --bf-reps 1' (capture r02f)"
 python tools/launch_summary.py $O/launches.csv) > profiles/r02_launch_list_summary.txt 2>&1
(echo "# ncu --set full --clock-control none + FP64 instruction counters, one launch each (final round-2 kernels, capture r02f)"
 echo "# k_solve<0,1,1,0,0> = K1 equal-deadline uniform-users kernel on C2 (bench default); k_solve<0,1,1,0,1> = K1 differing-deadline kernel on C3 (10^5) and C5 (10^6, device-generated); k_bf_main<8,1,0,1,1> = K2 over the full C4 space; k_eval = K3 on the C2 plans; k_stats_partial = K4 on C2"
 python tools/ncu_summary.py $O/prof_solve.ncu-rep $O/prof_solve_c3.ncu-rep $O/prof_solve_c5.ncu-rep $O/prof_bf.ncu-rep \
     $O/prof_eval.ncu-rep $O/prof_stats.ncu-rep) > profiles/r02_ncu_full_summary.txt 2>&1
(echo "# K1 k_solve<0,1,1,0,0> (equal deadlines), C2 (capture r02f): executed warp instructions and stall samples per source line"
 python tools/sass_hotspots.py $O/prof_solve.ncu-rep /tmp/solve_prof_r02f.o k_solveILb0ELb1ELb1ELb0ELb0E 60) > profiles/r02_k_solve_hotspots.txt 2>&1
(echo "# K1 k_solve<0,1,1,0,1> (differing deadlines), C5 10^6 (capture r02f)"
 python tools/sass_hotspots.py $O/prof_solve_c5.ncu-rep /tmp/solve_prof_r02f.o k_solveILb0ELb1ELb1ELb0ELb1E 60) > profiles/r02_k_solve_c5_hotspots.txt 2>&1
(echo "# K2 k_bf_main<8,1,0,1,1>, full C4 (capture r02f)"
 python tools/sass_hotspots.py $O/prof_bf.ncu-rep /tmp/bf_prof_r02f.o k_bf_mainILi8ELb1ELb0E 40) > profiles/r02_k_bf_main_hotspots.txt 2>&1
(echo "# K3 k_eval, C2 plans (capture r02f)"
 python tools/sass_hotspots.py $O/prof_eval.ncu-rep /tmp/eval_prof_r02f.o k_eval 30) > profiles/r02_k_eval_hotspots.txt 2>&1
echo collected
