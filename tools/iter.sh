#!/bin/bash
# Local build + GPU iteration: build default lib and variants, run GPU tests, time variants, profile k_solve.
# usage: tools/iter.sh TAG [variant flags pairs...]
set -e
cd /root/repo
TAG=$1; shift
python paper_2504_14611_b200/build.py > /dev/null
rm -f tools/libjdob_*.so
[ $# -ge 2 ] && tools/build_variants.sh "$@"
cp paper_2504_14611_b200/build/solve.o /tmp/solve_prof_$TAG.o
cp paper_2504_14611_b200/build/bruteforce.o /tmp/bf_prof_$TAG.o
timeout 3400 /usr/local/graft/bin/gpurun --timeout 1800 -- "timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3; bash tools/time_variants.sh 2>&1; timeout 600 ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-k_solve} -s ${KSKIP:-2} -c 1 -o gpurun_out/prof_$TAG -f ${PROFCMD:-python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-bf} > /dev/null 2>&1" > /tmp/gpurun_$TAG.log 2>&1 || true
tail -22 /tmp/gpurun_$TAG.log
