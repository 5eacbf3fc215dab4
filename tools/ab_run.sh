#!/bin/bash
# GPU parity suite, then kernel timings (tools/time_kernels.py) of the default build against
# tools/libjdob_<name>.so variants, then the executed n~ set-up fraction of C2 and C5.
# usage (on the GPU box): bash tools/ab_run.sh VARIANT [VARIANT ...]
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
for i in 1 2; do for L in default "$@"; do
  if [ $L = default ]; then python tools/time_kernels.py c2 c3 c5
  else JDOB_LIB=$PWD/tools/libjdob_$L.so python tools/time_kernels.py c2 c3 c5; fi
done; done
for W in c2 c5; do
  python bench.py --workload $W --steps 3 --warmup 3 --no-bf --no-cpu --no-e2e | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["config"]["workload"], d["ms_per_step"], d["roofline"]["n_tilde_setups_frac"], d["roofline"]["frac"])'
done
