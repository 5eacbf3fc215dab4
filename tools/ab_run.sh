#!/bin/bash
# GPU parity suite, then kernel timings (tools/time_kernels.py $WL, default "c2 c3 c5 bf") of the
# default build against tools/libjdob_<name>.so variants, then the executed n~ set-up fraction.
# usage (on the GPU box): [WL="c2 bf"] bash tools/ab_run.sh VARIANT [VARIANT ...]
WL=${WL:-c2 c3 c5 bf}
[ -z "$NOTEST" ] && timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
for i in 1 2; do for L in default "$@"; do
  if [ $L = default ]; then python tools/time_kernels.py $WL
  else JDOB_LIB=$PWD/tools/libjdob_$L.so python tools/time_kernels.py $WL; fi
done; done
