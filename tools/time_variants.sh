#!/bin/bash
# Time the default build and every tools/libjdob_*.so variant (tools/time_kernels.py).
python tools/time_kernels.py
for L in tools/libjdob_*.so; do [ -e "$L" ] && JDOB_LIB=$PWD/$L python tools/time_kernels.py; done
true
