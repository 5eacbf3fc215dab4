# A/B of whole bench steps (C2): default build vs tools/libjdob_<name>.so variants given as arguments
for i in 1 2; do for L in default "$@"; do
  if [ $L = default ]; then unset JDOB_LIB; else export JDOB_LIB=$PWD/tools/libjdob_$L.so; fi
  python bench.py --steps 10 --warmup 3 --no-bf --no-cpu --no-e2e | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print("'$L'", round(d["ms_per_step"],4), round(d["roofline"]["launch_ms"],4))'
done; done
