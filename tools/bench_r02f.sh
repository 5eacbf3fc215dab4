#!/bin/bash
# Round-2 final bench lines (one B200 under gpurun): C2 default (the driver's line), C3, C5 with 10^7
# instances generated on the device, and the N = 2 code path (two ranks on the one GPU over gloo --
# the torchrun plumbing and the exchanges, not a scaling number).  Outputs in $OUT.
set -x
OUT=${OUT:-gpurun_out/r02f}
mkdir -p $OUT
python __graft_entry__.py > $OUT/build_bench.log 2>&1
python bench.py > $OUT/bench_c2.jsonl 2> $OUT/bench_c2.err
python bench.py --workload c3 --no-bf > $OUT/bench_c3.jsonl 2> $OUT/bench_c3.err
python bench.py --workload c5 --scaling strong --no-bf > $OUT/bench_c5_1e7_devgen.jsonl 2> $OUT/bench_c5.err
JDOB_BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
    --master-port 29517 bench.py --gpus 2 --no-cpu > $OUT/bench_c2_n2_gloo.jsonl 2> $OUT/bench_c2_n2_gloo.err
JDOB_BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
    --master-port 29518 bench.py --gpus 2 --workload c3 --scaling strong --no-cpu --no-bf \
    > $OUT/bench_c3_strong_n2_gloo.jsonl 2> $OUT/bench_c3_strong_n2_gloo.err
python bench.py --impl reference --steps 3 --warmup 3 > $OUT/bench_reference.jsonl 2> $OUT/bench_reference.err
ls -la $OUT
