#!/bin/bash
# ncu full capture of the clustered fast train kernel (1 epoch launch) + launch list.
TAG=${1:-c}
OUT=gpurun_out
mkdir -p $OUT
timeout 300 python scripts/trace_step.py --mode fast > $OUT/trace_fast_$TAG.json 2>&1
timeout 600 python bench.py --no-cpu-baseline > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:train_cluster_kernel -s 1 -c 1 \
  -o $OUT/prof_cluster_$TAG -f python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > $OUT/ncu_cluster_$TAG.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_$TAG.csv \
  python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $OUT/ncu_launch_$TAG.log 2>&1
cat $OUT/trace_fast_$TAG.json; tail -3 $OUT/ncu_cluster_$TAG.log
