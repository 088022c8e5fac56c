#!/bin/bash
# ncu full capture of the persistent train kernel (fast and exact) + launch list.
TAG=${1:-n}
OUT=gpurun_out
mkdir -p $OUT
for M in fast exact; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:train_kernel -s 1 -c 1 \
    -o $OUT/prof_${M}_$TAG -f python bench.py --mode $M --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > $OUT/ncu_${M}_$TAG.log 2>&1
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_$TAG.csv \
  python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $OUT/ncu_launch_$TAG.log 2>&1
ls -la $OUT | tail -5
