#!/bin/bash
# Quick GPU iteration: parity tests + per-stage trace (fast & exact) + 1 bench line.
TAG=${1:-q}
OUT=gpurun_out
mkdir -p $OUT
timeout 900 python -u -m pytest tests -m gpu -x -v --timeout 300 > $OUT/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu_$TAG.log
for M in fast exact; do
  timeout 300 python scripts/trace_step.py --mode $M > $OUT/trace_${M}_$TAG.json 2>&1
done
timeout 600 python bench.py --no-cpu-baseline > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err
tail -3 $OUT/pytest_gpu_$TAG.log; cat $OUT/trace_fast_$TAG.json $OUT/trace_exact_$TAG.json
