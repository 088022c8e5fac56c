#!/bin/bash
# Quick GPU iteration: parity tests + per-stage trace (fast clustered, fast flat, exact) + 1 bench line.
TAG=${1:-q}
OUT=gpurun_out
mkdir -p $OUT
timeout 900 python -u -m pytest tests -m gpu -x -v --timeout 300 > $OUT/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu_$TAG.log
timeout 300 python scripts/trace_step.py --mode fast > $OUT/trace_fast_$TAG.json 2>&1
timeout 300 python scripts/trace_step.py --mode fast --flat > $OUT/trace_fastflat_$TAG.json 2>&1
timeout 300 python scripts/trace_step.py --mode exact > $OUT/trace_exact_$TAG.json 2>&1
timeout 600 python bench.py --no-cpu-baseline > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err
tail -3 $OUT/pytest_gpu_$TAG.log; cat $OUT/trace_fast_$TAG.json $OUT/trace_fastflat_$TAG.json $OUT/trace_exact_$TAG.json; tail -2 $OUT/bench_$TAG.err
