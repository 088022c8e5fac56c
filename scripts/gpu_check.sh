#!/bin/bash
# One GPU session: parity tests, smoke, bench, ncu launch list + full capture of the train kernel.
# Usage (from repo root, under gpurun): bash scripts/gpu_check.sh [tag]
set -x
TAG=${1:-r1}
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/nvsmi_$TAG.txt 2>&1
nproc > $OUT/nproc_$TAG.txt; lscpu | grep "Model name" >> $OUT/nproc_$TAG.txt
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_$TAG.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke_$TAG.log
timeout 300 python scripts/trace_step.py --mode fast > $OUT/trace_fast_$TAG.json 2>&1
timeout 300 python scripts/trace_step.py --mode exact > $OUT/trace_exact_$TAG.json 2>&1
timeout 600 python bench.py > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err
timeout 600 python bench.py --mode exact --no-cpu-baseline > $OUT/bench_exact_$TAG.json 2> $OUT/bench_exact_$TAG.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_$TAG.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline > $OUT/ncu_launch_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:train_kernel -s 1 -c 1 \
  -o $OUT/prof_train_$TAG -f python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > $OUT/ncu_full_$TAG.log 2>&1
ls -la $OUT
