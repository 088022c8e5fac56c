#!/bin/bash
# Full GPU evidence session: parity tests, smoke, per-stage trace, bench (fast + exact), sweep
# (configs[2]/[3]), ncu launch list and one full ncu capture of the train kernel.
# Usage (from repo root, under gpurun): bash scripts/gpu_check.sh [tag]
TAG=${1:-r1}
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/nvsmi_$TAG.txt 2>&1
(nproc; lscpu | grep "Model name") > $OUT/host_$TAG.txt
timeout 900 python -u -m pytest tests -m gpu -x -v --timeout 300 > $OUT/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_$TAG.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke_$TAG.log
for M in fast exact; do
  timeout 300 python scripts/trace_step.py --mode $M > $OUT/trace_${M}_$TAG.json 2>&1
done
timeout 600 python bench.py > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err
timeout 600 python bench.py --mode exact --no-cpu-baseline > $OUT/bench_exact_$TAG.json 2> $OUT/bench_exact_$TAG.err
timeout 900 python scripts/sweep.py --out $OUT/sweep_$TAG.json > $OUT/sweep_$TAG.log 2>&1
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $OUT/bench_ref_$TAG.json 2> $OUT/bench_ref_$TAG.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_$TAG.csv \
  python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $OUT/ncu_launch_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:train_kernel -s 1 -c 1 \
  -o $OUT/prof_train_$TAG -f python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > $OUT/ncu_full_$TAG.log 2>&1
ls -la $OUT | tail -20
