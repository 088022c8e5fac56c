#!/bin/bash
# Full GPU evidence session: parity tests, smoke, per-stage traces, bench (fast + exact + DP step at N=1),
# sweeps (configs[2]/[3]), widened CNN engines (configs[4]), the reference CPU arm, the ncu launch list and
# one full ncu capture of the bench kernel.
# Usage (from repo root, under gpurun): bash scripts/gpu_check.sh [tag]
TAG=${1:-r1}
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/nvsmi_$TAG.txt 2>&1
(nproc; lscpu | grep "Model name") > $OUT/host_$TAG.txt
timeout 900 python -u -m pytest tests -m gpu -x -v --timeout 300 > $OUT/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_$TAG.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke_$TAG.log
timeout 300 python scripts/trace_step.py --mode fast > $OUT/trace_fast_$TAG.json 2>&1
timeout 300 python scripts/trace_step.py --mode fast --flat > $OUT/trace_fastflat_$TAG.json 2>&1
timeout 300 python scripts/trace_step.py --mode exact > $OUT/trace_exact_$TAG.json 2>&1
timeout 600 python bench.py > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err
timeout 600 python bench.py --mode exact --no-cpu-baseline > $OUT/bench_exact_$TAG.json 2> $OUT/bench_exact_$TAG.err
timeout 600 python bench.py --force-dp --no-e2e --no-cpu-baseline > $OUT/bench_dp1_$TAG.json 2> $OUT/bench_dp1_$TAG.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $OUT/bench_ref_$TAG.json 2> $OUT/bench_ref_$TAG.err
timeout 900 python scripts/sweep.py --out $OUT/sweep_$TAG.json > $OUT/sweep_$TAG.log 2>&1
timeout 600 python scripts/wide_bench.py --batch 100 --n 1000 --steps 3 --out $OUT/wide_$TAG.jsonl > $OUT/wide_$TAG.log 2>&1
timeout 600 python scripts/wide_bench.py --batch 1000 --n 4000 --steps 3 --out $OUT/wide_$TAG.jsonl >> $OUT/wide_$TAG.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_$TAG.csv \
  python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $OUT/ncu_launch_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:train_cluster_kernel -s 1 -c 1 \
  -o $OUT/prof_cluster_$TAG -f python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > $OUT/ncu_cluster_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc_gemm_kernel -s 0 -c 3 \
  -o $OUT/prof_tc_$TAG -f python scripts/wide_bench.py --batch 100 --n 200 --steps 1 > $OUT/ncu_tc_$TAG.log 2>&1
ls -la $OUT | tail -30
