#!/bin/bash
# Full evidence session at HEAD (round 2): GPU tests, smoke, bench (+ reference arm), configs[3] line,
# sweeps, widened engines, same-GPU N=2 plumbing check, ncu launch list.
TAG=${1:-r2z}
OUT=gpurun_out; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/nvsmi_$TAG.txt 2>&1
(nproc; lscpu | grep "Model name") > $OUT/host_$TAG.txt
timeout 1200 python -u -m pytest tests -m gpu -x -q --timeout 400 > $OUT/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_$TAG.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke_$TAG.log
timeout 600 python bench.py > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $OUT/bench_ref_$TAG.json 2> $OUT/bench_ref_$TAG.err
timeout 600 python bench.py --mode exact --no-cpu-baseline --no-e2e > $OUT/bench_exact_$TAG.json 2> $OUT/bench_exact_$TAG.err
timeout 600 python bench.py --batch 16384 --n 32768 --steps 5 --no-cpu-baseline > $OUT/bench16k_$TAG.json 2> $OUT/bench16k_$TAG.err
TLB_BENCH_SAME_GPU=1 timeout 600 python bench.py --gpus 2 --batch 16 --n 800 --steps 3 --warmup 3 > $OUT/bench_same2_$TAG.json 2> $OUT/bench_same2_$TAG.err
timeout 300 python scripts/trace_step.py --mode fast > $OUT/trace_fast_$TAG.json 2>&1
timeout 900 python scripts/sweep.py --out $OUT/sweep_$TAG.json > $OUT/sweep_$TAG.log 2>&1
timeout 600 python scripts/wide_bench.py --batch 100 --n 1000 --steps 3 --out $OUT/wide_$TAG.jsonl > $OUT/wide_$TAG.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_$TAG.csv \
  python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $OUT/ncu_launch_$TAG.log 2>&1
tail -3 $OUT/pytest_gpu_$TAG.log; tail -2 $OUT/smoke_$TAG.log
for f in bench bench_ref bench_exact bench16k bench_same2; do python -c "
import json
try:
  d=json.loads(open('$OUT/${f}_$TAG.json').read().strip().splitlines()[-1])
  print('$f', d.get('value'), d.get('n_gpus'), d.get('ms_per_step'), (d.get('e2e') or {}).get('value'), (d.get('e2e_cpp') or {}).get('value'), (d.get('roofline') or {}).get('frac'), (d.get('cpu_baseline') or {}).get('value'), (d.get('impl_config') or {}).get('dp_note'))
except Exception as e: print('$f ERR', e)
"; done
cat $OUT/trace_fast_$TAG.json; tail -4 $OUT/wide_$TAG.log
TLB_CLUSTER_COOP=0 bash scripts/ncu_one.sh ncu_cluster_$TAG train_cluster_kernel python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
python scripts/ncu_lines.py $OUT/ncu_cluster_$TAG.ncu-rep 40 > $OUT/ncu_cluster_${TAG}_lines.txt 2>&1
grep -E "time_duration|dram__bytes|fma_cycles|issue_active" $OUT/ncu_cluster_${TAG}_keymetrics.csv | cut -d, -f2- | cut -c1-100
# the configs[3] / configs[2] kernels at HEAD: ncu of the batched train kernel (16k) and the inference kernel (1M),
# the batched kernel's per-CTA phase trace, the e2e call's host/device timeline
bash scripts/ncu_one.sh ncu_batch16k_$TAG train_batch_kernel python scripts/big_batch.py --what train --batch 16384 --n 32768 --reps 1 > /dev/null 2>&1
python scripts/ncu_lines.py $OUT/ncu_batch16k_$TAG.ncu-rep 40 > $OUT/ncu_batch16k_${TAG}_lines.txt 2>&1
bash scripts/ncu_one.sh ncu_infer1m_$TAG infer_kernel python scripts/big_batch.py --what eval --n 1048576 --reps 1 > /dev/null 2>&1
grep -E "time_duration|dram__bytes|fma_cycles|issue_active" $OUT/ncu_batch16k_${TAG}_keymetrics.csv $OUT/ncu_infer1m_${TAG}_keymetrics.csv | cut -c1-160
timeout 300 python scripts/trace_batch.py --batch 16384 --n 32768 > $OUT/trace_batch_16384_$TAG.json 2>&1
TLB_HOST_TRACE=1 timeout 300 python scripts/e2e_timeline.py --u8 --reps 4 > $OUT/e2e_timeline_$TAG.txt 2>&1
