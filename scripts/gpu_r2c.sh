#!/bin/bash
# Round-2: shard-layout tests, bench at N=1 (default + batch 16k), the N>1 plumbing on one GPU
# (TLB_BENCH_SAME_GPU, 2 ranks, gloo + CUDA IPC) and --force-dp at N=1.
TAG=${1:-r2c}
OUT=gpurun_out
mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_large.py -m gpu -x -q > $OUT/large_$TAG.log 2>&1; echo "rc=$?" >> $OUT/large_$TAG.log
timeout 600 python bench.py > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err
timeout 600 python bench.py --batch 16384 --n 32768 --steps 5 > $OUT/bench16k_$TAG.json 2> $OUT/bench16k_$TAG.err
timeout 600 python bench.py --force-dp --no-cpu-baseline > $OUT/bench_dp1_$TAG.json 2> $OUT/bench_dp1_$TAG.err
timeout 600 python bench.py --force-dp --dp-mode nccl --no-cpu-baseline > $OUT/bench_dp1nccl_$TAG.json 2> $OUT/bench_dp1nccl_$TAG.err
TLB_BENCH_SAME_GPU=1 timeout 600 python bench.py --gpus 2 --batch 16 --n 1600 --steps 3 --warmup 3 > $OUT/bench_same2_$TAG.json 2> $OUT/bench_same2_$TAG.err
TLB_BENCH_SAME_GPU=1 timeout 600 python bench.py --gpus 2 --batch 1024 --n 4096 --steps 3 --warmup 3 --no-cpu-baseline > $OUT/bench_same2big_$TAG.json 2> $OUT/bench_same2big_$TAG.err
tail -3 $OUT/large_$TAG.log
for f in bench bench16k bench_dp1 bench_dp1nccl bench_same2 bench_same2big; do echo "== $f"; python -c "
import json,sys
try:
  d=json.loads(open('$OUT/${f}_$TAG.json').read().strip().splitlines()[-1])
  print({k:d.get(k) for k in ['value','n_gpus','ms_per_step','gpu_launches']}, 'e2e', (d.get('e2e') or {}).get('value'), 'cpu', (d.get('cpu_baseline') or {}).get('value'), (d.get('impl_config') or {}).get('dp_note'), d['roofline']['frac'])
except Exception as e: print('ERR', e); print(open('$OUT/${f}_$TAG.err').read()[-1500:])
"; done
