#!/bin/bash
# Round-2: batch-100 A/B (cooperative vs plain cluster launch, repeated), N>1 plumbing on one GPU.
TAG=${1:-r2d}
OUT=gpurun_out
mkdir -p $OUT
for i in 1 2 3; do
  timeout 300 python bench.py --no-e2e --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('coop', d['value'], d['ms_per_step'])" >> $OUT/ab_$TAG.txt 2>&1
  TLB_CLUSTER_COOP=0 timeout 300 python bench.py --no-e2e --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('plain', d['value'], d['ms_per_step'])" >> $OUT/ab_$TAG.txt 2>&1
done
TLB_BENCH_SAME_GPU=1 timeout 600 python bench.py --gpus 2 --batch 16 --n 1600 --steps 3 --warmup 3 > $OUT/bench_same2_$TAG.json 2> $OUT/bench_same2_$TAG.err
TLB_BENCH_SAME_GPU=1 timeout 600 python bench.py --gpus 2 --batch 1024 --n 4096 --steps 3 --warmup 3 --no-cpu-baseline > $OUT/bench_same2big_$TAG.json 2> $OUT/bench_same2big_$TAG.err
cat $OUT/ab_$TAG.txt
for f in bench_same2 bench_same2big; do echo "== $f"; python -c "
import json,sys
try:
  d=json.loads(open('$OUT/${f}_$TAG.json').read().strip().splitlines()[-1])
  print({k:d.get(k) for k in ['value','n_gpus','ms_per_step','gpu_launches']}, 'e2e', (d.get('e2e') or {}).get('value'), 'cpu', (d.get('cpu_baseline') or {}).get('value'), (d.get('impl_config') or {}).get('dp_note'), d['roofline']['frac'], d['epoch_mean_loss'])
except Exception as e: print('ERR', e); print(open('$OUT/${f}_$TAG.err').read()[-1500:])
"; done
