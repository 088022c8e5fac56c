#!/bin/bash
TAG=${1:-r2e}
OUT=gpurun_out; mkdir -p $OUT
timeout 600 python -m pytest tests/test_ingest_bytes.py tests/test_gpu_large.py -m gpu -x -q > $OUT/tests_$TAG.log 2>&1; echo "rc=$?" >> $OUT/tests_$TAG.log
timeout 600 python bench.py > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err
timeout 600 python bench.py --batch 16384 --n 32768 --steps 5 > $OUT/bench16k_$TAG.json 2> $OUT/bench16k_$TAG.err
TLB_BENCH_SAME_GPU=1 timeout 600 python bench.py --gpus 2 --batch 16 --n 800 --steps 3 --warmup 3 > $OUT/bench_same2_$TAG.json 2> $OUT/bench_same2_$TAG.err
TLB_BENCH_SAME_GPU=1 timeout 600 python bench.py --gpus 2 --batch 1024 --n 4096 --steps 3 --warmup 3 --no-cpu-baseline > $OUT/bench_same2big_$TAG.json 2> $OUT/bench_same2big_$TAG.err
tail -3 $OUT/tests_$TAG.log
for f in bench bench16k bench_same2 bench_same2big; do echo "== $f"; python -c "
import json,sys
try:
  d=json.loads(open('$OUT/${f}_$TAG.json').read().strip().splitlines()[-1])
  print({k:d.get(k) for k in ['value','n_gpus','ms_per_step','gpu_launches']}, 'e2e', (d.get('e2e') or {}).get('value'), 'e2e_f32', (d.get('e2e_f32') or {}).get('value'), 'cpu', (d.get('cpu_baseline') or {}).get('value'), (d.get('impl_config') or {}).get('dp_note'), d['roofline']['frac'])
except Exception as e: print('ERR', e); print(open('$OUT/${f}_$TAG.err').read()[-1500:])
"; done
