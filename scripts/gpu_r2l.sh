#!/bin/bash
# verification after the packed-pair forward: GPU tests, smoke, bench (batch 100 and 16k), sweep
TAG=${1:-r2l}
OUT=gpurun_out; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/nvsmi_$TAG.txt 2>&1
timeout 1200 python -u -m pytest tests -m gpu -x -q --timeout 400 > $OUT/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_$TAG.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke_$TAG.log
timeout 600 python bench.py > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err
timeout 600 python bench.py --batch 16384 --n 32768 --steps 5 --no-cpu-baseline > $OUT/bench16k_$TAG.json 2> $OUT/bench16k_$TAG.err
timeout 900 python scripts/sweep.py --out $OUT/sweep_$TAG.json > $OUT/sweep_$TAG.log 2>&1
tail -3 $OUT/pytest_gpu_$TAG.log; tail -2 $OUT/smoke_$TAG.log
for f in bench bench16k; do python -c "
import json; d=json.loads(open('$OUT/${f}_$TAG.json').read().strip().splitlines()[-1]); print('$f', d['value'], d['ms_per_step'], (d.get('e2e') or {}).get('value'), (d.get('e2e_cpp') or {}).get('value'), d['roofline']['frac'], d['roofline']['peak'])"; done
tail -12 $OUT/sweep_$TAG.log
