#!/bin/bash
TAG=${1:-gk1}
OUT=gpurun_out; mkdir -p $OUT
for V in 0 1; do build/stage_bench_gk$V 200 > $OUT/sb_gk${V}_$TAG.txt 2>&1; echo "== gk$V"; grep -E '"fast"' $OUT/sb_gk${V}_$TAG.txt | grep -E 'product|forward_image'; done
timeout 300 python scripts/trace_step.py --mode fast > $OUT/trace_fast_$TAG.json 2>&1
timeout 600 python bench.py --no-cpu-baseline --no-e2e > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err
python -c "
import json; d=json.loads(open('$OUT/bench_$TAG.json').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['parity'], d['roofline']['frac'])"
cat $OUT/trace_fast_$TAG.json
timeout 1200 python -u -m pytest tests -m gpu -x -q --timeout 400 > $OUT/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu_$TAG.log
tail -3 $OUT/pytest_gpu_$TAG.log
