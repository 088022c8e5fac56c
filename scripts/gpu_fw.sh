#!/bin/bash
TAG=${1:-fw1}
OUT=gpurun_out; mkdir -p $OUT
for V in 0 1; do build/stage_bench_fw$V 200 > $OUT/sb_fw${V}_$TAG.txt 2>&1; done
timeout 1200 python -u -m pytest tests -m gpu -x -q --timeout 400 > $OUT/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_$TAG.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke_$TAG.log
timeout 600 python bench.py --no-cpu-baseline > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err
timeout 300 python scripts/trace_step.py --mode fast > $OUT/trace_fast_$TAG.json 2>&1
for V in 0 1; do echo "== fw$V"; grep -E '"fast"' $OUT/sb_fw${V}_$TAG.txt | grep -E '"conv1"|conv2_v2|forward_image|backward_product'; done
tail -3 $OUT/pytest_gpu_$TAG.log; tail -2 $OUT/smoke_$TAG.log
python -c "
import json; d=json.loads(open('$OUT/bench_$TAG.json').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['e2e']['value'], d['parity'], d['roofline']['frac'])"
cat $OUT/trace_fast_$TAG.json
