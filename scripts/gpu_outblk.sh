#!/bin/bash
TAG=${1:-ob}
OUT=gpurun_out; mkdir -p $OUT
TLB_HOST_TRACE=1 python scripts/e2e_timeline.py --u8 --reps 4 2>&1 | tail -3
timeout 2400 python -u -m pytest tests -m gpu -x -q --timeout 900 > $OUT/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu_$TAG.log
tail -3 $OUT/pytest_gpu_$TAG.log
for r in 1 2; do timeout 600 python bench.py > $OUT/bench_${r}_$TAG.json 2> $OUT/bench_${r}_$TAG.err
python -c "
import json; d=json.loads(open('$OUT/bench_${r}_$TAG.json').read().strip().splitlines()[-1]); print(d['value'], d['e2e']['value'], d['e2e_f32']['value'], d.get('e2e_cpp',{}).get('value'), d['parity']['epoch_loss_max_rel_vs_reference'], d['clocks'])"; done
