#!/bin/bash
TAG=${1:-share2}
OUT=gpurun_out; mkdir -p $OUT
timeout 1500 python -u -m pytest tests/test_gpu_sanitizer.py tests/test_gpu_large.py -m gpu -x -q --timeout 900 > $OUT/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_$TAG.log
tail -3 $OUT/pytest_$TAG.log
timeout 300 python scripts/batch_check.py --time > $OUT/bt_time_$TAG.jsonl 2>&1; grep batched $OUT/bt_time_$TAG.jsonl | cut -c1-150
timeout 600 python bench.py --batch 16384 --n 32768 > $OUT/bench16k_$TAG.json 2>&1
python -c "
import json; d=json.loads(open('$OUT/bench16k_$TAG.json').read().strip().splitlines()[-1]); print(d['value'], d['e2e']['value'], d['roofline']['frac'], d.get('parity'))"
