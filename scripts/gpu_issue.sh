#!/bin/bash
TAG=${1:-iss}
OUT=gpurun_out; mkdir -p $OUT
V=paper_1912_05234_b200/lib/variants/libtloom_b200_issue0.so
for r in 1 2; do
python scripts/batch_check.py --time --batches 1024,4096,16384,262144 > $OUT/bt_iss1_${r}_$TAG.jsonl 2>&1
TLB_LIB=$V python scripts/batch_check.py --time --batches 1024,4096,16384,262144 > $OUT/bt_iss0_${r}_$TAG.jsonl 2>&1
done
for f in iss1_1 iss0_1 iss1_2 iss0_2; do echo "$f $(grep batched $OUT/bt_${f}_$TAG.jsonl | python -c "
import sys, json; print([ (json.loads(l)['batch'], round(json.loads(l)['images_per_s']/1e6, 2)) for l in sys.stdin])")"; done
for r in 1 2; do
python bench.py --batch 16384 --n 32768 --steps 5 --no-cpu-baseline 2>/dev/null | tail -1 > $OUT/b16_iss1_${r}_$TAG.json
TLB_LIB=$V python bench.py --batch 16384 --n 32768 --steps 5 --no-cpu-baseline 2>/dev/null | tail -1 > $OUT/b16_iss0_${r}_$TAG.json
done
for f in iss1_1 iss0_1 iss1_2 iss0_2; do python -c "
import json; d=json.loads(open('$OUT/b16_${f}_$TAG.json').read()); print('$f', round(d['value']/1e6,2), round(d['e2e']['value']/1e6,2))"; done
TLB_BT_ONLY=1 python scripts/batch_check.py --parity 2>&1 | cut -c1-200
