#!/bin/bash
TAG=${1:-ilvb}
OUT=gpurun_out; mkdir -p $OUT
V=paper_1912_05234_b200/lib/variants/libtloom_b200_lossbase.so
for r in 1 2; do
python scripts/batch_check.py --time --batches 1024,2048,4096,16384 > $OUT/bt_ilv1_${r}_$TAG.jsonl 2>&1
TLB_LIB=$V python scripts/batch_check.py --time --batches 1024,2048,4096,16384 > $OUT/bt_ilv0_${r}_$TAG.jsonl 2>&1
done
for f in ilv1_1 ilv0_1 ilv1_2 ilv0_2; do echo "$f $(grep batched $OUT/bt_${f}_$TAG.jsonl | python -c "
import sys, json; print([ (json.loads(l)['batch'], round(json.loads(l)['images_per_s']/1e6, 2)) for l in sys.stdin])")"; done
