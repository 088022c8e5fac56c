#!/bin/bash
# channel-pair (FFMA2) batched kernel: parity vs oracle + timing A/B
TAG=${1:-p1}
OUT=gpurun_out; mkdir -p $OUT
for CFG in p4x640x1; do
  TLB_BT_ONLY=1 TLB_BATCH_CFG=$CFG timeout 300 python scripts/batch_check.py --parity >> $OUT/pair_parity_$TAG.jsonl 2>&1
done
for CFG in default p4x512x1 p4x640x1 p4x576x1 p3x384x1; do
  TLB_BT_ONLY=1 TLB_BATCH_CFG=$CFG timeout 300 python scripts/batch_check.py --time --batches 1024,16384,262144 >> $OUT/pair_time_$TAG.jsonl 2>&1
done
cat $OUT/pair_parity_$TAG.jsonl | cut -c1-330; cat $OUT/pair_time_$TAG.jsonl | cut -c1-200
