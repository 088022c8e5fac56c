#!/bin/bash
# warp-group batched kernel: parity vs oracle + timing A/B against the default batched kernel
TAG=${1:-wg1}
OUT=gpurun_out; mkdir -p $OUT
for CFG in wg4x192 wg3x192 wg4x160 wg3x256; do
  TLB_BT_ONLY=1 TLB_BATCH_CFG=$CFG timeout 300 python scripts/batch_check.py --parity >> $OUT/wg_parity_$TAG.jsonl 2>&1
done
for CFG in default wg4x192 wg3x192 wg4x160 wg3x256; do
  TLB_BT_ONLY=1 TLB_BATCH_CFG=$CFG timeout 300 python scripts/batch_check.py --time --batches 1024,16384,262144 >> $OUT/wg_time_$TAG.jsonl 2>&1
done
cat $OUT/wg_parity_$TAG.jsonl; cat $OUT/wg_time_$TAG.jsonl | cut -c1-200
