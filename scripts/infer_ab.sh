#!/bin/bash
# A/B of the batched inference kernel configurations (TLB_INFER_CFG) at 1M images + prediction parity.
TAG=${1:-ab}
OUT=gpurun_out
mkdir -p $OUT
for cfg in default 8x512x2 4x256x3 4x192x4 8x384x1 16x384x1; do
  TLB_INFER_CFG=$cfg timeout 40 python scripts/big_batch.py --what eval --n 1000000 --reps 5 --check 2>&1 | tail -3 | sed "s/^/$cfg /" >> $OUT/infer_ab_$TAG.txt
done
TLB_FAST_THREADS=256 timeout 40 python scripts/big_batch.py --what eval --n 1000000 --reps 5 --check | sed "s/^/old_eval_kernel /" >> $OUT/infer_ab_$TAG.txt 2>&1
cat $OUT/infer_ab_$TAG.txt
