#!/bin/bash
# A/B of the packed-pair (FFMA2) inference items against the scalar default at 1M images + prediction parity.
TAG=${1:-ipab}
OUT=gpurun_out
mkdir -p $OUT
for cfg in default 8x384x2; do
  TLB_INFER_CFG=$cfg timeout 60 python scripts/big_batch.py --what eval --n 1000000 --reps 5 --check 2>&1 | tail -1 | sed "s/^/$cfg /" >> $OUT/infer_pair_ab_$TAG.txt
done
cat $OUT/infer_pair_ab_$TAG.txt
