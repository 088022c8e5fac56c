#!/bin/bash
# Batched train kernel: config A/B timings + one ncu --set full capture (batch 16k) with source hot spots.
TAG=${1:-bt1}
OUT=gpurun_out
mkdir -p $OUT
timeout 300 python scripts/batch_check.py --parity > $OUT/bt_parity_$TAG.jsonl 2>&1
for CFG in default 2x512x1 3x384x1 4x512x1 4x768x1; do
  TLB_BATCH_CFG=$CFG timeout 300 python scripts/batch_check.py --time --batches 16384 2>&1 | head -1 >> $OUT/bt_ab_$TAG.jsonl
done
bash scripts/ncu_one.sh ncu_bt16k_$TAG train_batch_kernel python scripts/big_batch.py --what train --batch 16384 --n 32768 --reps 1 > /dev/null 2>&1
python scripts/ncu_lines.py $OUT/ncu_bt16k_${TAG}.ncu-rep 40 > $OUT/ncu_bt16k_${TAG}_srctop.txt 2>&1
cat $OUT/bt_parity_$TAG.jsonl $OUT/bt_ab_$TAG.jsonl; cat $OUT/ncu_bt16k_${TAG}_keymetrics.csv; head -60 $OUT/ncu_bt16k_${TAG}_srctop.txt
