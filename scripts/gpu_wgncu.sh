#!/bin/bash
TAG=${1:-wgn1}
OUT=gpurun_out; mkdir -p $OUT
TLB_BATCH_CFG=wg4x192 bash scripts/ncu_one.sh ncu_wg4x192_$TAG train_wg_kernel python scripts/big_batch.py --what train --batch 16384 --n 32768 --reps 1 > /dev/null 2>&1
python scripts/ncu_lines.py $OUT/ncu_wg4x192_$TAG.ncu-rep 45 > $OUT/ncu_wg4x192_${TAG}_lines.txt 2>&1
bash scripts/ncu_one.sh ncu_bt_$TAG train_batch_kernel python scripts/big_batch.py --what train --batch 16384 --n 32768 --reps 1 > /dev/null 2>&1
python scripts/ncu_lines.py $OUT/ncu_bt_$TAG.ncu-rep 45 > $OUT/ncu_bt_${TAG}_lines.txt 2>&1
paste -d, $OUT/ncu_wg4x192_${TAG}_keymetrics.csv $OUT/ncu_bt_${TAG}_keymetrics.csv | cut -c1-250
