#!/bin/bash
TAG=${1:-pn1}
OUT=gpurun_out; mkdir -p $OUT
for V in 0 1; do build/stage_bench_pair$V 200 > $OUT/sb_pair${V}_$TAG.txt 2>&1; done
TLB_BATCH_CFG=p2x256x2 bash scripts/ncu_one.sh ncu_p2_$TAG train_batch_kernel python scripts/big_batch.py --what train --batch 16384 --n 32768 --reps 1 > /dev/null 2>&1
python scripts/ncu_lines.py $OUT/ncu_p2_$TAG.ncu-rep 50 > $OUT/ncu_p2_${TAG}_lines.txt 2>&1
grep -E '"fast"' $OUT/sb_pair0_$TAG.txt | grep -E '"conv1"|conv2_v2|forward_image|product|backward_v14'
echo; grep -E '"fast"' $OUT/sb_pair1_$TAG.txt | grep -E '"conv1"|conv2_v2|forward_image|product'
cat $OUT/ncu_p2_${TAG}_keymetrics.csv | cut -c1-160
