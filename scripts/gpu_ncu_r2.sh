#!/bin/bash
# ncu --set full of the three default fast kernels after the packed-pair change + the bench launch list
TAG=${1:-r2m}
OUT=gpurun_out; mkdir -p $OUT
bash scripts/ncu_one.sh ncu_cluster_$TAG train_cluster_kernel python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
python scripts/ncu_lines.py $OUT/ncu_cluster_$TAG.ncu-rep 40 > $OUT/ncu_cluster_${TAG}_lines.txt 2>&1
bash scripts/ncu_one.sh ncu_batch16k_$TAG train_batch_kernel python scripts/big_batch.py --what train --batch 16384 --n 32768 --reps 1 > /dev/null 2>&1
python scripts/ncu_lines.py $OUT/ncu_batch16k_$TAG.ncu-rep 40 > $OUT/ncu_batch16k_${TAG}_lines.txt 2>&1
bash scripts/ncu_one.sh ncu_infer1m_$TAG infer_kernel python scripts/big_batch.py --what eval --n 1000000 --reps 1 > /dev/null 2>&1
python scripts/ncu_lines.py $OUT/ncu_infer1m_$TAG.ncu-rep 40 > $OUT/ncu_infer1m_${TAG}_lines.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_$TAG.csv \
  python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $OUT/ncu_launch_$TAG.log 2>&1
for k in cluster batch16k infer1m; do echo "== $k"; grep -E "time_duration|dram__bytes|fma_cycles|issue_active|warps_active|bank_conflicts|wavefronts|stalled_barrier|stalled_short" $OUT/ncu_${k}_${TAG}_keymetrics.csv | cut -d, -f2- | cut -c1-120; done
