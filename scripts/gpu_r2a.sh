#!/bin/bash
# Round-2 baseline: FFMA peak, large-batch train/eval timings, ncu --set full of train_kernel<false>
# (batch 16k) and eval_kernel<false> (1M images), the bench line.
TAG=${1:-r2a}
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/nvsmi_$TAG.txt 2>&1
(nproc; lscpu | grep "Model name") > $OUT/host_$TAG.txt
./build/ffma_peak 4096 20 > $OUT/ffma_peak_$TAG.json 2>&1
for B in 1024 16384 262144; do N=$(( B*2 > 32768 ? B*2 : 32768 ));
  timeout 300 python scripts/big_batch.py --what train --batch $B --n $N >> $OUT/big_$TAG.jsonl 2>&1; done
timeout 300 python scripts/big_batch.py --what eval --n 1000000 >> $OUT/big_$TAG.jsonl 2>&1
timeout 600 python bench.py --no-cpu-baseline > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:train_kernel -s 1 -c 1 \
  -o $OUT/prof_train16k_$TAG -f python scripts/big_batch.py --what train --batch 16384 --n 32768 --reps 1 > $OUT/ncu_train16k_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:eval_kernel -s 1 -c 1 \
  -o $OUT/prof_eval1m_$TAG -f python scripts/big_batch.py --what eval --n 1000000 --reps 1 > $OUT/ncu_eval1m_$TAG.log 2>&1
cat $OUT/ffma_peak_$TAG.json $OUT/big_$TAG.jsonl; tail -c 600 $OUT/bench_$TAG.json; tail -2 $OUT/ncu_train16k_$TAG.log $OUT/ncu_eval1m_$TAG.log
