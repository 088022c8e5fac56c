#!/bin/bash
OUT=gpurun_out; mkdir -p $OUT
timeout 300 python scripts/trace_step.py --mode fast > $OUT/trace_head.json 2>&1
(cd .ab_base && timeout 300 python scripts/trace_step.py --mode fast) > $OUT/trace_base.json 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:train_cluster -c 3 python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > $OUT/ncu_head.txt 2>&1
(cd .ab_base && timeout 300 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:train_cluster -c 3 python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline) > $OUT/ncu_base.txt 2>&1
grep -A3 "gpu__time\|inst_executed\|fma_cycles" $OUT/ncu_head.txt | grep -v "^--" | head -12; echo; grep "gpu__time\|inst_executed\|fma_cycles" $OUT/ncu_base.txt | head -12
