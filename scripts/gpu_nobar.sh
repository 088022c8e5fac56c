#!/bin/bash
TAG=${1:-push}
OUT=gpurun_out; mkdir -p $OUT
V=paper_1912_05234_b200/lib/variants/libtloom_b200_nobar0.so
for r in 1 2; do
timeout 300 python bench.py --no-cpu-baseline --no-e2e > $OUT/bench_nobar1_${r}_$TAG.json 2>&1
TLB_LIB=$V timeout 300 python bench.py --no-cpu-baseline --no-e2e > $OUT/bench_nobar0_${r}_$TAG.json 2>&1
done
timeout 300 python scripts/trace_step.py --mode fast > $OUT/trace_nobar1_$TAG.json 2>&1
for f in nobar1_1 nobar0_1 nobar1_2 nobar0_2; do python -c "
import json; d=json.loads(open('$OUT/bench_${f}_$TAG.json').read().strip().splitlines()[-1]); print('$f', d['value'], d['ms_per_step'], d['parity']['epoch_loss_max_rel_vs_reference'])"; done
cat $OUT/trace_nobar1_$TAG.json
timeout 1200 python -u -m pytest tests -m gpu -x -q --timeout 400 > $OUT/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu_$TAG.log
TLB_BENCH_SAME_GPU=1 timeout 600 python bench.py --gpus 2 --batch 16 --n 800 --steps 3 --warmup 3 > $OUT/bench_same2_$TAG.json 2> $OUT/bench_same2_$TAG.err
tail -3 $OUT/pytest_gpu_$TAG.log; tail -c 400 $OUT/bench_same2_$TAG.json
