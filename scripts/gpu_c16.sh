#!/bin/bash
TAG=${1:-c16}
OUT=gpurun_out; mkdir -p $OUT
V=paper_1912_05234_b200/lib/variants/libtloom_b200_c16.so
timeout 300 python bench.py --no-cpu-baseline --no-e2e > $OUT/bench_c8_$TAG.json 2>&1
TLB_LIB=$V timeout 300 python bench.py --no-cpu-baseline --no-e2e > $OUT/bench_c16_$TAG.json 2>&1
TLB_LIB=$V timeout 300 python scripts/trace_step.py --mode fast > $OUT/trace_c16_$TAG.json 2>&1
TLB_LIB=$V timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "fast or cluster" > $OUT/pytest_c16_$TAG.log 2>&1; echo "rc=$?" >> $OUT/pytest_c16_$TAG.log
for f in c8 c16; do python -c "
import json; d=json.loads(open('$OUT/bench_${f}_$TAG.json').read().strip().splitlines()[-1]); print('$f', d['value'], d['ms_per_step'], d['parity']['epoch_loss_max_rel_vs_reference'])" || tail -5 $OUT/bench_${f}_$TAG.json; done
cat $OUT/trace_c16_$TAG.json; tail -3 $OUT/pytest_c16_$TAG.log
