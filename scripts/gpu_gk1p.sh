#!/bin/bash
TAG=${1:-gk1p}
OUT=gpurun_out; mkdir -p $OUT
for V in 0 1; do build/stage_bench_gk1p$V 200 > $OUT/sb_gk1p${V}_$TAG.txt 2>&1; echo "== gk1p$V"; grep -E '"fast"' $OUT/sb_gk1p${V}_$TAG.txt | grep -E 'product|forward_image'; done
V=paper_1912_05234_b200/lib/variants/libtloom_b200_gk1p0.so
for r in 1 2; do
timeout 300 python bench.py --no-cpu-baseline --no-e2e > $OUT/bench_gk1p1_${r}_$TAG.json 2>&1
TLB_LIB=$V timeout 300 python bench.py --no-cpu-baseline --no-e2e > $OUT/bench_gk1p0_${r}_$TAG.json 2>&1
done
for f in gk1p1_1 gk1p0_1 gk1p1_2 gk1p0_2; do python -c "
import json; d=json.loads(open('$OUT/bench_${f}_$TAG.json').read().strip().splitlines()[-1]); print('$f', d['value'], d['ms_per_step'], d['parity']['epoch_loss_max_rel_vs_reference'])"; done
timeout 1200 python -u -m pytest tests -m gpu -x -q --timeout 400 > $OUT/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu_$TAG.log
tail -3 $OUT/pytest_gpu_$TAG.log
