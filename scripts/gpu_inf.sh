#!/bin/bash
# A/B: batched inference with rounds claimed from a counter vs static per-CTA chunks (TLB_INFER_STATIC=1).
TAG=${1:-inf}
OUT=gpurun_out; mkdir -p $OUT
for r in 1 2; do
TLB_INFER_STATIC=1 timeout 300 python scripts/big_batch.py --what eval --n 1048576 --check > $OUT/inf_static_${r}_$TAG.json 2>&1
timeout 300 python scripts/big_batch.py --what eval --n 1048576 --check > $OUT/inf_dyn_${r}_$TAG.json 2>&1
done
for f in static_1 dyn_1 static_2 dyn_2; do echo "$f $(tail -1 $OUT/inf_${f}_$TAG.json | cut -c1-300)"; done
timeout 1500 python -u -m pytest tests/test_gpu_sanitizer.py tests/test_gpu_large.py tests/test_gpu_parity.py -m gpu -x -q --timeout 900 > $OUT/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_$TAG.log
tail -3 $OUT/pytest_$TAG.log
