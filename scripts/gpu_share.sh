#!/bin/bash
# SM-pair mapping of the batched kernel: sweep the first CTA's share, trace, parity, tests.
TAG=${1:-share}
OUT=gpurun_out; mkdir -p $OUT
for S in 0 0.53 0.56; do
TLB_PAIR_SHARE=$S timeout 300 python scripts/trace_batch.py --batch 16384 --n 32768 > $OUT/trace_batch_16384_s${S}_$TAG.json 2>&1
python -c "
import json; d=json.loads(open('$OUT/trace_batch_16384_s${S}_$TAG.json').read().strip().splitlines()[-1]); print('share $S', d['coresidency'], d['epoch_ms'], [ (s['rounds_us_min_med_max'], s['idle_frac_before_barrier1']) for s in d['steps']])"
done
for S in 0 0.52 0.54 0.56 0.58 0.62; do
TLB_PAIR_SHARE=$S timeout 300 python scripts/batch_check.py --time --batches 16384,65536,262144 > $OUT/bt_time_s${S}_$TAG.jsonl 2>&1
echo "share $S: $(grep batched $OUT/bt_time_s${S}_$TAG.jsonl | python -c "
import sys, json; print([ (json.loads(l)['batch'], round(json.loads(l)['images_per_s']/1e6, 2)) for l in sys.stdin])")"
done
TLB_BT_ONLY=1 timeout 300 python scripts/batch_check.py --parity > $OUT/bt_parity_$TAG.jsonl 2>&1; echo "parity rc=$?"; cut -c1-330 $OUT/bt_parity_$TAG.jsonl
timeout 900 python -u -m pytest tests/test_ingest_bytes.py tests/test_gpu_parity.py -m gpu -x -q --timeout 400 > $OUT/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_$TAG.log
tail -3 $OUT/pytest_$TAG.log
