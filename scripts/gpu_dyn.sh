#!/bin/bash
# A/B: batched kernel with rounds claimed dynamically (TLB_BT_DYN=1 variant) vs static per-CTA chunks.
TAG=${1:-dyn}
OUT=gpurun_out; mkdir -p $OUT
V=paper_1912_05234_b200/lib/variants/libtloom_b200_btdyn.so
TLB_LIB=$V TLB_BT_ONLY=1 timeout 300 python scripts/batch_check.py --parity > $OUT/bt_parity_dyn_$TAG.jsonl 2>&1; echo "dyn parity rc=$?"
cat $OUT/bt_parity_dyn_$TAG.jsonl | cut -c1-300
for r in 1 2; do
timeout 300 python scripts/batch_check.py --time > $OUT/bt_time_base_${r}_$TAG.jsonl 2>&1
TLB_LIB=$V timeout 300 python scripts/batch_check.py --time > $OUT/bt_time_dyn_${r}_$TAG.jsonl 2>&1
done
for f in base_1 dyn_1 base_2 dyn_2; do echo "== $f"; grep -v "^$" $OUT/bt_time_${f}_$TAG.jsonl | cut -c1-200; done
TLB_LIB=$V timeout 600 python bench.py --batch 16384 --n 32768 --no-cpu-baseline > $OUT/bench16k_dyn_$TAG.json 2>&1
timeout 600 python bench.py --batch 16384 --n 32768 --no-cpu-baseline > $OUT/bench16k_base_$TAG.json 2>&1
for f in dyn base; do python -c "
import json; d=json.loads(open('$OUT/bench16k_${f}_$TAG.json').read().strip().splitlines()[-1]); print('$f', d['value'], d['e2e']['value'], d.get('parity'))"; done
TLB_LIB=$V timeout 900 python -u -m pytest tests/test_ingest_bytes.py tests/test_gpu_parity.py -m gpu -x -q --timeout 400 > $OUT/pytest_dyn_$TAG.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_dyn_$TAG.log
tail -3 $OUT/pytest_dyn_$TAG.log
