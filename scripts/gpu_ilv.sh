#!/bin/bash
# Interleaved round mapping in the batched kernel (+ sub-group ingestion chunks): device A/B vs the
# contiguous mapping (TLB_BT_INTERLEAVE=0 variant), e2e at 16k / 256k, parity, tests.
TAG=${1:-ilv}
OUT=gpurun_out; mkdir -p $OUT
V=paper_1912_05234_b200/lib/variants/libtloom_b200_ilv0.so
for r in 1 2; do
python scripts/batch_check.py --time --batches 1024,4096,16384,262144 > $OUT/bt_ilv1_${r}_$TAG.jsonl 2>&1
TLB_LIB=$V python scripts/batch_check.py --time --batches 1024,4096,16384,262144 > $OUT/bt_ilv0_${r}_$TAG.jsonl 2>&1
done
for f in ilv1_1 ilv0_1 ilv1_2 ilv0_2; do echo "$f $(grep batched $OUT/bt_${f}_$TAG.jsonl | python -c "
import sys, json; print([ (json.loads(l)['batch'], round(json.loads(l)['images_per_s']/1e6, 2)) for l in sys.stdin])")"; done
for r in 1 2; do python bench.py --batch 16384 --n 32768 --steps 5 --no-cpu-baseline 2>/dev/null | tail -1 > $OUT/b16_ilv_${r}_$TAG.json; python -c "
import json; d=json.loads(open('$OUT/b16_ilv_${r}_$TAG.json').read()); print('16k', round(d['value']/1e6,2), round(d['e2e']['value']/1e6,2), d['e2e']['call_ms'])"; done
python bench.py --batch 262144 --n 524288 --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 > $OUT/b256_ilv_$TAG.json; python -c "
import json; d=json.loads(open('$OUT/b256_ilv_$TAG.json').read()); print('256k', round(d['value']/1e6,2), round(d['e2e']['value']/1e6,2))"
TLB_BT_ONLY=1 python scripts/batch_check.py --parity 2>&1 | cut -c1-250
timeout 1800 python -m pytest tests/test_gpu_large.py tests/test_ingest_bytes.py tests/test_gpu_parity.py tests/test_gpu_sanitizer.py -m gpu -x -q --timeout 900 2>&1 | tail -2
