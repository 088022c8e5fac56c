#!/bin/bash
# A/B: first ingestion chunk enqueued before the kernel launch (default) vs after (TLB_FIRST_CHUNK_AHEAD=0).
TAG=${1:-ahead}
OUT=gpurun_out; mkdir -p $OUT
for r in 1 2 3; do
python bench.py --no-cpu-baseline 2>/dev/null | tail -1 > $OUT/b_ahead1_${r}_$TAG.json
TLB_FIRST_CHUNK_AHEAD=0 python bench.py --no-cpu-baseline 2>/dev/null | tail -1 > $OUT/b_ahead0_${r}_$TAG.json
done
for f in ahead1_1 ahead0_1 ahead1_2 ahead0_2 ahead1_3 ahead0_3; do python -c "
import json; d=json.loads(open('$OUT/b_${f}_$TAG.json').read()); print('$f', round(d['value']/1e6,3), round(d['e2e']['value']/1e6,3), round(d['e2e_f32']['value']/1e6,3), round(d['e2e_cpp']['value']/1e6,3), d['e2e']['call_ms']['median'])"; done
TLB_HOST_TRACE=1 python scripts/e2e_timeline.py --u8 --reps 4 2>&1 | grep "host us" | tail -2
python -m pytest tests/test_gpu_parity.py tests/test_ingest_bytes.py tests/test_tools.py -m gpu -q -x 2>&1 | tail -1
