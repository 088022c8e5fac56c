#!/bin/bash
TAG=${1:-poll}
OUT=gpurun_out; mkdir -p $OUT
L=paper_1912_05234_b200/lib/variants
for r in 1 2 3; do
python bench.py --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 > $OUT/b_p32_${r}_$TAG.json
TLB_LIB=$L/libtloom_b200_poll0.so python bench.py --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 > $OUT/b_p0_${r}_$TAG.json
TLB_LIB=$L/libtloom_b200_poll8.so python bench.py --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 > $OUT/b_p8_${r}_$TAG.json
done
for f in p32_1 p0_1 p8_1 p32_2 p0_2 p8_2 p32_3 p0_3 p8_3; do python -c "
import json; d=json.loads(open('$OUT/b_${f}_$TAG.json').read()); print('$f', round(d['value']/1e6,3))"; done
