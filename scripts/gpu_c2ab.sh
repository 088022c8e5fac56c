#!/bin/bash
TAG=${1:-c2k}
OUT=gpurun_out; mkdir -p $OUT
V=paper_1912_05234_b200/lib/variants/libtloom_b200_dprt.so
for r in 1 2 3; do
python bench.py --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 > $OUT/b_base_${r}_$TAG.json
TLB_LIB=$V python bench.py --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 > $OUT/b_direct_${r}_$TAG.json
done
for f in base_1 direct_1 base_2 direct_2 base_3 direct_3; do python -c "
import json; d=json.loads(open('$OUT/b_${f}_$TAG.json').read()); print('$f', round(d['value']/1e6,3), d['parity']['epoch_loss_max_rel_vs_reference'])"; done
