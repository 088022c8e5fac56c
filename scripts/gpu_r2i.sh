#!/bin/bash
# pageable (C++ drop-in) ingestion path + batched-kernel config A/B
TAG=${1:-r2i}
OUT=gpurun_out; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py -k "ingestion" tests/test_tools.py tests/test_gpu_acceptance.py -m gpu -x -q > $OUT/tests_$TAG.log 2>&1; echo "rc=$?" >> $OUT/tests_$TAG.log
timeout 600 python bench.py --no-cpu-baseline > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err
for T in 3 4 6; do TLB_INGEST_THREADS=$T timeout 300 paper_1912_05234_b200/bin/tloom-e2e-bench --steps 10 --warmup 3 > $OUT/cpp_e2e_t${T}_$TAG.json 2>&1; done
TLB_PAGEABLE_COPIES_FIRST=1 timeout 300 paper_1912_05234_b200/bin/tloom-e2e-bench --steps 10 --warmup 3 > $OUT/cpp_e2e_copiesfirst_$TAG.json 2>&1
for CFG in default 1x384x2 1x256x2 2x256x2 2x320x2 2x448x2; do
  echo "$CFG $(TLB_BATCH_CFG=$CFG timeout 300 python scripts/batch_check.py --time --batches 1024,16384 2>&1 | tr '\n' ' ')" >> $OUT/bt_ab_$TAG.txt
done
tail -3 $OUT/tests_$TAG.log; cat $OUT/bt_ab_$TAG.txt
for f in $OUT/cpp_e2e_*_$TAG.json; do echo "$f: $(cut -c1-400 $f)"; done
python -c "
import json; d=json.loads(open('$OUT/bench_$TAG.json').read().strip().splitlines()[-1]); print(d['value'], d['e2e']['value'], d.get('e2e_cpp'))"
