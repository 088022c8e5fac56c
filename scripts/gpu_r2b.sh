#!/bin/bash
# Round-2 verification of HEAD: GPU tests, smoke, bench (ours + reference arm), large-batch timings.
TAG=${1:-r2b}
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/nvsmi_$TAG.txt 2>&1
(nproc; lscpu | grep "Model name") > $OUT/host_$TAG.txt
timeout 900 python -u -m pytest tests -m gpu -x -q --timeout 300 > $OUT/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_$TAG.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke_$TAG.log
timeout 600 python bench.py > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $OUT/bench_ref_$TAG.json 2> $OUT/bench_ref_$TAG.err
for B in 1024 16384 262144; do N=$(( B*2 > 32768 ? B*2 : 32768 ));
  timeout 300 python scripts/big_batch.py --what train --batch $B --n $N >> $OUT/big_$TAG.jsonl 2>&1; done
timeout 300 python scripts/big_batch.py --what eval --n 1000000 >> $OUT/big_$TAG.jsonl 2>&1
tail -3 $OUT/pytest_gpu_$TAG.log; tail -2 $OUT/smoke_$TAG.log; cat $OUT/big_$TAG.jsonl; tail -c 400 $OUT/bench_$TAG.json; tail -c 300 $OUT/bench_ref_$TAG.json
