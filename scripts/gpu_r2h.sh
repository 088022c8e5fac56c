#!/bin/bash
# HEAD verification: GPU tests, smoke, bench (fast), reference arm, configs[3] 16k line.
TAG=${1:-r2h}
OUT=gpurun_out; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/nvsmi_$TAG.txt 2>&1
timeout 1200 python -u -m pytest tests -m gpu -x -q --timeout 400 > $OUT/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_$TAG.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke_$TAG.log
timeout 600 python bench.py > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $OUT/bench_ref_$TAG.json 2> $OUT/bench_ref_$TAG.err
timeout 600 python bench.py --batch 16384 --n 32768 --steps 5 --no-cpu-baseline > $OUT/bench16k_$TAG.json 2> $OUT/bench16k_$TAG.err
tail -3 $OUT/pytest_gpu_$TAG.log; tail -2 $OUT/smoke_$TAG.log
for f in bench bench_ref bench16k; do echo "== $f"; tail -c 600 $OUT/${f}_$TAG.json; tail -3 $OUT/${f}_$TAG.err; done
