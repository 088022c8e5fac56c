#!/bin/bash
TAG=${1:-trb}
OUT=gpurun_out; mkdir -p $OUT
for cfg in "16384 32768" "262144 524288"; do set -- $cfg
timeout 300 python scripts/trace_batch.py --batch $1 --n $2 > $OUT/trace_batch_${1}_$TAG.json 2>&1; echo "rc=$?"; cut -c1-300 $OUT/trace_batch_${1}_$TAG.json; done
