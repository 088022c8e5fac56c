#!/bin/bash
# Same-box A/B of the batch-100 bench: HEAD vs the worktree in .ab_base (an older commit), alternating.
OUT=gpurun_out; mkdir -p $OUT
for i in 1 2 3; do
  timeout 300 python bench.py --no-e2e --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('head', d['value'], d['ms_per_step'])" >> $OUT/ab_base.txt 2>&1
  (cd .ab_base && timeout 300 python bench.py --no-e2e --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('base', d['value'], d['ms_per_step'])") >> $OUT/ab_base.txt 2>&1
done
cat $OUT/ab_base.txt
