# Same-box A/B of library variants on the large-batch training sweep (flat kernel, 256-thread CTAs).
# usage: bash scripts/ab_sweep.sh MAXBATCH libA libB ...   (a lib of "-" = the in-tree default)
MB=$1; shift
OUT=gpurun_out; mkdir -p $OUT
for L in "$@"; do
  if [ "$L" = "-" ]; then unset TLB_LIB; else export TLB_LIB=$L; fi
  timeout 600 python scripts/sweep.py --modes fast --max-batch $MB --out /tmp/sw.json > /dev/null 2>&1
  python -c "
import json
for l in open('/tmp/sw.json'):
    d=json.loads(l)
    if d['config']=='batch_sweep': print('$L', d['batch'], round(d['images_per_s']))" | tee -a $OUT/ab_sweep.log
done
