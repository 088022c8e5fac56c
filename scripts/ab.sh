# Same-box A/B of library variants: bench.py kernel value (no e2e / CPU baseline), interleaved.
# usage: bash scripts/ab.sh ROUNDS libA libB ...   (a lib of "-" = the in-tree default)
R=$1; shift
OUT=gpurun_out; mkdir -p $OUT
for r in $(seq 1 $R); do
  for L in "$@"; do
    if [ "$L" = "-" ]; then unset TLB_LIB; else export TLB_LIB=$L; fi
    v=$(timeout 300 python bench.py --mode ${AB_MODE:-fast} --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step'],4))")
    echo "$r $L $v" | tee -a $OUT/ab.log
  done
done
