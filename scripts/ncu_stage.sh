# ncu --set full of selected fast stage-bench kernels; exports raw metrics + source-line stalls on the box.
# usage: bash scripts/ncu_stage.sh TAG 'regex of (int) stage ids, e.g. 0|2|4'
TAG=$1; IDS=$2; OUT=gpurun_out; mkdir -p $OUT
timeout 800 ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
  -k "regex:stage_kernel<\(bool\)0, \(int\)($IDS)>" -o /tmp/stage_$TAG ./paper_1912_05234_b200/_build/stage_bench ${ITERS:-200} > $OUT/ncu_stage_$TAG.log 2>&1
ncu -i /tmp/stage_$TAG.ncu-rep --page raw --csv > $OUT/ncu_stage_${TAG}_raw.csv 2>&1
for id in $(echo $IDS | tr '|' ' '); do
  ncu -i /tmp/stage_$TAG.ncu-rep --kernel-name-base demangled -k "regex:\(int\)$id>" --page source --csv --print-source sass,cuda \
    > $OUT/ncu_stage_${TAG}_src_$id.csv 2>&1
done
gzip -f $OUT/ncu_stage_${TAG}_src_*.csv
ls -la $OUT | grep ncu_stage_$TAG
