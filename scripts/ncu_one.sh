#!/bin/bash
# ncu --set full of one kernel (regex $2) launched by a python command ($3...), report -> gpurun_out/$1.ncu-rep
# plus the key-metrics CSV and source-line hot spots.  Usage: bash scripts/ncu_one.sh TAG REGEX cmd...
TAG=$1; RX=$2; shift 2
OUT=gpurun_out
mkdir -p $OUT
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$RX -s 1 -c 1 -o $OUT/$TAG -f "$@" > $OUT/$TAG.log 2>&1
python scripts/ncu_keymetrics.py $OUT/$TAG.ncu-rep > $OUT/${TAG}_keymetrics.csv 2>&1
ncu -i $OUT/$TAG.ncu-rep --page source --csv > $OUT/${TAG}_source.csv 2>/dev/null
tail -3 $OUT/$TAG.log; cat $OUT/${TAG}_keymetrics.csv
