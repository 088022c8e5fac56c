# e2e ingestion policy A/B on one box: pinned H2D bandwidth, then bench e2e with the default ramp vs
# fixed 2-group chunks (TLB_INGEST_CHUNK=200) vs geometric (0).
OUT=gpurun_out; mkdir -p $OUT
python scripts/h2d_probe.py > $OUT/h2d_probe.json 2>&1
for r in 1 2; do
  timeout 300 python bench.py --no-cpu-baseline > $OUT/e2e_ramp_$r.json 2>/dev/null
  TLB_INGEST_CHUNK=200 timeout 300 python bench.py --no-cpu-baseline > $OUT/e2e_fix2_$r.json 2>/dev/null
  TLB_INGEST_STREAMS=2 timeout 300 python bench.py --no-cpu-baseline > $OUT/e2e_str2_$r.json 2>/dev/null
done
cat $OUT/h2d_probe.json
for f in $OUT/e2e_*.json; do python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', round(d['value']), round(d['e2e']['value']), d['e2e']['call_ms']['median'], round(d['e2e']['h2d_GBps_measured'],1))"; done
