OUT=gpurun_out; mkdir -p $OUT
timeout 600 python -u -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "ingestion or train_fast or full_protocol" --timeout 300 > $OUT/pytest_ing.log 2>&1; echo "rc=$?" >> $OUT/pytest_ing.log
for r in 1 2 3; do
  timeout 300 python bench.py --no-cpu-baseline > $OUT/e2e_geo_$r.json 2>/dev/null
  TLB_INGEST_CHUNK=100 timeout 300 python bench.py --no-cpu-baseline > $OUT/e2e_fix_$r.json 2>/dev/null
done
tail -2 $OUT/pytest_ing.log
for f in $OUT/e2e_*.json; do python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', round(d['value']), round(d['e2e']['value']), d['e2e']['call_ms'])"; done
