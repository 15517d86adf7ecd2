set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q 2>&1 | tail -2
rm -f gpurun_out/r1_dbuf.jsonl
for cfg in r22 r64; do
  timeout 900 python bench.py --config $cfg --path densified --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | grep '^{' >> gpurun_out/r1_dbuf.jsonl
done
python - <<'PY'
import json
for l in open('gpurun_out/r1_dbuf.jsonl'):
    d=json.loads(l); c=d['config']
    print(c['workload'][:34], round(d['value'],2), round(d['ms_per_step'],2), d['e2e']['value'], d['phases_ms_per_step'], d['clocks']['sm_mhz'])
PY
