rm -f gpurun_out/r1_final_cfgs.jsonl
for a in "--config sp22" "--config sp64" "--config sq22 --path blocked" "--config r22 --path blocked" "--config r64 --path blocked"; do
  timeout 900 python bench.py $a --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | grep '^{' >> gpurun_out/r1_final_cfgs.jsonl
done
python - <<'PY'
import json
for l in open('gpurun_out/r1_final_cfgs.jsonl'):
    d=json.loads(l); c=d['config']
    print(c['workload'][:40], c['path'], round(d['value'],2), round(d['ms_per_step'],1), d['e2e']['value'], d['roofline']['frac'], d['roofline']['kernel'], d['clocks']['sm_mhz'])
PY
