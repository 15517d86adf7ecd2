set -x
timeout 1800 python -m pytest tests/test_multigpu.py -x -q 2>&1 | tail -2
run() { timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1 --master-port $2 bench.py --gpus $1 "${@:3}" 2>/dev/null | grep '^{' >> gpurun_out/r1_bench_n4n.jsonl; }
rm -f gpurun_out/r1_bench_n4n.jsonl
run 4 29541 --config r64 --steps 3 --warmup 3 --no-e2e
run 2 29543 --config r64 --steps 3 --warmup 3 --no-e2e
run 4 29544 --config r22 --path blocked --steps 3 --warmup 3 --no-e2e
run 4 29545 --config sq64 --steps 2 --warmup 3
python - <<'PY'
import json
for l in open('gpurun_out/r1_bench_n4n.jsonl'):
    d=json.loads(l); c=d['config']
    print(c['workload'][:30], c['path'], c['grid'], c['algorithm'], round(d['value'],1), round(d['ms_per_step'],1), (d.get('e2e') or {}).get('value'), d['phases_ms_per_step'], (d.get('exchange') or {}).get('uncovered_ms_per_step'))
PY
