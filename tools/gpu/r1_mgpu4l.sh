set -x
timeout 1800 python -m pytest tests/test_multigpu.py -x -q 2>&1 | tail -2
run() { timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1 --master-port $2 bench.py --gpus $1 "${@:3}" 2>/dev/null | grep '^{' >> gpurun_out/r1_bench_n4l.jsonl; }
rm -f gpurun_out/r1_bench_n4l.jsonl
run 4 29541 --config sq22 --path blocked --steps 2 --warmup 3 --no-e2e
run 4 29542 --config r22 --path blocked --steps 3 --warmup 3 --no-e2e
run 4 29543 --config sq22 --steps 2 --warmup 3 --no-e2e
run 2 29544 --config sq22 --path blocked --steps 1 --warmup 3 --no-e2e
python - <<'PY'
import json
for l in open('gpurun_out/r1_bench_n4l.jsonl'):
    d=json.loads(l); c=d['config']
    print(c['workload'][:30], c['path'], c['grid'], c['algorithm'], round(d['value'],1), round(d['ms_per_step'],1), (d.get('exchange') or {}).get('uncovered_ms_per_step'))
PY
