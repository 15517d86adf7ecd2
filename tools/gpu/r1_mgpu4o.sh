set -x
timeout 1800 python -m pytest tests/test_multigpu.py -x -q 2>&1 | tail -2
run() { timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1 --master-port $2 bench.py --gpus $1 "${@:3}" 2>/dev/null | grep '^{' >> gpurun_out/r1_bench_n4o.jsonl; }
rm -f gpurun_out/r1_bench_n4o.jsonl
run 4 29545 --config sq64 --steps 2 --warmup 3
run 2 29546 --config sq64 --steps 2 --warmup 3
python - <<'PY'
import json
for l in open('gpurun_out/r1_bench_n4o.jsonl'):
    d=json.loads(l); c=d['config']
    print(c['workload'][:30], c['grid'], round(d['value'],1), round(d['ms_per_step'],1), d['e2e']['value'], d['gpu_launches'], d['clocks'])
PY
