set -x
timeout 1800 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29531 tests/mp_worker.py > gpurun_out/r1_mp_worker4k.log 2>&1; echo "worker rc=$?"
grep '"host"' gpurun_out/r1_mp_worker4k.log | head -8
grep -c '"ok": true' gpurun_out/r1_mp_worker4k.log
run() { timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1 --master-port $2 bench.py --gpus $1 "${@:3}" --steps 3 --warmup 3 2>/dev/null | grep '^{' >> gpurun_out/r1_bench_n4k.jsonl; }
rm -f gpurun_out/r1_bench_n4k.jsonl
run 4 29541 --config sq64
run 2 29542 --config sq64
python - <<'PY'
import json
for l in open('gpurun_out/r1_bench_n4k.jsonl'):
    d=json.loads(l); c=d['config']
    print(c['workload'][:30], c['path'], c['grid'], round(d['value'],1), round(d['ms_per_step'],1), d['e2e'])
PY
