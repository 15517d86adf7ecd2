set -x
timeout 1800 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29531 tests/mp_worker.py > gpurun_out/r1_mp_worker4j.log 2>&1; echo "worker rc=$?"
grep -v '"ok": true, "bytes_ok": true' gpurun_out/r1_mp_worker4j.log | grep '^{' | head
grep -c '"ok": true, "bytes_ok": true' gpurun_out/r1_mp_worker4j.log
run() { timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1 --master-port $2 bench.py --gpus $1 "${@:3}" --steps 3 --warmup 3 --no-e2e 2>/dev/null | grep '^{' >> gpurun_out/r1_bench_n4j.jsonl; }
rm -f gpurun_out/r1_bench_n4j.jsonl
run 4 29541 --config r22 --path blocked
run 4 29542 --config r64 --path blocked
run 2 29543 --config r22 --path blocked
run 4 29544 --config r22 --path blocked --grid 1x4
python - <<'PY'
import json
for l in open('gpurun_out/r1_bench_n4j.jsonl'):
    d=json.loads(l); c=d['config']
    print(c['workload'][:30], c['path'], c['grid'], c['algorithm'], round(d['value'],1), round(d['ms_per_step'],1), d.get('exchange'))
PY
