set -x
timeout 1800 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29531 tests/mp_worker.py > gpurun_out/r1_mp_worker4g.log 2>&1; echo "worker rc=$?"
grep -v '"ok": true, "bytes_ok": true' gpurun_out/r1_mp_worker4g.log | grep '^{' | head
grep -c '"ok": true, "bytes_ok": true' gpurun_out/r1_mp_worker4g.log
run() { timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1 --master-port $2 bench.py --gpus $1 "${@:3}" --steps 3 --warmup 3 --no-e2e 2>/dev/null | grep '^{' >> gpurun_out/r1_bench_n4g.jsonl; }
rm -f gpurun_out/r1_bench_n4g.jsonl
run 4 29541 --config r64 --algorithm tallskinny
run 4 29542 --config r64 --grid 1x4 --algorithm tallskinny
run 4 29543 --config r22 --algorithm tallskinny
run 2 29547 --config r64 --algorithm tallskinny
run 4 29548 --config r64
python - <<'PY'
import json
for l in open('gpurun_out/r1_bench_n4g.jsonl'):
    d=json.loads(l); c=d['config']
    print(c['workload'][:30], c['path'], c['grid'], c['algorithm'], round(d['value'],1), round(d['ms_per_step'],1), d['phases_ms_per_step'], d.get('exchange'))
PY
