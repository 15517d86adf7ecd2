set -x
timeout 1500 python -m pytest tests/ -m gpu -x -q 2>&1 | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
rm -f gpurun_out/r1_final4.jsonl
run() { timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1 --master-port $2 bench.py --gpus $1 "${@:3}" 2>/dev/null | grep '^{' >> gpurun_out/r1_final4.jsonl; }
run 4 29571 --steps 2 --warmup 3
run 2 29572 --steps 2 --warmup 3
run 4 29573 --config sq22 --path blocked --steps 2 --warmup 3
python - <<'PY'
import json
for l in open('gpurun_out/r1_final4.jsonl'):
    d=json.loads(l); c=d['config']
    print(c['workload'][:34], c['grid'], c['path'], round(d['value'],2), round(d['ms_per_step'],1), d['e2e']['value'], d['roofline']['frac'], d['clocks']['sm_mhz'], d['clocks']['reasons'])
PY
