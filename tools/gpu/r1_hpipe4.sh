set -x
timeout 900 python -m pytest tests/test_multigpu.py -x -q 2>&1 | tail -2
rm -f gpurun_out/r1_hpipe4.jsonl
run() { timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1 --master-port $2 bench.py --gpus $1 "${@:3}" 2>/dev/null | grep '^{' >> gpurun_out/r1_hpipe4.jsonl; }
run 4 29561 --config sq64 --steps 2 --warmup 3
DBM_HOST_PIPE=0 run 4 29562 --config sq64 --steps 2 --warmup 3
run 4 29563 --config r64 --steps 5 --warmup 3
run 4 29564 --config sq22 --steps 2 --warmup 3
python - <<'PY'
import json
for l in open('gpurun_out/r1_hpipe4.jsonl'):
    d=json.loads(l); c=d['config']
    print(c['workload'][:34], c['grid'], c.get('algorithm'), round(d['value'],2), round(d['ms_per_step'],1), d['e2e']['value'], d['clocks']['sm_mhz'], d['clocks']['reasons'])
PY
