set -x
timeout 900 python -m pytest tests/test_multigpu.py -x -q 2>&1 | tail -3
timeout 600 python -m pytest tests/test_multigpu.py -x -q -s 2>&1 | grep '"host"' | head -20
rm -f gpurun_out/r1_hpipe2.jsonl
run() { timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1 --master-port $2 bench.py --gpus $1 "${@:3}" 2>gpurun_out/r1_hpipe2_err_$2.log | grep '^{' >> gpurun_out/r1_hpipe2.jsonl; }
run 2 29551 --config sq64 --steps 2 --warmup 3
DBM_HOST_PIPE=0 run 2 29552 --config sq64 --steps 2 --warmup 3
python - <<'PY'
import json
for l in open('gpurun_out/r1_hpipe2.jsonl'):
    d=json.loads(l); c=d['config']
    print(c['grid'], round(d['value'],2), round(d['ms_per_step'],1), d['e2e']['value'], d['clocks'])
PY
