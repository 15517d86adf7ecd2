timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1 --master-port=29534 tests/mp_worker.py > gpurun_out/r1_hpipe_blk.out 2> gpurun_out/r1_hpipe_blk.err
echo rc=$?
grep -v '"ok": true' gpurun_out/r1_hpipe_blk.out | head -20
grep '"host"' gpurun_out/r1_hpipe_blk.out | grep blocked | head -12
tail -5 gpurun_out/r1_hpipe_blk.err
rm -f gpurun_out/r1_hpipe_blk.jsonl
run() { timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1 --master-port $2 bench.py --gpus $1 "${@:3}" 2>/dev/null | grep '^{' >> gpurun_out/r1_hpipe_blk.jsonl; }
run 2 29581 --config sq22 --path blocked --steps 2 --warmup 3
DBM_HOST_PIPE=0 run 2 29582 --config sq22 --path blocked --steps 2 --warmup 3
python - <<'PY'
import json
for l in open('gpurun_out/r1_hpipe_blk.jsonl'):
    d=json.loads(l); c=d['config']
    print(c['workload'][:34], c['grid'], c['path'], round(d['value'],2), round(d['ms_per_step'],1), d['e2e']['value'])
PY
