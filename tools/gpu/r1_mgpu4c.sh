set -x
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29531 tests/mp_worker.py > gpurun_out/r1_mp_worker4c.log 2>&1; echo "worker rc=$?"
grep -v '"ok": true, "bytes_ok": true' gpurun_out/r1_mp_worker4c.log | grep '^{' | head
for cfg in r64 sq64; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29541 bench.py --gpus 4 --config $cfg --steps 2 --warmup 3 --no-e2e
done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29542 bench.py --gpus 4 --config r22 --steps 2 --warmup 3 --no-e2e
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29543 bench.py --gpus 2 --config r64 --steps 2 --warmup 3 --no-e2e
