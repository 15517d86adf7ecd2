set -x
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29531 tests/mp_worker.py > gpurun_out/r1_mp_worker4d.log 2>&1; echo "worker rc=$?"
grep -v '"ok": true, "bytes_ok": true' gpurun_out/r1_mp_worker4d.log | grep '^{' | head
grep -c '"ok": true, "bytes_ok": true' gpurun_out/r1_mp_worker4d.log
for g in 2x2 1x4; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29541 bench.py --gpus 4 --config r64 --grid $g --algorithm tallskinny --steps 3 --warmup 3 --no-e2e
done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29542 bench.py --gpus 4 --config r22 --path blocked --steps 2 --warmup 3 --no-e2e
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29543 bench.py --gpus 2 --config r64 --algorithm tallskinny --steps 3 --warmup 3 --no-e2e
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29544 bench.py --gpus 4 --steps 2 --warmup 3
