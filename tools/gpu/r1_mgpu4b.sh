set -x
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2
for shp in "1408 1408 1982464" "1408 704 991232" "704 704 495616" "704 384 495616" "704 320 495616"; do
set -- $shp
timeout 300 python tools/profile_dgemm.py --M $1 --N $2 --K $3 --reps 3 | tail -1
done
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29531 tests/mp_worker.py > gpurun_out/r1_mp_worker4b.log 2>&1; echo "worker rc=$?"
for cfg in sq64 r64; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29541 bench.py --gpus 4 --config $cfg --steps 2 --warmup 3 --no-e2e
done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29542 bench.py --gpus 4 --config r22 --path blocked --steps 2 --warmup 3 --no-e2e
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29543 bench.py --gpus 4 --config sq22 --path blocked --steps 1 --warmup 2 --no-e2e
for g in 1x4 4x1; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29544 bench.py --gpus 4 --config r64 --grid $g --steps 2 --warmup 3 --no-e2e
done
