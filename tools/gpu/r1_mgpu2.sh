set -x
nvidia-smi topo -m | head -5
timeout 1500 python -m pytest tests/test_multigpu.py -x -q -s 2>&1 | tail -40
for tr in ce nccl; do
for cfg in sq64 r64; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29541 bench.py --gpus 2 --config $cfg --steps 2 --warmup 3 --no-e2e --transport $tr
done
done
