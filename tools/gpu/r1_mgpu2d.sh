set -x
timeout 600 python -m pytest tests/test_gpu_sparse.py -x -q 2>&1 | tail -2
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29531 tests/mp_worker.py > gpurun_out/r1_mp_worker2d.log 2>&1
echo rc=$?
grep -c '"ok": true, "bytes_ok": true' gpurun_out/r1_mp_worker2d.log
grep -v '"ok": true, "bytes_ok": true' gpurun_out/r1_mp_worker2d.log | grep -v "^W1\|^\*\*\|^Setting\|^NCCL" | tail -20
timeout 900 python bench.py --config sp22 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r1_bench_sp22b.json 2> gpurun_out/r1_bench_sp22b.err; tail -2 gpurun_out/r1_bench_sp22b.err
