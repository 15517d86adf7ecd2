set -x
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29531 tests/mp_worker.py > gpurun_out/r1_mp_worker2c.log 2>&1
echo rc=$?
grep -c '"ok": true, "bytes_ok": true' gpurun_out/r1_mp_worker2c.log
grep -v '"ok": true, "bytes_ok": true' gpurun_out/r1_mp_worker2c.log | tail -30
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29532 bench.py --gpus 2 --config sp22 --steps 3 --warmup 3 > gpurun_out/r1_bench_sp22_n2.json 2> gpurun_out/r1_bench_sp22_n2.err
tail -3 gpurun_out/r1_bench_sp22_n2.err; cat gpurun_out/r1_bench_sp22_n2.json | cut -c1-600
