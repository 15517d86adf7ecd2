set -x
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29531 tests/mp_worker.py > gpurun_out/r1_mp_worker2.log 2>&1
grep -v '"ok": true, "bytes_ok": true' gpurun_out/r1_mp_worker2.log | tail -40
