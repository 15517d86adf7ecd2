set -x
timeout 1800 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29531 tests/mp_worker.py > gpurun_out/r1_mp_worker4e.log 2>&1; echo "worker rc=$?"
grep -v '"ok": true, "bytes_ok": true' gpurun_out/r1_mp_worker4e.log | grep '^{' | head
grep -c '"ok": true, "bytes_ok": true' gpurun_out/r1_mp_worker4e.log
for c in sp22 sp64; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29541 bench.py --gpus 4 --config $c --steps 3 --warmup 3 --no-e2e > gpurun_out/r1_bench_${c}_n4.json 2> gpurun_out/r1_bench_${c}_n4.err
grep '^{' gpurun_out/r1_bench_${c}_n4.json | cut -c1-400
done
