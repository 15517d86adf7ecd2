timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr=127.0.0.1 --master-port=29535 tests/mp_worker.py > gpurun_out/r1_mgpu4_final.out 2> gpurun_out/r1_mgpu4_final.err
echo rc=$?
grep -v '"ok": true' gpurun_out/r1_mgpu4_final.out | head -20
grep -c '"ok": true' gpurun_out/r1_mgpu4_final.out
tail -3 gpurun_out/r1_mgpu4_final.err
