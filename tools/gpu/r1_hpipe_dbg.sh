timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1 --master-port=29533 tests/mp_worker.py > gpurun_out/r1_hpipe_dbg.out 2> gpurun_out/r1_hpipe_dbg.err
echo rc=$?
grep -v '"ok": true' gpurun_out/r1_hpipe_dbg.out | head -30
tail -30 gpurun_out/r1_hpipe_dbg.err
