set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -3
DBM_DGEMM_WAVESYNC=32 timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "dgemm or multiply" 2>&1 | tail -3
for bs in 64; do
  timeout 300 python tools/profile_multiply.py --M 8192 --N 8192 --K 8192 --bs 64 --path blocked --reps 3 2>&1 | tail -2
  timeout 300 python tools/profile_multiply.py --M 31680 --N 31680 --K 31680 --bs 64 --path blocked --reps 2 2>&1 | tail -2
done
for w in 0 16 32 64 128; do
  DBM_DGEMM_WAVESYNC=$w timeout 300 python tools/profile_dgemm.py --M 63360 --N 63360 --K 16896 --reps 3 2>&1 | tail -1
done
DBM_DGEMM_WAVESYNC=32 timeout 300 python tools/profile_dgemm.py --M 63360 --N 63360 --K 16896 --reps 2 > gpurun_out/r1_pd10.txt 2>&1 && \
DBM_DGEMM_WAVESYNC=32 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_op_read_hit_rate.pct --clock-control none -k regex:dgemm -s 1 -c 1 --csv python tools/profile_dgemm.py --M 63360 --N 63360 --K 16896 --reps 2 > gpurun_out/r1_ncu10.csv 2>&1
tail -8 gpurun_out/r1_ncu10.csv; cat gpurun_out/r1_pd10.txt
