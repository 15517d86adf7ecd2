set -x
for rep in 1 2 3; do
for w in 0 64 256 1024; do
  DBM_DGEMM_WAVESYNC=$w timeout 300 python tools/profile_dgemm.py --M 63360 --N 63360 --K 15872 --reps 3 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w', round(d['ms'],2), round(d['tflops'],3))"
done
done
DBM_DGEMM_WAVESYNC=256 timeout 300 python tools/profile_dgemm.py --M 63360 --N 63360 --K 15872 --reps 2 > /dev/null 2>&1 && \
DBM_DGEMM_WAVESYNC=256 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_op_read_hit_rate.pct --clock-control none -k regex:dgemm -s 1 -c 1 --csv python tools/profile_dgemm.py --M 63360 --N 63360 --K 15872 --reps 2 > gpurun_out/r1_ncu28_256.csv 2>&1
grep -E "dram__bytes|hit_rate|duration" gpurun_out/r1_ncu28_256.csv | awk -F'","' '{print $(NF-2), $NF}'
