set -x
timeout 300 python tools/profile_dgemm.py --M 63360 --N 63360 --K 15872 --reps 2 > /dev/null 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_op_read_hit_rate.pct --clock-control none -k regex:dgemm -s 1 -c 1 --csv python tools/profile_dgemm.py --M 63360 --N 63360 --K 15872 --reps 2 > gpurun_out/r1_ncu29_0.csv 2>&1
grep -E "dram__bytes|hit_rate|duration" gpurun_out/r1_ncu29_0.csv | awk -F'","' '{print $(NF-2), $NF}'
