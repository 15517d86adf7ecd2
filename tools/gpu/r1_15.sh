set -x
for v in 0 1; do
  export DBM_SMM_SPARSE_V1=$v; [ $v = 0 ] && unset DBM_SMM_SPARSE_V1
  for occ in 0.1 0.5; do
    timeout 300 python tools/profile_multiply.py --M 11264 --N 11264 --K 11264 --bs 22 --path blocked --occ $occ --reps 3 2>&1 | tail -1
    timeout 300 python tools/profile_multiply.py --M 11264 --N 11264 --K 11264 --bs 64 --path blocked --occ $occ --reps 3 2>&1 | tail -1
  done
  timeout 300 python tools/profile_multiply.py --M 63360 --N 63360 --K 63360 --bs 22 --path blocked --occ 0.1 --reps 2 2>&1 | tail -1
  timeout 300 python tools/profile_multiply.py --M 63360 --N 63360 --K 63360 --bs 64 --path blocked --occ 0.1 --reps 2 2>&1 | tail -1
done
unset DBM_SMM_SPARSE_V1
timeout 300 python tools/smm_vs_batched.py --n 5632 --bs 22 2>&1 | tail -1
timeout 300 python tools/smm_vs_batched.py --n 8192 --bs 64 2>&1 | tail -1
timeout 300 python tools/profile_multiply.py --M 63360 --N 63360 --K 63360 --bs 22 --path blocked --occ 0.1 --reps 2 > gpurun_out/r1_sp15.txt 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_op_read_hit_rate.pct,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:smm_sparse -s 1 -c 3 --csv python tools/profile_multiply.py --M 63360 --N 63360 --K 63360 --bs 22 --path blocked --occ 0.1 --reps 2 > gpurun_out/r1_ncu15.csv 2>&1
grep -v "^==" gpurun_out/r1_ncu15.csv | tail -16
