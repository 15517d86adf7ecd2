set -x
timeout 300 python tools/profile_multiply.py --M 4094 --N 4094 --K 4094 --bs 23 --path blocked --reps 2 2>&1 | tail -1 || exit 1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:smm_sparse_run_kernel -c 1 -o gpurun_out/r1_ncu_smm_run23 -f python tools/profile_multiply.py --M 4094 --N 4094 --K 4094 --bs 23 --path blocked --reps 1 > gpurun_out/r1_ncu_smm_run23.log 2>&1
tail -3 gpurun_out/r1_ncu_smm_run23.log
