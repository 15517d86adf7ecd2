set -x
timeout 900 python -m pytest tests/test_gpu_sparse.py -x -q 2>&1 | tail -3
for occ in 0.1 0.5 1.0; do
  timeout 300 python tools/profile_multiply.py --M 11264 --N 11264 --K 11264 --bs 22 --path blocked --occ $occ --reps 3 2>&1 | tail -1
  timeout 300 python tools/profile_multiply.py --M 11264 --N 11264 --K 11264 --bs 64 --path blocked --occ $occ --reps 3 2>&1 | tail -1
done
timeout 300 python tools/profile_multiply.py --M 11264 --N 11264 --K 11264 --bs 22 --path blocked --occ 0.1 --reps 2 > gpurun_out/r1_sp14.txt 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:smm_sparse -s 1 -c 1 -o gpurun_out/r1_smm_sparse22b python tools/profile_multiply.py --M 11264 --N 11264 --K 11264 --bs 22 --path blocked --occ 0.1 --reps 2 > gpurun_out/r1_ncu14.log 2>&1
tail -2 gpurun_out/r1_ncu14.log
