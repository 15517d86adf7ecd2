set -x
timeout 900 python bench.py --config sp22 --steps 3 --warmup 3 > gpurun_out/r1_bench_sp22.json 2> gpurun_out/r1_bench_sp22.err; tail -3 gpurun_out/r1_bench_sp22.err
cat gpurun_out/r1_bench_sp22.json
timeout 900 python bench.py --config sp64 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r1_bench_sp64.json 2> gpurun_out/r1_bench_sp64.err; tail -3 gpurun_out/r1_bench_sp64.err
cat gpurun_out/r1_bench_sp64.json
timeout 300 python tools/profile_multiply.py --M 11264 --N 11264 --K 11264 --bs 22 --path blocked --occ 0.1 --reps 2 > gpurun_out/r1_sp13.txt 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:smm_sparse -s 1 -c 1 -o gpurun_out/r1_smm_sparse22 python tools/profile_multiply.py --M 11264 --N 11264 --K 11264 --bs 22 --path blocked --occ 0.1 --reps 2 > gpurun_out/r1_ncu13.log 2>&1
tail -3 gpurun_out/r1_ncu13.log
