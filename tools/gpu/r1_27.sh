set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sparse.py -x -q 2>&1 | tail -2
timeout 600 python tools/profile_multiply.py --M 1408 --N 1408 --K 1982464 --bs 64 --path densified --reps 3 2>&1 | tail -1
timeout 600 python tools/profile_multiply.py --M 31680 --N 31680 --K 31680 --bs 64 --path densified --reps 2 2>&1 | tail -1
timeout 1200 python bench.py --steps 3 --warmup 3 > gpurun_out/r1_bench27.json 2>/dev/null
grep '^{' gpurun_out/r1_bench27.json | python -c "
import json,sys
for l in sys.stdin: d=json.loads(l); print('sq64', d['value'], d['ms_per_step'], d['roofline']['frac'], d['phases_ms_per_step'], d['e2e']['value'], d['cpu_baseline'], d['clocks'])"
