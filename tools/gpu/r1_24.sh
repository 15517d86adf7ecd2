set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2
timeout 600 python tools/profile_multiply.py --M 5632 --N 5632 --K 5632 --bs 22 --path blocked --reps 3 2>&1 | tail -1
timeout 600 python tools/profile_multiply.py --M 15840 --N 15840 --K 15840 --bs 22 --path blocked --reps 2 2>&1 | tail -1
timeout 900 python bench.py --config sq22 --path blocked --steps 1 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | grep '^{' > gpurun_out/r1_bench_sq22_blocked.json
python -c "
import json
d=json.loads(open('gpurun_out/r1_bench_sq22_blocked.json').read())
print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['phases_ms_per_step'], d['clocks'])"
