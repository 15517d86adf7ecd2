set -x
timeout 900 python bench.py --config sq64 --path blocked --steps 1 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | grep '^{' > gpurun_out/r1_bench_sq64_blocked.json
python -c "
import json
d=json.loads(open('gpurun_out/r1_bench_sq64_blocked.json').read())
print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['phases_ms_per_step'])"
timeout 900 python bench.py --config r64 --path blocked --steps 3 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | grep '^{' > gpurun_out/r1_bench_r64_blocked.json
python -c "
import json
d=json.loads(open('gpurun_out/r1_bench_r64_blocked.json').read())
print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['phases_ms_per_step'])"
