set -x
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k host 2>&1 | tail -2
timeout 1500 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 2 2>/dev/null | grep '^{' > gpurun_out/r1_bench35.json
python -c "
import json
d=json.loads(open('gpurun_out/r1_bench35.json').read())
print(d['value'], d['e2e'])"
