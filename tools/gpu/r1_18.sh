set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sparse.py -x -q 2>&1 | tail -2
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 500 > gpurun_out/r1_bench18_clocks.csv &
CP=$!
timeout 1500 python bench.py > gpurun_out/r1_bench18_default.json 2> gpurun_out/r1_bench18_default.err
kill $CP
tail -2 gpurun_out/r1_bench18_default.err; grep '^{' gpurun_out/r1_bench18_default.json | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['e2e'], d['cpu_baseline'], d['clocks'], d['gpu_launches'])"
