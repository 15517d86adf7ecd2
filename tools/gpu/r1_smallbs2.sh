set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -k "small_block" tests/test_gpu_sparse.py -x -q 2>&1 | tail -3
rm -f gpurun_out/r1_smallbs2.jsonl
for bs in 26 32; do
  for n0 in 4096 8192; do
    n=$(( (n0 / bs) * bs ))
    timeout 300 python tools/profile_multiply.py --M $n --N $n --K $n --bs $bs --path blocked --reps 2 2>/dev/null | tail -1 | sed 's/^{/{"mode": "run-team2", /' >> gpurun_out/r1_smallbs2.jsonl
  done
done
timeout 300 python tools/profile_multiply.py --M 11264 --N 11264 --K 11264 --bs 22 --path blocked --occ 0.5 --reps 2 2>/dev/null | tail -1 | sed 's/^{/{"mode": "sp22-perm", /' >> gpurun_out/r1_smallbs2.jsonl
timeout 300 python tools/profile_multiply.py --M 63360 --N 63360 --K 63360 --bs 22 --path blocked --occ 0.1 --reps 2 2>/dev/null | tail -1 | sed 's/^{/{"mode": "sp22-perm", /' >> gpurun_out/r1_smallbs2.jsonl
python - <<'PY'
import json
for l in open('gpurun_out/r1_smallbs2.jsonl'):
    d=json.loads(l); print(d['mode'], d['bs'], d['M'], d['occ'], round(d['tflops'],2), {k: round(v,1) for k,v in d['phases_ms'].items() if v})
PY
timeout 600 python bench.py --config sp22 --steps 3 --warmup 3 2>/dev/null | grep '^{' > gpurun_out/r1_bench_sp22_perm.json
python -c "import json; d=json.load(open('gpurun_out/r1_bench_sp22_perm.json')); print(d['value'], d['roofline'], d['e2e']['value'])"
