set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sparse.py -x -q 2>&1 | tail -2
rm -f gpurun_out/r1_pitch.jsonl
for bs in 6 8 16 26 32; do
  n=$(( (4096 / bs) * bs ))
  timeout 300 python tools/profile_multiply.py --M $n --N $n --K $n --bs $bs --path blocked --reps 2 2>/dev/null | tail -1 | sed 's/^{/{"mode": "run-pitched", /' >> gpurun_out/r1_pitch.jsonl
done
python - <<'PY'
import json
for l in open('gpurun_out/r1_pitch.jsonl'):
    d=json.loads(l); print(d['mode'], d['bs'], d['M'], round(d['tflops'],2), {k: round(v,1) for k,v in d['phases_ms'].items() if v})
PY
