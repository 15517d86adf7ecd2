set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -k "small_block or matches_oracle or integer" tests/test_gpu_sparse.py -x -q 2>&1 | tail -3
rm -f gpurun_out/r1_smallbs.jsonl
for bs in 4 5 6 8 9 13 16 23 26 32; do
  n=$(( (4096 / bs) * bs ))
  for mode in run fma; do
    if [ $mode = fma ]; then export DBM_SMM_NO_RUN=1; else unset DBM_SMM_NO_RUN; fi
    timeout 300 python tools/profile_multiply.py --M $n --N $n --K $n --bs $bs --path blocked --reps 2 2>/dev/null | tail -1 | sed "s/^{/{\"mode\": \"$mode\", /" >> gpurun_out/r1_smallbs.jsonl
  done
done
unset DBM_SMM_NO_RUN
for bs in 13 23 32; do
  n=$(( (8192 / bs) * bs ))
  timeout 300 python tools/profile_multiply.py --M $n --N $n --K $n --bs $bs --path blocked --reps 2 2>/dev/null | tail -1 | sed 's/^{/{"mode": "run", /' >> gpurun_out/r1_smallbs.jsonl
  timeout 300 python tools/profile_multiply.py --M $n --N $n --K $n --bs $bs --path blocked --reps 2 --occ 0.3 2>/dev/null | tail -1 | sed 's/^{/{"mode": "run-sparse", /' >> gpurun_out/r1_smallbs.jsonl
done
python - <<'PY'
import json
for l in open('gpurun_out/r1_smallbs.jsonl'):
    d=json.loads(l); print(d['mode'], d['bs'], d['M'], d['occ'], round(d['tflops'],2), {k: round(v,1) for k,v in d['phases_ms'].items() if v})
PY
