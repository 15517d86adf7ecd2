set -x
timeout 1500 python -m pytest tests/ -m gpu -x -q 2>&1 | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/r1_final_bench.json 2> gpurun_out/r1_final_bench.err; echo bench rc=$?
cat gpurun_out/r1_final_bench.json
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r1_final_ref.json 2>/dev/null; echo ref rc=$?
cat gpurun_out/r1_final_ref.json
