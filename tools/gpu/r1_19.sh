set -x
timeout 1200 python -m pytest tests -x -q -m "gpu and not multigpu" 2>&1 | tail -3
timeout 600 python tools/profile_multiply.py --M 1408 --N 1408 --K 1982464 --bs 64 --path blocked --reps 2 2>&1 | tail -1
timeout 600 python tools/profile_multiply.py --M 1408 --N 1408 --K 1982464 --bs 22 --path blocked --reps 2 2>&1 | tail -1
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
