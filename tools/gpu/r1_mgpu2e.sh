set -x
timeout 300 python tools/microbench/ce_copy.py 2>&1 | tail -20
