"""Multi-GPU parity (NCCL over NVLink): torchrun tests/mp_worker.py on every visible GPU (2, 4 or 8),
all grid factorisations, both local paths, against the oracle (each case under a watchdog, so a hang
fails in minutes).  Skipped with fewer than 2 GPUs."""
import os
import subprocess
import sys

import pytest
import torch

pytestmark = [pytest.mark.gpu, pytest.mark.multigpu]
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_multirank_parity():
    n = torch.cuda.device_count() if torch.cuda.is_available() else 0
    if n < 2:
        pytest.skip("needs >= 2 GPUs")
    n = min(n, 8)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", "--master-port=29531", os.path.join(ROOT, "tests", "mp_worker.py"),
           "--groups", "cannon,sparse,host,nonuni"]  # (the host-pipeline sweep: tools/gpu/multigpu_check.sh)
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=2400, cwd=ROOT)
    print(r.stdout[-4000:])
    print(r.stderr[-4000:])
    assert r.returncode == 0
