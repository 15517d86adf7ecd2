"""The library's opt-in and measurement switches keep parity.

Every switch below is an environment variable the library reads once per process (DESIGN.md names the
measurement each one belongs to). The default tests never set them, so the code paths behind them would
otherwise go untested. Each variant re-runs a selection of the GPU parity tests in a fresh subprocess with
the switch set. Those tests compare the CUDA path against the host oracle: float inputs within 1e-12
normwise, integer inputs bit-exact.
"""
import os
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

# (switch, what it selects, test file, -k expression)
VARIANTS = [
    ("DBM_SP_BULK=0", "sparse bs 22 with the cp.async per-run kernel instead of TMA bulk staging",
     "tests/test_gpu_sparse.py", "multiply"),
    ("DBM_NU_KCAP=16", "non-uniform small-block kernel, entry groups of summed k <= 16",
     "tests/test_gpu_nonuniform.py", "multiply or product"),
    ("DBM_NU_KCAP=64", "non-uniform small-block kernel, entry groups of summed k <= 64",
     "tests/test_gpu_nonuniform.py", "multiply or product"),
    ("DBM_SMMQ=0", "padded small sizes on the per-run kernels instead of the R x R squares",
     "tests/test_gpu_parity.py", "smmq or small_block"),
    ("DBM_SMMQ=2", "R x R squares even when they do not fill the GPU",
     "tests/test_gpu_parity.py", "small_block or multiply_matches_oracle"),
    ("DBM_SMM_NO_RUN=1", "the FMA small-block kernels instead of the DMMA run kernels",
     "tests/test_gpu_parity.py", "small_block"),
    ("DBM_ZC_A=1", "zero-copy A (bs 64 blocks read through a TMA view)",
     "tests/test_gpu_parity.py", "multiply_matches_oracle or integer_bit_exact or k_chunking"),
    ("DBM_STACKGEN_DBUF=1", "double-buffered stack generation on a side stream",
     "tests/test_gpu_parity.py", "multiply_matches_oracle or smm22q or integer_bit_exact"),
    ("DBM_DGEMM_WAVESYNC=64", "the dgemm's fuzzy wave barrier (cooperative launch)",
     "tests/test_gpu_parity.py", "dgemm or multiply_matches_oracle or k_chunking"),
    ("DBM_SMM22Q_CENTRE=4", "the bs-22 square kernel's centre subtile on warp 4",
     "tests/test_gpu_parity.py", "smm22q or integer_bit_exact"),
    ("DBM_DENSIFY_B_ORDER=lj", "the vectorised B densify in column-major block order",
     "tests/test_gpu_parity.py", "densify or multiply_matches_oracle"),
]


@pytest.mark.parametrize("switch,what,path,kexpr", VARIANTS, ids=[v[0] for v in VARIANTS])
def test_switch_keeps_parity(switch, what, path, kexpr):
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    key, val = switch.split("=")
    env = dict(os.environ, **{key: val})
    r = subprocess.run([sys.executable, "-m", "pytest", path, "-q", "-x", "-m", "gpu", "-k", kexpr,
                        "-p", "no:cacheprovider"], env=env, cwd=ROOT, capture_output=True, text=True, timeout=1200)
    tail = (r.stdout[-4000:] + r.stderr[-2000:])
    assert r.returncode == 0, f"{switch} ({what}):\n{tail}"
    assert " passed" in r.stdout and " failed" not in r.stdout, f"{switch} ({what}):\n{tail}"
