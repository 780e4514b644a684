"""Multi-GPU parity: every factorisation of 2 and 4 GPUs against the oracle
(tests/mp_worker.py under torchrun, one process per GPU).  Skipped when the box
has fewer GPUs than the case needs."""
import os
import subprocess
import sys

import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.multigpu]
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("n", [2, 4])
def test_all_factorisations(n):
    import torch
    if torch.cuda.device_count() < n:
        pytest.skip(f"needs {n} GPUs, box has {torch.cuda.device_count()}")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={29600 + n}",
           os.path.join(ROOT, "tests", "mp_worker.py")]
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    out = p.stdout + p.stderr
    assert p.returncode == 0 and "MP_OK" in p.stdout, out[-4000:]


@pytest.mark.parametrize("n", [2, 4])
def test_full_size_sampled(n):
    """bench.py's launch configuration at full size (tests/mp_fullsize.py)."""
    import torch
    if torch.cuda.device_count() < n:
        pytest.skip(f"needs {n} GPUs, box has {torch.cuda.device_count()}")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={29640 + n}",
           os.path.join(ROOT, "tests", "mp_fullsize.py")]
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=1800, cwd=ROOT)
    assert p.returncode == 0 and "FULLSIZE_OK" in p.stdout, (p.stdout + p.stderr)[-4000:]
