"""Multi-GPU parity (2 GPUs -> 2x1x1; 4 GPUs -> the north star's 2x2x1 and the 1x2x2
sub-cube): runs tools/mp_parity.py under torchrun, one rank per GPU. Skipped when the
box has fewer GPUs."""
import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


@pytest.mark.parametrize("grid", ["2x1x1", "2x2x1", "1x2x2"])
def test_mp_parity(torch_cuda, grid):
    dims = [int(v) for v in grid.split("x")]
    n = dims[0] * dims[1] * dims[2]
    if torch_cuda.cuda.device_count() < n:
        pytest.skip(f"needs {n} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(29600 + n + dims[2]),
           str(ROOT / "tools" / "mp_parity.py"), grid]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600,
                       env={**os.environ, "PYTHONPATH": str(ROOT)})
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith(("PASS", "FAIL"))]
    assert r.returncode == 0 and lines and all(ln.startswith("PASS") for ln in lines), (
        r.stdout[-3000:] + r.stderr[-3000:])
