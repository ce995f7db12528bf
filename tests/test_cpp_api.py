"""The C++ drop-in (include/cube3d_b200.hpp over c3d.h): a compiled C++ caller with the
reference's call shapes (tests/cpp/test_cube3d_b200.cpp), built with g++ against the
in-tree libc3d.so. CPU: the header and the caller compile. GPU: the caller runs and
every known answer passes."""
import shutil
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
CPP = ROOT / "tests" / "cpp"


def _make(*targets):
    return subprocess.run(["make", "-s", "-C", str(CPP), *targets], capture_output=True, text=True,
                          timeout=300)


@pytest.mark.skipif(shutil.which("g++") is None, reason="needs g++")
def test_cpp_dropin_header_compiles():
    r = _make("syntax")
    assert r.returncode == 0, r.stdout + r.stderr


@pytest.mark.gpu
def test_cpp_dropin_caller_runs(torch_cuda):
    r = _make()
    assert r.returncode == 0, r.stdout + r.stderr
    out = subprocess.run([str(ROOT / "build" / "test_cube3d_b200")], capture_output=True, text=True,
                         timeout=600)
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith(("PASS", "FAIL"))]
    assert out.returncode == 0 and len(lines) >= 10 and all(ln.startswith("PASS") for ln in lines), (
        out.stdout + out.stderr)
