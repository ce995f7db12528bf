"""The reference's tooling surface: CUBE3D matrix files
(cube3d/matrix_io.hpp) and parameter checkpoints (transformer.hpp:259-293) pinned
byte-for-byte against the compiled reference (oracle/_ref), and the CLI
(tools/cube3d_main.cpp): `bench` reproduces the reference's modeled-cost table exactly
with --reference-traffic; `matmul` and `verify` run on the GPU."""
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

from oracle import cube3d_oracle as O
from oracle import ref
from paper_2105_14450_b200 import C3DError, cli, matrix_io as mio
from paper_2105_14450_b200 import cube3d as c3

ROOT = Path(__file__).resolve().parents[1]
needs_ref = pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built")


@pytest.mark.parametrize("kind", ["f32", "f64"])
def test_matrix_roundtrip_bit_exact(tmp_path, kind):
    m = np.random.default_rng(0).standard_normal((7, 5))
    m = m.astype(np.float32) if kind == "f32" else m
    p = tmp_path / "m.bin"
    mio.write_matrix(str(p), m, kind)
    back = mio.read_matrix(str(p))
    assert back.dtype == m.dtype and np.array_equal(back, m)
    assert mio.matrix_file_dtype(str(p)) == (1 if kind == "f32" else 0)


@needs_ref
@pytest.mark.parametrize("f32", [False, True])
def test_matrix_files_interchange_with_reference(tmp_path, f32):
    m = np.random.default_rng(1).standard_normal((9, 4))
    if f32:
        m = m.astype(np.float32).astype(np.float64)
    ref.write_matrix(tmp_path / "r.bin", m, f32=f32)
    mio.write_matrix(str(tmp_path / "o.bin"), m.astype(np.float32) if f32 else m)
    assert (tmp_path / "r.bin").read_bytes() == (tmp_path / "o.bin").read_bytes()
    assert np.array_equal(mio.read_matrix(str(tmp_path / "r.bin")).astype(np.float64), m)
    assert np.array_equal(ref.read_matrix(tmp_path / "o.bin", f32=f32), m)


def test_matrix_file_errors(tmp_path):
    bad = tmp_path / "bad.bin"
    bad.write_bytes(b"NOTCUBE" + bytes(20))
    for path, kw in ((bad, {}), (tmp_path / "missing.bin", {})):
        with pytest.raises(C3DError) as e:
            mio.read_matrix(str(path), **kw)
        assert e.value.name == "IoError"
    good = tmp_path / "g.bin"
    mio.write_matrix(str(good), np.ones((3, 3)))
    with pytest.raises(C3DError) as e:  # typed read of the other dtype
        mio.read_matrix(str(good), "f32")
    assert e.value.name == "IoError"
    good.write_bytes(good.read_bytes()[:-5])  # truncated payload
    with pytest.raises(C3DError) as e:
        mio.read_matrix(str(good))
    assert e.value.name == "IoError"


@needs_ref
def test_layer_checkpoints_interchange_with_reference(tmp_path):
    h = 16
    P = ref.init_layer_params(h, 3)
    gp = c3.GlobalLayerParams(**P)
    mio.save_layer_params(gp, str(tmp_path / "ours"))
    back = ref.load_layer_params(h, tmp_path / "ours")
    assert all(np.array_equal(back[f], P[f]) for f in O.FIELDS)
    ref.save_layer_params(P, h, tmp_path / "theirs")
    ours = mio.load_layer_params(str(tmp_path / "theirs"))
    assert all(np.array_equal(getattr(ours, f), P[f]) for f in O.FIELDS)
    for f in O.FIELDS:
        assert (tmp_path / f"ours.{f}.bin").read_bytes() == (tmp_path / f"theirs.{f}.bin").read_bytes()


@needs_ref
@pytest.mark.parametrize("mode,base,plist", [("weak", (2, 8, 2, 16), [1, 2]),
                                             ("weak", (2, 8, 2, 16), [1, 2, 4]),
                                             ("strong", (12, 36, 6, 144), [1, 2, 3])])
def test_cli_bench_reproduces_reference_table(tmp_path, capsys, mode, base, plist):
    b, s, n, h = base
    args = ["bench", "--mode", mode, "--p-list", ",".join(map(str, plist)), "--batch", str(b),
            "--seq", str(s), "--heads", str(n), "--hidden", str(h), "--reference-traffic"]
    assert cli.main(args) == 0
    got = capsys.readouterr().out
    assert got == ref.scaling_csv(mode == "weak", b, s, n, h, 1, plist)
    # this library's own traffic: the same forward, a cheaper backward
    assert cli.main(args[:-1] + ["--out", str(tmp_path / "t.csv")]) == 0
    ours = [ln.split(",") for ln in (tmp_path / "t.csv").read_text().splitlines()[1:]]
    theirs = [ln.split(",") for ln in got.splitlines()[1:]]
    for o, t in zip(ours, theirs):
        assert o[3] == t[3] and float(o[4]) <= float(t[4])


def test_cli_usage_errors_exit_2():
    assert cli.main(["bench", "--mode", "sideways"]) == 2
    assert cli.main(["nope"]) == 2
    # seq 8 on a 3-cube: ConfigInvalid, exit 2 (as the reference's bench, cube3d_main.cpp:51-58)
    assert cli.main(["bench", "--p-list", "1,3"]) == 2


@pytest.mark.gpu
def test_cli_matmul_and_verify(tmp_path, torch_cuda):
    r = np.random.default_rng(2)
    a = r.integers(0, 10, (128, 64)).astype(np.float64)
    b = r.integers(0, 10, (64, 192)).astype(np.float64)
    mio.write_matrix(str(tmp_path / "A.bin"), a)
    mio.write_matrix(str(tmp_path / "B.bin"), b)
    for extra in ([], ["--tc"]):
        rc = subprocess.run([sys.executable, "-m", "paper_2105_14450_b200.cli", "matmul", "--form",
                             "ab", "--a", str(tmp_path / "A.bin"), "--b", str(tmp_path / "B.bin"),
                             "--out", str(tmp_path / "C.bin"), *extra], cwd=ROOT,
                            capture_output=True, text=True, timeout=300)
        assert rc.returncode == 0, rc.stderr
        assert np.array_equal(mio.read_matrix(str(tmp_path / "C.bin")), a @ b)
    rc = subprocess.run([sys.executable, "-m", "paper_2105_14450_b200.cli", "verify"], cwd=ROOT,
                        capture_output=True, text=True, timeout=600)
    assert rc.returncode == 0 and "VERIFY PASS" in rc.stdout, rc.stdout + rc.stderr
