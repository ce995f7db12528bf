"""3-D cross-entropy head on one B200 against the oracle
(finite-difference-checked, tests/test_loss_oracle.py): fp32 mode within 1e-5
norm-wise, bf16 within 2e-2 on the same bf16-rounded inputs."""
import numpy as np
import pytest

from oracle import cube3d_oracle as O
from paper_2105_14450_b200 import cube3d as c3

from helpers import TOL_F32_NORM, bf16_round, to_np

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def cube(torch_cuda):
    c = c3.Cube((1, 1, 1), 0, 0)
    yield c
    c.close()


def run_loss(cube, x, w, b, t, batch, seq, dtype, mode):
    import torch
    dims = cube.dims
    X = c3.activation_to_device(cube, x, batch, seq, 0, dtype)
    d0 = c3.triple_for_group(0)
    W = c3.shard_to_device(cube, w, c3.WEIGHT, dtype, d0)
    B = c3.vector_to_device(cube, b, c3.F32)
    head = c3.LinearParams(W, B, 0)
    gs = c3.GroupState(0)
    loss, sv = c3.cross_entropy_fwd(cube, X, head, torch.tensor(t, dtype=torch.int32), gs, mode)
    dx, dw, db = c3.cross_entropy_bwd(cube, sv, head, mode)
    torch.cuda.synchronize()
    return (float(loss.item()), to_np(dx.local), to_np(dw.shard), to_np(db.shard))


@pytest.mark.parametrize("shape", [(2, 8, 16, 32), (4, 64, 128, 512)])
def test_cross_entropy_fp32(cube, shape):
    batch, seq, h, v = shape
    r = np.random.default_rng(11)
    x = r.uniform(-1, 1, (batch * seq, h))
    w = r.uniform(-0.5, 0.5, (h, v))
    b = r.uniform(-0.1, 0.1, v)
    t = r.integers(0, v, batch * seq)
    loss, dx, dw, db = run_loss(cube, x, w, b, t, batch, seq, c3.F32, c3.MODE_F32)
    lo, cache = O.cross_entropy_fwd(x, w, b, t)
    dxo, dwo, dbo = O.cross_entropy_bwd(cache)
    assert abs(loss - lo) / abs(lo) < TOL_F32_NORM
    assert O.normwise_err(dx, dxo) < TOL_F32_NORM
    assert O.normwise_err(dw, dwo) < TOL_F32_NORM
    assert O.normwise_err(db, dbo) < TOL_F32_NORM


def test_cross_entropy_bf16_tensor_cores(cube):
    batch, seq, h, v = 4, 128, 256, 1024
    r = np.random.default_rng(12)
    x = bf16_round(r.uniform(-1, 1, (batch * seq, h)))
    w = bf16_round(r.uniform(-0.2, 0.2, (h, v)))
    b = r.uniform(-0.1, 0.1, v)
    t = r.integers(0, v, batch * seq)
    loss, dx, dw, db = run_loss(cube, x, w, b, t, batch, seq, c3.BF16, c3.MODE_AUTO)
    lo, cache = O.cross_entropy_fwd(x, w, b, t)
    dxo, dwo, dbo = O.cross_entropy_bwd(cache)
    assert abs(loss - lo) / abs(lo) < 2e-3
    assert O.normwise_err(dx, dxo) < 2e-2
    assert O.normwise_err(dw, dwo) < 2e-2
    assert O.normwise_err(db, dbo) < 2e-2
