"""Standalone 3-D blocks on one B200 through the C ABI: c3d_linear_*, c3d_layernorm_*,
c3d_attention_*, c3d_mlp_* forward and backward against the dense oracle, and the
reference's edge-case known-answer tests (tests/test_nn_layers.cpp:117-160 linear
identity / zero input, :237-272 LayerNorm constant rows / gamma = 0, :295-331 zero Q/K
projections -> mean of V, :333-350 single key, :353-372 MLP zero input, :376-392 zero
blocks -> residual pass-through).

Gates: fp32 mode 1e-5 norm-wise (the reference's own KATs are exact where stated and
are kept exact here); bf16 tensor-core mode 2e-2 norm-wise vs fp64 on the same
bf16-rounded inputs plus 1e-2 vs the bf16-emulating oracle (helpers.check_bf16).
"""
import numpy as np
import pytest

from oracle import cube3d_oracle as O
from paper_2105_14450_b200 import cube3d as c3

from helpers import TOL_F32_NORM, bf16_round, check_bf16, oracle_params, to_np

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def cube(torch_cuda):
    c = c3.Cube((1, 1, 1), 0, 0)
    yield c
    c.close()


def sync():
    import torch
    torch.cuda.synchronize()


def linear_params(cube, w, b, dtype, group=0):
    W = c3.shard_to_device(cube, w, c3.WEIGHT, dtype, c3.triple_for_group(group))
    B = c3.vector_to_device(cube, b, c3.F32)
    return c3.LinearParams(W, B, group)


def gp_from(P, rnd=lambda a: a):
    return c3.GlobalLayerParams(**{f: rnd(np.asarray(getattr(P, f), dtype=np.float64))
                                   for f in O.FIELDS})


# ----------------------------------------------------------------- linear

def test_linear_identity_passes_through_bitwise(cube):
    """tests/test_nn_layers.cpp:117-137: identity weight, zero bias -> y == x, group toggles."""
    b, s, h = 2, 8, 16
    x = O.random_matrix(b * s, h, O.Rng(5))
    p = linear_params(cube, np.eye(h), np.zeros(h), c3.F32)
    X = c3.activation_to_device(cube, x, b, s, 0, c3.F32)
    gs = c3.GroupState(0)
    y, _ = c3.linear3d_fwd(cube, X, p, gs, c3.MODE_F32)
    sync()
    assert gs.input_group == 1 and y.group == 1
    assert np.array_equal(to_np(y.local), x.astype(np.float32).astype(np.float64))


def test_linear_zero_input_gives_bias(cube):
    """tests/test_nn_layers.cpp:139-160: zero input leaves the bias in every row."""
    b, s, h = 2, 8, 16
    r = O.Rng(7)
    w, bias = O.random_matrix(h, h, r), O.random_vector(h, r)
    p = linear_params(cube, w, bias, c3.F32)
    X = c3.activation_to_device(cube, np.zeros((b * s, h)), b, s, 0, c3.F32)
    y, _ = c3.linear3d_fwd(cube, X, p, c3.GroupState(0), c3.MODE_F32)
    sync()
    assert np.array_equal(to_np(y.local), np.tile(bias.astype(np.float32), (b * s, 1)))


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_linear_fwd_bwd_vs_dense(cube, dtype):
    """tests/test_nn_layers.cpp:162-196 (linear3d vs ref_linear_fwd/bwd), at a tcgen05 size."""
    b, s, h, o = 4, 128, 256, 512
    rnd = (lambda a: a) if dtype == "f32" else bf16_round
    dt, md = (c3.F32, c3.MODE_F32) if dtype == "f32" else (c3.BF16, c3.MODE_AUTO)
    r = O.Rng(11)
    w = rnd(O.random_matrix(h, o, r, -0.3, 0.3))
    bias = O.random_vector(o, r, -0.3, 0.3)
    x = rnd(O.random_matrix(b * s, h, r))
    gy = rnd(O.random_matrix(b * s, o, r))
    p = linear_params(cube, w, bias, dt)
    X = c3.activation_to_device(cube, x, b, s, 0, dt)
    GY = c3.activation_to_device(cube, gy, b, s, 1, dt)
    y, sv = c3.linear3d_fwd(cube, X, p, c3.GroupState(0), md)
    dx, dw, db = c3.linear3d_bwd(cube, GY, sv, p, md)
    sync()
    want = {"y": x @ w + bias, "dx": gy @ w.T, "dw": x.T @ gy, "db": gy.sum(axis=0)}
    got = {"y": to_np(y.local), "dx": to_np(dx.local), "dw": to_np(dw.shard), "db": to_np(db.shard)}
    assert dx.group == 0
    for k in want:
        if dtype == "f32":
            assert O.normwise_err(got[k], want[k]) < TOL_F32_NORM, k
        else:
            emul = {"y": rnd(want["y"]), "dx": rnd(want["dx"])}.get(k)
            check_bf16(got[k], want[k], k, emul)


# -------------------------------------------------------------- layernorm

@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_layernorm_fwd_bwd_vs_dense(cube, dtype):
    """tests/test_nn_layers.cpp:198-235."""
    b, s, h = 4, 64, 1024
    rnd = (lambda a: a) if dtype == "f32" else bf16_round
    dt = c3.F32 if dtype == "f32" else c3.BF16
    r = O.Rng(19)
    gamma, beta = O.random_vector(h, r, 0.5, 1.5), O.random_vector(h, r, -0.2, 0.2)
    x = rnd(O.random_matrix(b * s, h, O.Rng(23)))
    gy = rnd(O.random_matrix(b * s, h, O.Rng(29)))
    lp = c3.LayerNormParams(c3.vector_to_device(cube, gamma, c3.F32),
                            c3.vector_to_device(cube, beta, c3.F32))
    X = c3.activation_to_device(cube, x, b, s, 0, dt)
    GY = c3.activation_to_device(cube, gy, b, s, 0, dt)
    y, sv = c3.layernorm3d_fwd(cube, X, lp)
    dx, dg, dbt = c3.layernorm3d_bwd(cube, GY, sv)
    sync()
    yw, cache = O.layernorm_fwd(x, gamma, beta, 1e-5)
    dxw, dgw, dbw = O.layernorm_bwd(gy, cache)
    tol = TOL_F32_NORM if dtype == "f32" else 2e-2
    assert y.group == 0
    assert O.normwise_err(to_np(y.local), yw) < tol
    assert O.normwise_err(to_np(dx.local), dxw) < tol
    assert O.normwise_err(to_np(dg.shard), dgw) < tol
    assert O.normwise_err(to_np(dbt.shard), dbw) < tol


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_layernorm_trivial_rows(cube, dtype):
    """tests/test_nn_layers.cpp:237-272: constant rows -> exactly 0 (variance 0, eps floor);
    gamma = 0 -> exactly beta."""
    b, s, h = 2, 8, 16
    dt = c3.F32 if dtype == "f32" else c3.BF16
    x = np.repeat(np.arange(b * s, dtype=np.float64)[:, None], h, axis=1)
    one = c3.LayerNormParams(c3.vector_to_device(cube, np.ones(h), c3.F32),
                             c3.vector_to_device(cube, np.zeros(h), c3.F32))
    y, _ = c3.layernorm3d_fwd(cube, c3.activation_to_device(cube, x, b, s, 0, dt), one)
    sync()
    assert np.all(to_np(y.local) == 0.0)
    beta = O.random_vector(h, O.Rng(31))
    zero_g = c3.LayerNormParams(c3.vector_to_device(cube, np.zeros(h), c3.F32),
                                c3.vector_to_device(cube, beta, c3.F32))
    x2 = O.random_matrix(b * s, h, O.Rng(37))
    y2, _ = c3.layernorm3d_fwd(cube, c3.activation_to_device(cube, x2, b, s, 0, dt), zero_g)
    sync()
    want = beta.astype(np.float32) if dtype == "f32" else bf16_round(beta)
    assert np.array_equal(to_np(y2.local), np.tile(want, (b * s, 1)))


# -------------------------------------------------------------- attention

def run_attention(cube, gp, x, dy, b, s, n, h, dtype, mode):
    cfg = c3.TransformerConfig(b, s, n, h)
    params = c3.partition_layer_params(cube, gp, 0, dtype)
    X = c3.activation_to_device(cube, x, b, s, 0, dtype)
    DY = c3.activation_to_device(cube, dy, b, s, 0, dtype)
    gs = c3.GroupState(0)
    y, sv = c3.attention_fwd(cube, X, params, cfg, gs, mode)
    assert gs.input_group == 0  # two linears: the group is restored
    dx, g = c3.attention_bwd(cube, DY, sv, params, cfg, mode, grad_dtype=c3.F32)
    sync()
    grads = {f: to_np(getattr(g, f).shard) for f in ("w_qkv", "b_qkv", "w_out", "b_out")}
    return to_np(y.local), to_np(dx.local), grads


def attention_oracle(gp, x, dy, b, s, n, rnd=lambda a: a):
    P = oracle_params(gp)
    y, cache = O.attention_fwd(x, P, b, s, n, rnd)
    dx, dwq, dbq, dwo, dbo = O.attention_bwd(dy, cache, P, b, s, n, rnd)
    return y, dx, {"w_qkv": dwq, "b_qkv": dbq, "w_out": dwo, "b_out": dbo}


def test_attention_fp32_vs_dense_toy(cube):
    """tests/test_nn_layers.cpp:274-293 (toy config), fp32-exact mode."""
    b, s, n, h = 2, 8, 2, 16
    gp = gp_from(O.init_layer_params(h, 41))
    x = O.random_matrix(b * s, h, O.Rng(43))
    dy = O.random_matrix(b * s, h, O.Rng(44))
    y, dx, g = run_attention(cube, gp, x, dy, b, s, n, h, c3.F32, c3.MODE_F32)
    yw, dxw, gw = attention_oracle(gp, x, dy, b, s, n)
    assert O.normwise_err(y, yw) < TOL_F32_NORM
    assert O.normwise_err(dx, dxw) < TOL_F32_NORM
    for f in gw:
        assert O.normwise_err(g[f], gw[f].reshape(g[f].shape)) < TOL_F32_NORM, f


# (b, s, heads, hidden): head dim 64 and 128, sequence 128 .. 1024 (cfg4 has s = 1024,
# dh = 128), all on the flash tcgen05 kernels
FLASH_SHAPES = [(2, 128, 2, 128), (2, 256, 4, 256), (1, 512, 4, 256), (1, 1024, 2, 128),
                (2, 256, 2, 256), (1, 512, 2, 256), (1, 1024, 4, 512)]


@pytest.mark.parametrize("shape", FLASH_SHAPES)
def test_attention_bf16_flash_vs_oracle(cube, shape):
    b, s, n, h = shape
    gp = gp_from(O.init_layer_params(h, 7), bf16_round)
    r = O.Rng(9)
    x = bf16_round(O.random_matrix(b * s, h, r))
    dy = bf16_round(O.random_matrix(b * s, h, r))
    n0 = c3.launch_count()
    y, dx, g = run_attention(cube, gp, x, dy, b, s, n, h, c3.BF16, c3.MODE_AUTO)
    assert c3.launch_count() > n0
    yw, dxw, gw = attention_oracle(gp, x, dy, b, s, n)
    ye, dxe, ge = attention_oracle(gp, x, dy, b, s, n, bf16_round)
    check_bf16(y, yw, "y", ye)
    check_bf16(dx, dxw, "dx", dxe)
    for f in gw:
        check_bf16(g[f], gw[f].reshape(g[f].shape), f, ge[f].reshape(g[f].shape))


@pytest.mark.parametrize("shape", [(2, 256, 4, 256), (1, 512, 2, 256)])
def test_attention_flash_matches_unfused(cube, shape, monkeypatch):
    """The flash kernels (scores / probabilities never in HBM) against the unfused path
    (scores GEMM -> softmax kernel -> P V GEMM; dP GEMM -> softmax backward -> dQ, dK
    GEMMs) on the same bf16 inputs."""
    b, s, n, h = shape
    gp = gp_from(O.init_layer_params(h, 13), bf16_round)
    r = O.Rng(15)
    x = bf16_round(O.random_matrix(b * s, h, r))
    dy = bf16_round(O.random_matrix(b * s, h, r))
    flash = run_attention(cube, gp, x, dy, b, s, n, h, c3.BF16, c3.MODE_AUTO)
    monkeypatch.setenv("C3D_NO_FLASH", "1")
    monkeypatch.setenv("C3D_NO_FUSED_ATTN", "1")
    plain = run_attention(cube, gp, x, dy, b, s, n, h, c3.BF16, c3.MODE_AUTO)
    assert O.normwise_err(flash[0], plain[0]) < 5e-3
    assert O.normwise_err(flash[1], plain[1]) < 1e-2
    for f in flash[2]:
        assert O.normwise_err(flash[2][f], plain[2][f]) < 1e-2, f


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_attention_zero_qk_averages_values(cube, dtype):
    """tests/test_nn_layers.cpp:295-331: zeroed Q/K projections -> uniform weights 1/s,
    context = mean of the V rows of each batch item."""
    b, s, n, h = (2, 8, 2, 16) if dtype == "f32" else (2, 256, 2, 128)
    dt, md = (c3.F32, c3.MODE_F32) if dtype == "f32" else (c3.BF16, c3.MODE_AUTO)
    rnd = (lambda a: a) if dtype == "f32" else bf16_round
    P = O.init_layer_params(h, 47)
    dh = h // n
    for head in range(n):
        P.w_qkv[:, head * 3 * dh: head * 3 * dh + 2 * dh] = 0.0
        P.b_qkv[head * 3 * dh: head * 3 * dh + 2 * dh] = 0.0
    gp = gp_from(P, rnd)
    x = rnd(O.random_matrix(b * s, h, O.Rng(53)))
    cfg = c3.TransformerConfig(b, s, n, h)
    params = c3.partition_layer_params(cube, gp, 0, dt)
    y, _ = c3.attention_fwd(cube, c3.activation_to_device(cube, x, b, s, 0, dt), params, cfg,
                            c3.GroupState(0), md)
    sync()
    qkv = rnd(x @ gp.w_qkv + gp.b_qkv).reshape(b, s, n, 3, dh)
    ctx = np.repeat(qkv[:, :, :, 2].mean(axis=1, keepdims=True), s, axis=1).reshape(b * s, h)
    want = rnd(ctx) @ gp.w_out + gp.b_out
    tol = TOL_F32_NORM if dtype == "f32" else 1e-2
    assert O.normwise_err(to_np(y.local), want) < tol


def test_attention_single_key(cube):
    """tests/test_nn_layers.cpp:333-350: one key per softmax row (s = 1 on one rank):
    the probability is 1 and the attention reduces to the value path."""
    b, s, n, h = 4, 1, 2, 16
    gp = gp_from(O.init_layer_params(h, 59))
    x = O.random_matrix(b * s, h, O.Rng(61))
    dy = O.random_matrix(b * s, h, O.Rng(62))
    y, dx, g = run_attention(cube, gp, x, dy, b, s, n, h, c3.F32, c3.MODE_F32)
    yw, dxw, gw = attention_oracle(gp, x, dy, b, s, n)
    assert O.normwise_err(y, yw) < TOL_F32_NORM
    v = (x @ gp.w_qkv + gp.b_qkv).reshape(b * s, n, 3, h // n)[:, :, 2].reshape(b * s, h)
    assert O.normwise_err(y, v @ gp.w_out + gp.b_out) < TOL_F32_NORM
    assert O.normwise_err(dx, dxw) < TOL_F32_NORM


# -------------------------------------------------------------------- MLP

def mlp_oracle(gp, x, dy, rnd=lambda a: a):
    pre = x @ gp.w_fc1 + gp.b_fc1
    hact = rnd(O.gelu(pre))
    y = rnd(hact @ gp.w_fc2 + gp.b_fc2)
    dh = rnd((dy @ gp.w_fc2.T) * O.gelu_grad(rnd(pre)))
    return y, dh @ gp.w_fc1.T, {"w_fc1": x.T @ dh, "b_fc1": dh.sum(axis=0),
                                "w_fc2": hact.T @ dy, "b_fc2": dy.sum(axis=0)}


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_mlp_fwd_bwd_vs_dense(cube, dtype):
    """mlp_fwd/bwd (cube3d/transformer.hpp:44-70) against the dense composition."""
    b, s, n, h = 2, 128, 4, 256
    rnd = (lambda a: a) if dtype == "f32" else bf16_round
    dt, md = (c3.F32, c3.MODE_F32) if dtype == "f32" else (c3.BF16, c3.MODE_AUTO)
    gp = gp_from(O.init_layer_params(h, 71), rnd)
    x = rnd(O.random_matrix(b * s, h, O.Rng(73)))
    dy = rnd(O.random_matrix(b * s, h, O.Rng(79)))
    cfg = c3.TransformerConfig(b, s, n, h)
    params = c3.partition_layer_params(cube, gp, 0, dt)
    gs = c3.GroupState(0)
    y, sv = c3.mlp_fwd(cube, c3.activation_to_device(cube, x, b, s, 0, dt), params, cfg, gs, md)
    assert gs.input_group == 0
    dx, g = c3.mlp_bwd(cube, c3.activation_to_device(cube, dy, b, s, 0, dt), sv, params, cfg, md,
                       grad_dtype=c3.F32)
    sync()
    yw, dxw, gw = mlp_oracle(gp, x, dy)
    if dtype == "f32":
        assert O.normwise_err(to_np(y.local), yw) < TOL_F32_NORM
        assert O.normwise_err(to_np(dx.local), dxw) < TOL_F32_NORM
        for f in gw:
            got = to_np(getattr(g, f).shard)
            assert O.normwise_err(got, gw[f].reshape(got.shape)) < TOL_F32_NORM, f
    else:
        ye, dxe, ge = mlp_oracle(gp, x, dy, bf16_round)
        check_bf16(to_np(y.local), yw, "y", ye)
        check_bf16(to_np(dx.local), dxw, "dx", rnd(dxe))
        for f in gw:
            got = to_np(getattr(g, f).shard)
            check_bf16(got, gw[f].reshape(got.shape), f, ge[f].reshape(got.shape))


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_mlp_zero_input_zero_biases(cube, dtype):
    """tests/test_nn_layers.cpp:353-368: GELU(0) = 0, so the output is exactly zero."""
    b, s, n, h = (2, 8, 2, 16) if dtype == "f32" else (2, 128, 2, 256)
    dt, md = (c3.F32, c3.MODE_F32) if dtype == "f32" else (c3.BF16, c3.MODE_AUTO)
    P = O.init_layer_params(h, 59)
    P.b_fc1[:] = 0.0
    P.b_fc2[:] = 0.0
    params = c3.partition_layer_params(cube, gp_from(P), 0, dt)
    gs = c3.GroupState(0)
    y, _ = c3.mlp_fwd(cube, c3.activation_to_device(cube, np.zeros((b * s, h)), b, s, 0, dt),
                      params, c3.TransformerConfig(b, s, n, h), gs, md)
    sync()
    assert gs.input_group == 0
    assert np.all(to_np(y.local) == 0.0)


# ------------------------------------------------------------------ layer

@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_layer_zero_blocks_pass_residual(cube, dtype):
    """tests/test_nn_layers.cpp:376-392: zero weights and biases, unit LayerNorms ->
    y == x exactly, group restored."""
    b, s, n, h = (2, 8, 2, 16) if dtype == "f32" else (2, 256, 4, 256)
    dt, md = (c3.F32, c3.MODE_F32) if dtype == "f32" else (c3.BF16, c3.MODE_AUTO)
    rnd = (lambda a: a) if dtype == "f32" else bf16_round
    P = O.init_layer_params(h, 61)
    for f in ("w_qkv", "w_out", "w_fc1", "w_fc2", "b_qkv", "b_out", "b_fc1", "b_fc2"):
        getattr(P, f)[...] = 0.0
    P.ln1_gamma[:] = 1.0
    P.ln1_beta[:] = 0.0
    P.ln2_gamma[:] = 1.0
    P.ln2_beta[:] = 0.0
    x = rnd(O.random_matrix(b * s, h, O.Rng(67)))
    cfg = c3.TransformerConfig(b, s, n, h)
    params = c3.partition_layer_params(cube, gp_from(P), 0, dt)
    gs = c3.GroupState(0)
    y, _ = c3.transformer_layer_fwd(cube, c3.activation_to_device(cube, x, b, s, 0, dt), params,
                                    cfg, gs, md)
    sync()
    assert gs.input_group == 0
    want = x.astype(np.float32).astype(np.float64) if dtype == "f32" else x
    assert np.array_equal(to_np(y.local), want)
