"""3-D matmul and vector ops on one B200 (the p=1 cube) against the reference's
golden outputs and the pinned oracle. Integer inputs are bit-exact in both the
fp32 SIMT mode and the bf16 tcgen05 mode (ints < 10 are exact in bf16, sums stay
below 2^24); real inputs meet the stated tolerances."""
import numpy as np
import pytest

from oracle import cube3d_oracle as O
from paper_2105_14450_b200 import C3DError, cube3d as c3

from helpers import TOL_BF16_REL, TOL_F32_NORM, bf16_round, golden, to_np

pytestmark = pytest.mark.gpu

FORM_LAYOUTS = {
    "AB": (c3.INPUT, c3.WEIGHT, c3.OUTPUT, None),
    "ABt": (c3.INPUT, c3.WEIGHT_OF_TRANSPOSE, c3.OUTPUT, None),
    "AtB": (c3.INPUT, c3.INPUT, c3.WEIGHT, c3.canonical_directions().swapped()),
}
FWD = {"AB": c3.matmul_ab_fwd, "ABt": c3.matmul_abt_fwd, "AtB": c3.matmul_atb_fwd}
BWD = {"AB": c3.matmul_ab_bwd, "ABt": c3.matmul_abt_bwd, "AtB": c3.matmul_atb_bwd}


@pytest.fixture(scope="module")
def cube(torch_cuda):
    c = c3.Cube((1, 1, 1), 0, 0)
    yield c
    c.close()


def run_form(cube, form, a, b, g, dtype, mode, out_dtype=c3.F32):
    la, lb, lg, bdirs = FORM_LAYOUTS[form]
    A = c3.shard_to_device(cube, a, la, dtype)
    B = c3.shard_to_device(cube, b, lb, dtype, bdirs)
    Gd = c3.shard_to_device(cube, g, lg, dtype)
    C = FWD[form](cube, A, B, mode, out_dtype)
    dA, dB = BWD[form](cube, Gd, A, B, mode, out_dtype)
    import torch
    torch.cuda.synchronize()
    return to_np(C.shard), to_np(dA.shard), to_np(dB.shard), C


@pytest.mark.parametrize("p", [1, 2])
@pytest.mark.parametrize("form", ["AB", "ABt", "AtB"])
@pytest.mark.parametrize("mode,dtype", [(c3.MODE_F32, c3.F32), (c3.MODE_TC, c3.BF16)])
def test_matmul_integer_golden_bitwise(cube, p, form, mode, dtype):
    d = golden("matmul")
    a, b, g = d[f"int_p{p}_a"], d[f"int_p{p}_b"], d[f"int_p{p}_g"]
    c, da, db, C = run_form(cube, form, a, b, g, dtype, mode)
    assert np.array_equal(c, d[f"int_p{p}_{form}_c"])
    assert np.array_equal(da, d[f"int_p{p}_{form}_da"])
    assert np.array_equal(db, d[f"int_p{p}_{form}_db"])
    # direction closure: Output carries the swapped triple (test_ops3d.cpp:195-229)
    if form != "AtB":
        assert C.dirs == c3.canonical_directions().swapped() and C.layout == c3.OUTPUT


def test_cfg1_matmul_1024(cube):
    """Config 1: C = AB, M=N=K=1024, fp32 mode within 1e-5 norm-wise of fp64; integer
    inputs bitwise in fp32 and bf16 tensor-core modes."""
    r = O.Rng(O.Rng(7).next_u64(1)[0])
    a = O.random_matrix(1024, 1024, r)
    b = O.random_matrix(1024, 1024, r)
    g = O.random_matrix(1024, 1024, r)
    c, da, db, _ = run_form(cube, "AB", a, b, g, c3.F32, c3.MODE_F32)
    assert O.normwise_err(c, a @ b) < TOL_F32_NORM
    assert O.normwise_err(da, g @ b.T) < TOL_F32_NORM
    assert O.normwise_err(db, a.T @ g) < TOL_F32_NORM
    ab, bb, gb = bf16_round(a), bf16_round(b), bf16_round(g)
    c, da, db, _ = run_form(cube, "AB", a, b, g, c3.BF16, c3.MODE_TC)
    assert O.rel_err(c, ab @ bb) < 1e-3
    assert O.normwise_err(c, a @ b) < TOL_BF16_REL  # vs unrounded inputs
    ai = O.random_integer_matrix(1024, 1024, r)
    bi = O.random_integer_matrix(1024, 1024, r)
    gi = O.random_integer_matrix(1024, 1024, r)
    for mode, dt in ((c3.MODE_F32, c3.F32), (c3.MODE_TC, c3.BF16)):
        c, da, db, _ = run_form(cube, "AB", ai, bi, gi, dt, mode)
        assert np.array_equal(c, ai @ bi)
        assert np.array_equal(da, gi @ bi.T)
        assert np.array_equal(db, ai.T @ gi)


def test_matmul_real_golden(cube):
    d = golden("matmul")
    a, b, g = d["real_a"], d["real_b"], d["real_g"]
    c, da, db, _ = run_form(cube, "AB", a, b, g, c3.F32, c3.MODE_F32)
    assert O.normwise_err(c, d["real_f64_c"]) < TOL_F32_NORM
    assert O.normwise_err(da, d["real_f64_da"]) < TOL_F32_NORM
    assert O.normwise_err(db, d["real_f64_db"]) < TOL_F32_NORM


def test_matmul_errors(cube):
    a = c3.shard_to_device(cube, np.zeros((8, 8)), c3.INPUT, c3.F32)
    bw = c3.shard_to_device(cube, np.zeros((8, 8)), c3.WEIGHT, c3.F32,
                            c3.canonical_directions().swapped())
    with pytest.raises(C3DError) as e:
        c3.matmul_ab_fwd(cube, a, bw)
    assert e.value.name == "DirectionClash"
    bi = c3.shard_to_device(cube, np.zeros((8, 8)), c3.INPUT, c3.F32)
    with pytest.raises(C3DError) as e:
        c3.matmul_ab_fwd(cube, a, bi)
    assert e.value.name == "ShapeMismatch"


@pytest.mark.parametrize("mul", [False, True])
def test_vector_ops(cube, mul):
    rng = np.random.default_rng(5)
    n = 64
    a = rng.uniform(-1, 1, (n, n))
    bvec = rng.uniform(-1, 1, n)
    g = rng.uniform(-1, 1, (n, n))
    A = c3.shard_to_device(cube, a, c3.INPUT, c3.F32)
    Bv = c3.vector_to_device(cube, bvec, c3.F32)
    Gd = c3.shard_to_device(cube, g, c3.INPUT, c3.F32)
    if mul:
        Cm = c3.mul_vec_fwd(cube, A, Bv)
        dA, db = c3.mul_vec_bwd(cube, Gd, A, Bv)
        want_c, want_da, want_db = a * bvec, g * bvec, (g * a).sum(0)
    else:
        Cm = c3.add_vec_fwd(cube, A, Bv)
        dA, db = c3.add_vec_bwd(cube, Gd)
        want_c, want_da, want_db = a + bvec, g, g.sum(0)
    assert O.rel_err(to_np(Cm.shard), want_c) < 1e-6
    assert O.rel_err(to_np(dA.shard), want_da) < 1e-6
    assert O.rel_err(to_np(db.shard), want_db) < 1e-5


@pytest.mark.parametrize("form", ["ab", "abt", "atb"])
def test_batched_matmuls_equal_the_loop(cube, form):
    """batched_matmul_*_fwd/bwd (cube3d/ops3d.hpp:418-494): each slice equals its
    unbatched product bitwise and the counters equal the looped accounting
    (tests/test_ops3d.cpp:506-537); differing extents raise BatchMismatch."""
    import torch
    F = {"ab": "AB", "abt": "ABt", "atb": "AtB"}[form]
    la, lb, lg, bdirs = FORM_LAYOUTS[F]
    r = O.Rng(13)
    M, N, K = 128, 64, 192
    slices = []
    for _ in range(3):
        a = O.random_integer_matrix(M, N, r)
        b = O.random_integer_matrix(*((N, K) if F == "AB" else (K, N) if F == "ABt" else (M, K)), r)
        g = O.random_integer_matrix(*((M, K) if F != "AtB" else (N, K)), r)
        slices.append((c3.shard_to_device(cube, a, la, c3.BF16),
                       c3.shard_to_device(cube, b, lb, c3.BF16, bdirs),
                       c3.shard_to_device(cube, g, lg, c3.BF16)))
    A, B, G = ([s[k] for s in slices] for k in range(3))
    cube.reset_counters()
    cs = c3.batched_matmul_fwd(form, cube, A, B, c3.MODE_TC, c3.F32)
    das, dbs = c3.batched_matmul_bwd(form, cube, G, A, B, c3.MODE_TC, c3.F32)
    torch.cuda.synchronize()
    batched = cube.counters()
    cube.reset_counters()
    for t in range(3):
        c = FWD[F](cube, A[t], B[t], c3.MODE_TC, c3.F32)
        da, db = BWD[F](cube, G[t], A[t], B[t], c3.MODE_TC, c3.F32)
        torch.cuda.synchronize()
        assert np.array_equal(to_np(cs[t].shard), to_np(c.shard))
        assert np.array_equal(to_np(das[t].shard), to_np(da.shard))
        assert np.array_equal(to_np(dbs[t].shard), to_np(db.shard))
    assert cube.counters() == batched
    with pytest.raises(C3DError) as e:
        c3.batched_matmul_fwd(form, cube, A, B[:2], c3.MODE_TC, c3.F32)
    assert e.value.name == "BatchMismatch"
