"""tcgen05 GEMM (csrc/gemm_tc.cu) against a plain PyTorch fp32 reference of the same op.

Covers the four operand majors (K-major / MN-major for A and B), ragged shapes
(TMA out-of-bounds fill + masked epilogue), batching over two batch dims, split
operands (gathered column blocks / row blocks), and the fused epilogue. Integer
inputs are exact in bf16 and in fp32 accumulation, so those compare bitwise.
"""
import pytest

from paper_2105_14450_b200 import cube3d as c3

pytestmark = pytest.mark.gpu


def _store(torch, X, mn_major):
    # X: [batch][R][K] logical; return storage tensor and view dict
    B, R, K = X.shape
    if mn_major:
        st = X.transpose(1, 2).contiguous()  # [B][K][R]
        return st, dict(base=st.data_ptr(), dtype=c3.BF16, sr=1, sc=R, sb_lo=R * K, b_lo_n=B)
    st = X.contiguous()
    return st, dict(base=st.data_ptr(), dtype=c3.BF16, sr=K, sc=1, sb_lo=R * K, b_lo_n=B)


def _run(torch, M, N, K, a_mn, b_mn, batch=1, integer=False, mode=c3.MODE_TC, out_dtype=None,
         bias=False, act=0, alpha=1.0):
    g = torch.Generator(device="cuda").manual_seed(M * 7 + N * 13 + K)
    if integer:
        A = torch.randint(0, 10, (batch, M, K), device="cuda", generator=g).to(torch.bfloat16)
        Bm = torch.randint(0, 10, (batch, N, K), device="cuda", generator=g).to(torch.bfloat16)
    else:
        A = torch.rand((batch, M, K), device="cuda", generator=g).mul(2).sub(1).to(torch.bfloat16)
        Bm = torch.rand((batch, N, K), device="cuda", generator=g).mul(2).sub(1).to(torch.bfloat16)
    sa, va = _store(torch, A, a_mn)
    sb, vb = _store(torch, Bm, b_mn)
    odt = torch.float32 if out_dtype is None else out_dtype
    Cm = torch.full((batch, M, N), float("nan"), device="cuda", dtype=odt)
    vo = dict(base=Cm.data_ptr(), dtype=c3.F32 if odt == torch.float32 else c3.BF16, sr=N, sc=1,
              sb_lo=M * N, b_lo_n=batch)
    bvec = torch.rand(N, device="cuda", generator=g) if bias else None
    c3.gemm(M, N, K, va, vb, vo, alpha=alpha, bias=bvec.data_ptr() if bias else None, act=act,
            mode=mode, batch=batch)
    torch.cuda.synchronize()
    ref = torch.einsum("bmk,bnk->bmn", A.float(), Bm.float()) * alpha
    if bias:
        ref = ref + bvec
    if act == 1:
        ref = torch.nn.functional.gelu(ref)
    return Cm.float(), ref


@pytest.mark.parametrize("a_mn", [False, True])
@pytest.mark.parametrize("b_mn", [False, True])
@pytest.mark.parametrize("shape", [(128, 256, 64), (256, 512, 1024), (1024, 3072, 512),
                                   (64, 64, 64), (296, 200, 136), (512, 128, 2048)])
def test_gemm_majors_shapes(torch_cuda, a_mn, b_mn, shape):
    torch = torch_cuda
    M, N, K = shape
    got, ref = _run(torch, M, N, K, a_mn, b_mn)
    assert not torch.isnan(got).any()
    err = (got - ref).abs().max().item()
    assert err <= 1e-3 * max(1.0, ref.abs().max().item()), err


@pytest.mark.parametrize("a_mn,b_mn", [(False, False), (True, True), (False, True)])
def test_gemm_integer_exact(torch_cuda, a_mn, b_mn):
    torch = torch_cuda
    got, ref = _run(torch, 384, 256, 512, a_mn, b_mn, integer=True)
    assert torch.equal(got, ref)


def test_gemm_batched_exact(torch_cuda):
    torch = torch_cuda
    got, ref = _run(torch, 256, 64, 64, False, True, batch=6, integer=True)
    assert torch.equal(got, ref)
    got, ref = _run(torch, 128, 128, 256, True, True, batch=5, integer=True)
    assert torch.equal(got, ref)


def test_gemm_epilogue(torch_cuda):
    torch = torch_cuda
    got, ref = _run(torch, 256, 512, 256, False, True, bias=True, act=1, alpha=0.5)
    assert (got - ref).abs().max().item() < 2e-3
    got, ref = _run(torch, 256, 256, 128, False, False, out_dtype=torch.bfloat16)
    assert ((got - ref).abs() <= 1e-2 * ref.abs().clamp(min=1)).all()


def test_gemm_split_operands(torch_cuda):
    """B spread over 2 gathered column blocks ([q][K][N/2], MN-major, rsplit) and A over
    2 row blocks ([q][M/2][K], K-major, rsplit): the gather_cols / gather_rows layouts."""
    torch = torch_cuda
    M, N, K = 512, 512, 256
    g = torch.Generator(device="cuda").manual_seed(3)
    A = torch.randint(0, 10, (M, K), device="cuda", generator=g).to(torch.bfloat16)
    W = torch.randint(0, 10, (K, N), device="cuda", generator=g).to(torch.bfloat16)
    # gathered weight: [2][K][N/2] column blocks
    Wg = torch.stack([W[:, : N // 2], W[:, N // 2:]]).contiguous()
    Cm = torch.empty(M, N, device="cuda")
    c3.gemm(M, N, K, dict(base=A.data_ptr(), sr=K, sc=1),
            dict(base=Wg.data_ptr(), sr=1, sc=N // 2, rsplit=N // 2, s_hi=K * N // 2),
            dict(base=Cm.data_ptr(), dtype=c3.F32, sr=N, sc=1), mode=c3.MODE_TC)
    torch.cuda.synchronize()
    assert torch.equal(Cm, A.float() @ W.float())
    # dA-style: B K-major split along K ([2][N][K/2] column blocks of a row-major [N][K])
    Bk = torch.randint(0, 10, (N, K), device="cuda", generator=g).to(torch.bfloat16)
    Bs = torch.stack([Bk[:, : K // 2], Bk[:, K // 2:]]).contiguous()
    C2 = torch.empty(M, N, device="cuda")
    c3.gemm(M, N, K, dict(base=A.data_ptr(), sr=K, sc=1),
            dict(base=Bs.data_ptr(), sr=K // 2, sc=1, csplit=K // 2, s_hi=N * K // 2),
            dict(base=C2.data_ptr(), dtype=c3.F32, sr=N, sc=1), mode=c3.MODE_TC)
    torch.cuda.synchronize()
    assert torch.equal(C2, A.float() @ Bk.float().T)


def test_simt_matches(torch_cuda):
    torch = torch_cuda
    got, ref = _run(torch, 96, 80, 40, False, True, mode=c3.MODE_F32)
    assert (got - ref).abs().max().item() < 1e-4


@pytest.mark.parametrize("a_mn,b_mn", [(False, False), (False, True)])
def test_grouped_rasterisation_large_b(torch_cuda, a_mn, b_mn):
    """B larger than the grouping threshold (48 MB) switches to 16-row tile bands; with
    20 tile rows (one full band + a partial one) every output tile must be produced once
    (integer inputs: bitwise)."""
    torch = torch_cuda
    got, ref = _run(torch, 128 * 20, 4096, 8192, a_mn, b_mn, integer=True)
    assert not torch.isnan(got).any()
    assert torch.equal(got, ref)


@pytest.mark.parametrize("shape,a_mn,b_mn,segs", [((1024, 3072, 16384), True, True, None),
                                                  ((1024, 1024, 16384), True, True, "4"),
                                                  ((1024, 1024, 16384), True, True, "0"),
                                                  ((4096, 1024, 8192), True, False, "3"),
                                                  ((16384, 1024, 1024), False, True, "2")])
def test_k_segmented_exact(torch_cuda, monkeypatch, shape, a_mn, b_mn, segs):
    """Pair tiles that leave a poor last wave are cut into k segments (the 1024 x 3072 x
    16384 weight gradient takes 3 by itself; C3D_SK forces a count): the last segment of a
    tile to arrive adds the others' fp32 partials. Integer inputs keep every partial sum
    exact, so the result is bitwise the fp32 product."""
    torch = torch_cuda
    if segs:
        monkeypatch.setenv("C3D_SK", segs)
    M, N, K = shape
    got, ref = _run(torch, M, N, K, a_mn, b_mn, integer=True)
    assert not torch.isnan(got).any()
    assert torch.equal(got, ref)


def test_k_segmented_deterministic(torch_cuda):
    """The split tiles' partials are summed in k order whichever segment finishes last:
    two runs on real-valued inputs agree bitwise, and match fp32 to rounding."""
    torch = torch_cuda
    a, ref = _run(torch, 1024, 3072, 16384, True, True)
    b, _ = _run(torch, 1024, 3072, 16384, True, True)
    assert torch.equal(a, b)
    assert (a - ref).abs().max().item() <= 1e-3 * max(1.0, ref.abs().max().item())


def test_split_k_bf16_output(torch_cuda, monkeypatch):
    """Few tiles, long K: single-CTA split-K whose vectorised reduction writes bf16."""
    torch = torch_cuda
    monkeypatch.setenv("C3D_SK", "0")
    got, ref = _run(torch, 1024, 1024, 16384, True, True, out_dtype=torch.bfloat16)
    assert ((got - ref).abs() <= 1e-2 * ref.abs().clamp(min=1)).all()
