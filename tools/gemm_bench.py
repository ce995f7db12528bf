"""GEMM microbenchmark: the layer's linear GEMMs at cfg3 (p=1) with their operand
majors and epilogues. The GPU is warmed for ~0.5 s first (clocks ramp from idle);
each shape reports the median of per-launch CUDA-event times over back-to-back
launches, next to torch.matmul (cuBLAS) on the same shape."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2105_14450_b200 import cube3d as c3  # noqa: E402

R, H = 16384, 1024
SHAPES = [  # name, M, N, K, a_mn, b_mn, epilogue
    ("qkv_fwd", R, 3 * H, H, 0, 1, "bias"),
    ("out_fwd", R, H, H, 0, 1, "bias+resid"),
    ("fc1_fwd", R, 4 * H, H, 0, 1, "bias+gelu+pre"),
    ("fc2_fwd", R, H, 4 * H, 0, 1, "bias+resid"),
    ("fc2_dx", R, 4 * H, H, 0, 0, "gelu_grad"),
    ("fc1_dx", R, H, 4 * H, 0, 0, ""),
    ("out_dx", R, H, H, 0, 0, ""),
    ("qkv_dx", R, H, 3 * H, 0, 0, ""),
    ("fc2_dw", 4 * H, H, R, 1, 1, "f32"),
    ("fc1_dw", H, 4 * H, R, 1, 1, "f32"),
    ("out_dw", H, H, R, 1, 1, "f32"),
    ("qkv_dw", H, 3 * H, R, 1, 1, "f32"),
]


def timed(fn, n=20):
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(n)]
    for e0, e1 in evs:
        e0.record()
        fn()
        e1.record()
    torch.cuda.synchronize()
    ts = [e0.elapsed_time(e1) for e0, e1 in evs]
    return statistics.median(ts), min(ts), max(ts)


def run(name, M, N, K, a_mn, b_mn, epi):
    dev = "cuda"
    A = torch.randn((K, M) if a_mn else (M, K), device=dev).to(torch.bfloat16)
    B = torch.randn((K, N) if b_mn else (N, K), device=dev).to(torch.bfloat16)
    f32 = "f32" in epi
    C = torch.empty(M, N, device=dev, dtype=torch.float32 if f32 else torch.bfloat16)
    av = dict(base=A.data_ptr(), sr=1, sc=M) if a_mn else dict(base=A.data_ptr(), sr=K, sc=1)
    bv = dict(base=B.data_ptr(), sr=1, sc=N) if b_mn else dict(base=B.data_ptr(), sr=K, sc=1)
    ov = dict(base=C.data_ptr(), dtype=c3.F32 if f32 else c3.BF16, sr=N, sc=1)
    bias = torch.randn(N, device=dev) if "bias" in epi else None
    act = 1 if "gelu" in epi and "grad" not in epi else 0

    def go():
        c3.gemm(M, N, K, av, bv, ov, bias=bias.data_ptr() if bias is not None else None, act=act,
                mode=c3.MODE_TC)

    for _ in range(3):
        go()
    med, lo, hi = timed(go)
    Am = A.T if a_mn else A
    Bm = B if b_mn else B.T
    for _ in range(3):
        torch.matmul(Am, Bm)
    cmed, _, _ = timed(lambda: torch.matmul(Am, Bm))
    tf = 2 * M * N * K / (med * 1e-3) / 1e12
    tcb = 2 * M * N * K / (cmed * 1e-3) / 1e12
    print(f"{name:8s} M={M:5d} N={N:5d} K={K:5d} {epi:14s} {med * 1e3:7.1f} us "
          f"[{lo * 1e3:6.1f},{hi * 1e3:7.1f}] {tf:7.1f} TF/s | cuBLAS {cmed * 1e3:7.1f} us "
          f"{tcb:7.1f} TF/s", flush=True)
    return med


if __name__ == "__main__":
    sel = sys.argv[1:]
    x = torch.randn(8192, 8192, device="cuda", dtype=torch.bfloat16)
    torch.cuda.synchronize()
    import time
    t0 = time.time()
    while time.time() - t0 < 0.5:  # clock warm-up
        torch.matmul(x, x)
    torch.cuda.synchronize()
    tot = 0
    for s in SHAPES:
        if not sel or s[0] in sel:
            tot += run(*s)
    print(f"total {tot * 1e3:.1f} us")
