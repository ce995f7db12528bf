import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2105_14450_b200 import cube3d as c3
from paper_2105_14450_b200 import _lib
import ctypes as C
M, N, K = 1024, 4096, 16384
A = torch.randn((K, M), device="cuda").to(torch.bfloat16)
B = torch.randn((K, N), device="cuda").to(torch.bfloat16)
Cm = torch.empty(M, N, device="cuda")
av = dict(base=A.data_ptr(), sr=1, sc=M); bv = dict(base=B.data_ptr(), sr=1, sc=N)
ov = dict(base=Cm.data_ptr(), dtype=c3.F32, sr=N, sc=1)
def t(f, n=50):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(n): f()
    h = (time.perf_counter() - t0) / n
    torch.cuda.synchronize(); w = (time.perf_counter() - t0) / n
    return h * 1e6, w * 1e6
print("c3.gemm host/wall us", t(lambda: c3.gemm(M, N, K, av, bv, ov, mode=c3.MODE_TC)))
print("launch_count host us", t(lambda: _lib.lib().c3d_launch_count()))
print("torch.matmul host/wall", t(lambda: torch.matmul(A.T, B)))
print("tiny gemm host/wall", t(lambda: c3.gemm(128, 128, 64, dict(base=A.data_ptr(), sr=64, sc=1), dict(base=B.data_ptr(), sr=64, sc=1), dict(base=Cm.data_ptr(), dtype=c3.F32, sr=128, sc=1), mode=c3.MODE_TC)))
