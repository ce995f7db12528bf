import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2105_14450_b200 import cube3d as c3
M, N, K = 1024, 4096, 16384
A = torch.randn((K, M), device="cuda").to(torch.bfloat16)
B = torch.randn((K, N), device="cuda").to(torch.bfloat16)
C = torch.empty(M, N, device="cuda")
av = dict(base=A.data_ptr(), sr=1, sc=M); bv = dict(base=B.data_ptr(), sr=1, sc=N)
ov = dict(base=C.data_ptr(), dtype=c3.F32, sr=N, sc=1)
go = lambda: c3.gemm(M, N, K, av, bv, ov, mode=c3.MODE_TC)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for trial in range(3):
    for mode in ("back2back", "flush", "sync_then"):
        ts = []
        for _ in range(5):
            if mode == "flush": flush.zero_()
            if mode == "sync_then": torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); go(); e1.record(); torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3)
        print(trial, mode, " ".join(f"{t:7.1f}" for t in ts), flush=True)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20): go()
e1.record(); torch.cuda.synchronize()
print("20x back-to-back avg us", e0.elapsed_time(e1) * 1e3 / 20)
