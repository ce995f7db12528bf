"""The 1-D partition baseline BASELINE.json configs[4] compares the 3-D matmul against
(the paper's 1-D / Megatron-style row partition, which the reference does not implement,
SPEC.md:13): C = A B over a line of N GPUs with A and B row-partitioned (rank i holds
rows [i M/N, (i+1) M/N) of A and rows [i K/N, (i+1) K/N) of B), B all-gathered, and the
rank's row block of C computed locally, C row-partitioned like A. Communication per rank
is (N - 1)/N |B| against the 3-D algorithm's (p - 1)(|A| + |B| + |C|)/p^3 (cost_model.hpp:
33-45), and the local GEMM is (M/N) x K x N. It runs on this library's own peer-memory
all-gather and tcgen05 GEMM, so the comparison isolates the partitioning.
"""
from __future__ import annotations

from . import cube3d as c3


class OneDMatmul:
    """C = A B for M = N = K = n on a (N, 1, 1) grid (the cube's x axis as the 1-D line)."""

    def __init__(self, cube: c3.Cube, n: int, seed: int = 7):
        import torch
        self.cube = cube
        self.N = cube.dims[0]
        if cube.dims[1] != 1 or cube.dims[2] != 1:
            raise ValueError("the 1-D baseline runs on a (N, 1, 1) grid")
        if n % self.N:
            raise ValueError("n must be divisible by the number of GPUs")
        dev = cube.device_str()
        g = torch.Generator(device=dev).manual_seed(seed + cube.rank)
        self.n = n
        rows = n // self.N
        self.a = (torch.rand((rows, n), device=dev, generator=g) - 0.5).to(torch.bfloat16)
        self.b = (torch.rand((rows, n), device=dev, generator=g) - 0.5).to(torch.bfloat16)
        self.bfull = torch.empty((n, n), device=dev, dtype=torch.bfloat16)
        self.c = torch.empty((rows, n), device=dev, dtype=torch.bfloat16)

    def step(self):
        n, rows = self.n, self.n // self.N
        if self.N > 1:
            self.cube.all_gather(0, self.b, out=self.bfull)
        else:
            self.bfull.copy_(self.b)
        # C[rows][n] = A[rows][n] B[n][n]: A K-major, B as the (N, K) operand is MN-major
        c3.gemm(rows, n, n, {"base": self.a.data_ptr(), "sr": n, "sc": 1},
                {"base": self.bfull.data_ptr(), "sr": 1, "sc": n},
                {"base": self.c.data_ptr(), "sr": n, "sc": 1}, mode=c3.MODE_TC)

    def flops(self) -> float:
        return 2.0 * self.n ** 3
