"""BASELINE.json's other configurations on the current grid (run under torchrun for
N > 1): cfg1 (3-D C = A B, M=N=K=1024, fp32-exact mode and bf16), cfg2 (3-D Linear fwd+bwd,
batch*seq = 4096 (b=8, s=512), hidden 2048 -> 8192, bf16), cfg5 (3-D matmul sweep
M=N=K = 4096..32768, bf16, next to the 1-D row-partition baseline). Device-resident operands, CUDA graphs, CUDA events, max over
ranks; whole-job TFLOP/s. Prints one JSON line per measurement on rank 0.

usage: python tools/configs_bench.py [--sizes 4096,8192,16384,32768] [--iters 10]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2105_14450_b200 import cube3d as c3  # noqa: E402
from paper_2105_14450_b200 import dist  # noqa: E402


def timed(fn, iters):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(iters):
            fn()
    g.replay()
    torch.cuda.synchronize()
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    return dist.max_over_ranks(e0.elapsed_time(e1) / iters)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", default="4096,8192,16384,32768")
    ap.add_argument("--iters", type=int, default=10)
    args = ap.parse_args()
    rank, world, local = dist.init_process_group("nccl")
    torch.cuda.set_device(local)
    cube = dist.make_cube()
    dev = cube.device_str()
    g = torch.Generator(device=dev).manual_seed(5 + rank)
    d = c3.canonical_directions()
    grid = "x".join(map(str, cube.dims))

    def mat(n, k, layout, dt):
        shp = cube.local_shape(layout, n, k, d)
        return c3.ShardedMatrix((torch.rand(shp, device=dev, generator=g) - 0.5).to(dt), n, k,
                                layout, d)

    def out(line):
        if rank == 0:
            print(json.dumps({"grid": grid, "n_gpus": world, **line}), flush=True)

    # cfg1: M=N=K=1024, fp32-exact (SIMT) and bf16 tensor cores
    for name, dt, mode in (("fp32", torch.float32, c3.MODE_F32), ("bf16", torch.bfloat16, c3.MODE_AUTO)):
        a, b = mat(1024, 1024, c3.INPUT, dt), mat(1024, 1024, c3.WEIGHT, dt)
        ms = timed(lambda: c3.matmul_ab_fwd(cube, a, b, mode), args.iters)
        out({"config": "cfg1 matmul_ab_fwd M=N=K=1024", "dtype": name, "ms": ms,
             "tflops": 2 * 1024 ** 3 / (ms * 1e-3) / 1e12})
    # cfg2: Linear fwd + bwd, b*s = 4096 (b=8, s=512), 2048 -> 8192
    bsz, seq, hin, hout = 8, 512, 2048, 8192
    X = c3.Activation3D(torch.empty(cube.act_shape(bsz, seq, hin, 0), dtype=torch.bfloat16,
                                    device=dev).uniform_(-1, 1), bsz, seq, hin, 0)
    W = mat(hin, hout, c3.WEIGHT, torch.bfloat16)
    B = c3.DiagonalVector(torch.zeros(cube.diag_len(hout), device=dev), hout)
    lp = c3.LinearParams(W, B, 0)

    def linear_step():
        y, sv = c3.linear3d_fwd(cube, X, lp, c3.GroupState(0))
        c3.linear3d_bwd(cube, y, sv, lp)

    ms = timed(linear_step, args.iters)
    flops = 3 * 2.0 * bsz * seq * hin * hout
    out({"config": "cfg2 linear3d fwd+bwd b*s=4096 2048->8192", "dtype": "bf16", "ms": ms,
         "tflops": flops / (ms * 1e-3) / 1e12})
    # cfg5: matmul sweep, 3-D and the 1-D row-partition baseline (baselines.py) on a
    # (N, 1, 1) line of the same GPUs
    from paper_2105_14450_b200.baselines import OneDMatmul
    line = cube if cube.dims == (world, 1, 1) else dist.make_cube((world, 1, 1))
    # each size's 3-D and 1-D runs back to back (the same power / clock state)
    for n in (int(v) for v in args.sizes.split(",")):
        iters = max(2, args.iters // (n // 4096))
        try:
            a, b = mat(n, n, c3.INPUT, torch.bfloat16), mat(n, n, c3.WEIGHT, torch.bfloat16)
            ms = timed(lambda: c3.matmul_ab_fwd(cube, a, b), iters)
            out({"config": f"cfg5 matmul_ab_fwd M=N=K={n}", "dtype": "bf16", "ms": ms,
                 "tflops": 2.0 * n ** 3 / (ms * 1e-3) / 1e12})
            del a, b
            torch.cuda.empty_cache()
        except Exception as ex:
            out({"config": f"cfg5 matmul_ab_fwd M=N=K={n}", "error": str(ex)[:200]})
        try:
            od = OneDMatmul(line, n)
            ms = timed(od.step, iters)
            out({"config": f"cfg5 1-D row-partition matmul M=N=K={n}", "dtype": "bf16", "ms": ms,
                 "tflops": od.flops() / (ms * 1e-3) / 1e12, "grid_1d": f"{world}x1x1"})
            del od
            torch.cuda.empty_cache()
        except Exception as ex:
            out({"config": f"cfg5 1-D row-partition matmul M=N=K={n}", "error": str(ex)[:200]})
    torch.cuda.synchronize()
    dist.barrier()
    if line is not cube:
        line.close()
    cube.close()
    dist.destroy()


if __name__ == "__main__":
    main()
