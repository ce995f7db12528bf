"""Collective microbenchmark over the cube's axis lines (run under torchrun).

Times back-to-back all_gather / reduce_scatter / all_reduce calls on axis `--axis`
with CUDA events (max over ranks) for a range of payloads. The transport is the
peer-memory push kernels unless C3D_NCCL_COLL=1 (NCCL). busbw = payload*(p-1)/p / t.
"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2105_14450_b200 import cube3d as c3  # noqa: E402
from paper_2105_14450_b200 import dist as cdist  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--axis", type=int, default=0)
    ap.add_argument("--iters", type=int, default=50)
    ap.add_argument("--dtype", default="bf16")
    ap.add_argument("--graph", action="store_true", help="time a captured CUDA graph of the calls")
    ap.add_argument("--sizes", default="0.03,0.5,2,8,16,32,64")
    args = ap.parse_args()
    rank, world, local = cdist.init_process_group("nccl")
    torch.cuda.set_device(local)
    dims = c3.grid_for(world)
    cube = cdist.make_cube(dims)
    p = dims[args.axis]
    dt = torch.bfloat16 if args.dtype == "bf16" else torch.float32
    es = 2 if dt == torch.bfloat16 else 4
    # bring the SM clock up from idle before timing (about a second of GEMMs)
    w = torch.randn(4096, 4096, device="cuda", dtype=torch.bfloat16)
    t0 = time.time()
    while time.time() - t0 < 1.5:
        for _ in range(20):
            w @ w
        torch.cuda.synchronize()
    tag = "nccl" if os.environ.get("C3D_NCCL_COLL") else "symm"
    for mb in [float(v) for v in args.sizes.split(",")]:
        n = int(mb * 1e6 / es) // 64 * 64
        full = torch.ones(n, dtype=dt, device="cuda")
        shard = torch.ones(n // p, dtype=dt, device="cuda")
        out = torch.empty(n // p, dtype=dt, device="cuda")
        for name, fn in (("AG", lambda: cube.all_gather(args.axis, shard)),
                         ("RS", lambda: cube.reduce_scatter(args.axis, full)),
                         ("AR", lambda: cube.all_reduce(args.axis, out))):
            for _ in range(3):
                fn()
            torch.cuda.synchronize()
            g = None
            if args.graph:
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g):
                    for _ in range(args.iters):
                        fn()
                torch.cuda.synchronize()
                g.replay()
                torch.cuda.synchronize()
            cdist.barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            if g is not None:
                g.replay()
            else:
                for _ in range(args.iters):
                    fn()
            e1.record()
            torch.cuda.synchronize()
            us = cdist.max_over_ranks(e0.elapsed_time(e1) / args.iters * 1e3)
            payload = n * es if name != "AR" else (n // p) * es
            bus = payload * (p - 1) / p / (us * 1e-6) / 1e9 if name != "AR" else \
                2 * payload * (p - 1) / p / (us * 1e-6) / 1e9
            if rank == 0:
                print(f"{tag} axis{args.axis} p={p} {name} {payload / 1e6:8.3f} MB  "
                      f"{us:8.1f} us  busbw {bus:7.1f} GB/s", flush=True)
    cube.close()
    os._exit(0)


if __name__ == "__main__":
    main()
