"""Command line of the library, mirroring the reference's `cube3d` tool
(tools/cube3d_main.cpp:1-199): same subcommands, options and exit codes (0 success, 1
verification / runtime failure, 2 usage error).

    python -m paper_2105_14450_b200.cli verify --hidden 256 --seq 256 --batch 2 --heads 4
    python -m paper_2105_14450_b200.cli bench --mode weak --p-list 1,2 --out weak.csv
    python -m paper_2105_14450_b200.cli matmul --form ab --a A.bin --b B.bin --out C.bin

`verify` and `matmul` run on the GPUs of the process group (one process per GPU under
torchrun, grid by GPU count: 1 -> 1x1x1, 2 -> 2x1x1, 4 -> 2x2x1, 8 -> 2x2x2, or --grid);
`bench` prints the reference's modeled-cost scaling table (cube3d/bench.hpp) with this
library's traffic (or the reference's with --reference-traffic). Matrix files are the
reference's CUBE3D format (matrix_io.py).
"""
from __future__ import annotations

import argparse
import sys
from typing import List, Optional

import numpy as np

from . import traffic as T


def _p_list(s: str) -> List[int]:
    return [int(v) for v in s.split(",") if v]


def _grid(args, world):
    from . import cube3d as c3
    if args.grid:
        return tuple(int(v) for v in args.grid.split("x"))
    return c3.grid_for(world)


def _open_cube(args):
    import torch
    from . import dist
    rank, world, local = dist.init_process_group("nccl")
    torch.cuda.set_device(local)
    return dist.make_cube(_grid(args, world)), rank, world


def cmd_bench(args) -> int:
    try:
        rows = T.scaling_rows(args.mode, args.batch, args.seq, args.heads, args.hidden,
                              args.layers, args.p_list, args.lam, args.reference_traffic)
    except (ValueError, ZeroDivisionError) as e:
        print(f"ConfigInvalid: {e}", file=sys.stderr)
        return 2
    text = T.scaling_csv(rows)
    if args.out:
        try:
            with open(args.out, "w", newline="\n") as f:
                f.write(text)
        except OSError:
            print(f"cannot open {args.out} for writing", file=sys.stderr)
            return 1
    else:
        sys.stdout.write(text)
    return 0


def cmd_matmul(args) -> int:
    """Reads A and B, partitions them on the grid (Input / Weight / WeightOfTranspose /
    swapped-Input per form, tools/cube3d_main.cpp:85-99), runs the 3-D product in the
    files' precision class (f64 files in the fp32-exact mode, f32 files in the fp32-exact
    mode; --tc: bf16 tensor cores), collects C and writes it in the operands' dtype."""
    import torch
    from . import cube3d as c3
    from . import dist
    from .matrix_io import matrix_file_dtype, read_matrix, write_matrix
    if matrix_file_dtype(args.a) != matrix_file_dtype(args.b):
        print("operand files carry different dtypes", file=sys.stderr)
        return 2
    kind = "f32" if matrix_file_dtype(args.a) == 1 else "f64"
    a, b = read_matrix(args.a).astype(np.float64), read_matrix(args.b).astype(np.float64)
    cube, rank, world = _open_cube(args)
    try:
        dims = cube.dims
        dt, mode = (c3.BF16, c3.MODE_TC) if args.tc else (c3.F32, c3.MODE_F32)
        lay_b, dirs_b = {"ab": (c3.WEIGHT, None), "abt": (c3.WEIGHT_OF_TRANSPOSE, None),
                         "atb": (c3.INPUT, c3.canonical_directions().swapped())}[args.form]
        A = c3.shard_to_device(cube, a, c3.INPUT, dt)
        B = c3.shard_to_device(cube, b, lay_b, dt, dirs_b)
        fwd = {"ab": c3.matmul_ab_fwd, "abt": c3.matmul_abt_fwd, "atb": c3.matmul_atb_fwd}
        C = fwd[args.form](cube, A, B, mode, c3.F32)
        torch.cuda.synchronize()
        shards = [None] * world
        local = C.shard.double().cpu().numpy()
        if world > 1:
            import torch.distributed as tdist
            tdist.all_gather_object(shards, local)
        else:
            shards = [local]
        if rank == 0:
            full = c3.collect(shards, C.layout, dims, C.global_rows, C.global_cols, C.dirs)
            write_matrix(args.out, full, kind)
        cube.close()
        dist.destroy()
    except Exception:
        cube.close()
        raise
    return 0


def cmd_verify(args) -> int:
    """Property suite on the GPUs (the reference's run_verify checks that need no serial
    oracle, cube3d/verify.hpp:345-744): integer products exact in every form and mode,
    forward / backward of a layer deterministic and group-preserving, every ranks' traffic
    equal to the traffic model and sent == received (zero unaccounted traffic), layer
    gradients finite. Prints PASS / FAIL lines; exit 0 iff all pass."""
    import torch
    from . import cube3d as c3
    from . import dist
    cube, rank, world = _open_cube(args)
    dims = cube.dims
    fails = []

    def report(name, ok, detail=""):
        if rank == 0:
            print(("PASS " if ok else "FAIL ") + name + (f": {detail}" if detail else ""),
                  flush=True)
        if not ok:
            fails.append(name)

    def gather(x):
        if world == 1:
            return [x]
        import torch.distributed as tdist
        out = [None] * world
        tdist.all_gather_object(out, x)
        return out

    rng = np.random.default_rng(args.seed)
    q = dims[0] * dims[1] * dims[2]
    m = 16 * q * q
    for form in ("ab", "abt", "atb"):
        for dt, mode, tag in ((c3.F32, c3.MODE_F32, "f32"), (c3.BF16, c3.MODE_TC, "bf16")):
            a = rng.integers(0, 10, (m, m)).astype(np.float64)
            b = rng.integers(0, 10, (m, m)).astype(np.float64)
            lay_b, dirs_b = {"ab": (c3.WEIGHT, None), "abt": (c3.WEIGHT_OF_TRANSPOSE, None),
                             "atb": (c3.INPUT, c3.canonical_directions().swapped())}[form]
            A = c3.shard_to_device(cube, a, c3.INPUT, dt)
            B = c3.shard_to_device(cube, b, lay_b, dt, dirs_b)
            fwd = {"ab": c3.matmul_ab_fwd, "abt": c3.matmul_abt_fwd, "atb": c3.matmul_atb_fwd}
            C = fwd[form](cube, A, B, mode, c3.F32)
            torch.cuda.synchronize()
            full = c3.collect(gather(C.shard.double().cpu().numpy()), C.layout, dims,
                              C.global_rows, C.global_cols, C.dirs)
            want = a @ b if form == "ab" else a @ b.T if form == "abt" else a.T @ b
            report(f"matmul-{form}-{tag}-integer-exact", bool(np.array_equal(full, want)))
    bsz, seq, heads, hid = args.batch, args.seq, args.heads, args.hidden
    cfg = c3.TransformerConfig(bsz, seq, heads, hid)
    gp = c3.init_layer_params(cfg, args.seed)
    for dt, mode, tag in ((c3.F32, c3.MODE_F32, "f32"), (c3.BF16, c3.MODE_AUTO, "bf16")):
        x = rng.uniform(-1, 1, (bsz * seq, hid))
        dy = rng.uniform(-1, 1, (bsz * seq, hid))
        params = c3.partition_layer_params(cube, gp, 0, dt)
        X = c3.activation_to_device(cube, x, bsz, seq, 0, dt)
        DY = c3.activation_to_device(cube, dy, bsz, seq, 0, dt)
        runs = []
        for _ in range(2):
            cube.reset_counters()
            gs = c3.GroupState(0)
            y, sv = c3.transformer_layer_fwd(cube, X, params, cfg, gs, mode)
            torch.cuda.synchronize()
            cf = cube.counters()
            cube.reset_counters()
            dx, g = c3.transformer_layer_bwd(cube, DY, sv, params, cfg, mode, grad_dtype=c3.F32)
            torch.cuda.synchronize()
            cb = cube.counters()
            runs.append((y.local.double().cpu().numpy(), dx.local.double().cpu().numpy(),
                         gs.input_group, cf, cb))
        (y0, dx0, g0, cf, cb), (y1, dx1, _, _, _) = runs
        report(f"layer-{tag}-deterministic", bool(np.array_equal(y0, y1) and np.array_equal(dx0, dx1)))
        report(f"layer-{tag}-group-preserved", g0 == 0)
        report(f"layer-{tag}-finite", bool(np.isfinite(y0).all() and np.isfinite(dx0).all()))
        model = T.layer_traffic(bsz, seq, heads, hid, dims,
                                flash=T.flash_applies(seq, heads, hid, dims, dt == c3.BF16))
        for which, c in (("fwd", cf), ("bwd", cb)):
            tot = gather((c["elements_sent"], c["elements_received"]))
            sent, recv = sum(t[0] for t in tot), sum(t[1] for t in tot)
            want = model[0 if which == "fwd" else 1]
            report(f"layer-{tag}-{which}-traffic", sent == want and sent == recv,
                   f"sent {sent} received {recv} model {want}")
    if rank == 0:
        print(f"VERIFY {'PASS' if not fails else 'FAIL'} ({len(fails)} failure(s))", flush=True)
    cube.close()
    dist.destroy()
    return 0 if not fails else 1


def main(argv: Optional[List[str]] = None) -> int:
    ap = argparse.ArgumentParser(prog="cube3d_b200", description="3-D tensor-parallel Transformer "
                                 "linear algebra on B200 (the reference cube3d tool's commands)")
    sub = ap.add_subparsers(dest="cmd", required=True)
    v = sub.add_parser("verify", help="property suite on this process group's GPUs")
    v.add_argument("--batch", type=int, default=2)
    v.add_argument("--seq", type=int, default=256)
    v.add_argument("--heads", type=int, default=4)
    v.add_argument("--hidden", type=int, default=256)
    v.add_argument("--seed", type=int, default=7)
    v.add_argument("--grid", default=None, help="px x py x pz")
    bch = sub.add_parser("bench", help="modeled weak/strong scaling table (CSV)")
    bch.add_argument("--mode", choices=["weak", "strong"], default="weak")
    bch.add_argument("--p-list", type=_p_list, default=[1, 2])
    bch.add_argument("--batch", type=int, default=2)
    bch.add_argument("--seq", type=int, default=8)
    bch.add_argument("--heads", type=int, default=2)
    bch.add_argument("--hidden", type=int, default=16)
    bch.add_argument("--layers", type=int, default=1)
    bch.add_argument("--lambda", dest="lam", type=float, default=1.0)
    bch.add_argument("--out", default="")
    bch.add_argument("--reference-traffic", action="store_true",
                     help="charge the reference's traffic model instead of this library's")
    mm = sub.add_parser("matmul", help="one 3-D product over CUBE3D matrix files")
    mm.add_argument("--form", choices=["ab", "abt", "atb"], default="ab")
    mm.add_argument("--a", required=True)
    mm.add_argument("--b", required=True)
    mm.add_argument("--out", required=True)
    mm.add_argument("--tc", action="store_true", help="bf16 tensor-core mode")
    mm.add_argument("--grid", default=None, help="px x py x pz")
    try:
        args = ap.parse_args(argv)
    except SystemExit as e:
        return 0 if e.code == 0 else 2
    from ._lib import C3DError
    try:
        return {"verify": cmd_verify, "bench": cmd_bench, "matmul": cmd_matmul}[args.cmd](args)
    except C3DError as e:
        print(str(e), file=sys.stderr)
        return 2 if e.name in ("ConfigInvalid", "HeadsIndivisible") else 1


if __name__ == "__main__":
    sys.exit(main())
