"""Multi-GPU parity driver (run under torchrun, one rank per GPU): 3-D matmuls and the
Transformer layer on the grid for WORLD_SIZE, collected on rank 0 and compared with
the reference's golden outputs / the pinned oracle. Prints PASS/FAIL lines; exit 1
on failure. Used by tests/test_multigpu_gpu.py."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from oracle import cube3d_oracle as O  # noqa: E402
from paper_2105_14450_b200 import cube3d as c3  # noqa: E402
from paper_2105_14450_b200 import dist as cdist  # noqa: E402
from helpers import bf16_round, golden, to_np  # noqa: E402

FAILS = []


def report(name, ok, detail=""):
    if dist.get_rank() == 0:
        print(("PASS " if ok else "FAIL ") + name + (f": {detail}" if detail else ""), flush=True)
    if not ok:
        FAILS.append(name)


def gather_all(arr):
    out = [None] * dist.get_world_size()
    dist.all_gather_object(out, arr)
    return out


def collective_checks(cube, dims):
    """Endpoint collectives: the reference's transport KATs (tests/test_transport.cpp:
    66-111) on every axis with extent 2, plus large payloads (multi-block, chunked
    through the mailbox) against torch-computed expectations, f32 and bf16."""
    dev = cube.device_str()
    for axis in range(3):
        if dims[axis] != 2:
            continue
        pos = cube.coords[axis]
        f = torch.float32
        base = 1.0 if pos == 0 else 3.0
        ag = cube.all_gather(axis, torch.tensor([base, base + 1], dtype=f, device=dev))
        mine = torch.tensor([1, 2, 3, 4] if pos == 0 else [10, 20, 30, 40], dtype=f, device=dev)
        rs = cube.reduce_scatter(axis, mine)
        ar = cube.all_reduce(axis, torch.tensor([1, 2] if pos == 0 else [3, 4], dtype=f,
                                                device=dev))
        mx = cube.all_reduce(axis, torch.tensor([1, 9] if pos == 0 else [3, 4], dtype=f,
                                                device=dev), op="max")
        bc = torch.tensor([1, 2, 3, 4] if pos == 1 else [0, 0, 0, 0], dtype=f, device=dev)
        cube.broadcast(axis, 1, bc)
        torch.cuda.synchronize()
        ok = (ag.tolist() == [1, 2, 3, 4] and rs.tolist() == ([11, 22] if pos == 0 else [33, 44])
              and ar.tolist() == [4, 6] and mx.tolist() == [3, 9] and bc.tolist() == [1, 2, 3, 4])
        oks = gather_all(ok)
        report(f"collectives-kat-axis{axis}", all(oks))
        # large integer-valued payloads (exact in bf16 and f32), odd sizes hit the
        # scalar path; 40M f32 elements exceed one mailbox slot and are chunked
        for dt in (torch.float32, torch.bfloat16):
            for n in (1000003, 4 << 20, 40 << 20 if dt == torch.float32 else 8 << 20):
                g = torch.Generator(device="cpu").manual_seed(7 + n)
                full = torch.randint(0, 8, (2, 2 * n if n < (40 << 20) else n), generator=g)
                full = full.to(dt)
                m = full.shape[1]
                mine = full[pos].to(dev)
                got_ag = cube.all_gather(axis, mine)
                got_rs = cube.reduce_scatter(axis, mine)
                got_ar = cube.all_reduce(axis, mine.clone())
                torch.cuda.synchronize()
                exp_sum = (full[0].float() + full[1].float()).to(dt)
                ok = (torch.equal(got_ag.cpu(), full.reshape(-1))
                      and torch.equal(got_rs.cpu(), exp_sum[pos * (m // 2):(pos + 1) * (m // 2)])
                      and torch.equal(got_ar.cpu(), exp_sum))
                oks = gather_all(bool(ok))
                report(f"collectives-axis{axis}-{str(dt)[6:]}-n{m}", all(oks))


def matmul_checks(cube, dims):
    q = dims[0] * dims[1] * dims[2]
    n = 4 * q * q if q > 1 else 32
    rng = O.Rng(500 + q)
    a = O.random_integer_matrix(n, n, rng)
    b = O.random_integer_matrix(n, n, rng)
    g = O.random_integer_matrix(n, n, rng)
    forms = {"AB": (c3.INPUT, c3.WEIGHT, c3.OUTPUT, None, c3.matmul_ab_fwd, c3.matmul_ab_bwd,
                    a @ b, g @ b.T, a.T @ g),
             "ABt": (c3.INPUT, c3.WEIGHT_OF_TRANSPOSE, c3.OUTPUT, None, c3.matmul_abt_fwd,
                     c3.matmul_abt_bwd, a @ b.T, g @ b, g.T @ a),
             "AtB": (c3.INPUT, c3.INPUT, c3.WEIGHT, c3.canonical_directions().swapped(),
                     c3.matmul_atb_fwd, c3.matmul_atb_bwd, a.T @ b, b @ g.T, a @ g)}
    for mode, dt in ((c3.MODE_F32, c3.F32), (c3.MODE_AUTO, c3.BF16)):
        for form, (la, lb, lg, bd, fwd, bwd, wc, wda, wdb) in forms.items():
            A = c3.shard_to_device(cube, a, la, dt)
            B = c3.shard_to_device(cube, b, lb, dt, bd)
            G = c3.shard_to_device(cube, g, lg, dt)
            C = fwd(cube, A, B, mode, c3.F32)
            dA, dB = bwd(cube, G, A, B, mode, c3.F32)
            torch.cuda.synchronize()
            res = []
            for M, glob in ((C, wc), (dA, wda), (dB, wdb)):
                fam = gather_all(to_np(M.shard))
                got = c3.collect(fam, M.layout, dims, glob.shape[0], glob.shape[1], M.dirs)
                res.append(np.array_equal(got, glob))
            report(f"matmul-{form}-{'f32' if dt == c3.F32 else 'bf16'}-integer-bitwise", all(res),
                   str(res))
    if dims[1] != dims[2]:
        return
    # vector ops along the diagonal
    vec = O.Rng(9).uniform(-1, 1, n)
    am = O.Rng(10).uniform(-1, 1, n * n).reshape(n, n)
    A = c3.shard_to_device(cube, am, c3.INPUT, c3.F32)
    V = c3.vector_to_device(cube, vec, c3.F32)
    C = c3.add_vec_fwd(cube, A, V)
    dA, db = c3.add_vec_bwd(cube, A)
    torch.cuda.synchronize()
    got = c3.collect(gather_all(to_np(C.shard)), c3.INPUT, dims, n, n)
    gdb = c3.collect_diagonal(gather_all(to_np(db.shard)), dims, n)
    report("add_vec-fwd-bwd", O.rel_err(got, am + vec) < 1e-6 and O.rel_err(gdb, am.sum(0)) < 1e-5)


def traffic_check(cube, dims, tag, b, s, n, h, bf16, which):
    """Zero unaccounted traffic (cube3d/verify.hpp:671-682): the elements all ranks sent
    during one layer forward (which=0) or backward (1) equal the library's closed-form
    model (paper_2105_14450_b200/traffic.py), and sent == received."""
    from paper_2105_14450_b200 import traffic as T
    cnt = gather_all(cube.counters())
    sent = sum(c["elements_sent"] for c in cnt)
    recv = sum(c["elements_received"] for c in cnt)
    want = T.layer_traffic(b, s, n, h, dims, flash=T.flash_applies(s, n, h, dims, bf16))[which]
    report(f"traffic-model-{tag}", sent == want and sent == recv,
           f"measured {sent} (received {recv}), model {want}")


def layer_check(cube, dims, name, dtype, mode):
    d = golden(name)
    _, b, s, n, h, seed = (int(v) for v in d["cfg"])
    gp = c3.GlobalLayerParams(**{f: np.array(d["p_" + f]) for f in O.FIELDS})
    x, dy = d["x"], d["dy"]
    if dtype == c3.BF16:
        gp = c3.GlobalLayerParams(**{f: bf16_round(getattr(gp, f)) for f in O.FIELDS})
        x, dy = bf16_round(x), bf16_round(dy)
    cfg = c3.TransformerConfig(b, s, n, h)
    params = c3.partition_layer_params(cube, gp, 0, dtype)
    X = c3.activation_to_device(cube, x, b, s, 0, dtype)
    DY = c3.activation_to_device(cube, dy, b, s, 0, dtype)
    gs = c3.GroupState(0)
    cube.reset_counters()
    y, saved = c3.transformer_layer_fwd(cube, X, params, cfg, gs, mode)
    torch.cuda.synchronize()
    traffic_check(cube, dims, f"{name}-{'f32' if dtype == c3.F32 else 'bf16'}-fwd", b, s, n, h,
                  dtype == c3.BF16, 0)
    cube.reset_counters()
    dx, grads = c3.transformer_layer_bwd(cube, DY, saved, params, cfg, mode, grad_dtype=c3.F32)
    torch.cuda.synchronize()
    traffic_check(cube, dims, f"{name}-{'f32' if dtype == c3.F32 else 'bf16'}-bwd", b, s, n, h,
                  dtype == c3.BF16, 1)
    Y = c3.activation_to_global(gather_all(to_np(y.local)), b, s, h, 0, dims)
    DX = c3.activation_to_global(gather_all(to_np(dx.local)), b, s, h, 0, dims)
    G = {}
    for f in O.FIELDS:
        v = getattr(grads, f)
        fam = gather_all(to_np(v.shard))
        if f.startswith("w_"):
            G[f] = c3.collect(fam, c3.WEIGHT, dims, v.global_rows, v.global_cols, v.dirs)
        else:
            G[f] = c3.collect_diagonal(fam, dims, v.global_len)
    if dtype == c3.F32:
        errs = {"y": O.normwise_err(Y, d["y"]), "dx": O.normwise_err(DX, d["dx"])}
        for f in O.FIELDS:
            errs[f] = O.normwise_err(G[f], d["g_" + f].reshape(G[f].shape))
        ok = all(e < 1e-5 for e in errs.values())
    else:
        P = O.LayerParams(**{f: getattr(gp, f) for f in O.FIELDS})
        yo, cache = O.layer_fwd(x, P, b, s, n)
        dxo, Go = O.layer_bwd(dy, cache, P, b, s, n)
        errs = {"y": O.normwise_err(Y, yo), "dx": O.normwise_err(DX, dxo)}
        for f in O.FIELDS:
            errs[f] = O.normwise_err(G[f], getattr(Go, f).reshape(G[f].shape))
        ok = all(e < 2e-2 for e in errs.values())
    worst = max(errs, key=errs.get)
    report(f"layer-{name}-{'f32' if dtype == c3.F32 else 'bf16'}", ok,
           f"worst {worst}={errs[worst]:.2e}")


def layer_tc_check(cube, dims):
    """bf16 layer at a shape that takes the flash tcgen05 attention kernels (dh = 64,
    256 / 512 keys per rank; with the seq axis split, the distributed-softmax passes)
    against the fp64 oracle on the same bf16-rounded inputs."""
    b, s, n, h = 2, 512, 8, 512
    P = O.init_layer_params(h, 41)
    gp = c3.GlobalLayerParams(**{f: bf16_round(getattr(P, f)) for f in O.FIELDS})
    r = O.Rng(42)
    x = bf16_round(O.random_matrix(b * s, h, r))
    dy = bf16_round(O.random_matrix(b * s, h, r))
    cfg = c3.TransformerConfig(b, s, n, h)
    params = c3.partition_layer_params(cube, gp, 0, c3.BF16)
    X = c3.activation_to_device(cube, x, b, s, 0, c3.BF16)
    DY = c3.activation_to_device(cube, dy, b, s, 0, c3.BF16)
    cube.reset_counters()
    y, saved = c3.transformer_layer_fwd(cube, X, params, cfg, c3.GroupState(0))
    torch.cuda.synchronize()
    traffic_check(cube, dims, "flash-shape-fwd", b, s, n, h, True, 0)
    cube.reset_counters()
    dx, grads = c3.transformer_layer_bwd(cube, DY, saved, params, cfg, grad_dtype=c3.F32)
    torch.cuda.synchronize()
    traffic_check(cube, dims, "flash-shape-bwd", b, s, n, h, True, 1)
    Y = c3.activation_to_global(gather_all(to_np(y.local)), b, s, h, 0, dims)
    DX = c3.activation_to_global(gather_all(to_np(dx.local)), b, s, h, 0, dims)
    PO = O.LayerParams(**{f: getattr(gp, f) for f in O.FIELDS})
    yo, cache = O.layer_fwd(x, PO, b, s, n)
    dxo, Go = O.layer_bwd(dy, cache, PO, b, s, n)
    errs = {"y": O.normwise_err(Y, yo), "dx": O.normwise_err(DX, dxo)}
    for f in O.FIELDS:
        v = getattr(grads, f)
        fam = gather_all(to_np(v.shard))
        if f.startswith("w_"):
            G = c3.collect(fam, c3.WEIGHT, dims, v.global_rows, v.global_cols, v.dirs)
        else:
            G = c3.collect_diagonal(fam, dims, v.global_len)
        errs[f] = O.normwise_err(G, getattr(Go, f).reshape(G.shape))
    worst = max(errs, key=errs.get)
    report("layer-bf16-fused-attention-shape", all(e < 2e-2 for e in errs.values()),
           f"worst {worst}={errs[worst]:.2e}")


def loss_check(cube, dims):
    """3-D cross-entropy on the grid vs the (finite-difference-checked) oracle."""
    q = dims[0] * dims[1] * dims[2]
    batch, seq, h, v = 4, 64, 64, 256
    r = np.random.default_rng(21)
    x = r.uniform(-1, 1, (batch * seq, h))
    w = r.uniform(-0.5, 0.5, (h, v))
    b = r.uniform(-0.1, 0.1, v)
    t = r.integers(0, v, batch * seq)
    X = c3.activation_to_device(cube, x, batch, seq, 0, c3.F32)
    d0 = c3.triple_for_group(0)
    W = c3.shard_to_device(cube, w, c3.WEIGHT, c3.F32, d0)
    B = c3.vector_to_device(cube, b, c3.F32)
    head = c3.LinearParams(W, B, 0)
    loss, sv = c3.cross_entropy_fwd(cube, X, head, torch.tensor(t, dtype=torch.int32),
                                    c3.GroupState(0), c3.MODE_F32)
    dx, dw, db = c3.cross_entropy_bwd(cube, sv, head, c3.MODE_F32)
    torch.cuda.synchronize()
    lo, cache = O.cross_entropy_fwd(x, w, b, t)
    dxo, dwo, dbo = O.cross_entropy_bwd(cache)
    losses = gather_all(float(loss.item()))
    gdx = c3.activation_to_global(gather_all(to_np(dx.local)), batch, seq, h, 0, dims)
    gdw = c3.collect(gather_all(to_np(dw.shard)), c3.WEIGHT, dims, h, v, d0)
    gdb = c3.collect_diagonal(gather_all(to_np(db.shard)), dims, v)
    ok = (all(abs(l - lo) / abs(lo) < 1e-5 for l in losses) and O.normwise_err(gdx, dxo) < 1e-5
          and O.normwise_err(gdw, dwo) < 1e-5 and O.normwise_err(gdb, dbo) < 1e-5)
    report(f"cross-entropy-f32-{q}ranks", ok, f"loss={losses[0]:.6f} oracle={lo:.6f}")


def desync_checks(dims):
    """Recoverable failures (cube3d/transport.hpp:32-40, 67-78, 305-319): a collective whose
    members disagree on the length, and a member that never arrives, both surface as
    C3D_ERR_DESYNC on the affected ranks (no trap, no hang), and the cube stays poisoned."""
    from paper_2105_14450_b200 import C3DError
    axis = next((a for a in range(3) if dims[a] > 1), None)
    if axis is None:
        return
    os.environ["C3D_PEER_TIMEOUT_MS"] = "2000"
    for case in ("header", "timeout"):
        cube = cdist.make_cube(dims)
        dev = cube.device_str()
        pos = cube.coords[axis]
        names = []
        try:
            if case == "header":  # one member gathers 16 more elements than the others
                n = 1000 + (16 if pos == 1 else 0)
                cube.all_gather(axis, torch.ones(n, dtype=torch.float32, device=dev))
            elif pos == 0:  # position 1 never joins this all-gather
                cube.all_gather(axis, torch.ones(1000, dtype=torch.float32, device=dev))
            cube.check()
        except C3DError as e:
            names.append(e.name)
        try:  # poisoned: the next call fails too
            cube.all_reduce(axis, torch.ones(8, dtype=torch.float32, device=dev))
            cube.check()
        except C3DError as e:
            names.append(e.name)
        got = gather_all((pos, names))
        dist.barrier()
        cube.close()
        if case == "header":
            ok = all(nm == ["Desync", "Desync"] for _, nm in got)
        else:  # the waiting members report it; the absent one never waited
            ok = all((nm == ["Desync", "Desync"]) if p == 0 else True for p, nm in got)
        report(f"desync-{case}-detected", ok, str(got))
    os.environ.pop("C3D_PEER_TIMEOUT_MS", None)


def main():
    rank, world, local = cdist.init_process_group("nccl")
    torch.cuda.set_device(local)
    dims = c3.grid_for(world) if len(sys.argv) < 2 else tuple(int(v) for v in sys.argv[1].split("x"))
    cube = cdist.make_cube(dims)
    collective_checks(cube, dims)
    if os.environ.get("MP_SKIP_MATMUL") is None:
        matmul_checks(cube, dims)
    if dims[1] == dims[2] or 1 in dims[1:]:  # layer grids: py == pz or one of them 1
        loss_check(cube, dims)
        layer_tc_check(cube, dims)
        for name in ("layer_toy", "layer_small"):
            layer_check(cube, dims, name, c3.F32, c3.MODE_F32)
            layer_check(cube, dims, name, c3.BF16, c3.MODE_AUTO)
    cube.close()
    dist.barrier()
    if os.environ.get("C3D_NCCL_COLL") is None:
        desync_checks(dims)
    dist.destroy_process_group()
    return 1 if FAILS else 0


if __name__ == "__main__":
    sys.exit(main())
