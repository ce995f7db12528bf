"""Generates tests/golden/*.npz from the reference itself (oracle/_ref, built from
/root/reference by oracle/Makefile). Run here, where /root/reference exists:

    make -C oracle && python tests/golden/make_golden.py

The fixtures pin the numpy oracle (tests/test_oracle_golden.py) and are the
parity targets of the GPU tests (tests/test_layer_gpu.py); /root/reference is
never read at test time.
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from oracle import ref  # noqa: E402

OUT = Path(__file__).resolve().parent
LAYOUTS = [0, 1, 2, 3]
CANON = (1, 0, 2)
SWAP = (2, 0, 1)


def rng_fixtures():
    d = {}
    d["u64_seed7"] = ref.rng_u64(7, 2000)
    d["u64_seed123"] = ref.rng_u64(123, 700)
    d["uniform_seed7"] = ref.rng_uniform(7, 1000, -1.0, 1.0)
    d["uniform_seed5_p1"] = ref.rng_uniform(5, 333, -0.1, 0.1)
    d["intmat_seed5"] = ref.random_integer_matrix(5, 4, 4)
    for k, v in ref.init_layer_params(16, 7).items():
        d["init16_" + k] = v
    np.savez_compressed(OUT / "rng.npz", **d)


def layout_fixtures():
    d = {}
    for p in (1, 2, 3):
        rows, cols = p * p * 2, p * p * 3
        for lay in LAYOUTS:
            for tag, dirs in (("c", None), ("s", SWAP)):
                dd = dirs or ((2, 0, 1) if lay == 2 else CANON)
                tab = []
                for r in range(p ** 3):
                    c = (r // (p * p), (r // p) % p, r % p)
                    (r0, r1), (c0, c1) = ref.shard_bounds(lay, p, c, rows, cols, dd)
                    tab.append([r0, r1, c0, c1])
                d[f"bounds_p{p}_l{lay}_{tag}"] = np.array(tab, dtype=np.int64)
        n = p * p * 2
        tab = []
        for r in range(p ** 3):
            c = (r // (p * p), (r // p) % p, r % p)
            holds, (b0, b1) = ref.diagonal_slice(p, c, n)
            tab.append([int(holds), b0, b1])
        d[f"diag_p{p}"] = np.array(tab, dtype=np.int64)
    for g in (0, 1):
        d[f"act_p2_g{g}"] = ref.activation_map(2, 4, 4, 8, g)
        d[f"act_p2_big_g{g}"] = ref.activation_map(2, 4, 8, 16, g)
    np.savez_compressed(OUT / "layout.npz", **d)


def matmul_fixtures():
    d = {}
    for p in (1, 2):
        n = p * p * 2 * 4  # 8 or 32
        a = ref.random_integer_matrix(100 + p, n, n)
        b = ref.random_integer_matrix(200 + p, n, n)
        g = ref.random_integer_matrix(300 + p, n, n)
        d[f"int_p{p}_a"], d[f"int_p{p}_b"], d[f"int_p{p}_g"] = a, b, g
        for form in ("AB", "ABt", "AtB"):
            c, da, db, cnt = ref.run_matmul(p, form, a, b, g)
            d[f"int_p{p}_{form}_c"], d[f"int_p{p}_{form}_da"], d[f"int_p{p}_{form}_db"] = c, da, db
            d[f"int_p{p}_{form}_counters"] = cnt
    # real-valued p=2, 64^3, f64 and f32 paths of the reference
    rng = np.random.default_rng(11)
    a, b, g = (rng.uniform(-1, 1, (64, 64)) for _ in range(3))
    d["real_a"], d["real_b"], d["real_g"] = a, b, g
    for f32 in (0, 1):
        c, da, db, _ = ref.run_matmul(2, "AB", a, b, g, f32=bool(f32))
        d[f"real_f{32 if f32 else 64}_c"], d[f"real_f{32 if f32 else 64}_da"] = c, da
        d[f"real_f{32 if f32 else 64}_db"] = db
    np.savez_compressed(OUT / "matmul.npz", **d)


def layer_fixture(name, p, b, s, n, h, seed):
    # verify.hpp:578-581: params from init_layer_params(cfg, seed); x, dy from Rng(seed)
    params = ref.init_layer_params(h, seed)
    u = ref.rng_uniform(seed, 2 * b * s * h, -1.0, 1.0)
    x = u[: b * s * h].reshape(b * s, h)
    dy = u[b * s * h:].reshape(b * s, h)
    y, dx, dps, cnt, _ = ref.run_layer(p, b, s, n, h, params, x, dy)
    ys, dxs, dpss = ref.layer_serial(b, s, n, h, params, x, dy)
    d = {"cfg": np.array([p, b, s, n, h, seed]), "x": x, "dy": dy, "y": y, "dx": dx,
         "y_serial": ys, "dx_serial": dxs, "counters": cnt}
    for k in ref.FIELDS:
        d["p_" + k] = params[k]
        d["g_" + k] = dps[k]
    traf = ref.layer_costs(p, b, s, n, h)
    d["costs"] = np.array(traf, dtype=np.uint64)
    np.savez_compressed(OUT / f"{name}.npz", **d)


def costs_fixture():
    d = {}
    for (p, b, s, n, h) in [(2, 32, 512, 16, 1024), (2, 2, 8, 2, 16), (2, 4, 32, 4, 64),
                            (1, 32, 512, 16, 1024), (2, 64, 1024, 16, 2048)]:
        d[f"layer_{p}_{b}_{s}_{n}_{h}"] = np.array(ref.layer_costs(p, b, s, n, h), dtype=np.uint64)
    np.savez_compressed(OUT / "costs.npz", **d)


if __name__ == "__main__":
    if not ref.available():
        sys.exit("build oracle/_ref first: make -C oracle")
    rng_fixtures()
    layout_fixtures()
    matmul_fixtures()
    layer_fixture("layer_toy", 2, 2, 8, 2, 16, 7)
    layer_fixture("layer_small", 2, 4, 32, 4, 64, 11)
    costs_fixture()
    ok, txt = ref.run_verify()
    (OUT / "reference_verify.txt").write_text(txt)
    print("golden fixtures written; reference verify:", "PASS" if ok else "FAIL")
