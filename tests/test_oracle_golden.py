"""Pins the numpy oracle (oracle/cube3d_oracle.py) to golden vectors produced by the
reference itself (tests/golden/make_golden.py over oracle/_ref). CPU only."""
from pathlib import Path

import numpy as np
import pytest

from oracle import cube3d_oracle as O

G = Path(__file__).resolve().parent / "golden"


def load(name):
    return np.load(G / f"{name}.npz")


def test_rng_streams_bitwise():
    d = load("rng")
    assert np.array_equal(O.Rng(7).next_u64(2000), d["u64_seed7"])
    assert np.array_equal(O.Rng(123).next_u64(700), d["u64_seed123"])
    assert np.array_equal(O.Rng(7).uniform(-1.0, 1.0, 1000), d["uniform_seed7"])
    assert np.array_equal(O.Rng(5).uniform(-0.1, 0.1, 333), d["uniform_seed5_p1"])
    assert np.array_equal(O.random_integer_matrix(4, 4, O.Rng(5)), d["intmat_seed5"])


def test_init_layer_params_bitwise():
    d = load("rng")
    p = O.init_layer_params(16, 7)
    for f in O.FIELDS:
        assert np.array_equal(getattr(p, f).ravel(), d["init16_" + f].ravel()), f


@pytest.mark.parametrize("p", [1, 2, 3])
def test_shard_bounds_tables(p):
    d = load("layout")
    rows, cols = p * p * 2, p * p * 3
    for lay in range(4):
        for tag, dirs in (("c", None), ("s", (2, 0, 1))):
            tab = []
            for r in range(p ** 3):
                (r0, r1), (c0, c1) = O.shard_bounds(lay, O.coords_of(p, r), rows, cols, p, dirs)
                tab.append([r0, r1, c0, c1])
            assert np.array_equal(np.array(tab), d[f"bounds_p{p}_l{lay}_{tag}"]), (lay, tag)


@pytest.mark.parametrize("p", [1, 2, 3])
def test_diagonal_tables(p):
    d = load("layout")
    tab = []
    for r in range(p ** 3):
        holds, (b0, b1) = O.diagonal_slice(O.coords_of(p, r), p * p * 2, p)
        tab.append([int(holds), b0, b1])
    assert np.array_equal(np.array(tab), d[f"diag_p{p}"])


@pytest.mark.parametrize("g", [0, 1])
def test_activation_map(g):
    d = load("layout")
    for tag, (b, s, h) in (("", (4, 4, 8)), ("_big", (4, 8, 16))):
        iota = np.arange(b * s * h, dtype=np.float64).reshape(b * s, h)
        fam = O.activation_from_global(iota, b, s, g, 2)
        got = np.stack([f.ravel() for f in fam])
        assert np.array_equal(got, d[f"act_p2{tag}_g{g}"])


@pytest.mark.parametrize("p", [1, 2])
def test_matmul_integer_exact(p):
    d = load("matmul")
    a, b, g = d[f"int_p{p}_a"], d[f"int_p{p}_b"], d[f"int_p{p}_g"]
    grads = {"AB": (g @ b.T, a.T @ g), "ABt": (g @ b, g.T @ a), "AtB": (b @ g.T, a @ g)}
    for form in ("AB", "ABt", "AtB"):
        assert np.array_equal(O.serial_matmul(a, b, form), d[f"int_p{p}_{form}_c"])
        da, db = grads[form]
        assert np.array_equal(da, d[f"int_p{p}_{form}_da"])
        assert np.array_equal(db, d[f"int_p{p}_{form}_db"])


def test_matmul_real_f64_and_reference_f32_gap():
    d = load("matmul")
    a, b, g = d["real_a"], d["real_b"], d["real_g"]
    assert O.rel_err(O.serial_matmul(a, b), d["real_f64_c"]) < 1e-13
    # the reference's own fp32 3-D path vs fp64: the scale of fp32 rounding at K=64
    assert O.normwise_err(d["real_f32_c"], a @ b) < 1e-6


@pytest.mark.parametrize("name", ["layer_toy", "layer_small"])
def test_layer_oracle_matches_reference(name):
    d = load(name)
    p, b, s, n, h, seed = (int(v) for v in d["cfg"])
    P = O.init_layer_params(h, seed)
    for f in O.FIELDS:
        assert np.array_equal(getattr(P, f).ravel(), d["p_" + f].ravel())
    u = O.Rng(seed).uniform(-1.0, 1.0, 2 * b * s * h)
    x, dy = u[: b * s * h].reshape(b * s, h), u[b * s * h:].reshape(b * s, h)
    assert np.array_equal(x, d["x"]) and np.array_equal(dy, d["dy"])
    y, cache = O.layer_fwd(x, P, b, s, n)
    dx, G = O.layer_bwd(dy, cache, P, b, s, n)
    # reference's own layer tolerance in f64 is 1e-10 (cube3d/verify.hpp:312)
    assert O.rel_err(y, d["y"]) < 1e-10
    assert O.rel_err(dx, d["dx"]) < 1e-10
    for f in O.FIELDS:
        assert O.rel_err(getattr(G, f), d["g_" + f].reshape(getattr(G, f).shape)) < 1e-10, f


@pytest.mark.parametrize("name", ["layer_toy", "layer_small"])
def test_traffic_model_matches_reference(name):
    d = load(name)
    p, b, s, n, h, _ = (int(v) for v in d["cfg"])
    fwd, bwd = O.traffic_layer(b, s, n, h, p)
    assert (fwd, bwd) == (int(d["costs"][0]), int(d["costs"][1]))
    mf, mb = O.layer_madds(b, s, n, h, p)
    assert (mf, mb) == (int(d["costs"][2]), int(d["costs"][3]))
    # measured reference counters: every rank's sent/received sum to the model
    cnt = d["counters"].astype(np.int64)
    assert int(cnt[:, 0].sum()) == fwd + bwd and int(cnt[:, 1].sum()) == fwd + bwd


def test_cfg3_costs():
    d = load("costs")
    for key in d.files:
        _, p, b, s, n, h = key.split("_")
        fwd, bwd = O.traffic_layer(int(b), int(s), int(n), int(h), int(p))
        assert (fwd, bwd) == (int(d[key][0]), int(d[key][1])), key
