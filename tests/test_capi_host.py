"""C-ABI library on the CPU: it loads, exports every symbol include/c3d.h declares,
and its pure-host placement / topology / RNG functions reproduce the reference's
known-answer tests (proj/tests/test_topology.cpp, test_sharding.cpp) and the
golden tables bit-exactly. No GPU compute is called here."""
import re
from pathlib import Path

import numpy as np
import pytest

from oracle import cube3d_oracle as O
from paper_2105_14450_b200 import C3DError, cube3d as c3
from paper_2105_14450_b200 import _lib

ROOT = Path(__file__).resolve().parents[1]
G = ROOT / "tests" / "golden"


def test_library_exports_every_declared_symbol():
    text = (ROOT / "include" / "c3d.h").read_text()
    declared = set(re.findall(r"^\s*(?:const char\*|int|long long)\s+(c3d_\w+)\(", text, re.M))
    assert len(declared) >= 40
    L = _lib.lib()
    missing = [s for s in declared if not hasattr(L, s)]
    assert not missing, missing
    assert set(_lib.SIGNATURES) == declared


def test_topology_kats():
    # test_topology.cpp:20-53
    assert c3.rank_of((2, 2, 2), (0, 0, 0)) == 0
    assert c3.rank_of((2, 2, 2), (1, 0, 1)) == 5
    assert c3.rank_of((2, 2, 2), (1, 1, 1)) == 7
    with pytest.raises(C3DError) as e:
        c3.rank_of((2, 2, 2), (2, 0, 0))
    assert e.value.name == "OutOfRange"
    assert c3.axis_group((2, 2, 2), 0, c3.Y) == ([0, 2], 0)
    assert c3.axis_group((2, 2, 2), 7, c3.Z) == ([6, 7], 1)
    assert c3.build_cube(8) == 2 and c3.build_cube(1) == 1 and c3.build_cube(27) == 3
    for bad in (12, 0):
        with pytest.raises(C3DError) as e:
            c3.build_cube(bad)
        assert e.value.name == "NotACube"


@pytest.mark.parametrize("p", [1, 2, 3])
def test_topology_matches_oracle(p):
    dims = (p, p, p)
    for r in range(p ** 3):
        c = c3.coords_of(dims, r)
        assert c == O.coords_of(p, r)
        assert c3.rank_of(dims, c) == r
        for ax in range(3):
            m, pos = c3.axis_group(dims, r, ax)
            assert m == O.axis_group(p, c, ax) and pos == c[ax]
            assert c3.line_index(dims, r, ax) == O.line_index(p, c, ax)


def test_sharding_kats():
    # test_sharding.cpp:25-50
    iota = np.arange(16, dtype=np.float64).reshape(4, 4)
    sh = c3.partition(iota, c3.INPUT, (2, 2, 2))
    assert sh[c3.rank_of((2, 2, 2), (1, 0, 1))].ravel().tolist() == [10, 11]
    assert c3.shard_bounds(c3.WEIGHT, (2, 2, 2), (0, 1, 0), 4, 4) == ((0, 2), (2, 3))
    assert c3.shard_bounds(c3.OUTPUT, (2, 2, 2), (0, 0, 0), 4, 4) == ((0, 1), (0, 2))
    assert c3.shard_bounds(c3.OUTPUT, (2, 2, 2), (1, 0, 1), 4, 4) == ((3, 4), (0, 2))
    with pytest.raises(C3DError) as e:
        c3.partition(np.zeros((6, 8)), c3.INPUT, (2, 2, 2))
    assert e.value.name == "IndivisibleShape" and "rows=6" in str(e.value)
    with pytest.raises(C3DError) as e:
        c3.shard_bounds(c3.INPUT, (2, 2, 2), (0, 0, 0), 4, 4, c3.DirectionTriple(1, 1, 2))
    assert e.value.name == "DirectionClash"


def test_diagonal_kat():
    # test_sharding.cpp:121-136
    dims = (2, 2, 2)
    fam = c3.partition_diagonal(np.array([0.0, 1, 2, 3]), dims)
    want = {(0, 0, 0): [0], (1, 0, 0): [1], (0, 1, 1): [2], (1, 1, 1): [3], (0, 1, 0): [],
            (0, 0, 1): []}
    for c, w in want.items():
        assert fam[c3.rank_of(dims, c)].tolist() == w
    assert c3.collect_diagonal(fam, dims, 4).tolist() == [0, 1, 2, 3]


@pytest.mark.parametrize("p", [1, 2, 3])
def test_shard_bounds_golden(p):
    d = np.load(G / "layout.npz")
    rows, cols = p * p * 2, p * p * 3
    for lay in range(4):
        for tag, dirs in (("c", None), ("s", c3.DirectionTriple(2, 0, 1))):
            tab = []
            for r in range(p ** 3):
                (r0, r1), (c0, c1) = c3.shard_bounds(lay, (p, p, p), c3.coords_of((p, p, p), r),
                                                     rows, cols, dirs)
                tab.append([r0, r1, c0, c1])
            assert np.array_equal(np.array(tab), d[f"bounds_p{p}_l{lay}_{tag}"])
        tab = []
        for r in range(p ** 3):
            holds, (b0, b1) = c3.diagonal_slice((p, p, p), c3.coords_of((p, p, p), r), p * p * 2)
            tab.append([int(holds), b0, b1])
        assert np.array_equal(np.array(tab), d[f"diag_p{p}"])


@pytest.mark.parametrize("g", [0, 1])
def test_activation_map_golden(g):
    d = np.load(G / "layout.npz")
    for tag, (b, s, h) in (("", (4, 4, 8)), ("_big", (4, 8, 16))):
        iota = np.arange(b * s * h, dtype=np.float64).reshape(b * s, h)
        fam = c3.activation_from_global(iota, b, s, g, (2, 2, 2))
        assert np.array_equal(np.stack([f.ravel() for f in fam]), d[f"act_p2{tag}_g{g}"])
        back = c3.activation_to_global(fam, b, s, h, g, (2, 2, 2))
        assert np.array_equal(back, iota)


def test_rng_bitwise():
    d = np.load(G / "rng.npz")
    assert np.array_equal(c3.Rng(7).next_u64(2000), d["u64_seed7"])
    assert np.array_equal(c3.Rng(7).uniform(-1.0, 1.0, 1000), d["uniform_seed7"])
    assert np.array_equal(c3.random_integer_matrix(4, 4, c3.Rng(5)), d["intmat_seed5"])
    cfg = c3.TransformerConfig(2, 8, 2, 16)
    gp = c3.init_layer_params(cfg, 7)
    for f in O.FIELDS:
        assert np.array_equal(getattr(gp, f).ravel(), d["init16_" + f].ravel())


@pytest.mark.parametrize("dims", [(1, 1, 1), (2, 2, 2), (3, 3, 3), (2, 1, 1), (1, 2, 2),
                                  (2, 2, 1), (4, 2, 2)])
def test_partition_collect_and_balance(dims):
    # partition/collect inverse, disjoint cover, perfect balance (test_sharding.cpp:71-119)
    q = dims[0] * dims[1] * dims[2]
    rows, cols = 2 * q * q, 3 * q * q
    m = np.random.default_rng(1).uniform(size=(rows, cols))
    for lay in range(4):
        fam = c3.partition(m, lay, dims)
        assert len({f.size for f in fam}) == 1
        assert sum(f.size for f in fam) == m.size
        assert np.array_equal(c3.collect(fam, lay, dims, rows, cols), m)


@pytest.mark.parametrize("dims", [(2, 1, 1), (1, 2, 2), (2, 2, 2)])
def test_activation_roundtrip_subgrids(dims):
    b, s, h = 4, 8, 16
    m = np.arange(b * s * h, dtype=np.float64).reshape(b * s, h)
    for g in (0, 1):
        fam = c3.activation_from_global(m, b, s, g, dims)
        assert len({f.size for f in fam}) == 1
        assert np.array_equal(c3.activation_to_global(fam, b, s, h, g, dims), m)


def test_diagonal_subgrids_tile_once():
    # the reference's diagonal on cubes and py == pz grids; every rank holds one slice on
    # sub-grids with py or pz equal to 1 (2x2x1, the north star's 4-GPU grid)
    for dims in [(2, 1, 1), (1, 2, 2), (2, 2, 2), (3, 2, 2), (2, 2, 1), (2, 1, 2), (1, 4, 1)]:
        n = 48
        fam = c3.partition_diagonal(np.arange(n, dtype=np.float64), dims)
        assert c3.collect_diagonal(fam, dims, n).tolist() == list(range(n))
        holders = [c for c in c3._ranks(dims) if c3.diagonal_slice(dims, c, n)[0]]
        if dims[1] == dims[2]:
            assert all(c[1] == c[2] for c in holders)
        else:
            assert len(holders) == dims[0] * dims[1] * dims[2]
    # 2x2x1: rank (i, j, 0) holds b[j*N/2 + i*N/4, +N/4)
    assert c3.diagonal_slice((2, 2, 1), (1, 0, 0), 8) == (True, (2, 4))
    assert c3.diagonal_slice((2, 2, 1), (0, 1, 0), 8) == (True, (4, 6))
    with pytest.raises(C3DError) as e:
        c3.diagonal_slice((1, 2, 4), (0, 0, 0), 16)
    assert e.value.name == "ConfigInvalid"


def test_grid_for_gpu_counts():
    """BASELINE.json north star: 2 and 4 GPUs as the 2x1x1 and 2x2x1 sub-cubes."""
    assert c3.grid_for(1) == (1, 1, 1) and c3.grid_for(8) == (2, 2, 2)
    assert c3.grid_for(2) == (2, 1, 1) and c3.grid_for(4) == (2, 2, 1)
