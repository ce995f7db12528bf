"""Shared test helpers: golden fixtures, oracle parameter conversion, tolerances."""
from pathlib import Path

import numpy as np

from oracle import cube3d_oracle as O
from paper_2105_14450_b200 import cube3d as c3

G = Path(__file__).resolve().parent / "golden"

# Tolerances (north star, BASELINE.json): fp32 mode 1e-5 norm-wise against an fp64
# oracle (the reference's own max-rel metric gives ~3e-5 at K=1024
# in fp32, so 1e-5 is stated norm-wise); bf16 tensor-core mode 2e-2 norm-wise
# against the fp64 oracle on the same bf16-rounded inputs and parameters. The
# reference's element-wise max-rel metric (cube3d/verify.hpp:268-279) is not a
# usable bf16 gate: the reference init gives attention logits of std ~3 after
# LayerNorm, so per-element bf16 storage error is amplified on small elements.
# A second gate (1e-2 norm-wise) compares against the fp64 oracle that
# rounds to bf16 at the same storage points as the product (oracle `rnd` hook):
# that one catches indexing/layout bugs that the loose gate could hide.
TOL_F32_NORM = 1e-5
TOL_BF16_NORM = 2e-2
TOL_BF16_EMUL = 1e-2
TOL_BF16_REL = 2e-2  # matmul-level max-rel gate (no attention amplification)


def check_bf16(got, want, what="", emulated=None):
    ne = O.normwise_err(got, want)
    assert ne < TOL_BF16_NORM, (what, "vs fp64", ne, O.rel_err(got, want))
    if emulated is not None:
        ee = O.normwise_err(got, emulated)
        assert ee < TOL_BF16_EMUL, (what, "vs bf16-emulating oracle", ee)


def golden(name):
    return np.load(G / f"{name}.npz")


def bf16_round(a: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even to bf16, returned as float64."""
    import torch
    return torch.tensor(np.asarray(a, dtype=np.float32)).to(torch.bfloat16).double().numpy()


def global_params_from(d, prefix="p_", h=None) -> c3.GlobalLayerParams:
    vals = {f: np.array(d[prefix + f], dtype=np.float64) for f in O.FIELDS}
    return c3.GlobalLayerParams(**vals)


def oracle_params(gp) -> O.LayerParams:
    return O.LayerParams(**{f: np.asarray(getattr(gp, f), dtype=np.float64) for f in O.FIELDS})


def map_params(gp, fn):
    return c3.GlobalLayerParams(**{f: fn(getattr(gp, f)) for f in O.FIELDS})


def to_np(t):
    return t.detach().double().cpu().numpy()


def collect_grads(cube, grads, dims=(1, 1, 1)):
    """Global gradients from a single-rank (p=1) LayerParams."""
    out = {}
    for f in O.FIELDS:
        v = getattr(grads, f)
        out[f] = to_np(v.shard)
    return out
