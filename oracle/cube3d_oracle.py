"""CPU oracle for the 3-D matmul / Transformer-layer path -- TEST INFRASTRUCTURE ONLY.

A numpy (float64) restatement of the reference library's algorithm for this
path, each function citing the reference file:line it follows (paths relative
to /root/reference/proj/include/). Only tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline leg may import this module, and only as the checker;
the product never routes through it.

Pinned: tests/test_oracle_golden.py checks every function here against golden
vectors produced by the reference itself (oracle/_ref, built from the
reference headers by oracle/Makefile; fixtures and generator in tests/golden/).

Numerics note: the reference's serial oracle accumulates each product in
ascending k with one accumulator (cube3d/reference.hpp:44-52); numpy's matmul
uses a different (blocked) order, so float64 results agree to ~1e-15 relative,
and integer-valued inputs agree exactly.
"""
from __future__ import annotations

import math
from dataclasses import dataclass
from typing import List, Tuple

import numpy as np

try:  # erf for the exact-erf GELU (cube3d/nn.hpp:44-56)
    from scipy.special import erf as _erf
except Exception:  # pragma: no cover
    _erf = np.vectorize(math.erf)

M64 = (1 << 64) - 1

# --------------------------------------------------------------------------- Rng
# cube3d/rng.hpp:17-34: std::mt19937_64 plus an explicit 53-bit mapping.

_N, _M = 312, 156
_MATRIX_A = np.uint64(0xB5026F5AA96619E9)
_UPPER = np.uint64(0xFFFFFFFF80000000)
_LOWER = np.uint64(0x000000007FFFFFFF)


class MT19937_64:
    """std::mt19937_64 (the standard's parameters), twist vectorised in 3 chunks."""

    def __init__(self, seed: int):
        mt = [0] * _N
        mt[0] = int(seed) & M64
        for i in range(1, _N):
            mt[i] = (6364136223846793005 * (mt[i - 1] ^ (mt[i - 1] >> 62)) + i) & M64
        self.mt = np.array(mt, dtype=np.uint64)
        self.idx = _N

    def _twist(self):
        mt = self.mt
        one = np.uint64(1)

        def step(lo, hi, nxt, far):
            x = (mt[lo:hi] & _UPPER) | (nxt & _LOWER)
            xa = x >> one
            xa = np.where((x & one) == one, xa ^ _MATRIX_A, xa)
            mt[lo:hi] = far ^ xa

        step(0, _N - _M, mt[1:_N - _M + 1].copy(), mt[_M:_N].copy())
        step(_N - _M, _N - 1, mt[_N - _M + 1:_N].copy(), mt[0:_M - 1].copy())
        step(_N - 1, _N, mt[0:1].copy(), mt[_M - 1:_M].copy())
        self.idx = 0

    @staticmethod
    def _temper(y: np.ndarray) -> np.ndarray:
        y = y ^ ((y >> np.uint64(29)) & np.uint64(0x5555555555555555))
        y = y ^ ((y << np.uint64(17)) & np.uint64(0x71D67FFFEDA60000))
        y = y ^ ((y << np.uint64(37)) & np.uint64(0xFFF7EEE000000000))
        return y ^ (y >> np.uint64(43))

    def next(self, n: int) -> np.ndarray:
        out = np.empty(n, dtype=np.uint64)
        got = 0
        while got < n:
            if self.idx >= _N:
                self._twist()
            take = min(n - got, _N - self.idx)
            out[got:got + take] = self._temper(self.mt[self.idx:self.idx + take])
            self.idx += take
            got += take
        return out


class Rng:
    """cube3d/rng.hpp:17-34."""

    def __init__(self, seed: int):
        self.gen = MT19937_64(seed)

    def next_u64(self, n: int = 1) -> np.ndarray:
        return self.gen.next(n)

    def next_unit(self, n: int) -> np.ndarray:
        # static_cast<double>(gen_() >> 11) * 0x1.0p-53  (rng.hpp:24)
        return (self.gen.next(n) >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)

    def uniform(self, lo: float, hi: float, n: int) -> np.ndarray:
        # lo + (hi - lo) * next_unit()  (rng.hpp:26)
        return lo + (hi - lo) * self.next_unit(n)

    def below(self, bound: int, n: int) -> np.ndarray:
        # gen_() % bound  (rng.hpp:30)
        return (self.gen.next(n) % np.uint64(bound)).astype(np.float64)


def random_matrix(rows, cols, rng: Rng, lo=-1.0, hi=1.0):
    """cube3d/rng.hpp:36-42 (row-major fill order)."""
    return rng.uniform(lo, hi, rows * cols).reshape(rows, cols)


def random_integer_matrix(rows, cols, rng: Rng, bound=10):
    """cube3d/rng.hpp:46-52."""
    return rng.below(bound, rows * cols).reshape(rows, cols)


def random_vector(n, rng: Rng, lo=-1.0, hi=1.0):
    """cube3d/rng.hpp:54-59."""
    return rng.uniform(lo, hi, n)


# --------------------------------------------------------------------- topology
# cube3d/topology.hpp:57-127 for a p x p x p cube.

X, Y, Z = 0, 1, 2


def rank_of(p: int, c) -> int:
    """topology.hpp:68-71."""
    return (c[0] * p + c[1]) * p + c[2]


def coords_of(p: int, r: int) -> Tuple[int, int, int]:
    """topology.hpp:73-77."""
    return (r // (p * p), (r // p) % p, r % p)


def axis_group(p: int, c, axis: int) -> List[int]:
    """topology.hpp:79-95: ascending along `axis`."""
    out = []
    for q in range(p):
        cc = list(c)
        cc[axis] = q
        out.append(rank_of(p, cc))
    return out


def line_index(p: int, c, axis: int) -> int:
    """topology.hpp:99-107."""
    i, j, l = c
    return [j * p + l, i * p + l, i * p + j][axis]


# ---------------------------------------------------------------------- layouts
INPUT, WEIGHT, OUTPUT, WEIGHT_OF_TRANSPOSE = 0, 1, 2, 3
CANONICAL = (Y, X, Z)


def swapped(d):
    """layout.hpp:57: input and output roles swap, weight stays."""
    return (d[2], d[1], d[0])


def default_dirs(layout):
    """layout.hpp:67-69."""
    return swapped(CANONICAL) if layout == OUTPUT else CANONICAL


class IndivisibleShape(ValueError):
    pass


def shard_bounds(layout, c, rows, cols, p, dirs=None):
    """layout.hpp:93-123 -> ((r0, r1), (c0, c1))."""
    d = dirs or default_dirs(layout)
    if rows % (p * p) or cols % (p * p):
        raise IndivisibleShape(f"rows={rows} cols={cols} must be divisible by {p * p}")
    r2, c2 = rows // (p * p), cols // (p * p)
    a, w, o = c[d[0]], c[d[1]], c[d[2]]
    if layout in (INPUT, OUTPUT):
        r0, c0 = (w * p + a) * r2, o * (cols // p)
        return (r0, r0 + r2), (c0, c0 + cols // p)
    if layout == WEIGHT:
        r0, c0 = o * (rows // p), (a * p + w) * c2
        return (r0, r0 + rows // p), (c0, c0 + c2)
    r0, c0 = (a * p + w) * r2, o * (cols // p)
    return (r0, r0 + r2), (c0, c0 + cols // p)


def diagonal_slice(c, n, p):
    """layout.hpp:134-142 -> (holds, (b0, b1))."""
    if n % (p * p):
        raise IndivisibleShape(f"vector length={n}")
    n2 = n // (p * p)
    b0 = c[1] * n2 * p + c[0] * n2
    return c[1] == c[2], (b0, b0 + n2)


def group_axes(group):
    """activation.hpp:28-35: (input axis, output axis) of a group."""
    return (Y, Z) if group == 0 else (Z, Y)


def activation_index(p, c, batch, seq, hidden, group):
    """activation.hpp:119-134: global rows of the local rows and the column block."""
    ia, oa = group_axes(group)
    bl, sl, hl = batch // p, seq // p, hidden // p
    w, a, o = c[X], c[ia], c[oa]
    rows = np.array([(w * bl + bi) * seq + a * sl + si for bi in range(bl) for si in range(sl)],
                    dtype=np.int64)
    return rows, o * hl, hl


def activation_from_global(g, batch, seq, group, p):
    """activation.hpp:103-138 (rank order)."""
    out = []
    for r in range(p ** 3):
        rows, c0, hl = activation_index(p, coords_of(p, r), batch, seq, g.shape[1], group)
        out.append(g[rows][:, c0:c0 + hl])
    return out


# ---------------------------------------------------------------- serial oracle
# cube3d/reference.hpp, float64.

def serial_matmul(a, b, form="AB"):
    """reference.hpp:24-55."""
    if form == "AB":
        return a @ b
    if form == "ABt":
        return a @ b.T
    return a.T @ b


def gelu(x):
    """nn.hpp:44-48: exact erf form."""
    return 0.5 * x * (1.0 + _erf(x * 0.7071067811865476))


def gelu_grad(x):
    """nn.hpp:50-56."""
    cdf = 0.5 * (1.0 + _erf(x * 0.7071067811865476))
    pdf = np.exp(-0.5 * x * x) * 0.3989422804014327
    return cdf + x * pdf


def layernorm_fwd(x, gamma, beta, eps):
    """reference.hpp:95-126: two-pass mean / centred variance."""
    h = x.shape[1]
    mean = x.sum(axis=1, keepdims=True) * (1.0 / h)
    d = x - mean
    inv = 1.0 / np.sqrt((d * d).sum(axis=1, keepdims=True) * (1.0 / h) + eps)
    xhat = d * inv
    return gamma * xhat + beta, (xhat, inv, gamma)


def layernorm_bwd(dy, cache):
    """reference.hpp:135-159."""
    xhat, inv, gamma = cache
    h = dy.shape[1]
    dbeta = dy.sum(axis=0)
    dgamma = (dy * xhat).sum(axis=0)
    dxh = dy * gamma
    rs = dxh.sum(axis=1, keepdims=True)
    rd = (dxh * xhat).sum(axis=1, keepdims=True)
    dx = inv * (dxh - rs * (1.0 / h) - xhat * rd * (1.0 / h))
    return dx, dgamma, dbeta


def cross_entropy_fwd(x, w, b, targets):
    """The loss row X1 of SURVEY.md §8(a) -- NOT IN THE REFERENCE (its only loss is
    <dY, Y>, cube3d/verify.hpp:611-617), so parity is unpinned by reference outputs: the
    linear is the reference's ref_linear_fwd (cube3d/reference.hpp:65-73), the
    log-softmax the max-shifted stable form, and tests/test_oracle_golden.py checks the
    gradients against central finite differences (the reference's finite_diff,
    cube3d/reference.hpp:389-405). -> (mean loss, cache)."""
    logits = x @ w + b
    m = logits.max(axis=1, keepdims=True)
    e = np.exp(logits - m)
    se = e.sum(axis=1, keepdims=True)
    n = x.shape[0]
    loss = float(np.mean(np.log(se[:, 0]) + m[:, 0] - logits[np.arange(n), targets]))
    return loss, (x, w, e / se, targets)


def cross_entropy_bwd(cache):
    """-> (dx, dw, db) of the mean loss."""
    x, w, p, targets = cache
    n = x.shape[0]
    dl = p.copy()
    dl[np.arange(n), targets] -= 1.0
    dl /= n
    return dl @ w.T, x.T @ dl, dl.sum(axis=0)


@dataclass
class LayerParams:
    """GlobalLayerParams (transformer.hpp:182-194), float64."""

    ln1_gamma: np.ndarray
    ln1_beta: np.ndarray
    w_qkv: np.ndarray
    b_qkv: np.ndarray
    w_out: np.ndarray
    b_out: np.ndarray
    ln2_gamma: np.ndarray
    ln2_beta: np.ndarray
    w_fc1: np.ndarray
    b_fc1: np.ndarray
    w_fc2: np.ndarray
    b_fc2: np.ndarray


FIELDS = ["ln1_gamma", "ln1_beta", "w_qkv", "b_qkv", "w_out", "b_out", "ln2_gamma", "ln2_beta",
          "w_fc1", "b_fc1", "w_fc2", "b_fc2"]


def init_layer_params(hidden: int, seed: int) -> LayerParams:
    """transformer.hpp:198-218: U[-0.1, 0.1], fixed draw order, gammas + 1."""
    rng = Rng(seed)
    h = hidden
    v = lambda n: rng.uniform(-0.1, 0.1, n)
    m = lambda r, c: rng.uniform(-0.1, 0.1, r * c).reshape(r, c)
    ln1g = v(h) + 1.0
    ln1b = v(h)
    wqkv = m(h, 3 * h)
    bqkv = v(3 * h)
    wout = m(h, h)
    bout = v(h)
    ln2g = v(h) + 1.0
    ln2b = v(h)
    w1 = m(h, 4 * h)
    b1 = v(4 * h)
    w2 = m(4 * h, h)
    b2 = v(h)
    return LayerParams(ln1g, ln1b, wqkv, bqkv, wout, bout, ln2g, ln2b, w1, b1, w2, b2)


# `rnd` (default identity) rounds every tensor a low-precision implementation
# stores (activations, probabilities, activation gradients) -- the test suite
# passes a bf16 round-to-nearest-even to emulate storage precision while keeping
# float64 arithmetic; weight/bias/LN-parameter gradients stay unrounded.
_ident = lambda a: a  # noqa: E731


def attention_fwd(x, P: LayerParams, batch, seq, heads, rnd=_ident, resid=None):
    """reference.hpp:174-213: fused QKV with head-major [head][q|k|v][dim] columns.
    `resid` (the layer's residual, transformer.hpp:120) is added before rounding."""
    h = x.shape[1]
    dh = h // heads
    scale = 1.0 / math.sqrt(dh)
    qkv = rnd(x @ P.w_qkv + P.b_qkv)
    t = qkv.reshape(batch, seq, heads, 3, dh)
    q, k, v = t[:, :, :, 0], t[:, :, :, 1], t[:, :, :, 2]           # [b, s, H, dh]
    scores = np.einsum("bihd,bjhd->bhij", q, k) * scale               # [b, H, s, s]
    m = scores.max(axis=-1, keepdims=True)
    e = np.exp(scores - m)
    probs = rnd(e / e.sum(axis=-1, keepdims=True))
    ctx = rnd(np.einsum("bhij,bjhd->bihd", probs, v).reshape(batch * seq, h))
    y = ctx @ P.w_out + P.b_out
    if resid is not None:
        y = y + resid
    return rnd(y), (x, qkv, probs, ctx)


def attention_bwd(dy, cache, P: LayerParams, batch, seq, heads, rnd=_ident):
    """reference.hpp:222-280."""
    x, qkv, probs, ctx = cache
    h = x.shape[1]
    dh = h // heads
    scale = 1.0 / math.sqrt(dh)
    dctx = rnd(dy @ P.w_out.T)
    dw_out = ctx.T @ dy
    db_out = dy.sum(axis=0)
    t = qkv.reshape(batch, seq, heads, 3, dh)
    q, k, v = t[:, :, :, 0], t[:, :, :, 1], t[:, :, :, 2]
    dc = dctx.reshape(batch, seq, heads, dh)
    dprobs = np.einsum("bihd,bjhd->bhij", dc, v)
    dv = rnd(np.einsum("bhij,bihd->bjhd", probs, dc))
    rowdot = (dprobs * probs).sum(axis=-1, keepdims=True)
    ds = rnd(probs * (dprobs - rowdot) * scale)
    dq = rnd(np.einsum("bhij,bjhd->bihd", ds, k))
    dk = rnd(np.einsum("bhij,bihd->bjhd", ds, q))
    dqkv = np.stack([dq, dk, dv], axis=3).reshape(batch * seq, 3 * h)
    dx = rnd(dqkv @ P.w_qkv.T)
    dw_qkv = x.T @ dqkv
    db_qkv = dqkv.sum(axis=0)
    return dx, dw_qkv, db_qkv, dw_out, db_out


def layer_fwd(x, P: LayerParams, batch, seq, heads, eps=1e-5, rnd=_ident):
    """reference.hpp:301-317 (pre-norm residual, transformer.hpp:115-128)."""
    n1, (xh1, inv1, g1) = layernorm_fwd(x, P.ln1_gamma, P.ln1_beta, eps)
    n1, ln1 = rnd(n1), (rnd(xh1), inv1, g1)
    y1, attn = attention_fwd(n1, P, batch, seq, heads, rnd, resid=x)
    n2, (xh2, inv2, g2) = layernorm_fwd(y1, P.ln2_gamma, P.ln2_beta, eps)
    n2, ln2 = rnd(n2), (rnd(xh2), inv2, g2)
    pre_full = n2 @ P.w_fc1 + P.b_fc1
    pre, hact = rnd(pre_full), rnd(gelu(pre_full))
    y = rnd(hact @ P.w_fc2 + P.b_fc2 + y1)
    return y, (ln1, attn, ln2, n2, pre, hact)


def layer_bwd(dy, cache, P: LayerParams, batch, seq, heads, rnd=_ident):
    """reference.hpp:325-354 -> (dx, LayerParams of gradients)."""
    ln1, attn, ln2, n2, pre, hact = cache
    dw2 = hact.T @ dy
    db2 = dy.sum(axis=0)
    dh = rnd((dy @ P.w_fc2.T) * gelu_grad(pre))
    dw1 = n2.T @ dh
    db1 = dh.sum(axis=0)
    dn2 = rnd(dh @ P.w_fc1.T)
    dxl2, dg2, db2n = layernorm_bwd(dn2, ln2)
    dy1 = rnd(dy + dxl2)
    dn1, dwqkv, dbqkv, dwout, dbout = attention_bwd(dy1, attn, P, batch, seq, heads, rnd)
    dxl1, dg1, db1n = layernorm_bwd(dn1, ln1)
    dx = rnd(dy1 + dxl1)
    return dx, LayerParams(dg1, db1n, dwqkv, dbqkv, dwout, dbout, dg2, db2n, dw1, db1, dw2, db2)


# ------------------------------------------------------------------ cost model
# cube3d/cost_model.hpp:54-165 (global element totals, sent == received).

def traffic_matmul(m, n, k, p):
    return (p - 1) * (m * n + n * k + m * k)


def traffic_diag_expand(n, p):
    return (p - 1) * n + (p - 1) * n * p


def traffic_diag_reduce(n, p):
    return 2 * (p - 1) * n * p


def traffic_layer(b, s, n_heads, h, p):
    """(fwd, bwd) of traffic::transformer_layer_fwd/bwd (cost_model.hpp:155-163)."""
    p3 = p ** 3
    rows = b * s
    rl = rows // (p * p)
    dh = h // n_heads
    lin_f = lambda hi, ho: traffic_matmul(rows, hi, ho, p) + traffic_diag_expand(ho, p)
    lin_b = lambda hi, ho: 2 * traffic_matmul(rows, hi, ho, p) + traffic_diag_reduce(ho, p)
    ln_f = 2 * p3 * (p - 1) * rl + 2 * traffic_diag_expand(h, p)
    ln_b = 2 * p3 * (p - 1) * rl + 2 * traffic_diag_reduce(h, p)
    slices = (b // p) * (n_heads // p)
    shard = (s // p) * dh
    core_f = p3 * slices * (p - 1) * (2 * shard + 2 * s)
    core_b = p3 * slices * (p - 1) * (2 * shard + s)
    fwd = 2 * ln_f + lin_f(h, 3 * h) + core_f + lin_f(h, h) + lin_f(h, 4 * h) + lin_f(4 * h, h)
    bwd = 2 * ln_b + lin_b(h, h) + core_b + lin_b(h, 3 * h) + lin_b(4 * h, h) + lin_b(h, 4 * h)
    return fwd, bwd


def layer_madds(b, s, n_heads, h, p):
    """madds::transformer_layer_fwd/bwd (cost_model.hpp:195-208), per rank."""
    rows = b * s
    mm = lambda m, n, k: (m // p) * (n // p) * (k // p)
    slices = (b // p) * (n_heads // p)
    core = slices * 2 * s * (s // p) * (h // n_heads)
    fwd = mm(rows, h, 3 * h) + core + mm(rows, h, h) + mm(rows, h, 4 * h) + mm(rows, 4 * h, h)
    return fwd, 2 * fwd


# ------------------------------------------------------------------ error metrics

def rel_err(got, want) -> float:
    """verify.hpp:268-279: max |got - want| / max(1, |want|)."""
    got = np.asarray(got, dtype=np.float64)
    want = np.asarray(want, dtype=np.float64)
    if got.shape != want.shape:
        return 1e300
    if want.size == 0:
        return 0.0
    return float((np.abs(got - want) / np.maximum(1.0, np.abs(want))).max())


def normwise_err(got, want) -> float:
    """||got - want||_2 / ||want||_2 (SURVEY.md §8(c) recommendation)."""
    got = np.asarray(got, dtype=np.float64)
    want = np.asarray(want, dtype=np.float64)
    den = np.linalg.norm(want)
    return float(np.linalg.norm(got - want) / (den if den > 0 else 1.0))
