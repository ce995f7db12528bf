"""Traffic accounting of this library's Transformer layer.

Every collective the library issues charges the rank's CostCounters with the reference's
ring convention (cube3d/counters.hpp:32-36): all_gather / reduce_scatter / all_reduce over
p ranks charge (p - 1) x the per-rank count to every member, a broadcast charges its root
(p - 1) x len. `layer_traffic` is the closed form of what one layer forward and backward
charge, summed over all ranks, on any supported px x py x pz grid (py == pz or one of them
1). The GPU tests compare it with the measured counters (zero unaccounted traffic, the
reference's check at cube3d/verify.hpp:671-682).

On a p x p x p cube the forward equals the reference's traffic::transformer_layer_fwd
(cube3d/cost_model.hpp:155-158) exactly. The backward moves less than
traffic::transformer_layer_bwd by the terms of `reference_deviation`, each a deliberate
reuse:

* ``reuse_weight_gather``  matmul_ab_bwd re-gathers B along x (ops3d.hpp:152); the layer
  gathers its four weights once per layer, packed, and the backward reuses them:
  - (p - 1) * Win * Wout per linear.
* ``reuse_input_gather``   matmul_ab_bwd re-gathers A for dB = A^T dC (ops3d.hpp:158); the
  forward's gathered input is kept: - (p - 1) * rows * Win per linear.
* ``reuse_output_grad_gather``  dC is gathered twice (ops3d.hpp:143, 161); once here:
  - (p - 1) * rows * Wout per linear.
* ``rowdot_gather``  the softmax backward all-reduces a full-length row dot per slice
  (attention.hpp:161-169, (p - 1) * s per slice and rank); here D = rowsum(dO * O) is
  computed for the rank's own query rows and all-gathered: (p - 1) * s / p per slice.

Packing (several vectors per broadcast / all-gather, the LayerNorm moments in one
all-gather instead of two all-reduces) changes call counts, not element counts.
"""
from __future__ import annotations

from typing import Dict, Sequence, Tuple


def _expand(P: int, Pi: int, Po: int, px: int, S: float) -> float:
    """expand_diagonal_multi over S packed slice elements (ops3d.cpp): total sent."""
    t = 0.0
    if Pi == Po and Pi > 1:
        t += (P / Pi) * (Pi - 1) * S  # one broadcast per input-axis line, root sends
    if px > 1:
        t += P * (px - 1) * S
    if Pi > Po:
        t += P * (Pi - 1) * S * px
    return t


def _reduce(P: int, Pi: int, Po: int, px: int, S: float) -> float:
    """reduce_to_diagonal_multi over S packed slice elements: total sent."""
    t = 0.0
    if Pi > Po:
        t += P * (Pi - 1) * S * px
    if px > 1:
        t += P * (px - 1) * S
    if Pi == Po and Pi > 1:
        t += P * (Pi - 1) * S
    return t


def layer_traffic(b: int, s: int, n: int, h: int, dims: Sequence[int],
                  flash: bool = True) -> Tuple[int, int]:
    """(forward, backward) elements sent, summed over all ranks, by one layer
    (transformer_layer_fwd / _bwd) with group-0 input. `flash`: the bf16 flash attention
    path (rowdot all-gathered); False: the unfused path (fp32-exact mode), whose softmax
    backward all-reduces the full row dot like the reference."""
    px, py, pz = (int(v) for v in dims)
    P = px * py * pz
    Q = max(py, pz)
    rows0 = (b // px) * (s // py)          # group-0 activation rows per rank
    rows1 = (b // px) * (s // pz)          # group-1 activation rows per rank
    T = 12 * h * h / P                     # packed weight shard elements
    S0 = 6 * h / (Q * px)                  # ln1 g|b, b_out, ln2 g|b, b_fc2 slices
    S1 = 7 * h / (Q * px)                  # b_qkv, b_fc1 slices
    H = n // py
    hd = H * (h // n)
    slices = (b // px) * H
    Ps = pz

    def lin_fwd(g_in, win, wout):
        # gather A along the input axis, reduce-scatter C along the output axis
        if g_in == 0:
            return P * (py - 1) * rows0 * win / pz + P * (pz - 1) * rows1 * wout / py
        return P * (pz - 1) * rows1 * win / py + P * (py - 1) * rows0 * wout / pz

    def lin_bwd(g_in, win, wout):
        # gather dC along the output axis, reduce-scatter dA along the input axis (dW below)
        if g_in == 0:
            return P * (pz - 1) * rows1 * wout / py + P * (py - 1) * rows0 * win / pz
        return P * (py - 1) * rows0 * wout / pz + P * (pz - 1) * rows1 * win / py

    ln = P * (pz - 1) * 2 * rows0
    fwd = (_expand(P, py, pz, px, S0) + _expand(P, pz, py, px, S1) + P * (px - 1) * T
           + 2 * ln + lin_fwd(0, h, 3 * h) + lin_fwd(1, h, h) + lin_fwd(0, h, 4 * h)
           + lin_fwd(1, 4 * h, h))
    if Ps > 1:
        fwd += P * (Ps - 1) * (2 * rows1 * hd + 2 * slices * s)
    bwd = (lin_bwd(1, 4 * h, h) + lin_bwd(0, h, 4 * h) + 2 * ln + lin_bwd(1, h, h)
           + lin_bwd(0, h, 3 * h) + _reduce(P, py, pz, px, S0) + _reduce(P, pz, py, px, S1)
           + P * (px - 1) * T)
    if Ps > 1:
        bwd += P * (Ps - 1) * (2 * rows1 * hd + slices * (s // Ps if flash else s))
    return int(round(fwd)), int(round(bwd))


def flash_applies(s: int, n: int, h: int, dims: Sequence[int], bf16: bool) -> bool:
    """Whether the layer's attention takes the flash kernels (flash_supported, flash.cu):
    bf16, head dim 64 / 128, queries and per-rank keys multiples of 128."""
    keys = s // int(dims[2])
    return bf16 and (h // n) in (64, 128) and s % 128 == 0 and keys % 128 == 0


def reference_deviation(b: int, s: int, n: int, h: int, p: int,
                        flash: bool = True) -> Dict[str, int]:
    """Named terms by which the backward's traffic is below the reference's
    traffic::transformer_layer_bwd on a p-cube (the forward has none)."""
    rows = b * s
    lins = [(h, 3 * h), (h, h), (h, 4 * h), (4 * h, h)]
    slices_per_rank = (b // p) * (n // p)
    return {
        "reuse_weight_gather": sum((p - 1) * wi * wo for wi, wo in lins),
        "reuse_input_gather": sum((p - 1) * rows * wi for wi, _ in lins),
        "reuse_output_grad_gather": sum((p - 1) * rows * wo for _, wo in lins),
        "rowdot_gather": p ** 3 * slices_per_rank * (p - 1) * (s - s // p) if flash else 0,
    }


def layer_madds(b: int, s: int, n: int, h: int, p: int) -> Tuple[int, int]:
    """Per-rank multiply-adds of one layer (fwd, bwd) on a p-cube: madds::transformer_layer_*
    (cube3d/cost_model.hpp:172-208); the library charges the same counts."""
    rows = b * s
    mm = lambda m, k, nn: (m // p) * (k // p) * (nn // p)  # noqa: E731
    slices = (b // p) * (n // p)
    core = slices * 2 * s * (s // p) * (h // n)
    fwd = mm(rows, h, 3 * h) + core + mm(rows, h, h) + mm(rows, h, 4 * h) + mm(rows, 4 * h, h)
    return fwd, 2 * fwd


def scaling_rows(mode: str, b: int, s: int, n: int, h: int, layers: int, p_list: Sequence[int],
                 lam: float = 1.0, reference_traffic: bool = False):
    """The CLI bench table (cube3d/bench.hpp:41-93): modeled cost units per rank per step
    (multiply-adds + lam x communicated elements) for each cube side; weak scaling grows
    batch x p, hidden x p^2, heads x p. `reference_traffic`: charge the reference's traffic
    model (this library's plus the documented reuse terms) instead of this library's."""
    rows = []
    for p in p_list:
        if p < 1:
            raise ValueError("cube side must be positive")
        bb, hh, nn = (b * p, h * p * p, n * p) if mode == "weak" else (b, h, n)
        # TransformerConfig::validate (cube3d/nn.hpp:29-40)
        if bb % p or s % p or hh % (p * p) or (4 * hh) % (p * p) or nn % p or hh % nn:
            raise ValueError(f"configuration (b={bb}, s={s}, heads={nn}, h={hh}) is not "
                             f"divisible on the p={p} cube")
        f, bw = layer_traffic(bb, s, nn, hh, (p, p, p),
                              flash=flash_applies(s, nn, hh, (p, p, p), True))
        if reference_traffic and p > 1:
            bw += sum(reference_deviation(bb, s, nn, hh, p, flash_applies(s, nn, hh, (p, p, p),
                                                                          True)).values())
        p3 = p ** 3
        mf, mb = layer_madds(bb, s, nn, hh, p)
        fc = layers * (mf + lam * (f // p3))
        bc = layers * (mb + lam * (bw // p3))
        rows.append((p3, bb, hh, float(fc), float(bc), (fc + bc) / bb))
    return rows


def scaling_csv(rows) -> str:
    out = ["gpus,batch,hidden,forward_cost,backward_cost,avg_step_cost"]
    for g, b, h, f, bw, a in rows:
        out.append(f"{g},{b},{h},{f:.6f},{bw:.6f},{a:.6f}")
    return "\n".join(out) + "\n"
