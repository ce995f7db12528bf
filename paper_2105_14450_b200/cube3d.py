"""Python mirror of the reference ``cube3d`` operator API over the C ABI.

Names, argument meaning and error behaviour follow the reference headers
(/root/reference/proj/include/cube3d/*.hpp, cited per function) so callers and
parity tests read like the reference's own. Device tensors are torch CUDA
tensors (plumbing only); every op runs in ``libc3d.so`` -- sm_100a kernels and
NCCL over NVLink. Host-side placement helpers (partition/collect, the
"test/CLI side of the transport", cube3d/sharding.hpp:49-98) use numpy.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import List, Optional, Sequence, Tuple

import numpy as np

from . import _lib as L
from ._lib import C3DError, call, lib

# ------------------------------------------------------------------ enums

X, Y, Z = 0, 1, 2  # Axis (cube3d/topology.hpp:15)
INPUT, WEIGHT, OUTPUT, WEIGHT_OF_TRANSPOSE = 0, 1, 2, 3  # Layout (cube3d/layout.hpp:29)
F32, BF16 = L.F32, L.BF16
MODE_AUTO, MODE_TC, MODE_F32 = L.MODE_AUTO, L.MODE_TC, L.MODE_F32
LAYOUT_NAMES = {0: "Input", 1: "Weight", 2: "Output", 3: "WeightOfTranspose"}


@dataclass(frozen=True)
class DirectionTriple:
    """cube3d/layout.hpp:44-61: gather axes of input / weight, scatter axis of output."""

    input: int = Y
    weight: int = X
    output: int = Z

    def swapped(self) -> "DirectionTriple":
        return DirectionTriple(self.output, self.weight, self.input)

    def as_c(self):
        return (C.c_int * 3)(self.input, self.weight, self.output)


def canonical_directions() -> DirectionTriple:
    return DirectionTriple(Y, X, Z)


def default_directions(layout: int) -> DirectionTriple:
    """cube3d/layout.hpp:67-69: Output comes out of the canonical matmul swapped."""
    return canonical_directions().swapped() if layout == OUTPUT else canonical_directions()


def axis_of_group(group: int) -> int:
    """cube3d/activation.hpp:28-31."""
    if group not in (0, 1):
        raise C3DError(10, "GroupMismatch: group index must be 0 or 1")
    return Y if group == 0 else Z


def triple_for_group(group: int) -> DirectionTriple:
    """cube3d/activation.hpp:33-35: group 0 -> (y,x,z), group 1 -> (z,x,y)."""
    return DirectionTriple(axis_of_group(group), X, axis_of_group(1 - group))


@dataclass
class GroupState:
    """cube3d/activation.hpp:20-26."""

    input_group: int = 0

    def toggle(self) -> None:
        self.input_group = 1 - self.input_group


def _i3(v: Sequence[int]):
    return (C.c_int * 3)(*[int(t) for t in v])


# ------------------------------------------------------------ topology

def rank_of(dims, coords) -> int:
    r = C.c_int()
    call("c3d_grid_rank_of", _i3(dims), _i3(coords), C.byref(r))
    return r.value


def coords_of(dims, rank: int) -> Tuple[int, int, int]:
    out = (C.c_int * 3)()
    call("c3d_grid_coords_of", _i3(dims), int(rank), out)
    return tuple(out)


def axis_group(dims, rank: int, axis: int) -> Tuple[List[int], int]:
    """CubeTopology::axis_group (cube3d/topology.hpp:79-95): (members, my_position)."""
    n = int(dims[axis]) if 0 <= axis < 3 else 1
    m = (C.c_int * max(n, 1))()
    pos = C.c_int()
    call("c3d_grid_axis_group", _i3(dims), int(rank), int(axis), m, C.byref(pos))
    return list(m)[:n], pos.value


def line_index(dims, rank: int, axis: int) -> int:
    out = C.c_int()
    call("c3d_grid_line_index", _i3(dims), int(rank), int(axis), C.byref(out))
    return out.value


def build_cube(total_ranks: int) -> int:
    out = C.c_int()
    call("c3d_build_cube", int(total_ranks), C.byref(out))
    return out.value


def grid_for(n_gpus: int) -> Tuple[int, int, int]:
    """Grid used for n GPUs (north star): 1 -> 1x1x1, 2 -> 2x1x1, 4 -> 2x2x1 sub-cubes,
    8 -> the 2x2x2 cube."""
    table = {1: (1, 1, 1), 2: (2, 1, 1), 4: (2, 2, 1), 8: (2, 2, 2)}
    if n_gpus in table:
        return table[n_gpus]
    p = build_cube(n_gpus)
    return (p, p, p)


# ------------------------------------------------------------ layouts

def shard_bounds(layout: int, dims, coords, rows: int, cols: int,
                 dirs: Optional[DirectionTriple] = None):
    """cube3d/layout.hpp:93-123 -> ((row_begin, row_end), (col_begin, col_end))."""
    d = dirs or default_directions(layout)
    out = (C.c_int64 * 4)()
    call("c3d_shard_bounds", int(layout), _i3(dims), _i3(coords), int(rows), int(cols), d.as_c(),
         out)
    return (out[0], out[1]), (out[2], out[3])


def diagonal_slice(dims, coords, n: int):
    """cube3d/layout.hpp:134-142 -> (holds, (begin, end))."""
    holds = C.c_int()
    out = (C.c_int64 * 2)()
    call("c3d_diagonal_slice", _i3(dims), _i3(coords), int(n), C.byref(holds), out)
    return bool(holds.value), (out[0], out[1])


def activation_rows(dims, coords, batch, seq, hidden, group):
    """Index map of activation_from_global (cube3d/activation.hpp:119-134)."""
    dummy = np.zeros(1, dtype=np.int64)
    cb, lc = C.c_int64(), C.c_int64()
    call("c3d_activation_rows", _i3(dims), _i3(coords), int(batch), int(seq), int(hidden),
         int(group), None, C.byref(cb), C.byref(lc))
    px, pin = dims[0], dims[axis_of_group(group)]
    n = (batch // px) * (seq // pin)
    rows = np.zeros(max(n, 1), dtype=np.int64) if n else dummy
    call("c3d_activation_rows", _i3(dims), _i3(coords), int(batch), int(seq), int(hidden),
         int(group), rows.ctypes.data_as(C.POINTER(C.c_int64)), None, None)
    return rows[:n], cb.value, lc.value


def _ranks(dims):
    return [coords_of(dims, r) for r in range(dims[0] * dims[1] * dims[2])]


def partition(gm: np.ndarray, layout: int, dims, dirs: Optional[DirectionTriple] = None):
    """cube3d/sharding.hpp:51-77: one shard per rank (rank order)."""
    out = []
    for c in _ranks(dims):
        (r0, r1), (c0, c1) = shard_bounds(layout, dims, c, gm.shape[0], gm.shape[1], dirs)
        out.append(np.ascontiguousarray(gm[r0:r1, c0:c1]))
    return out


def collect(shards, layout: int, dims, rows: int, cols: int,
            dirs: Optional[DirectionTriple] = None) -> np.ndarray:
    """cube3d/sharding.hpp:80-98."""
    if len(shards) != dims[0] * dims[1] * dims[2]:
        raise C3DError(6, f"InconsistentFamily: family has {len(shards)} shards")
    gm = np.zeros((rows, cols), dtype=np.asarray(shards[0]).dtype)
    for c, s in zip(_ranks(dims), shards):
        (r0, r1), (c0, c1) = shard_bounds(layout, dims, c, rows, cols, dirs)
        s = np.asarray(s)
        if s.shape != (r1 - r0, c1 - c0):
            raise C3DError(6, "InconsistentFamily: shard shape does not match its bounds")
        gm[r0:r1, c0:c1] = s
    return gm


def partition_diagonal(vec: np.ndarray, dims):
    """cube3d/sharding.hpp:100-119 (empty off the diagonal)."""
    out = []
    for c in _ranks(dims):
        holds, (b, e) = diagonal_slice(dims, c, len(vec))
        out.append(np.ascontiguousarray(vec[b:e]) if holds else vec[:0].copy())
    return out


def collect_diagonal(family, dims, n: int) -> np.ndarray:
    """cube3d/sharding.hpp:121-146."""
    out = np.zeros(n, dtype=np.float64)
    seen = np.zeros(n, dtype=bool)
    for c, s in zip(_ranks(dims), family):
        holds, (b, e) = diagonal_slice(dims, c, n)
        if not holds:
            continue
        if seen[b:e].any():
            raise C3DError(6, "InconsistentFamily: diagonal slices overlap")
        seen[b:e] = True
        out[b:e] = np.asarray(s, dtype=np.float64)
    if not seen.all():
        raise C3DError(6, "InconsistentFamily: diagonal slices do not cover the vector")
    return out


def activation_from_global(gm: np.ndarray, batch: int, seq: int, group: int, dims):
    """cube3d/activation.hpp:103-138."""
    out = []
    for c in _ranks(dims):
        rows, cb, lc = activation_rows(dims, c, batch, seq, gm.shape[1], group)
        out.append(np.ascontiguousarray(gm[rows][:, cb:cb + lc]))
    return out


def activation_to_global(locals_, batch: int, seq: int, hidden: int, group: int, dims):
    """cube3d/activation.hpp:141-164."""
    gm = np.zeros((batch * seq, hidden), dtype=np.asarray(locals_[0]).dtype)
    for c, a in zip(_ranks(dims), locals_):
        rows, cb, lc = activation_rows(dims, c, batch, seq, hidden, group)
        gm[rows, cb:cb + lc] = np.asarray(a)
    return gm


# ------------------------------------------------------------ rng

class Rng:
    """cube3d/rng.hpp:17-34 (mt19937_64, 53-bit unit mapping), host side in libc3d."""

    def __init__(self, seed: int):
        self._h = C.c_void_p()
        call("c3d_rng_create", C.c_uint64(seed & (2**64 - 1)), C.byref(self._h))

    def __del__(self):
        try:
            if self._h:
                lib().c3d_rng_destroy(self._h)
        except Exception:
            pass

    def next_u64(self, n: int = 1) -> np.ndarray:
        out = np.zeros(n, dtype=np.uint64)
        call("c3d_rng_next_u64", self._h, out.ctypes.data_as(C.POINTER(C.c_uint64)), n)
        return out

    def uniform(self, lo: float, hi: float, n: int) -> np.ndarray:
        out = np.zeros(n, dtype=np.float64)
        call("c3d_rng_uniform", self._h, lo, hi, out.ctypes.data_as(C.POINTER(C.c_double)), n)
        return out

    def below(self, bound: int, n: int) -> np.ndarray:
        out = np.zeros(n, dtype=np.float64)
        call("c3d_rng_below", self._h, C.c_uint64(bound), out.ctypes.data_as(C.POINTER(C.c_double)),
             n)
        return out


def random_matrix(rows, cols, rng: Rng, lo=-1.0, hi=1.0) -> np.ndarray:
    return rng.uniform(lo, hi, rows * cols).reshape(rows, cols)


def random_integer_matrix(rows, cols, rng: Rng, bound=10) -> np.ndarray:
    return rng.below(bound, rows * cols).reshape(rows, cols)


def random_vector(n, rng: Rng, lo=-1.0, hi=1.0) -> np.ndarray:
    return rng.uniform(lo, hi, n)


# ------------------------------------------------------------ device tensors

def _torch():
    import torch
    return torch


def torch_dtype(dt: int):
    torch = _torch()
    return torch.float32 if dt == F32 else torch.bfloat16


def c3d_dtype(t) -> int:
    torch = _torch()
    if t.dtype == torch.float32:
        return F32
    if t.dtype == torch.bfloat16:
        return BF16
    raise C3DError(12, f"ConfigInvalid: unsupported dtype {t.dtype}")


def _stream(stream=None):
    torch = _torch()
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


@dataclass
class ShardedMatrix:
    """cube3d/sharding.hpp:18-34 with a device-resident shard."""

    shard: object  # torch tensor, local rows x cols, contiguous
    global_rows: int
    global_cols: int
    layout: int
    dirs: DirectionTriple

    def c(self) -> L.c3d_matrix:
        m = L.c3d_matrix()
        m.data = self.shard.data_ptr() if self.shard.numel() else None
        m.dtype = c3d_dtype(self.shard)
        m.global_rows = self.global_rows
        m.global_cols = self.global_cols
        m.layout = self.layout
        m.dirs = (C.c_int * 3)(self.dirs.input, self.dirs.weight, self.dirs.output)
        return m


@dataclass
class DiagonalVector:
    """cube3d/sharding.hpp:38-47 (shard empty off the diagonal)."""

    shard: object
    global_len: int

    def c(self) -> L.c3d_vector:
        v = L.c3d_vector()
        v.data = self.shard.data_ptr() if self.shard.numel() else None
        v.dtype = c3d_dtype(self.shard)
        v.global_len = self.global_len
        return v


@dataclass
class Activation3D:
    """cube3d/activation.hpp:41-62: local [(b/px)(s/p_in), h/p_out]."""

    local: object
    batch: int
    seq: int
    hidden: int
    group: int

    def c(self) -> L.c3d_activation:
        a = L.c3d_activation()
        a.data = self.local.data_ptr() if self.local.numel() else None
        a.dtype = c3d_dtype(self.local)
        a.batch, a.seq, a.hidden, a.group = self.batch, self.seq, self.hidden, self.group
        return a


def _empty(shape, dt: int, device):
    torch = _torch()
    return torch.empty(shape, dtype=torch_dtype(dt), device=device)


# ------------------------------------------------------------ the cube

class Cube:
    """One rank's handle (the reference Endpoint, cube3d/transport.hpp:138-290)."""

    def __init__(self, dims=(1, 1, 1), rank: int = 0, device: int = 0,
                 uid: Optional[bytes] = None):
        self.dims = tuple(int(d) for d in dims)
        self.rank = int(rank)
        self.device = int(device)
        self._h = C.c_void_p()
        buf = C.create_string_buffer(uid, 128) if uid is not None else None
        call("c3d_cube_create", _i3(self.dims), self.rank, self.device, buf, C.byref(self._h))
        self.coords = coords_of(self.dims, self.rank)

    @staticmethod
    def unique_id() -> bytes:
        buf = C.create_string_buffer(128)
        call("c3d_unique_id", buf)
        return buf.raw

    def close(self):
        if self._h:
            call("c3d_cube_destroy", self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def handle(self):
        return self._h

    def p(self, axis: int) -> int:
        return self.dims[axis]

    def barrier(self, stream=None):
        call("c3d_cube_barrier", self._h, _stream(stream))

    def check(self, stream=None):
        """c3d_cube_check: synchronise and raise C3DError("Desync", ...) when a peer wait of
        this cube failed (timeout or mismatched collective header)."""
        call("c3d_cube_check", self._h, _stream(stream))

    def counters(self) -> dict:
        c = L.c3d_counters()
        call("c3d_counters_get", self._h, C.byref(c))
        return {"elements_sent": c.elements_sent, "elements_received": c.elements_received,
                "sent_by_kind": list(c.sent_by_kind), "received_by_kind": list(c.received_by_kind),
                "calls_by_kind": list(c.calls_by_kind), "multiply_adds": c.multiply_adds}

    def reset_counters(self):
        call("c3d_counters_reset", self._h)

    # --- Endpoint collectives along one axis (cube3d/transport.hpp:160-257)
    def broadcast(self, axis: int, root_position: int, buf, stream=None):
        """In place: every member of the axis line receives root_position's buf."""
        call("c3d_broadcast", self._h, axis, root_position, C.c_void_p(buf.data_ptr()),
             buf.numel(), c3d_dtype(buf), _stream(stream))
        return buf

    def all_gather(self, axis: int, shard, stream=None, out=None):
        """-> (p * numel,) tensor (or `out`): the members' shards in ascending position
        order."""
        torch = _torch()
        if out is None:
            out = torch.empty(self.dims[axis] * shard.numel(), dtype=shard.dtype,
                              device=shard.device)
        call("c3d_all_gather", self._h, axis, C.c_void_p(shard.data_ptr()),
             C.c_void_p(out.data_ptr()), shard.numel(), c3d_dtype(shard), _stream(stream))
        return out

    def reduce_scatter(self, axis: int, full, stream=None):
        """full holds p equal blocks; -> this position's block of the elementwise sum."""
        torch = _torch()
        p = self.dims[axis]
        if full.numel() % p:
            raise C3DError(3, f"LengthMismatch: {full.numel()} elements not divisible by {p}")
        out = torch.empty(full.numel() // p, dtype=full.dtype, device=full.device)
        call("c3d_reduce_scatter", self._h, axis, C.c_void_p(full.data_ptr()),
             C.c_void_p(out.data_ptr()), out.numel(), c3d_dtype(full), _stream(stream))
        return out

    def all_reduce(self, axis: int, buf, op: str = "sum", stream=None):
        """In place sum (or max) over the axis line."""
        call("c3d_all_reduce", self._h, axis, C.c_void_p(buf.data_ptr()), buf.numel(),
             c3d_dtype(buf), 1 if op == "max" else 0, _stream(stream))
        return buf

    def device_str(self):
        return f"cuda:{self.device}"

    # --- placement helpers for this rank
    def bounds(self, layout, rows, cols, dirs=None):
        return shard_bounds(layout, self.dims, self.coords, rows, cols, dirs)

    def local_shape(self, layout, rows, cols, dirs=None):
        (r0, r1), (c0, c1) = self.bounds(layout, rows, cols, dirs)
        return (r1 - r0, c1 - c0)

    def act_shape(self, batch, seq, hidden, group):
        _, _, lc = activation_rows(self.dims, self.coords, batch, seq, hidden, group)
        pin = self.dims[axis_of_group(group)]
        return ((batch // self.dims[0]) * (seq // pin), lc)

    def diag_len(self, n):
        holds, (b, e) = diagonal_slice(self.dims, self.coords, n)
        return (e - b) if holds else 0


def shard_to_device(cube: Cube, gm: np.ndarray, layout: int, dtype: int,
                    dirs: Optional[DirectionTriple] = None) -> ShardedMatrix:
    """This rank's shard of a global host matrix, uploaded (host-side test/CLI helper)."""
    torch = _torch()
    (r0, r1), (c0, c1) = cube.bounds(layout, gm.shape[0], gm.shape[1], dirs)
    t = torch.tensor(np.ascontiguousarray(gm[r0:r1, c0:c1]), dtype=torch.float64)
    return ShardedMatrix(t.to(device=cube.device_str(), dtype=torch_dtype(dtype)).contiguous(),
                         gm.shape[0], gm.shape[1], layout, dirs or default_directions(layout))


def vector_to_device(cube: Cube, vec: np.ndarray, dtype: int) -> DiagonalVector:
    torch = _torch()
    holds, (b, e) = diagonal_slice(cube.dims, cube.coords, len(vec))
    part = vec[b:e] if holds else vec[:0]
    t = torch.tensor(np.ascontiguousarray(part), dtype=torch.float64)
    return DiagonalVector(t.to(device=cube.device_str(), dtype=torch_dtype(dtype)), len(vec))


def activation_to_device(cube: Cube, gm: np.ndarray, batch, seq, group, dtype) -> Activation3D:
    torch = _torch()
    rows, cb, lc = activation_rows(cube.dims, cube.coords, batch, seq, gm.shape[1], group)
    t = torch.tensor(np.ascontiguousarray(gm[rows][:, cb:cb + lc]), dtype=torch.float64)
    return Activation3D(t.to(device=cube.device_str(), dtype=torch_dtype(dtype)).contiguous(),
                        batch, seq, gm.shape[1], group)


# ------------------------------------------------------------ 3-D matmuls

def _out_matrix(cube: Cube, rows, cols, layout, dirs, dtype) -> ShardedMatrix:
    shape = cube.local_shape(layout, rows, cols, dirs)
    return ShardedMatrix(_empty(shape, dtype, cube.device_str()), rows, cols, layout, dirs)


def _fwd(name, cube, a, b, c, mode, stream):
    ca, cb, cc = a.c(), b.c(), c.c()
    call(name, cube.handle, mode, C.byref(ca), C.byref(cb), C.byref(cc), _stream(stream))
    return c


def matmul_ab_fwd(cube: Cube, a: ShardedMatrix, b: ShardedMatrix, mode=MODE_AUTO,
                  out_dtype: Optional[int] = None, stream=None) -> ShardedMatrix:
    """cube3d/ops3d.hpp:114-132: C = A B, Output layout with the swapped triple."""
    dt = c3d_dtype(a.shard) if out_dtype is None else out_dtype
    c = _out_matrix(cube, a.global_rows, b.global_cols, OUTPUT, a.dirs.swapped(), dt)
    return _fwd("c3d_matmul_ab_fwd", cube, a, b, c, mode, stream)


def matmul_abt_fwd(cube, a, b, mode=MODE_AUTO, out_dtype=None, stream=None):
    """cube3d/ops3d.hpp:174-193: C = A B^T."""
    dt = c3d_dtype(a.shard) if out_dtype is None else out_dtype
    c = _out_matrix(cube, a.global_rows, b.global_rows, OUTPUT, a.dirs.swapped(), dt)
    return _fwd("c3d_matmul_abt_fwd", cube, a, b, c, mode, stream)


def matmul_atb_fwd(cube, a, b, mode=MODE_AUTO, out_dtype=None, stream=None):
    """cube3d/ops3d.hpp:230-249: C = A^T B, Weight layout under A's triple."""
    dt = c3d_dtype(a.shard) if out_dtype is None else out_dtype
    c = _out_matrix(cube, a.global_cols, b.global_cols, WEIGHT, a.dirs, dt)
    return _fwd("c3d_matmul_atb_fwd", cube, a, b, c, mode, stream)


def _bwd(name, cube, dc, a, b, mode, out_dtype, stream):
    dt = c3d_dtype(dc.shard) if out_dtype is None else out_dtype
    da = _out_matrix(cube, a.global_rows, a.global_cols, a.layout, a.dirs, dt)
    db = _out_matrix(cube, b.global_rows, b.global_cols, b.layout, b.dirs, dt)
    cdc, ca, cb, cda, cdb = dc.c(), a.c(), b.c(), da.c(), db.c()
    call(name, cube.handle, mode, C.byref(cdc), C.byref(ca), C.byref(cb), C.byref(cda),
         C.byref(cdb), _stream(stream))
    return da, db


def matmul_ab_bwd(cube, dc, a, b, mode=MODE_AUTO, out_dtype=None, stream=None):
    """cube3d/ops3d.hpp:137-168 -> (dA, dB)."""
    return _bwd("c3d_matmul_ab_bwd", cube, dc, a, b, mode, out_dtype, stream)


def matmul_abt_bwd(cube, dc, a, b, mode=MODE_AUTO, out_dtype=None, stream=None):
    """cube3d/ops3d.hpp:196-223."""
    return _bwd("c3d_matmul_abt_bwd", cube, dc, a, b, mode, out_dtype, stream)


def matmul_atb_bwd(cube, dc, a, b, mode=MODE_AUTO, out_dtype=None, stream=None):
    """cube3d/ops3d.hpp:252-277."""
    return _bwd("c3d_matmul_atb_bwd", cube, dc, a, b, mode, out_dtype, stream)


# ------------------------------------------------------------ batched matmuls
# cube3d/ops3d.hpp:418-494 (BatchedShardedMatrix = a list of ShardedMatrix slices)

_FWD_SHAPE = {"ab": lambda a, b: (a.global_rows, b.global_cols, OUTPUT, a.dirs.swapped()),
              "abt": lambda a, b: (a.global_rows, b.global_rows, OUTPUT, a.dirs.swapped()),
              "atb": lambda a, b: (a.global_cols, b.global_cols, WEIGHT, a.dirs)}


def _arr(ms):
    return (L.c3d_matrix * max(1, len(ms)))(*[m.c() for m in ms])


def batched_matmul_fwd(form: str, cube: Cube, a: Sequence[ShardedMatrix],
                       b: Sequence[ShardedMatrix], mode=MODE_AUTO, out_dtype=None, stream=None):
    """batched_matmul_{ab,abt,atb}_fwd: one 3-D product per slice; BatchMismatch when the
    slice counts differ."""
    outs = []
    for x, y in zip(a, b):
        r, c, lay, d = _FWD_SHAPE[form](x, y)
        dt = c3d_dtype(x.shard) if out_dtype is None else out_dtype
        outs.append(_out_matrix(cube, r, c, lay, d, dt))
    ca, cb, cc = _arr(a), _arr(b), _arr(outs)
    call(f"c3d_batched_matmul_{form}_fwd", cube.handle, mode, len(a), ca, len(b), cb, cc,
         _stream(stream))
    return outs


def batched_matmul_bwd(form: str, cube: Cube, dc, a, b, mode=MODE_AUTO, out_dtype=None,
                       stream=None):
    """batched_matmul_{ab,abt,atb}_bwd -> (list of dA, list of dB)."""
    das, dbs = [], []
    for g, x, y in zip(dc, a, b):
        dt = c3d_dtype(g.shard) if out_dtype is None else out_dtype
        das.append(_out_matrix(cube, x.global_rows, x.global_cols, x.layout, x.dirs, dt))
        dbs.append(_out_matrix(cube, y.global_rows, y.global_cols, y.layout, y.dirs, dt))
    call(f"c3d_batched_matmul_{form}_bwd", cube.handle, mode, len(dc), _arr(dc), len(a), _arr(a),
         len(b), _arr(b), _arr(das), _arr(dbs), _stream(stream))
    return das, dbs


# ------------------------------------------------------------ vector ops

def _vec_out(cube, n, dtype):
    return DiagonalVector(_empty((cube.diag_len(n),), dtype, cube.device_str()), n)


def add_vec_fwd(cube, a: ShardedMatrix, b: DiagonalVector, stream=None) -> ShardedMatrix:
    """cube3d/ops3d.hpp:347-357."""
    c = _out_matrix(cube, a.global_rows, a.global_cols, a.layout, a.dirs, c3d_dtype(a.shard))
    ca, cb, cc = a.c(), b.c(), c.c()
    call("c3d_add_vec_fwd", cube.handle, C.byref(ca), C.byref(cb), C.byref(cc), _stream(stream))
    return c


def add_vec_bwd(cube, dc: ShardedMatrix, db_dtype=F32, stream=None):
    """cube3d/ops3d.hpp:361-372 -> (dA, db)."""
    da = _out_matrix(cube, dc.global_rows, dc.global_cols, dc.layout, dc.dirs, c3d_dtype(dc.shard))
    db = _vec_out(cube, dc.global_cols, db_dtype)
    cdc, cda, cdb = dc.c(), da.c(), db.c()
    call("c3d_add_vec_bwd", cube.handle, C.byref(cdc), C.byref(cda), C.byref(cdb), _stream(stream))
    return da, db


def mul_vec_fwd(cube, a, b, stream=None):
    """cube3d/ops3d.hpp:382-396."""
    c = _out_matrix(cube, a.global_rows, a.global_cols, a.layout, a.dirs, c3d_dtype(a.shard))
    ca, cb, cc = a.c(), b.c(), c.c()
    call("c3d_mul_vec_fwd", cube.handle, C.byref(ca), C.byref(cb), C.byref(cc), _stream(stream))
    return c


def mul_vec_bwd(cube, dc, a, b, db_dtype=F32, stream=None):
    """cube3d/ops3d.hpp:401-416 (re-expands b instead of a saved copy) -> (dA, db)."""
    da = _out_matrix(cube, dc.global_rows, dc.global_cols, dc.layout, dc.dirs, c3d_dtype(dc.shard))
    db = _vec_out(cube, dc.global_cols, db_dtype)
    cdc, ca, cb, cda, cdb = dc.c(), a.c(), b.c(), da.c(), db.c()
    call("c3d_mul_vec_bwd", cube.handle, C.byref(cdc), C.byref(ca), C.byref(cb), C.byref(cda),
         C.byref(cdb), _stream(stream))
    return da, db


# ------------------------------------------------------------ NN blocks

@dataclass
class TransformerConfig:
    """cube3d/nn.hpp:16-41."""

    batch: int
    seq: int
    heads: int
    hidden: int
    layers: int = 1
    eps: float = 1e-5

    def head_dim(self) -> int:
        return self.hidden // self.heads

    def c(self) -> L.c3d_config:
        return L.c3d_config(self.batch, self.seq, self.heads, self.hidden, self.eps)


class Saved:
    """Opaque saved-for-backward state (library-owned device buffers)."""

    def __init__(self, handle):
        self._h = handle

    def __del__(self):
        try:
            if self._h:
                lib().c3d_saved_free(self._h)
        except Exception:
            pass


@dataclass
class GlobalLayerParams:
    """cube3d/transformer.hpp:182-194 (host, float64)."""

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


def init_layer_params(cfg: TransformerConfig, seed: int) -> GlobalLayerParams:
    """cube3d/transformer.hpp:198-218: U[-0.1, 0.1] in a fixed draw order, gammas + 1."""
    rng = Rng(seed)
    h = cfg.hidden
    vec = lambda n: rng.uniform(-0.1, 0.1, n)
    mat = lambda r, c: rng.uniform(-0.1, 0.1, r * c).reshape(r, c)
    ln1_gamma = vec(h) + 1.0
    ln1_beta = vec(h)
    w_qkv = mat(h, 3 * h)
    b_qkv = vec(3 * h)
    w_out = mat(h, h)
    b_out = vec(h)
    ln2_gamma = vec(h) + 1.0
    ln2_beta = vec(h)
    w_fc1 = mat(h, 4 * h)
    b_fc1 = vec(4 * h)
    w_fc2 = mat(4 * h, h)
    b_fc2 = vec(h)
    return GlobalLayerParams(ln1_gamma, ln1_beta, w_qkv, b_qkv, w_out, b_out, ln2_gamma, ln2_beta,
                             w_fc1, b_fc1, w_fc2, b_fc2)


@dataclass
class LayerParams:
    """One rank's LayerParams (cube3d/transformer.hpp:78-85); also used for grads."""

    ln1_gamma: DiagonalVector
    ln1_beta: DiagonalVector
    w_qkv: ShardedMatrix
    b_qkv: DiagonalVector
    w_out: ShardedMatrix
    b_out: DiagonalVector
    ln2_gamma: DiagonalVector
    ln2_beta: DiagonalVector
    w_fc1: ShardedMatrix
    b_fc1: DiagonalVector
    w_fc2: ShardedMatrix
    b_fc2: DiagonalVector

    def c(self) -> L.c3d_layer_params:
        p = L.c3d_layer_params()
        for n in L.LAYER_FIELDS:
            setattr(p, n, getattr(self, n).c())
        return p


def partition_layer_params(cube: Cube, gp: GlobalLayerParams, input_group: int = 0,
                           dtype: int = BF16, vec_dtype: int = F32) -> LayerParams:
    """cube3d/transformer.hpp:223-254 for this rank: QKV/FC1 under the input triple,
    OUT/FC2 under the swapped triple, vectors on the diagonal."""
    d_in, d_sw = triple_for_group(input_group), triple_for_group(1 - input_group)
    W = lambda m, d: shard_to_device(cube, m, WEIGHT, dtype, d)
    V = lambda v: vector_to_device(cube, v, vec_dtype)
    return LayerParams(V(gp.ln1_gamma), V(gp.ln1_beta), W(gp.w_qkv, d_in), V(gp.b_qkv),
                       W(gp.w_out, d_sw), V(gp.b_out), V(gp.ln2_gamma), V(gp.ln2_beta),
                       W(gp.w_fc1, d_in), V(gp.b_fc1), W(gp.w_fc2, d_sw), V(gp.b_fc2))


def empty_like_params(cube: Cube, p: LayerParams, dtype: Optional[int] = None,
                      vec_dtype: int = F32) -> LayerParams:
    torch = _torch()
    out = {}
    for n in L.LAYER_FIELDS:
        f = getattr(p, n)
        if isinstance(f, ShardedMatrix):
            dt = torch_dtype(dtype) if dtype is not None else f.shard.dtype
            out[n] = ShardedMatrix(torch.empty_like(f.shard, dtype=dt), f.global_rows,
                                   f.global_cols, f.layout, f.dirs)
        else:
            out[n] = DiagonalVector(torch.empty(f.shard.shape, dtype=torch_dtype(vec_dtype),
                                                device=f.shard.device), f.global_len)
    return LayerParams(**out)


def _act_out(cube, batch, seq, hidden, group, dtype):
    shape = cube.act_shape(batch, seq, hidden, group)
    return Activation3D(_empty(shape, dtype, cube.device_str()), batch, seq, hidden, group)


def transformer_layer_fwd(cube: Cube, x: Activation3D, params: LayerParams,
                          cfg: TransformerConfig, gs: GroupState, mode=MODE_AUTO,
                          stream=None, save: bool = True):
    """cube3d/transformer.hpp:115-128 -> (y, saved)."""
    y = _act_out(cube, x.batch, x.seq, x.hidden, x.group, c3d_dtype(x.local))
    cx, cy, cp, cc = x.c(), y.c(), params.c(), cfg.c()
    g = C.c_int(gs.input_group)
    h = C.c_void_p()
    call("c3d_layer_fwd", cube.handle, mode, C.byref(cc), C.byref(cx), C.byref(cp), C.byref(g),
         C.byref(cy), C.byref(h) if save else None, _stream(stream))
    gs.input_group = g.value
    y.group = cy.group
    return y, (Saved(h) if save else None)


def transformer_layer_bwd(cube: Cube, dy: Activation3D, saved: Saved, params: LayerParams,
                          cfg: TransformerConfig, mode=MODE_AUTO, grad_dtype: Optional[int] = None,
                          stream=None, grads: Optional[LayerParams] = None):
    """cube3d/transformer.hpp:130-148 -> (dx, grads)."""
    dx = _act_out(cube, dy.batch, dy.seq, dy.hidden, dy.group, c3d_dtype(dy.local))
    if grads is None:
        grads = empty_like_params(cube, params, grad_dtype)
    cdy, cdx, cp, cg, cc = dy.c(), dx.c(), params.c(), grads.c(), cfg.c()
    call("c3d_layer_bwd", cube.handle, mode, C.byref(cc), C.byref(cdy), saved._h, C.byref(cp),
         C.byref(cdx), C.byref(cg), _stream(stream))
    return dx, grads


def transformer_stack_fwd(cube: Cube, x: Activation3D, layers: Sequence["LayerParams"],
                          cfg: TransformerConfig, gs: GroupState, mode=MODE_AUTO, stream=None):
    """cube3d/transformer.hpp:150-163 -> (y, saved)."""
    y = _act_out(cube, x.batch, x.seq, x.hidden, x.group, c3d_dtype(x.local))
    arr = (L.c3d_layer_params * len(layers))(*[p.c() for p in layers])
    cx, cy, cc = x.c(), y.c(), cfg.c()
    g = C.c_int(gs.input_group)
    h = C.c_void_p()
    call("c3d_stack_fwd", cube.handle, mode, C.byref(cc), C.byref(cx), arr, len(layers),
         C.byref(g), C.byref(cy), C.byref(h), _stream(stream))
    gs.input_group = g.value
    return y, Saved(h)


def transformer_stack_bwd(cube: Cube, dy: Activation3D, saved: Saved, layers: Sequence["LayerParams"],
                          cfg: TransformerConfig, mode=MODE_AUTO, grad_dtype: Optional[int] = None,
                          stream=None):
    """cube3d/transformer.hpp:165-176 (reverse order) -> (dx, [grads per layer])."""
    dx = _act_out(cube, dy.batch, dy.seq, dy.hidden, dy.group, c3d_dtype(dy.local))
    grads = [empty_like_params(cube, p, grad_dtype) for p in layers]
    arr = (L.c3d_layer_params * len(layers))(*[p.c() for p in layers])
    garr = (L.c3d_layer_params * len(layers))(*[g.c() for g in grads])
    cdy, cdx, cc = dy.c(), dx.c(), cfg.c()
    call("c3d_stack_bwd", cube.handle, mode, C.byref(cc), C.byref(cdy), saved._h, arr, len(layers),
         C.byref(cdx), garr, _stream(stream))
    return dx, grads


def _block_fwd(name, cube, x, params, cfg, gs, mode, stream):
    y = _act_out(cube, x.batch, x.seq, x.hidden, x.group, c3d_dtype(x.local))
    cx, cy, cp, cc = x.c(), y.c(), params.c(), cfg.c()
    g = C.c_int(gs.input_group)
    h = C.c_void_p()
    call(name, cube.handle, mode, C.byref(cc), C.byref(cx), C.byref(cp), C.byref(g), C.byref(cy),
         C.byref(h), _stream(stream))
    gs.input_group = g.value
    return y, Saved(h)


def _block_bwd(name, cube, dy, saved, params, cfg, mode, grad_dtype, stream):
    dx = _act_out(cube, dy.batch, dy.seq, dy.hidden, dy.group, c3d_dtype(dy.local))
    grads = empty_like_params(cube, params, grad_dtype)
    cdy, cdx, cp, cg, cc = dy.c(), dx.c(), params.c(), grads.c(), cfg.c()
    call(name, cube.handle, mode, C.byref(cc), C.byref(cdy), saved._h, C.byref(cp), C.byref(cdx),
         C.byref(cg), _stream(stream))
    return dx, grads


def attention_fwd(cube, x, params, cfg, gs, mode=MODE_AUTO, stream=None):
    """cube3d/attention.hpp:78-136."""
    return _block_fwd("c3d_attention_fwd", cube, x, params, cfg, gs, mode, stream)


def attention_bwd(cube, dy, saved, params, cfg, mode=MODE_AUTO, grad_dtype=None, stream=None):
    """cube3d/attention.hpp:138-189 (fills w_qkv, b_qkv, w_out, b_out of the grads)."""
    return _block_bwd("c3d_attention_bwd", cube, dy, saved, params, cfg, mode, grad_dtype, stream)


def mlp_fwd(cube, x, params, cfg, gs, mode=MODE_AUTO, stream=None):
    """cube3d/transformer.hpp:44-53."""
    return _block_fwd("c3d_mlp_fwd", cube, x, params, cfg, gs, mode, stream)


def mlp_bwd(cube, dy, saved, params, cfg, mode=MODE_AUTO, grad_dtype=None, stream=None):
    """cube3d/transformer.hpp:55-70 (fills w_fc1, b_fc1, w_fc2, b_fc2)."""
    return _block_bwd("c3d_mlp_bwd", cube, dy, saved, params, cfg, mode, grad_dtype, stream)


@dataclass
class LinearParams:
    """cube3d/nn.hpp:62-67."""

    weight: ShardedMatrix
    bias: DiagonalVector
    input_group: int = 0

    def c(self):
        return L.c3d_linear_params(self.weight.c(), self.bias.c(), self.input_group)


def linear3d_fwd(cube, x: Activation3D, params: LinearParams, gs: GroupState, mode=MODE_AUTO,
                 stream=None):
    """cube3d/nn.hpp:81-97 -> (y, saved)."""
    y = _act_out(cube, x.batch, x.seq, params.weight.global_cols, 1 - x.group,
                 c3d_dtype(x.local))
    cx, cy, cp = x.c(), y.c(), params.c()
    g = C.c_int(gs.input_group)
    h = C.c_void_p()
    call("c3d_linear_fwd", cube.handle, mode, C.byref(cx), C.byref(cp), C.byref(g), C.byref(cy),
         C.byref(h), _stream(stream))
    gs.input_group = g.value
    return y, Saved(h)


def linear3d_bwd(cube, dy: Activation3D, saved: Saved, params: LinearParams, mode=MODE_AUTO,
                 stream=None, db_dtype=F32):
    """cube3d/nn.hpp:99-112 -> (dx, dweight, dbias)."""
    w = params.weight
    dx = _act_out(cube, dy.batch, dy.seq, w.global_rows, params.input_group, c3d_dtype(dy.local))
    torch = _torch()
    dw = ShardedMatrix(torch.empty_like(w.shard), w.global_rows, w.global_cols, w.layout, w.dirs)
    db = _vec_out(cube, w.global_cols, db_dtype)
    cdy, cp, cdx, cdw, cdb = dy.c(), params.c(), dx.c(), dw.c(), db.c()
    call("c3d_linear_bwd", cube.handle, mode, C.byref(cdy), saved._h, C.byref(cp), C.byref(cdx),
         C.byref(cdw), C.byref(cdb), _stream(stream))
    return dx, dw, db


def cross_entropy_fwd(cube, x: Activation3D, head: LinearParams, targets, gs: GroupState,
                      mode=MODE_AUTO, stream=None):
    """3-D cross-entropy: mean over the batch*seq tokens of
    logsumexp(x W + b) - (x W + b)[target]. `targets`: global int32 device tensor
    [batch * seq] (kept alive by the returned state). -> (loss device scalar, saved)."""
    torch = _torch()
    t = targets.to(device=x.local.device, dtype=torch.int32).contiguous()
    loss = torch.zeros(1, dtype=torch.float32, device=x.local.device)
    cx, cp = x.c(), head.c()
    g = C.c_int(gs.input_group)
    h = C.c_void_p()
    call("c3d_loss_fwd", cube.handle, mode, C.byref(cx), C.byref(cp), C.c_void_p(t.data_ptr()),
         C.byref(g), C.c_void_p(loss.data_ptr()), C.byref(h), _stream(stream))
    gs.input_group = g.value
    sv = Saved(h)
    sv.keep = (t, x.batch, x.seq, x.hidden, x.group, c3d_dtype(x.local))
    return loss, sv


def cross_entropy_bwd(cube, saved: Saved, head: LinearParams, mode=MODE_AUTO, stream=None,
                      db_dtype=F32):
    """-> (dx, dweight, dbias) of cross_entropy_fwd."""
    _, batch, seq, hidden, group, dt = saved.keep
    w = head.weight
    dx = _act_out(cube, batch, seq, hidden, group, dt)
    torch = _torch()
    dw = ShardedMatrix(torch.empty_like(w.shard), w.global_rows, w.global_cols, w.layout, w.dirs)
    db = _vec_out(cube, w.global_cols, db_dtype)
    cp, cdx, cdw, cdb = head.c(), dx.c(), dw.c(), db.c()
    call("c3d_loss_bwd", cube.handle, mode, saved._h, C.byref(cp), C.byref(cdx), C.byref(cdw),
         C.byref(cdb), _stream(stream))
    return dx, dw, db


@dataclass
class LayerNormParams:
    """cube3d/nn.hpp:119-124."""

    gamma: DiagonalVector
    beta: DiagonalVector
    eps: float = 1e-5


def layernorm3d_fwd(cube, x: Activation3D, params: LayerNormParams, stream=None):
    """cube3d/nn.hpp:140-185 -> (y, saved)."""
    y = _act_out(cube, x.batch, x.seq, x.hidden, x.group, c3d_dtype(x.local))
    cx, cy = x.c(), y.c()
    cp = L.c3d_layernorm_params(params.gamma.c(), params.beta.c(), params.eps)
    h = C.c_void_p()
    call("c3d_layernorm_fwd", cube.handle, C.byref(cx), C.byref(cp), C.byref(cy), C.byref(h),
         _stream(stream))
    return y, Saved(h)


def layernorm3d_bwd(cube, dy: Activation3D, saved: Saved, stream=None, vec_dtype=F32):
    """cube3d/nn.hpp:187-222 -> (dx, dgamma, dbeta)."""
    dx = _act_out(cube, dy.batch, dy.seq, dy.hidden, dy.group, c3d_dtype(dy.local))
    dg, dbt = _vec_out(cube, dy.hidden, vec_dtype), _vec_out(cube, dy.hidden, vec_dtype)
    cdy, cdx, cdg, cdb = dy.c(), dx.c(), dg.c(), dbt.c()
    call("c3d_layernorm_bwd", cube.handle, C.byref(cdy), saved._h, C.byref(cdx), C.byref(cdg),
         C.byref(cdb), _stream(stream))
    return dx, dg, dbt


def gemm(M, N, K, a_view: dict, b_view: dict, out_view: dict, alpha=1.0, bias=None, act=0,
         accumulate=False, mode=MODE_AUTO, batch=1, stream=None):
    """Local GEMM over strided views (csrc/gemm.hpp); views are dicts of c3d_view fields."""
    def mk(d):
        v = L.c3d_view()
        v.base = d["base"]
        v.dtype = d.get("dtype", BF16)
        for k in ("sr", "sc", "s_hi", "rsplit", "csplit", "sb_lo", "sb_hi"):
            setattr(v, k, int(d.get(k, 0)))
        v.b_lo_n = int(d.get("b_lo_n", 1))
        return v
    va, vb, vo = mk(a_view), mk(b_view), mk(out_view)
    call("c3d_gemm", int(M), int(N), int(K), int(batch), C.byref(va), C.byref(vb), C.byref(vo),
         float(alpha), C.c_void_p(bias) if bias else None, int(act), int(accumulate), int(mode),
         _stream(stream))


def launch_count() -> int:
    return int(lib().c3d_launch_count())


def prof_enable(on: bool = True) -> None:
    call("c3d_prof_enable", int(on))


def prof_read():
    """-> (sum of tcgen05 GEMM launch times in ms, sum of their flops, launches)."""
    ms, fl, n = C.c_double(), C.c_double(), C.c_longlong()
    call("c3d_prof_read", C.byref(ms), C.byref(fl), C.byref(n))
    return ms.value, fl.value, n.value


def prof_read_comm():
    """-> (sum of collective times in ms, sum of payload bytes, calls)."""
    ms, by, n = C.c_double(), C.c_double(), C.c_longlong()
    call("c3d_prof_read_comm", C.byref(ms), C.byref(by), C.byref(n))
    return ms.value, by.value, n.value
