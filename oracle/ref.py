"""ctypes access to the compiled reference (oracle/_ref/libcube3d_ref.so) -- TEST INFRASTRUCTURE.

The library is the reference's own code (headers under /root/reference, built
in place by oracle/Makefile). ``available()`` is False when it has not been
built (e.g. a box without the prebuilt file): callers then skip, never fall back.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "_ref" / "libcube3d_ref.so"
FIELDS = ["ln1_gamma", "ln1_beta", "w_qkv", "b_qkv", "w_out", "b_out", "ln2_gamma", "ln2_beta",
          "w_fc1", "b_fc1", "w_fc2", "b_fc2"]
_lib = None


def available() -> bool:
    return LIB.exists()


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(str(LIB))
        _lib.ref_last_error.restype = C.c_char_p
    return _lib


def _dp(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _chk(code):
    if code != 0:
        raise RuntimeError(lib().ref_last_error().decode())


def param_shapes(h):
    return [(h,), (h,), (h, 3 * h), (3 * h,), (h, h), (h,), (h,), (h,), (h, 4 * h), (4 * h,),
            (4 * h, h), (h,)]


def _pp(arrs):
    ptrs = (C.POINTER(C.c_double) * 12)(*[_dp(a) for a in arrs])
    return ptrs


def rng_uniform(seed, n, lo=-1.0, hi=1.0, skip=0):
    out = np.zeros(n)
    _chk(lib().ref_rng_uniform(C.c_uint64(seed), C.c_int64(skip), C.c_double(lo), C.c_double(hi),
                               C.c_int64(n), _dp(out)))
    return out


def rng_u64(seed, n):
    out = np.zeros(n, dtype=np.uint64)
    _chk(lib().ref_rng_u64(C.c_uint64(seed), C.c_int64(n),
                           out.ctypes.data_as(C.POINTER(C.c_uint64))))
    return out


def random_integer_matrix(seed, rows, cols):
    out = np.zeros((rows, cols))
    _chk(lib().ref_random_integer_matrix(C.c_uint64(seed), C.c_int64(rows), C.c_int64(cols),
                                         _dp(out)))
    return out


def init_layer_params(hidden, seed):
    arrs = [np.zeros(s) for s in param_shapes(hidden)]
    _chk(lib().ref_init_layer_params(C.c_int64(hidden), C.c_uint64(seed), _pp(arrs)))
    return dict(zip(FIELDS, arrs))


def shard_bounds(layout, p, c, rows, cols, dirs):
    out = (C.c_int64 * 4)()
    _chk(lib().ref_shard_bounds(layout, p, c[0], c[1], c[2], C.c_int64(rows), C.c_int64(cols),
                                dirs[0], dirs[1], dirs[2], out))
    return (out[0], out[1]), (out[2], out[3])


def diagonal_slice(p, c, n):
    holds = C.c_int()
    out = (C.c_int64 * 2)()
    _chk(lib().ref_diagonal_slice(p, c[0], c[1], c[2], C.c_int64(n), C.byref(holds), out))
    return bool(holds.value), (out[0], out[1])


def activation_map(p, batch, seq, hidden, group):
    out = np.zeros(batch * seq * hidden)
    _chk(lib().ref_activation_map(p, C.c_int64(batch), C.c_int64(seq), C.c_int64(hidden), group,
                                  _dp(out)))
    return out.reshape(p ** 3, -1)


def run_matmul(p, form, a, b, g, f32=False):
    """verify_detail::run_matmul (cube3d/verify.hpp:60-114): (C, dA, dB, counters[P][3])."""
    fi = {"AB": 0, "ABt": 1, "AtB": 2}[form]
    M, N = a.shape
    K = b.shape[1] if form in ("AB", "AtB") else b.shape[0]
    cshape = (M, K) if form != "AtB" else (N, K)
    c = np.zeros(cshape)
    da = np.zeros(a.shape)
    db = np.zeros(b.shape)
    cnt = np.zeros((p ** 3, 3), dtype=np.uint64)
    a, b, g = (np.ascontiguousarray(t, dtype=np.float64) for t in (a, b, g))
    _chk(lib().ref_run_matmul(p, fi, int(f32), C.c_int64(M), C.c_int64(N), C.c_int64(K), _dp(a),
                              _dp(b), _dp(g), _dp(c), _dp(da), _dp(db),
                              cnt.ctypes.data_as(C.POINTER(C.c_uint64))))
    return c, da, db, cnt


def run_layer(p, b, s, n, h, params, x, dy, f32=False):
    """verify_detail::run_layer (cube3d/verify.hpp:181-232) through the 3-D path."""
    ps = [np.ascontiguousarray(params[f], dtype=np.float64) for f in FIELDS]
    x = np.ascontiguousarray(x, dtype=np.float64)
    dy = np.ascontiguousarray(dy, dtype=np.float64)
    y = np.zeros_like(x)
    dx = np.zeros_like(x)
    dps = [np.zeros(sh) for sh in param_shapes(h)]
    cnt = np.zeros((p ** 3, 3), dtype=np.uint64)
    secs = C.c_double()
    _chk(lib().ref_run_layer(p, int(f32), C.c_int64(b), C.c_int64(s), C.c_int64(n), C.c_int64(h),
                             _pp(ps), _dp(x), _dp(dy), _dp(y), _dp(dx), _pp(dps),
                             cnt.ctypes.data_as(C.POINTER(C.c_uint64)), C.byref(secs)))
    return y, dx, dict(zip(FIELDS, dps)), cnt, secs.value


def layer_serial(b, s, n, h, params, x, dy):
    ps = [np.ascontiguousarray(params[f], dtype=np.float64) for f in FIELDS]
    x = np.ascontiguousarray(x, dtype=np.float64)
    dy = np.ascontiguousarray(dy, dtype=np.float64)
    y = np.zeros_like(x)
    dx = np.zeros_like(x)
    dps = [np.zeros(sh) for sh in param_shapes(h)]
    _chk(lib().ref_layer_serial(C.c_int64(b), C.c_int64(s), C.c_int64(n), C.c_int64(h), _pp(ps),
                                _dp(x), _dp(dy), _dp(y), _dp(dx), _pp(dps)))
    return y, dx, dict(zip(FIELDS, dps))


def layer_costs(p, b, s, n, h):
    out = (C.c_uint64 * 4)()
    _chk(lib().ref_layer_costs(p, C.c_int64(b), C.c_int64(s), C.c_int64(n), C.c_int64(h), out))
    return tuple(out)


def run_verify(p=2, b=2, s=8, n=2, h=16, seed=7, f32=False):
    buf = C.create_string_buffer(1 << 16)
    rc = lib().ref_run_verify(p, C.c_int64(b), C.c_int64(s), C.c_int64(n), C.c_int64(h),
                              C.c_uint64(seed), int(f32), buf, C.c_int64(1 << 16))
    return rc == 0, buf.value.decode()


def time_layer(p, b, s, n, h, params, x, dy):
    """The reference's 3-D layer fwd and bwd in float on p^3 rank threads, timed
    separately with an Endpoint barrier between them: (fwd_seconds, bwd_seconds)."""
    ps = [np.ascontiguousarray(params[f], dtype=np.float64) for f in FIELDS]
    x = np.ascontiguousarray(x, dtype=np.float64)
    dy = np.ascontiguousarray(dy, dtype=np.float64)
    secs = (C.c_double * 2)()
    _chk(lib().ref_time_layer(p, C.c_int64(b), C.c_int64(s), C.c_int64(n), C.c_int64(h),
                              _pp(ps), _dp(x), _dp(dy), secs))
    return secs[0], secs[1]


def write_matrix(path, m, f32=False):
    """The reference's write_matrix_file (cube3d/matrix_io.hpp:83-108)."""
    m = np.ascontiguousarray(np.atleast_2d(m), dtype=np.float64)
    _chk(lib().ref_write_matrix(str(path).encode(), C.c_int64(m.shape[0]), C.c_int64(m.shape[1]),
                                _dp(m), int(f32)))


def read_matrix(path, f32=False, cap=1 << 24):
    rows, cols = C.c_int64(), C.c_int64()
    buf = np.zeros(cap)
    _chk(lib().ref_read_matrix(str(path).encode(), int(f32), C.byref(rows), C.byref(cols), _dp(buf),
                               C.c_int64(cap)))
    return buf[:rows.value * cols.value].reshape(rows.value, cols.value)


def save_layer_params(params, h, prefix):
    ps = [np.ascontiguousarray(params[f], dtype=np.float64) for f in FIELDS]
    _chk(lib().ref_save_layer_params(C.c_int64(h), _pp(ps), str(prefix).encode()))


def load_layer_params(h, prefix):
    arrs = [np.zeros(s) for s in param_shapes(h)]
    _chk(lib().ref_load_layer_params(C.c_int64(h), str(prefix).encode(), _pp(arrs)))
    return dict(zip(FIELDS, arrs))


def scaling_csv(weak, b, s, n, h, layers, p_list, lam=1.0):
    """cube3d/bench.hpp run_scaling + write_scaling_csv (the CLI's bench subcommand)."""
    ps = (C.c_int * len(p_list))(*p_list)
    buf = C.create_string_buffer(1 << 16)
    _chk(lib().ref_scaling_csv(int(weak), C.c_int64(b), C.c_int64(s), C.c_int64(n), C.c_int64(h),
                               C.c_int64(layers), ps, len(p_list), C.c_double(lam), buf,
                               C.c_int64(1 << 16)))
    return buf.value.decode()
