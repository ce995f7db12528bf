"""ctypes binding of the C ABI (include/c3d.h).

This is the reference-side binding a Python caller of the library uses; the
same declarations are what a C or C++ host includes. Loading fails loudly when
``libc3d.so`` is missing -- there is no CPU fallback anywhere in the package.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

_PKG = Path(__file__).resolve().parent
LIB_PATH = Path(os.environ.get("C3D_LIB", _PKG / "libc3d.so"))

# status codes (c3d_status), same order as cube3d/errors.hpp:24-37
STATUS_NAMES = {
    0: "OK", 1: "NotACube", 2: "OutOfRange", 3: "LengthMismatch", 4: "Desync",
    5: "IndivisibleShape", 6: "InconsistentFamily", 7: "ShapeMismatch", 8: "DirectionClash",
    9: "BatchMismatch", 10: "GroupMismatch", 11: "HeadsIndivisible", 12: "ConfigInvalid",
    13: "NonFinite", 14: "IoError", 100: "CudaError", 101: "NcclError", 102: "InternalError",
}

F32, BF16 = 0, 1
MODE_AUTO, MODE_TC, MODE_F32 = 0, 1, 2


class c3d_matrix(C.Structure):
    _fields_ = [("data", C.c_void_p), ("dtype", C.c_int), ("global_rows", C.c_int64),
                ("global_cols", C.c_int64), ("layout", C.c_int), ("dirs", C.c_int * 3)]


class c3d_vector(C.Structure):
    _fields_ = [("data", C.c_void_p), ("dtype", C.c_int), ("global_len", C.c_int64)]


class c3d_activation(C.Structure):
    _fields_ = [("data", C.c_void_p), ("dtype", C.c_int), ("batch", C.c_int64),
                ("seq", C.c_int64), ("hidden", C.c_int64), ("group", C.c_int)]


class c3d_view(C.Structure):
    _fields_ = [("base", C.c_void_p), ("dtype", C.c_int), ("sr", C.c_int64), ("sc", C.c_int64),
                ("s_hi", C.c_int64), ("rsplit", C.c_int64), ("csplit", C.c_int64),
                ("sb_lo", C.c_int64), ("sb_hi", C.c_int64), ("b_lo_n", C.c_int)]


class c3d_counters(C.Structure):
    _fields_ = [("elements_sent", C.c_uint64), ("elements_received", C.c_uint64),
                ("sent_by_kind", C.c_uint64 * 5), ("received_by_kind", C.c_uint64 * 5),
                ("calls_by_kind", C.c_uint64 * 5), ("multiply_adds", C.c_uint64)]


class c3d_config(C.Structure):
    _fields_ = [("batch", C.c_int64), ("seq", C.c_int64), ("heads", C.c_int64),
                ("hidden", C.c_int64), ("eps", C.c_double)]


class c3d_linear_params(C.Structure):
    _fields_ = [("weight", c3d_matrix), ("bias", c3d_vector), ("input_group", C.c_int)]


class c3d_layernorm_params(C.Structure):
    _fields_ = [("gamma", c3d_vector), ("beta", c3d_vector), ("eps", C.c_double)]


LAYER_FIELDS = ["ln1_gamma", "ln1_beta", "w_qkv", "b_qkv", "w_out", "b_out", "ln2_gamma",
                "ln2_beta", "w_fc1", "b_fc1", "w_fc2", "b_fc2"]


class c3d_layer_params(C.Structure):
    _fields_ = [(n, c3d_matrix if n.startswith("w_") else c3d_vector) for n in LAYER_FIELDS]


P = C.POINTER
VP = C.c_void_p
I3 = C.c_int * 3

# name -> argtypes (every symbol declared in include/c3d.h)
SIGNATURES = {
    "c3d_last_error": [],
    "c3d_version": [],
    "c3d_launch_count": [],
    "c3d_prof_enable": [C.c_int],
    "c3d_prof_read": [P(C.c_double), P(C.c_double), P(C.c_longlong)],
    "c3d_prof_read_comm": [P(C.c_double), P(C.c_double), P(C.c_longlong)],
    "c3d_rng_create": [C.c_uint64, P(VP)],
    "c3d_rng_destroy": [VP],
    "c3d_rng_next_u64": [VP, P(C.c_uint64), C.c_int64],
    "c3d_rng_uniform": [VP, C.c_double, C.c_double, P(C.c_double), C.c_int64],
    "c3d_rng_below": [VP, C.c_uint64, P(C.c_double), C.c_int64],
    "c3d_grid_rank_of": [I3, I3, P(C.c_int)],
    "c3d_grid_coords_of": [I3, C.c_int, I3],
    "c3d_grid_axis_group": [I3, C.c_int, C.c_int, P(C.c_int), P(C.c_int)],
    "c3d_grid_line_index": [I3, C.c_int, C.c_int, P(C.c_int)],
    "c3d_build_cube": [C.c_int, P(C.c_int)],
    "c3d_shard_bounds": [C.c_int, I3, I3, C.c_int64, C.c_int64, I3, P(C.c_int64)],
    "c3d_diagonal_slice": [I3, I3, C.c_int64, P(C.c_int), P(C.c_int64)],
    "c3d_activation_rows": [I3, I3, C.c_int64, C.c_int64, C.c_int64, C.c_int, P(C.c_int64),
                            P(C.c_int64), P(C.c_int64)],
    "c3d_unique_id": [C.c_char_p],
    "c3d_cube_create": [I3, C.c_int, C.c_int, C.c_char_p, P(VP)],
    "c3d_cube_destroy": [VP],
    "c3d_cube_info": [VP, P(C.c_int), I3, I3],
    "c3d_cube_barrier": [VP, VP],
    "c3d_counters_get": [VP, P(c3d_counters)],
    "c3d_counters_reset": [VP],
    "c3d_cube_check": [VP, VP],
    "c3d_broadcast": [VP, C.c_int, C.c_int, VP, C.c_size_t, C.c_int, VP],
    "c3d_all_gather": [VP, C.c_int, VP, VP, C.c_size_t, C.c_int, VP],
    "c3d_reduce_scatter": [VP, C.c_int, VP, VP, C.c_size_t, C.c_int, VP],
    "c3d_all_reduce": [VP, C.c_int, VP, C.c_size_t, C.c_int, C.c_int, VP],
    "c3d_gemm": [C.c_int64, C.c_int64, C.c_int64, C.c_int, P(c3d_view), P(c3d_view),
                 P(c3d_view), C.c_float, VP, C.c_int, C.c_int, C.c_int, VP],
    "c3d_matmul_ab_fwd": [VP, C.c_int, P(c3d_matrix), P(c3d_matrix), P(c3d_matrix), VP],
    **{f"c3d_batched_matmul_{k}_fwd": [VP, C.c_int, C.c_int, P(c3d_matrix), C.c_int,
                                       P(c3d_matrix), P(c3d_matrix), VP]
       for k in ("ab", "abt", "atb")},
    **{f"c3d_batched_matmul_{k}_bwd": [VP, C.c_int, C.c_int, P(c3d_matrix), C.c_int,
                                       P(c3d_matrix), C.c_int, P(c3d_matrix), P(c3d_matrix),
                                       P(c3d_matrix), VP]
       for k in ("ab", "abt", "atb")},
    "c3d_matmul_ab_bwd": [VP, C.c_int, P(c3d_matrix), P(c3d_matrix), P(c3d_matrix),
                          P(c3d_matrix), P(c3d_matrix), VP],
    "c3d_matmul_abt_fwd": [VP, C.c_int, P(c3d_matrix), P(c3d_matrix), P(c3d_matrix), VP],
    "c3d_matmul_abt_bwd": [VP, C.c_int, P(c3d_matrix), P(c3d_matrix), P(c3d_matrix),
                           P(c3d_matrix), P(c3d_matrix), VP],
    "c3d_matmul_atb_fwd": [VP, C.c_int, P(c3d_matrix), P(c3d_matrix), P(c3d_matrix), VP],
    "c3d_matmul_atb_bwd": [VP, C.c_int, P(c3d_matrix), P(c3d_matrix), P(c3d_matrix),
                           P(c3d_matrix), P(c3d_matrix), VP],
    "c3d_add_vec_fwd": [VP, P(c3d_matrix), P(c3d_vector), P(c3d_matrix), VP],
    "c3d_add_vec_bwd": [VP, P(c3d_matrix), P(c3d_matrix), P(c3d_vector), VP],
    "c3d_mul_vec_fwd": [VP, P(c3d_matrix), P(c3d_vector), P(c3d_matrix), VP],
    "c3d_mul_vec_bwd": [VP, P(c3d_matrix), P(c3d_matrix), P(c3d_vector), P(c3d_matrix),
                        P(c3d_vector), VP],
    "c3d_saved_free": [VP],
    "c3d_linear_fwd": [VP, C.c_int, P(c3d_activation), P(c3d_linear_params), P(C.c_int),
                       P(c3d_activation), P(VP), VP],
    "c3d_linear_bwd": [VP, C.c_int, P(c3d_activation), VP, P(c3d_linear_params),
                       P(c3d_activation), P(c3d_matrix), P(c3d_vector), VP],
    "c3d_stack_fwd": [VP, C.c_int, P(c3d_config), P(c3d_activation), P(c3d_layer_params),
                      C.c_int, P(C.c_int), P(c3d_activation), P(VP), VP],
    "c3d_stack_bwd": [VP, C.c_int, P(c3d_config), P(c3d_activation), VP, P(c3d_layer_params),
                      C.c_int, P(c3d_activation), P(c3d_layer_params), VP],
    "c3d_loss_fwd": [VP, C.c_int, P(c3d_activation), P(c3d_linear_params), VP, P(C.c_int), VP,
                     P(VP), VP],
    "c3d_loss_bwd": [VP, C.c_int, VP, P(c3d_linear_params), P(c3d_activation), P(c3d_matrix),
                     P(c3d_vector), VP],
    "c3d_layernorm_fwd": [VP, P(c3d_activation), P(c3d_layernorm_params), P(c3d_activation),
                          P(VP), VP],
    "c3d_layernorm_bwd": [VP, P(c3d_activation), VP, P(c3d_activation), P(c3d_vector),
                          P(c3d_vector), VP],
    "c3d_attention_fwd": [VP, C.c_int, P(c3d_config), P(c3d_activation), P(c3d_layer_params),
                          P(C.c_int), P(c3d_activation), P(VP), VP],
    "c3d_attention_bwd": [VP, C.c_int, P(c3d_config), P(c3d_activation), VP,
                          P(c3d_layer_params), P(c3d_activation), P(c3d_layer_params), VP],
    "c3d_mlp_fwd": [VP, C.c_int, P(c3d_config), P(c3d_activation), P(c3d_layer_params),
                    P(C.c_int), P(c3d_activation), P(VP), VP],
    "c3d_mlp_bwd": [VP, C.c_int, P(c3d_config), P(c3d_activation), VP, P(c3d_layer_params),
                    P(c3d_activation), P(c3d_layer_params), VP],
    "c3d_layer_fwd": [VP, C.c_int, P(c3d_config), P(c3d_activation), P(c3d_layer_params),
                      P(C.c_int), P(c3d_activation), P(VP), VP],
    "c3d_layer_bwd": [VP, C.c_int, P(c3d_config), P(c3d_activation), VP, P(c3d_layer_params),
                      P(c3d_activation), P(c3d_layer_params), VP],
}
RESTYPES = {"c3d_last_error": C.c_char_p, "c3d_version": C.c_char_p,
            "c3d_launch_count": C.c_longlong}


class C3DError(RuntimeError):
    """Raised for every non-zero status; ``name`` is the reference error class name."""

    def __init__(self, code: int, message: str):
        super().__init__(message)
        self.code = code
        self.name = STATUS_NAMES.get(code, "InternalError")


_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise ImportError(f"{LIB_PATH} is missing: build it with "
                              "`python -m paper_2105_14450_b200.build` (no CPU fallback exists)")
        L = C.CDLL(str(LIB_PATH))
        for name, args in SIGNATURES.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = RESTYPES.get(name, C.c_int)
        _lib = L
    return _lib


def check(code: int) -> None:
    if code != 0:
        msg = lib().c3d_last_error().decode()
        raise C3DError(code, msg)


def call(name: str, *args) -> None:
    check(getattr(lib(), name)(*args))
