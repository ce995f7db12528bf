"""B200-native 3-D parallel matmul and 3-D Transformer layer (arXiv 2105.14450).

The compute lives in ``libc3d.so`` (sm_100a CUDA kernels + NCCL, C ABI in
``include/c3d.h``); :mod:`.cube3d` mirrors the reference ``cube3d`` operator API.
"""
from . import cube3d  # noqa: F401
from ._lib import C3DError, LIB_PATH  # noqa: F401

__all__ = ["cube3d", "C3DError", "LIB_PATH"]
