// Device helpers shared by the GEMM epilogues and the elementwise kernels.
#pragma once

#include <cuda_bf16.h>

#include "gemm.hpp"

namespace c3d {

// gelu / gelu_grad: the exact erf form of cube3d/nn.hpp:44-56, in fp32.
__device__ __forceinline__ float gelu_f(float x) {
  return 0.5f * x * (1.f + erff(x * 0.70710678118654752f));
}
__device__ __forceinline__ float gelu_grad_f(float x) {
  const float cdf = 0.5f * (1.f + erff(x * 0.70710678118654752f));
  const float pdf = expf(-0.5f * x * x) * 0.3989422804014327f;
  return cdf + x * pdf;
}

__device__ __forceinline__ float ld_any(const void* base, int dtype, long long off) {
  if (dtype == kF32) return static_cast<const float*>(base)[off];
  return __bfloat162float(static_cast<const __nv_bfloat16*>(base)[off]);
}

__device__ __forceinline__ void st_any(void* base, int dtype, long long off, float v) {
  if (dtype == kF32) static_cast<float*>(base)[off] = v;
  else static_cast<__nv_bfloat16*>(base)[off] = __float2bfloat16_rn(v);
}

// Scalar epilogue of one element at output offset `off`, column n.
__device__ __forceinline__ void epi_scalar(const Epilogue& e, long long off, long long n,
                                           float acc) {
  float v = acc * e.alpha;
  if (e.bias) v += e.bias[n];
  if (e.pre_act) st_any(e.pre_act, e.pre_dtype, off, v);
  if (e.act == kActGelu) v = gelu_f(v);
  else if (e.act == kActGeluGrad) v *= gelu_grad_f(ld_any(e.aux, e.aux_dtype, off));
  if (e.resid) v += ld_any(e.resid, e.resid_dtype, off);
  if (e.accumulate) v += ld_any(e.out.base, e.out.dtype, off);
  st_any(e.out.base, e.out.dtype, off, v);
}

}  // namespace c3d
