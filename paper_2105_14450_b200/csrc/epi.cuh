// Device helpers shared by the GEMM epilogues and the elementwise kernels.
#pragma once

#include <cuda_bf16.h>

#include "gemm.hpp"

namespace c3d {

// gelu / gelu_grad: the erf form of cube3d/nn.hpp:44-56 in fp32. erf(z) by
// Abramowitz & Stegun 7.1.26 (|error| < 1.5e-7): one reciprocal, one exp and five FMAs,
// and the exp e^{-z^2} = e^{-x^2/2} is the Gaussian density gelu' needs as well.
__device__ __forceinline__ void phi_both(float x, float& cdf, float& pdf) {
  // t = 1 / (1 + p z), z = |x| / sqrt(2); e = e^{-z^2} = 2^{-x^2 log2(e) / 2}. MUFU.RCP and
  // MUFU.EX2 with flush-to-zero (the IEEE-rounded reciprocal and the denormal-preserving
  // exp add a slow path / range fix-up per element; e underflows only where erf is 1).
  float t, e;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(t) : "f"(fmaf(0.3275911f * 0.70710678118654752f, fabsf(x), 1.f)));
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(x * x * -0.72134752044448170f));
  const float poly =
      t * fmaf(t, fmaf(t, fmaf(t, fmaf(t, 1.061405429f, -1.453152027f), 1.421413741f),
                      -0.284496736f),
               0.254829592f);
  const float erf_abs = 1.f - poly * e;
  cdf = 0.5f + 0.5f * copysignf(erf_abs, x);
  pdf = e * 0.3989422804014327f;
}
__device__ __forceinline__ float gelu_f(float x) {
  float c, p;
  phi_both(x, c, p);
  return x * c;
}
__device__ __forceinline__ float gelu_grad_f(float x) {
  float c, p;
  phi_both(x, c, p);
  return c + x * p;
}
// gelu(x) and gelu'(x) sharing one erf.
__device__ __forceinline__ void gelu_both(float x, float& g, float& gd) {
  float c, p;
  phi_both(x, c, p);
  g = x * c;
  gd = c + x * p;
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
  if (e.act == kActGeluSave) {
    float g, gd;
    gelu_both(v, g, gd);
    if (e.pre_act) st_any(e.pre_act, e.pre_dtype, off, gd);
    v = g;
  } else if (e.pre_act) {
    st_any(e.pre_act, e.pre_dtype, off, v);
  }
  if (e.act == kActGelu) v = gelu_f(v);
  else if (e.act == kActGeluGrad) v *= gelu_grad_f(ld_any(e.aux, e.aux_dtype, off));
  else if (e.act == kActMulAux) v *= ld_any(e.aux, e.aux_dtype, off);
  else if (e.act == kActSoftmaxBwd)
    v = ld_any(e.aux, e.aux_dtype, off) * (v - e.alpha * e.rowvec[off / e.rv_div]);
  if (e.resid) v += ld_any(e.resid, e.resid_dtype, off);
  if (e.accumulate) v += ld_any(e.out.base, e.out.dtype, off);
  st_any(e.out.base, e.out.dtype, off, v);
}

}  // namespace c3d
