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

// Packed fp32 pairs (FFMA2 / FMUL2 on sm_100): half the issue slots of scalar math.
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
  float2 d;
  asm("{\n\t.reg .b64 ra, rb, rc, rd;\n\tmov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t"
      "mov.b64 rc, {%6, %7};\n\tfma.rn.f32x2 rd, ra, rb, rc;\n\tmov.b64 {%0, %1}, rd;\n\t}"
      : "=f"(d.x), "=f"(d.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
  return d;
}
__device__ __forceinline__ float2 fmul2(float2 a, float2 b) {
  float2 d;
  asm("{\n\t.reg .b64 ra, rb, rd;\n\tmov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t"
      "mul.rn.f32x2 rd, ra, rb;\n\tmov.b64 {%0, %1}, rd;\n\t}"
      : "=f"(d.x), "=f"(d.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return d;
}
__device__ __forceinline__ float2 fadd2(float2 a, float2 b) {
  float2 d;
  asm("{\n\t.reg .b64 ra, rb, rd;\n\tmov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t"
      "add.rn.f32x2 rd, ra, rb;\n\tmov.b64 {%0, %1}, rd;\n\t}"
      : "=f"(d.x), "=f"(d.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return d;
}

// gelu_both on a pair, in packed fp32 (same formula and rounding sequence per element as
// phi_both / gelu_both: the packed ops round each lane like their scalar forms).
__device__ __forceinline__ void gelu_both2(float2 x, float2& g, float2& gd) {
  const float2 ax = make_float2(fabsf(x.x), fabsf(x.y));
  const float2 tin = ffma2(make_float2(0.3275911f * 0.70710678118654752f, 0.3275911f * 0.70710678118654752f),
                           ax, make_float2(1.f, 1.f));
  const float2 ea = fmul2(fmul2(x, x), make_float2(-0.72134752044448170f, -0.72134752044448170f));
  float2 t, e;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(t.x) : "f"(tin.x));
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(t.y) : "f"(tin.y));
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e.x) : "f"(ea.x));
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e.y) : "f"(ea.y));
  auto c2 = [](float v) { return make_float2(v, v); };
  float2 poly = ffma2(t, c2(1.061405429f), c2(-1.453152027f));
  poly = ffma2(t, poly, c2(1.421413741f));
  poly = ffma2(t, poly, c2(-0.284496736f));
  poly = ffma2(t, poly, c2(0.254829592f));
  poly = fmul2(t, poly);
  const float2 erf_abs = ffma2(make_float2(-poly.x, -poly.y), e, c2(1.f));
  const float2 cdf = ffma2(c2(0.5f), make_float2(copysignf(erf_abs.x, x.x), copysignf(erf_abs.y, x.y)),
                           c2(0.5f));
  const float2 pdf = fmul2(e, c2(0.3989422804014327f));
  g = fmul2(x, cdf);
  gd = ffma2(x, pdf, cdf);
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
