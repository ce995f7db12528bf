// Distributed attention softmax (cube3d/attention.hpp:106-126) and its adjoint
// (:161-169), batched over every local (batch, head) slice: one warp per score row.
// Scores and dP arrive in fp32; P and dS leave in the activation dtype.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "common.hpp"
#include "epi.cuh"
#include "kernels.hpp"

namespace c3d {

namespace {

constexpr int kWarps = 8;

__device__ __forceinline__ float wsum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float wmax(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

inline unsigned blocks_for(int64_t rows) { return static_cast<unsigned>((rows + kWarps - 1) / kWarps); }

#define ROW_PROLOGUE                                                                   \
  const int64_t r = blockIdx.x * static_cast<int64_t>(kWarps) + threadIdx.x / 32;      \
  const int lane = threadIdx.x % 32;                                                   \
  if (r >= rows) return;                                                               \
  const float* srow = sc + r * cols;

__global__ void rowmax_kernel(const float* sc, int64_t rows, int64_t cols, float* mx) {
  ROW_PROLOGUE
  float m = -INFINITY;
  for (int64_t c = lane; c < cols; c += 32) m = fmaxf(m, srow[c]);
  m = wmax(m);
  if (lane == 0) mx[r] = m;
}

__global__ void rowexpsum_kernel(const float* sc, int64_t rows, int64_t cols, const float* mx,
                                 float* sum) {
  ROW_PROLOGUE
  const float m = mx[r];
  float s = 0.f;
  for (int64_t c = lane; c < cols; c += 32) s += expf(srow[c] - m);
  s = wsum(s);
  if (lane == 0) sum[r] = s;
}

__global__ void norm_kernel(const float* sc, int64_t rows, int64_t cols, const float* mx,
                            const float* sum, void* p, int pdt) {
  ROW_PROLOGUE
  const float m = mx[r], inv = 1.f / sum[r];
  for (int64_t c = lane; c < cols; c += 32) st_any(p, pdt, r * cols + c, expf(srow[c] - m) * inv);
}

__global__ void fused_kernel(const float* sc, int64_t rows, int64_t cols, void* p, int pdt) {
  ROW_PROLOGUE
  float m = -INFINITY;
  for (int64_t c = lane; c < cols; c += 32) m = fmaxf(m, srow[c]);
  m = wmax(m);
  float s = 0.f;
  for (int64_t c = lane; c < cols; c += 32) s += expf(srow[c] - m);
  const float inv = 1.f / wsum(s);
  for (int64_t c = lane; c < cols; c += 32) st_any(p, pdt, r * cols + c, expf(srow[c] - m) * inv);
}

__global__ void bwd_rowdot_kernel(const float* sc, const void* p, int pdt, int64_t rows,
                                  int64_t cols, float* rowdot) {
  ROW_PROLOGUE
  float s = 0.f;
  for (int64_t c = lane; c < cols; c += 32) s += srow[c] * ld_any(p, pdt, r * cols + c);
  s = wsum(s);
  if (lane == 0) rowdot[r] = s;
}

__global__ void bwd_ds_kernel(const float* sc, const void* p, int pdt, int64_t rows,
                              int64_t cols, const float* rowdot, float scale, void* ds,
                              int dsdt) {
  ROW_PROLOGUE
  const float rd = rowdot[r];
  for (int64_t c = lane; c < cols; c += 32) {
    const float pv = ld_any(p, pdt, r * cols + c);
    st_any(ds, dsdt, r * cols + c, pv * (srow[c] - rd) * scale);
  }
}

__global__ void bwd_fused_kernel(const float* sc, const void* p, int pdt, int64_t rows,
                                 int64_t cols, float scale, void* ds, int dsdt) {
  ROW_PROLOGUE
  float s = 0.f;
  for (int64_t c = lane; c < cols; c += 32) s += srow[c] * ld_any(p, pdt, r * cols + c);
  const float rd = wsum(s);
  for (int64_t c = lane; c < cols; c += 32) {
    const float pv = ld_any(p, pdt, r * cols + c);
    st_any(ds, dsdt, r * cols + c, pv * (srow[c] - rd) * scale);
  }
}

#undef ROW_PROLOGUE

// D[b*S + q] = sum_d dO[b][q][d] * O[b][q][d] over packed [bi][q][head][dh] context
// buffers: the softmax-backward row dot product sum_j P_ij dP_ij (dP = dO V^T, O = P V).
__global__ void attn_rowdot_kernel(const void* d_o, const void* o, int dt, int64_t rows,
                                   int64_t S, int64_t H, int64_t dh, int64_t sb_hi, float* out) {
  const int64_t r = blockIdx.x * static_cast<int64_t>(kWarps) + threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  if (r >= rows) return;
  const int64_t b = r / S, q = r - (r / S) * S;
  const int64_t base = (b / H) * sb_hi + q * (H * dh) + (b % H) * dh;
  float acc = 0.f;
  for (int64_t d = lane; d < dh; d += 32) acc += ld_any(d_o, dt, base + d) * ld_any(o, dt, base + d);
  acc = wsum(acc);
  if (lane == 0) out[r] = acc;
}

}  // namespace

#define LAUNCH_ROWS(kern, name, ...)                                               \
  do {                                                                             \
    if (rows == 0) return;                                                         \
    kern<<<blocks_for(rows), 32 * kWarps, 0, s>>>(__VA_ARGS__);                    \
    check_launch(name);                                                            \
  } while (0)

void k_softmax_rowmax(const float* sc, int64_t rows, int64_t cols, float* mx, cudaStream_t s) {
  LAUNCH_ROWS(rowmax_kernel, "softmax_rowmax", sc, rows, cols, mx);
}
void k_softmax_rowexpsum(const float* sc, int64_t rows, int64_t cols, const float* mx,
                         float* sum, cudaStream_t s) {
  LAUNCH_ROWS(rowexpsum_kernel, "softmax_rowexpsum", sc, rows, cols, mx, sum);
}
void k_softmax_norm(const float* sc, int64_t rows, int64_t cols, const float* mx,
                    const float* sum, void* p, int pdt, cudaStream_t s) {
  LAUNCH_ROWS(norm_kernel, "softmax_norm", sc, rows, cols, mx, sum, p, pdt);
}
void k_softmax_fused(const float* sc, int64_t rows, int64_t cols, void* p, int pdt,
                     cudaStream_t s) {
  LAUNCH_ROWS(fused_kernel, "softmax_fused", sc, rows, cols, p, pdt);
}
void k_softmax_bwd_rowdot(const float* dp, const void* p, int pdt, int64_t rows, int64_t cols,
                          float* rowdot, cudaStream_t s) {
  LAUNCH_ROWS(bwd_rowdot_kernel, "softmax_bwd_rowdot", dp, p, pdt, rows, cols, rowdot);
}
void k_softmax_bwd_ds(const float* dp, const void* p, int pdt, int64_t rows, int64_t cols,
                      const float* rowdot, float scale, void* ds, int dsdt, cudaStream_t s) {
  LAUNCH_ROWS(bwd_ds_kernel, "softmax_bwd_ds", dp, p, pdt, rows, cols, rowdot, scale, ds, dsdt);
}
// dh = 64, bf16: 8 threads per row, one 16-B vector of each operand per thread.
__global__ void attn_rowdot64_kernel(const __nv_bfloat16* d_o, const __nv_bfloat16* o,
                                     int64_t rows, int64_t S, int64_t H, int64_t sb_hi,
                                     float* out) {
  const int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  const int64_t r = t / 8;
  const int part = static_cast<int>(t % 8);
  float acc = 0.f;
  if (r < rows) {
    const int64_t b = r / S, q = r - (r / S) * S;
    const int64_t base = (b / H) * sb_hi + q * (H * 64) + (b % H) * 64 + part * 8;
    const uint4 x = *reinterpret_cast<const uint4*>(d_o + base);
    const uint4 y = *reinterpret_cast<const uint4*>(o + base);
    const __nv_bfloat162* hx = reinterpret_cast<const __nv_bfloat162*>(&x);
    const __nv_bfloat162* hy = reinterpret_cast<const __nv_bfloat162*>(&y);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float2 a = __bfloat1622float2(hx[i]);
      const float2 c = __bfloat1622float2(hy[i]);
      acc += a.x * c.x + a.y * c.y;
    }
  }
#pragma unroll
  for (int off = 4; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
  if (r < rows && part == 0) out[r] = acc;
}

void k_attn_rowdot(const void* d_o, const void* o, int dt, int64_t nslices, int64_t S, int64_t H,
                   int64_t dh, int64_t sb_hi, float* out, cudaStream_t s) {
  const int64_t rows = nslices * S;
  if (rows == 0) return;
  if (dt == kBF16 && dh == 64 && reinterpret_cast<uintptr_t>(d_o) % 16 == 0 &&
      reinterpret_cast<uintptr_t>(o) % 16 == 0 && sb_hi % 8 == 0) {
    const int64_t threads = rows * 8;
    attn_rowdot64_kernel<<<static_cast<unsigned>((threads + 255) / 256), 256, 0, s>>>(
        static_cast<const __nv_bfloat16*>(d_o), static_cast<const __nv_bfloat16*>(o), rows, S, H,
        sb_hi, out);
    check_launch("attn_rowdot64");
    return;
  }
  attn_rowdot_kernel<<<blocks_for(rows), kWarps * 32, 0, s>>>(d_o, o, dt, rows, S, H, dh, sb_hi, out);
  check_launch("attn_rowdot");
}
void k_softmax_bwd_fused(const float* dp, const void* p, int pdt, int64_t rows, int64_t cols,
                         float scale, void* ds, int dsdt, cudaStream_t s) {
  LAUNCH_ROWS(bwd_fused_kernel, "softmax_bwd_fused", dp, p, pdt, rows, cols, scale, ds, dsdt);
}

}  // namespace c3d
