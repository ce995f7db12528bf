// Row / column / elementwise kernels of the layer path (HBM-bound). Row
// reductions use one warp per row with shuffles; column sums use a fixed
// two-stage tree so results are run-to-run deterministic (the reference's
// "run-determinism" check, cube3d/verify.hpp:738-744).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <type_traits>

#include "common.hpp"
#include "epi.cuh"
#include "kernels.hpp"

namespace c3d {

namespace {

constexpr int kWarpsPerBlock = 8;

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

inline unsigned row_blocks(int64_t rows) {
  return static_cast<unsigned>((rows + kWarpsPerBlock - 1) / kWarpsPerBlock);
}

// ------------------------------------------------------------ elementwise
__global__ void apply_epilogue_kernel(const void* in, int in_dt, int64_t rows, int64_t cols,
                                      Epilogue e) {
  const int64_t n = rows * cols;
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < n;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = t / cols, c = t % cols;
    const float v = ld_any(in, in_dt, t);
    epi_scalar(e, view_offset(e.out, 0, r, c), c, v);
  }
}

__global__ void convert_batch_kernel(ConvBatch b) {
  const ConvSeg& g = b.seg[blockIdx.y];
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < g.n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    st_any(g.dst, g.ddt, i, ld_any(g.src, g.sdt, i));
}

__global__ void convert_kernel(const void* src, int sdt, void* dst, int ddt, int64_t n) {
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < n;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x)
    st_any(dst, ddt, t, ld_any(src, sdt, t));
}

// y = gelu(x); x <- gelu'(x) in place (the MLP's saved pre-activation becomes the
// factor its backward multiplies by). Vector path: 8 bf16 / 4+4 fp32 per thread.
__global__ void gelu_save_kernel(void* x, int xdt, void* y, int ydt, int64_t n, int vec) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  const int64_t t0 = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (vec) {
    for (int64_t t = t0; t < n / 8; t += stride) {
      float v[8], g[8], d[8];
      if (xdt == kBF16) {
        const uint4 q = reinterpret_cast<const uint4*>(x)[t];
        const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&q);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const float2 f = __bfloat1622float2(h[i]);
          v[2 * i] = f.x;
          v[2 * i + 1] = f.y;
        }
      } else {
        const float4 a = reinterpret_cast<const float4*>(x)[2 * t];
        const float4 b = reinterpret_cast<const float4*>(x)[2 * t + 1];
        v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
        v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
      }
#pragma unroll
      for (int i = 0; i < 8; i += 2) {
        float2 g2, d2;
        gelu_both2(make_float2(v[i], v[i + 1]), g2, d2);
        g[i] = g2.x;
        g[i + 1] = g2.y;
        d[i] = d2.x;
        d[i + 1] = d2.y;
      }
      auto put = [&](void* base, int dt, const float* w) {
        if (dt == kBF16) {
          uint4 q;
          __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&q);
#pragma unroll
          for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(w[2 * i], w[2 * i + 1]);
          reinterpret_cast<uint4*>(base)[t] = q;
        } else {
          reinterpret_cast<float4*>(base)[2 * t] = make_float4(w[0], w[1], w[2], w[3]);
          reinterpret_cast<float4*>(base)[2 * t + 1] = make_float4(w[4], w[5], w[6], w[7]);
        }
      };
      put(y, ydt, g);
      put(x, xdt, d);
    }
    return;
  }
  for (int64_t t = t0; t < n; t += stride) {
    float g, d;
    gelu_both(ld_any(x, xdt, t), g, d);
    st_any(y, ydt, t, g);
    st_any(x, xdt, t, d);
  }
}

__global__ void mul_cols_kernel(const void* a, int adt, const float* b, void* c, int cdt,
                                int64_t rows, int64_t cols) {
  const int64_t n = rows * cols;
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < n;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x)
    st_any(c, cdt, t, ld_any(a, adt, t) * b[t % cols]);
}

// stage 1: partial[chunk][c] = sum over rows of chunk; stage 2: ordered sum of chunks.
constexpr int kColChunkRows = 64;
__global__ void colsum_partial_kernel(const void* x, int xdt, const void* y, int ydt,
                                      int64_t rows, int64_t cols, float* partial) {
  const int64_t c = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (c >= cols) return;
  const int64_t r0 = static_cast<int64_t>(blockIdx.y) * kColChunkRows;
  const int64_t r1 = min(rows, r0 + kColChunkRows);
  float acc = 0.f;
  for (int64_t r = r0; r < r1; ++r) {
    float v = ld_any(x, xdt, r * cols + c);
    if (y) v *= ld_any(y, ydt, r * cols + c);
    acc += v;
  }
  partial[blockIdx.y * cols + c] = acc;
}
// Column sums at HBM speed: a CTA of 32 warps covers 256 columns (8 per lane, 16-B loads)
// x `rows_per_cta` rows (the launcher sizes the grid to one wave, one CTA per SM; a warp
// issues 2-8 row loads before summing them), so >= 64 KB per SM stay in flight. Warps combine through shared memory in a
// fixed order into a per-chunk partial; the last CTA of each column tile (counter) sums
// the chunks in chunk order -- deterministic, and no second launch. With DUAL, one pass
// over x yields both colsum(x * y) (out) and colsum(x) (out2): LayerNorm's dgamma and
// dbeta.
constexpr int kCsWarps = 32;
template <int XDT, int YDT, bool DUAL>
__global__ void __launch_bounds__(32 * kCsWarps, 1) colsum_chunk_kernel(const void* x, const void* y, int64_t rows,
                                                              int64_t cols, int64_t rows_per_cta,
                                                              float* partial, unsigned* counters,
                                                              float* out, float* out2) {
  constexpr int NS = DUAL ? 2 : 1;
  __shared__ float red[kCsWarps][256];
  __shared__ unsigned last;
  const int lane = threadIdx.x % 32, w = threadIdx.x / 32;
  const int64_t c8 = blockIdx.x * 256LL + lane * 8;
  const int64_t rbeg = static_cast<int64_t>(blockIdx.y) * rows_per_cta;
  const int64_t rend = min(rows, rbeg + rows_per_cta);
  // raw 16-B words stay in registers until summed (8 values: one word bf16, two fp32)
  constexpr int QX = XDT == kBF16 ? 1 : 2, QY = YDT == kF32 ? 2 : 1;
  // 8 values of a raw word group: bf16 -> fp32 is a shift / mask of the 32-bit pair
  auto val = [](int dt, const uint4* q, int i) -> float {
    if (dt == kBF16) {
      const uint32_t u = reinterpret_cast<const uint32_t*>(q)[i / 2];
      return __uint_as_float((i & 1) ? (u & 0xffff0000u) : (u << 16));
    }
    return reinterpret_cast<const float*>(q)[i];
  };
  float acc[NS][8];
#pragma unroll
  for (int k = 0; k < NS; ++k)
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[k][i] = 0.f;
  const int64_t r0 = rbeg + w;
  const int64_t nr = r0 < rend ? (rend - r0 + kCsWarps - 1) / kCsWarps : 0;  // this warp's rows
  if (c8 < cols && nr > 0) {
    // row loads in flight per lane: 32 registers of raw words
    constexpr int U = 8 / (QX + (YDT >= 0 ? QY : 0));
    const int64_t stride = kCsWarps * cols;  // elements between this warp's rows
    const char* px = static_cast<const char*>(x) + (r0 * cols + c8) * (XDT == kBF16 ? 2 : 4);
    const char* py = YDT >= 0 ? static_cast<const char*>(y) + (r0 * cols + c8) * (YDT == kBF16 ? 2 : 4)
                              : nullptr;
    const int64_t sx = stride * (XDT == kBF16 ? 2 : 4), sy = stride * (YDT == kBF16 ? 2 : 4);
    auto step = [&](int n) {  // n <= U rows: loads first, then the sums
      uint4 qx[U][QX], qy[U][QY];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (u < n) {
#pragma unroll
          for (int i = 0; i < QX; ++i) qx[u][i] = __ldg(reinterpret_cast<const uint4*>(px + u * sx) + i);
          if (YDT >= 0) {
#pragma unroll
            for (int i = 0; i < QY; ++i) qy[u][i] = __ldg(reinterpret_cast<const uint4*>(py + u * sy) + i);
          }
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (u < n) {
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const float v = val(XDT, qx[u], i);
            if (YDT >= 0) {
              if (DUAL) acc[1][i] += v;
              acc[0][i] = fmaf(v, val(YDT, qy[u], i), acc[0][i]);
            } else {
              acc[0][i] += v;
            }
          }
        }
      }
      px += n * sx;
      if (YDT >= 0) py += n * sy;
    };
    int64_t k = 0;
#pragma unroll 1
    for (; k + U <= nr; k += U) step(U);
    if (k < nr) step(static_cast<int>(nr - k));
  }
  const int64_t c = blockIdx.x * 256LL + threadIdx.x;  // threads < 256: one column each
  const int64_t nchunks = gridDim.y;
  // warps combine through shared memory in warp order into this chunk's partial
#pragma unroll
  for (int k = 0; k < NS; ++k) {
    if (k) __syncthreads();
#pragma unroll
    for (int i = 0; i < 8; ++i) red[w][lane * 8 + i] = acc[k][i];
    __syncthreads();
    if (threadIdx.x < 256 && c < cols) {
      float t = 0.f;
#pragma unroll 8
      for (int q = 0; q < kCsWarps; ++q) t += red[q][threadIdx.x];
      partial[(k * nchunks + blockIdx.y) * cols + c] = t;
    }
  }
  // the last chunk CTA of this column tile reduces the tile's chunks in order
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned prev = atomicAdd(counters + blockIdx.x, 1u);
    last = prev + 1 == static_cast<unsigned>(nchunks) ? 1u : 0u;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  // warp w sums chunks w, w + kCsWarps, ... (8 columns per lane, 4 chunks in flight), then
  // the warps combine in order: a fixed association, so the result is deterministic
#pragma unroll
  for (int k = 0; k < NS; ++k) {
    float t[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    if (c8 < cols) {
      const float* base = partial + k * nchunks * cols + c8;
#pragma unroll 1
      for (int64_t q0 = w; q0 < nchunks; q0 += 4 * kCsWarps) {
        float4 v[4][2];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int64_t q = q0 + kCsWarps * u;
          if (q < nchunks) {
            v[u][0] = __ldcg(reinterpret_cast<const float4*>(base + q * cols));
            v[u][1] = __ldcg(reinterpret_cast<const float4*>(base + q * cols + 4));
          } else {
            v[u][0] = v[u][1] = make_float4(0.f, 0.f, 0.f, 0.f);
          }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          t[0] += v[u][0].x; t[1] += v[u][0].y; t[2] += v[u][0].z; t[3] += v[u][0].w;
          t[4] += v[u][1].x; t[5] += v[u][1].y; t[6] += v[u][1].z; t[7] += v[u][1].w;
        }
      }
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < 8; ++i) red[w][lane * 8 + i] = t[i];
    __syncthreads();
    if (threadIdx.x < 256 && c < cols) {
      float sum = 0.f;
#pragma unroll 8
      for (int q = 0; q < kCsWarps; ++q) sum += red[q][threadIdx.x];
      (k == 0 ? out : out2)[c] = sum;
    }
  }
}

__global__ void colsum_final_kernel(const float* partial, int64_t chunks, int64_t cols,
                                    float* out) {
  const int64_t c = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (c >= cols) return;
  float acc = 0.f;
  for (int64_t k = 0; k < chunks; ++k) acc += partial[k * cols + c];
  out[c] = acc;
}

// ------------------------------------------------------------ LayerNorm
__global__ void row_sum_kernel(const void* x, int dt, int64_t rows, int64_t cols,
                               const float* sums, float inv_h, float* out) {
  const int64_t r = blockIdx.x * static_cast<int64_t>(kWarpsPerBlock) + threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  if (r >= rows) return;
  const float mean = sums ? sums[r] * inv_h : 0.f;
  float acc = 0.f;
  for (int64_t c = lane; c < cols; c += 32) {
    const float v = ld_any(x, dt, r * cols + c);
    if (sums) {
      const float d = v - mean;
      acc += d * d;
    } else {
      acc += v;
    }
  }
  acc = warp_sum(acc);
  if (lane == 0) out[r] = acc;
}

__global__ void ln_apply_kernel(const void* x, int dt, int64_t rows, int64_t cols,
                                const float* sums, const float* sq, float inv_h, float eps,
                                const float* gamma, const float* beta, void* y, int ydt,
                                void* xhat, int xhdt, float* inv_std) {
  const int64_t r = blockIdx.x * static_cast<int64_t>(kWarpsPerBlock) + threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  if (r >= rows) return;
  const float mean = sums[r] * inv_h;
  const float inv = 1.f / sqrtf(sq[r] * inv_h + eps);
  if (lane == 0 && inv_std) inv_std[r] = inv;
  for (int64_t c = lane; c < cols; c += 32) {
    const float xh = (ld_any(x, dt, r * cols + c) - mean) * inv;
    if (xhat) st_any(xhat, xhdt, r * cols + c, xh);
    st_any(y, ydt, r * cols + c, gamma[c] * xh + beta[c]);
  }
}

__global__ void ln_fwd_fused_kernel(const void* x, int dt, int64_t rows, int64_t cols,
                                    float eps, const float* gamma, const float* beta, void* y,
                                    int ydt, void* xhat, int xhdt, float* inv_std) {
  const int64_t r = blockIdx.x * static_cast<int64_t>(kWarpsPerBlock) + threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  if (r >= rows) return;
  const float inv_h = 1.f / static_cast<float>(cols);
  float s = 0.f;
  for (int64_t c = lane; c < cols; c += 32) s += ld_any(x, dt, r * cols + c);
  const float mean = warp_sum(s) * inv_h;
  float q = 0.f;
  for (int64_t c = lane; c < cols; c += 32) {
    const float d = ld_any(x, dt, r * cols + c) - mean;
    q += d * d;
  }
  const float inv = 1.f / sqrtf(warp_sum(q) * inv_h + eps);
  if (lane == 0 && inv_std) inv_std[r] = inv;
  for (int64_t c = lane; c < cols; c += 32) {
    const float xh = (ld_any(x, dt, r * cols + c) - mean) * inv;
    if (xhat) st_any(xhat, xhdt, r * cols + c, xh);
    st_any(y, ydt, r * cols + c, gamma[c] * xh + beta[c]);
  }
}

__global__ void ln_bwd_rows_kernel(const void* dy, int dt, const void* xhat, int xdt,
                                   const float* gamma, int64_t rows, int64_t cols, float* rs) {
  const int64_t r = blockIdx.x * static_cast<int64_t>(kWarpsPerBlock) + threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  if (r >= rows) return;
  float s = 0.f, d = 0.f;
  for (int64_t c = lane; c < cols; c += 32) {
    const float g = ld_any(dy, dt, r * cols + c) * gamma[c];
    s += g;
    d += g * ld_any(xhat, xdt, r * cols + c);
  }
  s = warp_sum(s);
  d = warp_sum(d);
  if (lane == 0) {
    rs[r] = s;
    rs[rows + r] = d;
  }
}

__global__ void ln_bwd_dx_kernel(const void* dy, int dt, const void* xhat, int xdt,
                                 const float* gamma, const float* inv_std, const float* rs,
                                 float inv_h, int64_t rows, int64_t cols, const void* resid,
                                 int rdt, void* dx, int dxdt) {
  const int64_t n = rows * cols;
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < n;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = t / cols, c = t % cols;
    const float g = ld_any(dy, dt, t) * gamma[c];
    float v = inv_std[r] * (g - rs[r] * inv_h - ld_any(xhat, xdt, t) * rs[rows + r] * inv_h);
    if (resid) v += ld_any(resid, rdt, t);
    st_any(dx, dxdt, t, v);
  }
}

// ---- vectorised LayerNorm: a warp per row, the row held in registers (8 values per
// 16-B vector, VPL vectors per lane, cols = 256 * VPL); same arithmetic as above.
__device__ __forceinline__ void vload8(const void* base, int dt, int64_t off, float (&v)[8]) {
  if (dt == kBF16) {
    const uint4 q = *reinterpret_cast<const uint4*>(static_cast<const __nv_bfloat16*>(base) + off);
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&q);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float2 f = __bfloat1622float2(h[i]);
      v[2 * i] = f.x;
      v[2 * i + 1] = f.y;
    }
  } else {
    const float4 a = *reinterpret_cast<const float4*>(static_cast<const float*>(base) + off);
    const float4 b = *reinterpret_cast<const float4*>(static_cast<const float*>(base) + off + 4);
    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
    v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
  }
}
__device__ __forceinline__ void vstore8(void* base, int dt, int64_t off, const float (&v)[8]) {
  if (dt == kBF16) {
    uint4 q;
    __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&q);
#pragma unroll
    for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(v[2 * i], v[2 * i + 1]);
    *reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(base) + off) = q;
  } else {
    *reinterpret_cast<float4*>(static_cast<float*>(base) + off) = make_float4(v[0], v[1], v[2], v[3]);
    *reinterpret_cast<float4*>(static_cast<float*>(base) + off + 4) = make_float4(v[4], v[5], v[6], v[7]);
  }
}

template <int VPL>
__global__ void ln_fwd_vec_kernel(const void* x, int dt, int64_t rows, float eps,
                                  const float* gamma, const float* beta, void* y, int ydt,
                                  void* xhat, int xhdt, float* inv_std, const float* gsums,
                                  const float* gsq, float ginv_h) {
  constexpr int64_t cols = 256 * VPL;
  const int64_t r = blockIdx.x * static_cast<int64_t>(kWarpsPerBlock) + threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  if (r >= rows) return;
  float v[VPL][8];
  float s = 0.f;
#pragma unroll
  for (int k = 0; k < VPL; ++k) {
    vload8(x, dt, r * cols + (k * 32 + lane) * 8, v[k]);
#pragma unroll
    for (int i = 0; i < 8; ++i) s += v[k][i];
  }
  float mean, inv;
  if (gsums) {  // statistics all-reduced along the output axis
    mean = gsums[r] * ginv_h;
    inv = 1.f / sqrtf(gsq[r] * ginv_h + eps);
  } else {
    const float inv_h = 1.f / static_cast<float>(cols);
    mean = warp_sum(s) * inv_h;
    float q = 0.f;
#pragma unroll
    for (int k = 0; k < VPL; ++k)
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float d = v[k][i] - mean;
        q += d * d;
      }
    inv = 1.f / sqrtf(warp_sum(q) * inv_h + eps);
  }
  if (lane == 0 && inv_std) inv_std[r] = inv;
#pragma unroll
  for (int k = 0; k < VPL; ++k) {
    const int64_t c = (k * 32 + lane) * 8;
    float xh[8], o[8];
    const float4 g0 = __ldg(reinterpret_cast<const float4*>(gamma + c));
    const float4 g1 = __ldg(reinterpret_cast<const float4*>(gamma + c + 4));
    const float4 b0 = __ldg(reinterpret_cast<const float4*>(beta + c));
    const float4 b1 = __ldg(reinterpret_cast<const float4*>(beta + c + 4));
    const float g[8] = {g0.x, g0.y, g0.z, g0.w, g1.x, g1.y, g1.z, g1.w};
    const float bb[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      xh[i] = (v[k][i] - mean) * inv;
      o[i] = g[i] * xh[i] + bb[i];
    }
    if (xhat) vstore8(xhat, xhdt, r * cols + c, xh);
    vstore8(y, ydt, r * cols + c, o);
  }
}

// Row sum (sums == null) or centred sum of squares of a row held in registers.
template <int VPL>
__global__ void row_sum_vec_kernel(const void* x, int dt, int64_t rows, const float* sums,
                                   float inv_h, float* out) {
  constexpr int64_t cols = 256 * VPL;
  const int64_t r = blockIdx.x * static_cast<int64_t>(kWarpsPerBlock) + threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  if (r >= rows) return;
  const float mean = sums ? sums[r] * inv_h : 0.f;
  float acc = 0.f;
#pragma unroll
  for (int k = 0; k < VPL; ++k) {
    float v[8];
    vload8(x, dt, r * cols + (k * 32 + lane) * 8, v);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (sums) {
        const float d = v[i] - mean;
        acc += d * d;
      } else {
        acc += v[i];
      }
    }
  }
  acc = warp_sum(acc);
  if (lane == 0) out[r] = acc;
}

template <int VPL>
__global__ void ln_bwd_rows_vec_kernel(const void* dy, int dt, const void* xhat, int xdt,
                                       const float* gamma, int64_t rows, float* rs) {
  constexpr int64_t cols = 256 * VPL;
  const int64_t r = blockIdx.x * static_cast<int64_t>(kWarpsPerBlock) + threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  if (r >= rows) return;
  float s = 0.f, d = 0.f;
#pragma unroll
  for (int k = 0; k < VPL; ++k) {
    const int64_t c = (k * 32 + lane) * 8;
    float g[8], xh[8];
    vload8(dy, dt, r * cols + c, g);
    vload8(xhat, xdt, r * cols + c, xh);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const float gg = g[i] * __ldg(gamma + c + i);
      s += gg;
      d += gg * xh[i];
    }
  }
  s = warp_sum(s);
  d = warp_sum(d);
  if (lane == 0) {
    rs[r] = s;
    rs[rows + r] = d;
  }
}

// Local row moments over this rank's column block: st[2r] = mean, st[2r+1] = centred
// sum of squares (Chan et al.'s pairwise combination then merges the blocks exactly).
template <int VPL>
__global__ void row_moments_vec_kernel(const void* x, int dt, int64_t rows, float* st) {
  constexpr int64_t cols = 256 * VPL;
  const int64_t r = blockIdx.x * static_cast<int64_t>(kWarpsPerBlock) + threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  if (r >= rows) return;
  float v[VPL][8];
  float s = 0.f;
#pragma unroll
  for (int k = 0; k < VPL; ++k) {
    vload8(x, dt, r * cols + (k * 32 + lane) * 8, v[k]);
#pragma unroll
    for (int i = 0; i < 8; ++i) s += v[k][i];
  }
  const float mean = warp_sum(s) * (1.f / static_cast<float>(cols));
  float q = 0.f;
#pragma unroll
  for (int k = 0; k < VPL; ++k)
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const float d = v[k][i] - mean;
      q += d * d;
    }
  q = warp_sum(q);
  if (lane == 0) {
    st[2 * r] = mean;
    st[2 * r + 1] = q;
  }
}

// Merges the P gathered (mean, M2) pairs of each row (equal block sizes n) into the
// full-row sum and centred sum of squares.
__global__ void combine_moments_kernel(const float* st, int P, int64_t rows, float n,
                                       float* sums, float* sq) {
  const int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (r >= rows) return;
  float m = 0.f;
  for (int p = 0; p < P; ++p) m += st[p * 2 * rows + 2 * r];
  m /= static_cast<float>(P);
  float q = 0.f;
  for (int p = 0; p < P; ++p) {
    const float d = st[p * 2 * rows + 2 * r] - m;
    q += st[p * 2 * rows + 2 * r + 1] + n * d * d;
  }
  sums[r] = m * n * static_cast<float>(P);
  sq[r] = q;
}

// Row statistics and dx in one pass when they need no all-reduce (p_out = 1):
// g = dy * gamma, s = sum g, d = sum g * xhat, dx = inv_std * (g - s/h - xhat * d/h) (+ resid).
// With `grs` the row sums come all-reduced ([s | d], scaled by ginv_h).
template <int VPL>
__global__ void __launch_bounds__(256, 2) ln_bwd_vec_kernel(const void* dy, int dt, const void* xhat, int xdt,
                                  const float* gamma, const float* inv_std, int64_t rows,
                                  const void* resid, int rdt, void* dx, int dxdt,
                                  const float* grs, float ginv_h) {
  constexpr int64_t cols = 256 * VPL;
  const int64_t r = blockIdx.x * static_cast<int64_t>(kWarpsPerBlock) + threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  if (r >= rows) return;
  float g[VPL][8], xh[VPL][8];
  float s = 0.f, d = 0.f;
#pragma unroll
  for (int k = 0; k < VPL; ++k) {
    const int64_t c = (k * 32 + lane) * 8;
    vload8(dy, dt, r * cols + c, g[k]);
    vload8(xhat, xdt, r * cols + c, xh[k]);
    const float4 g0 = __ldg(reinterpret_cast<const float4*>(gamma + c));
    const float4 g1 = __ldg(reinterpret_cast<const float4*>(gamma + c + 4));
    const float gm[8] = {g0.x, g0.y, g0.z, g0.w, g1.x, g1.y, g1.z, g1.w};
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      g[k][i] *= gm[i];
      s += g[k][i];
      d += g[k][i] * xh[k][i];
    }
  }
  if (grs) {
    s = grs[r] * ginv_h;
    d = grs[rows + r] * ginv_h;
  } else {
    const float inv_h = 1.f / static_cast<float>(cols);
    s = warp_sum(s) * inv_h;
    d = warp_sum(d) * inv_h;
  }
  const float inv = inv_std[r];
#pragma unroll
  for (int k = 0; k < VPL; ++k) {
    const int64_t c = (k * 32 + lane) * 8;
    float o[8], rr[8];
    if (resid) vload8(resid, rdt, r * cols + c, rr);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      o[i] = inv * (g[k][i] - s - xh[k][i] * d);
      if (resid) o[i] += rr[i];
    }
    vstore8(dx, dxdt, r * cols + c, o);
  }
}

// LayerNorm backward with its column sums (bf16 rows): dx as ln_bwd_vec_kernel, plus
// dgamma = sum dy * xhat, dbeta = sum dy and, with RES, sum resid (the bias gradient of the
// linear whose output gradient the residual carries) -- one read of every operand instead
// of a separate column-sum pass. Persistent: a CTA's warps stride the rows, keep their
// lanes' column sums in registers, combine them in warp order through shared memory and
// write one partial row per CTA (partial[cta][k][cols]); colsum_parts_kernel sums those.
template <int VPL, bool RES>
__global__ void __launch_bounds__(256, 1) ln_bwd_sums_kernel(
    const __nv_bfloat16* dy, const __nv_bfloat16* xhat, const float* gamma, const float* inv_std,
    int64_t rows, const __nv_bfloat16* resid, __nv_bfloat16* dx, float* partial) {
  constexpr int cols = 256 * VPL;
  constexpr int NS = RES ? 3 : 2;
  __shared__ float red[kWarpsPerBlock][cols];
  const int lane = threadIdx.x % 32, w = threadIdx.x / 32;
  auto lo = [](uint32_t u) { return __uint_as_float(u << 16); };
  auto hi = [](uint32_t u) { return __uint_as_float(u & 0xffff0000u); };
  float gm[VPL][8], acc[NS][VPL][8];
#pragma unroll
  for (int k = 0; k < VPL; ++k) {
    const int c = (k * 32 + lane) * 8;
    const float4 g0 = __ldg(reinterpret_cast<const float4*>(gamma + c));
    const float4 g1 = __ldg(reinterpret_cast<const float4*>(gamma + c + 4));
    gm[k][0] = g0.x; gm[k][1] = g0.y; gm[k][2] = g0.z; gm[k][3] = g0.w;
    gm[k][4] = g1.x; gm[k][5] = g1.y; gm[k][6] = g1.z; gm[k][7] = g1.w;
#pragma unroll
    for (int j = 0; j < NS; ++j)
#pragma unroll
      for (int i = 0; i < 8; ++i) acc[j][k][i] = 0.f;
  }
  const float inv_h = 1.f / static_cast<float>(cols);
  for (int64_t r = static_cast<int64_t>(blockIdx.x) * kWarpsPerBlock + w; r < rows;
       r += static_cast<int64_t>(gridDim.x) * kWarpsPerBlock) {
    uint4 qd[VPL], qx[VPL], qr[VPL];
#pragma unroll
    for (int k = 0; k < VPL; ++k) {
      const int64_t off = r * cols + (k * 32 + lane) * 8;
      qd[k] = __ldg(reinterpret_cast<const uint4*>(dy + off));
      qx[k] = __ldg(reinterpret_cast<const uint4*>(xhat + off));
      if (RES) qr[k] = __ldg(reinterpret_cast<const uint4*>(resid + off));
    }
    const float inv = __ldg(inv_std + r);
    float sg = 0.f, sd = 0.f;
#pragma unroll
    for (int k = 0; k < VPL; ++k) {
      const uint32_t* ud = reinterpret_cast<const uint32_t*>(&qd[k]);
      const uint32_t* ux = reinterpret_cast<const uint32_t*>(&qx[k]);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float d = (i & 1) ? hi(ud[i / 2]) : lo(ud[i / 2]);
        const float x = (i & 1) ? hi(ux[i / 2]) : lo(ux[i / 2]);
        acc[0][k][i] = fmaf(d, x, acc[0][k][i]);
        acc[1][k][i] += d;
        const float g = d * gm[k][i];
        sg += g;
        sd = fmaf(g, x, sd);
      }
    }
    sg = warp_sum(sg) * inv_h;
    sd = warp_sum(sd) * inv_h;
#pragma unroll
    for (int k = 0; k < VPL; ++k) {
      const uint32_t* ud = reinterpret_cast<const uint32_t*>(&qd[k]);
      const uint32_t* ux = reinterpret_cast<const uint32_t*>(&qx[k]);
      const uint32_t* ur = reinterpret_cast<const uint32_t*>(&qr[k]);
      uint4 o;
      uint32_t* uo = reinterpret_cast<uint32_t*>(&o);
#pragma unroll
      for (int i = 0; i < 8; i += 2) {
        float v[2];
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const float d = e ? hi(ud[i / 2]) : lo(ud[i / 2]);
          const float x = e ? hi(ux[i / 2]) : lo(ux[i / 2]);
          v[e] = inv * (d * gm[k][i + e] - sg - x * sd);
          if (RES) {
            const float rv = e ? hi(ur[i / 2]) : lo(ur[i / 2]);
            acc[NS - 1][k][i + e] += rv;
            v[e] += rv;
          }
        }
        const __nv_bfloat162 h2 = __floats2bfloat162_rn(v[0], v[1]);
        uo[i / 2] = *reinterpret_cast<const uint32_t*>(&h2);
      }
      *reinterpret_cast<uint4*>(dx + r * cols + (k * 32 + lane) * 8) = o;
    }
  }
  // warps combine in warp order; thread t owns columns t, t + 256, ...
#pragma unroll
  for (int j = 0; j < NS; ++j) {
    if (j) __syncthreads();
#pragma unroll
    for (int k = 0; k < VPL; ++k)
#pragma unroll
      for (int i = 0; i < 8; ++i) red[w][(k * 32 + lane) * 8 + i] = acc[j][k][i];
    __syncthreads();
#pragma unroll
    for (int q = 0; q < VPL; ++q) {
      const int c = q * 256 + threadIdx.x;
      float t = 0.f;
#pragma unroll
      for (int ww = 0; ww < kWarpsPerBlock; ++ww) t += red[ww][c];
      partial[(static_cast<int64_t>(blockIdx.x) * NS + j) * cols + c] = t;
    }
  }
}

// out[j] for j < width: sum over parts p of partial[p][j], in part order (32 part groups
// per column, then the groups in order: a fixed association). Block: 32 columns x 32 groups.
__global__ void __launch_bounds__(1024) colsum_parts_kernel(const float* partial, int parts,
                                                            int64_t width, int64_t seg,
                                                            float* out0, float* out1, float* out2) {
  __shared__ float red[32][33];
  const int tx = threadIdx.x % 32, ty = threadIdx.x / 32;
  const int64_t j = blockIdx.x * 32LL + tx;
  float t = 0.f;
  if (j < width) {
    float v[8];
    for (int p0 = ty; p0 < parts; p0 += 32 * 8) {
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int p = p0 + 32 * u;
        v[u] = p < parts ? __ldcg(partial + static_cast<int64_t>(p) * width + j) : 0.f;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) t += v[u];
    }
  }
  red[ty][tx] = t;
  __syncthreads();
  if (ty == 0 && j < width) {
    float sum = 0.f;
#pragma unroll 8
    for (int q = 0; q < 32; ++q) sum += red[q][tx];
    const int64_t k = j / seg;
    float* o = k == 0 ? out0 : k == 1 ? out1 : out2;
    o[j % seg] = sum;
  }
}

__global__ void copy_heads_kernel(const void* src, int64_t src_ld, int64_t src_hs, void* dst,
                                  int64_t dst_ld, int64_t dst_hs, int64_t rows, int64_t heads,
                                  int64_t dh, int dt) {
  const int64_t n = rows * heads * dh;
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < n;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t k = t % dh, h = (t / dh) % heads, r = t / (dh * heads);
    st_any(dst, dt, r * dst_ld + h * dst_hs + k, ld_any(src, dt, r * src_ld + h * src_hs + k));
  }
}

unsigned grid_for(int64_t n) {
  const int64_t b = (n + 255) / 256;
  return static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>(b, 148 * 16)));
}

}  // namespace

void k_apply_epilogue(const void* in, int in_dtype, int64_t rows, int64_t cols,
                      const Epilogue& e, cudaStream_t s) {
  if (rows * cols == 0) return;
  apply_epilogue_kernel<<<grid_for(rows * cols), 256, 0, s>>>(in, in_dtype, rows, cols, e);
  check_launch("apply_epilogue");
}


void k_colsum(const void* x, int xdt, const void* y, int ydt, int64_t rows, int64_t cols,
              float* out, cudaStream_t s, float* out_x) {
  if (cols == 0) return;
  auto al = [](const void* q) { return reinterpret_cast<uintptr_t>(q) % 16 == 0; };
  const bool vec = cols % 8 == 0 && al(x) && (!y || al(y)) && rows > 0;
  if (!vec) {
    // generic path: two-stage partial / final kernels (and a second pass for out_x)
    const int64_t chunks = std::max<int64_t>(1, (rows + kColChunkRows - 1) / kColChunkRows);
    float* partial = nullptr;
    C3D_CUDA(cudaMallocAsync(&partial, chunks * cols * sizeof(float), s));
    for (int pass = 0; pass < (out_x && y ? 2 : 1); ++pass) {
      const void* yy = pass == 0 ? y : nullptr;
      float* o = pass == 0 ? out : out_x;
      if (rows == 0) {
        C3D_CUDA(cudaMemsetAsync(partial, 0, chunks * cols * sizeof(float), s));
      } else {
        dim3 g1(static_cast<unsigned>((cols + 127) / 128), static_cast<unsigned>(chunks));
        colsum_partial_kernel<<<g1, 128, 0, s>>>(x, xdt, yy, ydt, rows, cols, partial);
        check_launch("colsum_partial");
      }
      colsum_final_kernel<<<static_cast<unsigned>((cols + 127) / 128), 128, 0, s>>>(partial, chunks,
                                                                                    cols, o);
      check_launch("colsum_final");
    }
    C3D_CUDA(cudaFreeAsync(partial, s));
    return;
  }
  const bool dual = out_x && y;
  const int64_t tiles = (cols + 255) / 256;
  // one wave of 1024-thread CTAs, one per SM, each summing a contiguous block of rows (a
  // multiple of 32): no partial second wave, and few chunk partials for the finishing CTA
  static int num_sms = 0;
  if (num_sms == 0) {
    int dev = 0;
    C3D_CUDA(cudaGetDevice(&dev));
    C3D_CUDA(cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, dev));
  }
  int64_t chunks = std::max<int64_t>(1, std::min<int64_t>(num_sms / tiles, (rows + 31) / 32));
  const int64_t rows_per_cta = ((rows + chunks - 1) / chunks + 31) / 32 * 32;
  chunks = std::max<int64_t>(1, (rows + rows_per_cta - 1) / rows_per_cta);
  char* scratch = nullptr;
  const size_t pbytes = static_cast<size_t>((dual ? 2 : 1) * chunks * cols) * sizeof(float);
  C3D_CUDA(cudaMallocAsync(&scratch, pbytes + tiles * sizeof(unsigned), s));
  unsigned* counters = reinterpret_cast<unsigned*>(scratch + pbytes);
  C3D_CUDA(cudaMemsetAsync(counters, 0, tiles * sizeof(unsigned), s));
  float* partial = reinterpret_cast<float*>(scratch);
  dim3 g(static_cast<unsigned>(tiles), static_cast<unsigned>(chunks));
  const int yk = y ? ydt : -1;
#define C3D_COLSUM(XD, YD, DU) \
  colsum_chunk_kernel<XD, YD, DU><<<g, 32 * kCsWarps, 0, s>>>(x, y, rows, cols, rows_per_cta, partial, \
                                                     counters, out, out_x)
  if (dual) {
    if (xdt == kBF16 && yk == kBF16) C3D_COLSUM(kBF16, kBF16, true);
    else if (xdt == kBF16) C3D_COLSUM(kBF16, kF32, true);
    else if (yk == kBF16) C3D_COLSUM(kF32, kBF16, true);
    else C3D_COLSUM(kF32, kF32, true);
  } else {
    if (xdt == kBF16 && yk == -1) C3D_COLSUM(kBF16, -1, false);
    else if (xdt == kBF16 && yk == kBF16) C3D_COLSUM(kBF16, kBF16, false);
    else if (xdt == kBF16 && yk == kF32) C3D_COLSUM(kBF16, kF32, false);
    else if (xdt == kF32 && yk == -1) C3D_COLSUM(kF32, -1, false);
    else if (xdt == kF32 && yk == kBF16) C3D_COLSUM(kF32, kBF16, false);
    else C3D_COLSUM(kF32, kF32, false);
  }
#undef C3D_COLSUM
  check_launch("colsum_chunk");
  if (out_x && !y) C3D_CUDA(cudaMemcpyAsync(out_x, out, cols * sizeof(float), cudaMemcpyDeviceToDevice, s));
  C3D_CUDA(cudaFreeAsync(scratch, s));
}

void k_convert_batch(const ConvSeg* segs, int n, cudaStream_t s) {
  for (int i0 = 0; i0 < n; i0 += ConvBatch::kMax) {
    ConvBatch b;
    const int m = std::min(n - i0, ConvBatch::kMax);
    int64_t most = 0;
    for (int i = 0; i < m; ++i) {
      b.seg[i] = segs[i0 + i];
      most = std::max(most, segs[i0 + i].n);
    }
    if (most == 0) continue;
    const unsigned bx = static_cast<unsigned>(std::min<int64_t>((most + 255) / 256, 148 * 4));
    convert_batch_kernel<<<dim3(bx, static_cast<unsigned>(m)), 256, 0, s>>>(b);
    check_launch("convert_batch");
  }
}

void k_convert(const void* src, int sdt, void* dst, int ddt, int64_t n, cudaStream_t s) {
  if (n == 0) return;
  convert_kernel<<<grid_for(n), 256, 0, s>>>(src, sdt, dst, ddt, n);
  check_launch("convert");
}

void k_gelu_save(void* x, int xdt, void* y, int ydt, int64_t n, cudaStream_t s) {
  if (n == 0) return;
  const bool vec = n % 8 == 0 && reinterpret_cast<uintptr_t>(x) % 16 == 0 &&
                   reinterpret_cast<uintptr_t>(y) % 16 == 0;
  const int64_t work = vec ? n / 8 : n;
  const int blocks = static_cast<int>(std::min<int64_t>((work + 255) / 256, 148 * 16));
  gelu_save_kernel<<<blocks, 256, 0, s>>>(x, xdt, y, ydt, n, vec ? 1 : 0);
  check_launch("gelu_save");
}

void k_mul_cols(const void* a, int adt, const float* b, void* c, int cdt, int64_t rows,
                int64_t cols, cudaStream_t s) {
  if (rows * cols == 0) return;
  mul_cols_kernel<<<grid_for(rows * cols), 256, 0, s>>>(a, adt, b, c, cdt, rows, cols);
  check_launch("mul_cols");
}

namespace {
bool al16(const void* p) { return reinterpret_cast<uintptr_t>(p) % 16 == 0; }
int ln_vpl(int64_t cols) {
  return (cols == 256 || cols == 512 || cols == 1024 || cols == 2048) ? static_cast<int>(cols / 256) : 0;
}
template <typename F>
void by_vpl(int vpl, F&& f) {
  if (vpl == 1) f(std::integral_constant<int, 1>{});
  else if (vpl == 2) f(std::integral_constant<int, 2>{});
  else if (vpl == 4) f(std::integral_constant<int, 4>{});
  else f(std::integral_constant<int, 8>{});
}
}  // namespace

bool k_row_moments(const void* x, int dt, int64_t rows, int64_t cols, float* st, cudaStream_t s) {
  const int vpl = ln_vpl(cols);
  if (!vpl || !al16(x)) return false;
  if (rows == 0) return true;
  by_vpl(vpl, [&](auto V) {
    row_moments_vec_kernel<decltype(V)::value><<<row_blocks(rows), 32 * kWarpsPerBlock, 0, s>>>(
        x, dt, rows, st);
  });
  check_launch("row_moments");
  return true;
}

void k_combine_moments(const float* st, int P, int64_t rows, int64_t n, float* sums, float* sq,
                       cudaStream_t s) {
  if (rows == 0) return;
  combine_moments_kernel<<<static_cast<unsigned>((rows + 255) / 256), 256, 0, s>>>(
      st, P, rows, static_cast<float>(n), sums, sq);
  check_launch("combine_moments");
}

void k_row_sum(const void* x, int dt, int64_t rows, int64_t cols, const float* sums,
               float inv_h, float* out, cudaStream_t s) {
  if (rows == 0) return;
  if (const int vpl = ln_vpl(cols); vpl && al16(x)) {
    by_vpl(vpl, [&](auto V) {
      row_sum_vec_kernel<decltype(V)::value><<<row_blocks(rows), 32 * kWarpsPerBlock, 0, s>>>(
          x, dt, rows, sums, inv_h, out);
    });
    check_launch("row_sum_vec");
    return;
  }
  row_sum_kernel<<<row_blocks(rows), 32 * kWarpsPerBlock, 0, s>>>(x, dt, rows, cols, sums, inv_h,
                                                                  out);
  check_launch("row_sum");
}

void k_ln_apply(const void* x, int dt, int64_t rows, int64_t cols, const float* sums,
                const float* sq, float inv_h, float eps, const float* gamma, const float* beta,
                void* y, int ydt, void* xhat, int xhdt, float* inv_std, cudaStream_t s) {
  if (rows == 0) return;
  if (const int vpl = ln_vpl(cols);
      vpl && al16(x) && al16(y) && (!xhat || al16(xhat)) && al16(gamma) && al16(beta)) {
    by_vpl(vpl, [&](auto V) {
      ln_fwd_vec_kernel<decltype(V)::value><<<row_blocks(rows), 32 * kWarpsPerBlock, 0, s>>>(
          x, dt, rows, eps, gamma, beta, y, ydt, xhat, xhdt, inv_std, sums, sq, inv_h);
    });
    check_launch("ln_apply_vec");
    return;
  }
  ln_apply_kernel<<<row_blocks(rows), 32 * kWarpsPerBlock, 0, s>>>(
      x, dt, rows, cols, sums, sq, inv_h, eps, gamma, beta, y, ydt, xhat, xhdt, inv_std);
  check_launch("ln_apply");
}

void k_ln_fwd_fused(const void* x, int dt, int64_t rows, int64_t cols, float eps,
                    const float* gamma, const float* beta, void* y, int ydt, void* xhat,
                    int xhdt, float* inv_std, cudaStream_t s) {
  if (rows == 0) return;
  const int vpl = ln_vpl(cols);
  if (vpl && al16(x) && al16(y) && (!xhat || al16(xhat)) && al16(gamma) && al16(beta)) {
    auto launch = [&](auto kern) {
      kern<<<row_blocks(rows), 32 * kWarpsPerBlock, 0, s>>>(x, dt, rows, eps, gamma, beta, y, ydt,
                                                            xhat, xhdt, inv_std, nullptr, nullptr,
                                                            0.f);
    };
    if (vpl == 1) launch(ln_fwd_vec_kernel<1>);
    else if (vpl == 2) launch(ln_fwd_vec_kernel<2>);
    else if (vpl == 4) launch(ln_fwd_vec_kernel<4>);
    else launch(ln_fwd_vec_kernel<8>);
    check_launch("ln_fwd_vec");
    return;
  }
  ln_fwd_fused_kernel<<<row_blocks(rows), 32 * kWarpsPerBlock, 0, s>>>(
      x, dt, rows, cols, eps, gamma, beta, y, ydt, xhat, xhdt, inv_std);
  check_launch("ln_fwd_fused");
}

bool k_ln_bwd_fused(const void* dy, int dt, const void* xhat, int xdt, const float* gamma,
                    const float* inv_std, int64_t rows, int64_t cols, const void* resid, int rdt,
                    void* dx, int dxdt, cudaStream_t s) {
  const int vpl = ln_vpl(cols);
  if (!vpl || !al16(dy) || !al16(xhat) || !al16(gamma) || !al16(dx) || (resid && !al16(resid)))
    return false;
  if (rows == 0) return true;
  auto launch = [&](auto kern) {
    kern<<<row_blocks(rows), 32 * kWarpsPerBlock, 0, s>>>(dy, dt, xhat, xdt, gamma, inv_std, rows,
                                                          resid, rdt, dx, dxdt, nullptr, 0.f);
  };
  if (vpl == 1) launch(ln_bwd_vec_kernel<1>);
  else if (vpl == 2) launch(ln_bwd_vec_kernel<2>);
  else if (vpl == 4) launch(ln_bwd_vec_kernel<4>);
  else launch(ln_bwd_vec_kernel<8>);
  check_launch("ln_bwd_vec");
  return true;
}

void k_colsum_parts(const float* partial, int parts, int64_t width, float* out, cudaStream_t s) {
  if (width == 0) return;
  colsum_parts_kernel<<<static_cast<unsigned>((width + 31) / 32), 1024, 0, s>>>(
      partial, parts, width, width, out, nullptr, nullptr);
  check_launch("colsum_parts");
}

bool k_ln_bwd_sums(const void* dy, int dt, const void* xhat, int xdt, const float* gamma,
                   const float* inv_std, int64_t rows, int64_t cols, const void* resid, int rdt,
                   void* dx, int dxdt, float* dgamma, float* dbeta, float* dresid,
                   cudaStream_t s) {
  const int vpl = ln_vpl(cols);
  // the per-lane column sums live in registers: up to 1024 columns (VPL 4)
  if (!vpl || vpl > 4 || dt != kBF16 || xdt != kBF16 || dxdt != kBF16 || (resid && rdt != kBF16) ||
      (resid != nullptr) != (dresid != nullptr) || !al16(dy) || !al16(xhat) || !al16(gamma) || !al16(dx) ||
      (resid && !al16(resid)))
    return false;
  if (rows == 0) {
    C3D_CUDA(cudaMemsetAsync(dgamma, 0, cols * sizeof(float), s));
    C3D_CUDA(cudaMemsetAsync(dbeta, 0, cols * sizeof(float), s));
    if (dresid) C3D_CUDA(cudaMemsetAsync(dresid, 0, cols * sizeof(float), s));
    return true;
  }
  static int num_sms = 0;
  if (num_sms == 0) {
    int dev = 0;
    C3D_CUDA(cudaGetDevice(&dev));
    C3D_CUDA(cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, dev));
  }
  const int ns = dresid ? 3 : 2;
  const int grid = static_cast<int>(std::min<int64_t>(num_sms, (rows + kWarpsPerBlock - 1) / kWarpsPerBlock));
  float* partial = nullptr;
  C3D_CUDA(cudaMallocAsync(&partial, static_cast<size_t>(grid) * ns * cols * sizeof(float), s));
  const auto* d16 = static_cast<const __nv_bfloat16*>(dy);
  const auto* x16 = static_cast<const __nv_bfloat16*>(xhat);
  const auto* r16 = static_cast<const __nv_bfloat16*>(resid);
  auto* o16 = static_cast<__nv_bfloat16*>(dx);
  auto go = [&](auto V) {
    constexpr int VV = decltype(V)::value;
    if (dresid)
      ln_bwd_sums_kernel<VV, true><<<grid, 32 * kWarpsPerBlock, 0, s>>>(d16, x16, gamma, inv_std,
                                                                        rows, r16, o16, partial);
    else
      ln_bwd_sums_kernel<VV, false><<<grid, 32 * kWarpsPerBlock, 0, s>>>(d16, x16, gamma, inv_std,
                                                                         rows, nullptr, o16, partial);
  };
  if (vpl == 1) go(std::integral_constant<int, 1>{});
  else if (vpl == 2) go(std::integral_constant<int, 2>{});
  else go(std::integral_constant<int, 4>{});
  check_launch("ln_bwd_sums");
  const int64_t width = static_cast<int64_t>(ns) * cols;
  colsum_parts_kernel<<<static_cast<unsigned>((width + 31) / 32), 1024, 0, s>>>(
      partial, grid, width, cols, dgamma, dbeta, dresid);
  check_launch("colsum_parts");
  C3D_CUDA(cudaFreeAsync(partial, s));
  return true;
}

void k_ln_bwd_rows(const void* dy, int dt, const void* xhat, int xdt, const float* gamma,
                   int64_t rows, int64_t cols, float* rs, cudaStream_t s) {
  if (rows == 0) return;
  if (const int vpl = ln_vpl(cols); vpl && al16(dy) && al16(xhat)) {
    by_vpl(vpl, [&](auto V) {
      ln_bwd_rows_vec_kernel<decltype(V)::value><<<row_blocks(rows), 32 * kWarpsPerBlock, 0, s>>>(
          dy, dt, xhat, xdt, gamma, rows, rs);
    });
    check_launch("ln_bwd_rows_vec");
    return;
  }
  ln_bwd_rows_kernel<<<row_blocks(rows), 32 * kWarpsPerBlock, 0, s>>>(dy, dt, xhat, xdt, gamma,
                                                                      rows, cols, rs);
  check_launch("ln_bwd_rows");
}

void k_ln_bwd_dx(const void* dy, int dt, const void* xhat, int xdt, const float* gamma,
                 const float* inv_std, const float* rs, float inv_h, int64_t rows, int64_t cols,
                 const void* resid, int rdt, void* dx, int dxdt, cudaStream_t s) {
  if (rows * cols == 0) return;
  if (const int vpl = ln_vpl(cols);
      vpl && al16(dy) && al16(xhat) && al16(gamma) && al16(dx) && (!resid || al16(resid))) {
    by_vpl(vpl, [&](auto V) {
      ln_bwd_vec_kernel<decltype(V)::value><<<row_blocks(rows), 32 * kWarpsPerBlock, 0, s>>>(
          dy, dt, xhat, xdt, gamma, inv_std, rows, resid, rdt, dx, dxdt, rs, inv_h);
    });
    check_launch("ln_bwd_dx_vec");
    return;
  }
  ln_bwd_dx_kernel<<<grid_for(rows * cols), 256, 0, s>>>(dy, dt, xhat, xdt, gamma, inv_std, rs,
                                                         inv_h, rows, cols, resid, rdt, dx, dxdt);
  check_launch("ln_bwd_dx");
}

void k_copy_heads(const void* src, int64_t src_ld, int64_t src_hs, void* dst, int64_t dst_ld,
                  int64_t dst_hs, int64_t rows, int64_t heads, int64_t dh, int dt,
                  cudaStream_t s) {
  const int64_t n = rows * heads * dh;
  if (n == 0) return;
  copy_heads_kernel<<<grid_for(n), 256, 0, s>>>(src, src_ld, src_hs, dst, dst_ld, dst_hs, rows,
                                                heads, dh, dt);
  check_launch("copy_heads");
}

}  // namespace c3d
