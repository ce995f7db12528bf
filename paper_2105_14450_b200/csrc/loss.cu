// 3-D cross-entropy over a (hidden -> vocab) linear head: the loss row of SURVEY.md
// §8(a) (X1; not in the reference, whose only loss is <dY, Y>, cube3d/verify.hpp:
// 611-617). Logits are fp32 with rows split along x and the group's input axis and
// vocabulary columns split along its output axis; the row max and the
// (sum exp, target logit) pairs are all-reduced along the column axis, the mean over
// tokens along the two row axes.
#include <cuda_runtime.h>

#include <cmath>

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

// local row -> global token (activation_from_global, cube3d/activation.hpp:119-134)
__device__ __forceinline__ int64_t global_row(int64_t r, const LossMap& m) {
  const int64_t bi = r / m.sl, si = r - (r / m.sl) * m.sl;
  return (m.w * m.bl + bi) * m.seq + m.a * m.sl + si;
}

// st[r] = sum_c exp(l - m[r]); st[rows + r] = l[target - col0] if the target column is
// local, else 0.
__global__ void loss_stats_kernel(const float* logits, int64_t rows, int64_t cols,
                                  const float* mx, const int32_t* targets, LossMap map,
                                  float* st) {
  const int64_t r = blockIdx.x * static_cast<int64_t>(kWarps) + threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  if (r >= rows) return;
  const float* row = logits + r * cols;
  const float m = mx[r];
  float s = 0.f;
  for (int64_t c = lane; c < cols; c += 32) s += expf(row[c] - m);
  s = wsum(s);
  if (lane == 0) {
    const int64_t t = targets[global_row(r, map)] - map.col0;
    st[r] = s;
    st[rows + r] = (t >= 0 && t < cols) ? row[t] : 0.f;
  }
}

// One block: sum_r (log(se_r) + m_r - tl_r) * scale, fixed order (deterministic).
__global__ void loss_reduce_kernel(const float* mx, const float* st, int64_t rows, float scale,
                                   float* out) {
  __shared__ float part[256];
  float acc = 0.f;
  for (int64_t r = threadIdx.x; r < rows; r += blockDim.x)
    acc += logf(st[r]) + mx[r] - st[rows + r];
  part[threadIdx.x] = acc;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if (static_cast<int>(threadIdx.x) < w) part[threadIdx.x] += part[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = part[0] * scale;
}

// dlogits = (softmax - onehot(target)) * scale, in the gradient dtype.
__global__ void loss_grad_kernel(const float* logits, int64_t rows, int64_t cols, const float* mx,
                                 const float* st, const int32_t* targets, LossMap map,
                                 float scale, void* out, int dt) {
  const int64_t n = rows * cols;
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < n;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = t / cols, c = t - (t / cols) * cols;
    float g = expf(logits[t] - mx[r]) / st[r];
    if (targets[global_row(r, map)] - map.col0 == c) g -= 1.f;
    st_any(out, dt, t, g * scale);
  }
}

}  // namespace

void k_loss_stats(const float* logits, int64_t rows, int64_t cols, const float* mx,
                  const int32_t* targets, const LossMap& map, float* st, cudaStream_t s) {
  if (rows == 0) return;
  loss_stats_kernel<<<static_cast<unsigned>((rows + kWarps - 1) / kWarps), 32 * kWarps, 0, s>>>(
      logits, rows, cols, mx, targets, map, st);
  check_launch("loss_stats");
}

void k_loss_reduce(const float* mx, const float* st, int64_t rows, float scale, float* out,
                   cudaStream_t s) {
  loss_reduce_kernel<<<1, 256, 0, s>>>(mx, st, rows, scale, out);
  check_launch("loss_reduce");
}

void k_loss_grad(const float* logits, int64_t rows, int64_t cols, const float* mx, const float* st,
                 const int32_t* targets, const LossMap& map, float scale, void* out, int dt,
                 cudaStream_t s) {
  const int64_t n = rows * cols;
  if (n == 0) return;
  const int blocks = static_cast<int>(std::min<int64_t>((n + 255) / 256, 148 * 16));
  loss_grad_kernel<<<blocks, 256, 0, s>>>(logits, rows, cols, mx, st, targets, map, scale, out, dt);
  check_launch("loss_grad");
}

}  // namespace c3d
