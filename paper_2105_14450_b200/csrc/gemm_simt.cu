// SIMT fp32 GEMM over arbitrary views: the "fp32-exact" mode used for oracle
// comparison (north star: fp32 within 1e-5) and for shapes TMA cannot address
// (tiny or misaligned shards). Every output accumulates its products in
// ascending k, like `multiply_accumulate` (cube3d/matrix.hpp:79-90); products
// are fused (FMA), so results differ from the -ffp-contract=off reference only
// in the last bit of each step.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "gemm.hpp"
#include "epi.cuh"
#include "gemm_tc.hpp"

namespace c3d {

namespace {

constexpr int kTM = 64, kTN = 64, kTK = 16;

__global__ void __launch_bounds__(256) simt_gemm_kernel(GemmProblem p) {
  __shared__ float As[kTK][kTM + 4];
  __shared__ float Bs[kTK][kTN + 4];
  const int b = blockIdx.z;
  const long long m0 = static_cast<long long>(blockIdx.y) * kTM;
  const long long n0 = static_cast<long long>(blockIdx.x) * kTN;
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  float acc[4][4] = {};
  for (long long k0 = 0; k0 < p.K; k0 += kTK) {
    for (int e = threadIdx.x; e < kTM * kTK; e += 256) {
      const int kk = e % kTK, rr = e / kTK;
      const long long m = m0 + rr, k = k0 + kk;
      As[kk][rr] = (m < p.M && k < p.K) ? ld_any(p.a.base, p.a.dtype, view_offset(p.a, b, m, k)) : 0.f;
      const long long n = n0 + rr;
      Bs[kk][rr] = (n < p.N && k < p.K) ? ld_any(p.b.base, p.b.dtype, view_offset(p.b, b, n, k)) : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < kTK; ++kk) {
      float av[4], bv[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) av[i] = As[kk][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) bv[j] = Bs[kk][tx * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
    }
    __syncthreads();
  }
  const Epilogue& e = p.epi;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const long long m = m0 + ty * 4 + i;
    if (m >= p.M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const long long n = n0 + tx * 4 + j;
      if (n >= p.N) continue;
      epi_scalar(e, view_offset(e.out, b, m, n), n, acc[i][j]);
    }
  }
}

}  // namespace

void simt_gemm_launch(const GemmProblem& p, cudaStream_t stream) {
  dim3 grid(static_cast<unsigned>((p.N + kTN - 1) / kTN), static_cast<unsigned>((p.M + kTM - 1) / kTM),
            static_cast<unsigned>(p.batch));
  simt_gemm_kernel<<<grid, 256, 0, stream>>>(p);
}

}  // namespace c3d
