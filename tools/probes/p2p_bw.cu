// NVLink peer bandwidth probe (single process, 2 GPUs): SM push (remote stores),
// SM pull (remote loads) and copy-engine peer copies, one-way and both ways at once.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o p2p_bw p2p_bw.cu
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

template <int U>
__global__ void copy_kernel(const uint4* __restrict__ src, uint4* __restrict__ dst, size_t n) {
  size_t i0 = (size_t)blockIdx.x * blockDim.x * U + threadIdx.x;
  const size_t stride = (size_t)gridDim.x * blockDim.x * U;
  for (; i0 < n; i0 += stride) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) if (i0 + u * blockDim.x < n) v[u] = src[i0 + u * blockDim.x];
#pragma unroll
    for (int u = 0; u < U; ++u) if (i0 + u * blockDim.x < n) dst[i0 + u * blockDim.x] = v[u];
  }
}

int main() {
  int nd = 0;
  CK(cudaGetDeviceCount(&nd));
  if (nd < 2) { printf("need 2 GPUs\n"); return 1; }
  const size_t bytes = 256ull << 20;
  void *a[2], *b[2];
  cudaStream_t s[2];
  cudaEvent_t e0[2], e1[2];
  for (int d = 0; d < 2; ++d) {
    CK(cudaSetDevice(d));
    CK(cudaDeviceEnablePeerAccess(1 - d, 0));
    CK(cudaMalloc(&a[d], bytes));
    CK(cudaMalloc(&b[d], bytes));
    CK(cudaMemset(a[d], 1, bytes));
    CK(cudaStreamCreate(&s[d]));
    CK(cudaEventCreate(&e0[d]));
    CK(cudaEventCreate(&e1[d]));
  }
  int ac = 0;
  cudaDeviceCanAccessPeer(&ac, 0, 1);
  printf("canAccessPeer %d\n", ac);
  const size_t n = bytes / 16;
  // mode 0: push (dev d runs, src local a[d], dst remote b[1-d]); 1: pull (src remote a[1-d], dst local b[d]); 2: CE
  const char* names[] = {"SM push", "SM pull", "CE copy"};
  for (int mode = 0; mode < 3; ++mode) {
    for (int both = 0; both < 2; ++both) {
      for (int grid : {32, 64, 148, 296, 592}) {
        if (mode == 2 && grid != 148) continue;
        for (int threads : {256, 512, 1024}) {
          if (mode == 2 && threads != 512) continue;
          float best = 1e9;
          for (int it = 0; it < 5; ++it) {
            for (int d = 0; d < (both ? 2 : 1); ++d) {
              CK(cudaSetDevice(d));
              CK(cudaEventRecord(e0[d], s[d]));
              const uint4* src = (const uint4*)(mode == 1 ? a[1 - d] : a[d]);
              uint4* dst = (uint4*)(mode == 1 ? b[d] : b[1 - d]);
              if (mode == 2) CK(cudaMemcpyPeerAsync(dst, mode == 1 ? d : 1 - d, src, d, bytes, s[d]));
              else copy_kernel<4><<<grid, threads, 0, s[d]>>>(src, dst, n);
              CK(cudaEventRecord(e1[d], s[d]));
            }
            float worst = 0;
            for (int d = 0; d < (both ? 2 : 1); ++d) {
              CK(cudaSetDevice(d));
              CK(cudaEventSynchronize(e1[d]));
              float ms;
              CK(cudaEventElapsedTime(&ms, e0[d], e1[d]));
              worst = ms > worst ? ms : worst;
            }
            best = worst < best ? worst : best;
          }
          printf("%s %s grid=%d threads=%d: %.1f GB/s per direction\n", names[mode],
                 both ? "bidir" : "oneway", grid, threads, bytes / (best * 1e-3) / 1e9);
        }
      }
    }
  }
  return 0;
}
