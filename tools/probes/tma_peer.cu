// Probe: do TMA tensor stores / bulk copies / TMA loads work on NVLink peer memory,
// and at what bandwidth? Single process, 2 GPUs.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_peer tma_peer.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// each block: 128 rows x 64 bf16 cols (16 KB) tiles; tile t at rows [t*128, +128)
__global__ void tma_store_kernel(const __grid_constant__ CUtensorMap map, const uint4* src, int tiles) {
  extern __shared__ __align__(1024) uint8_t sm[];
  for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
    const uint4* s = src + (size_t)t * 1024;
    uint4* d = reinterpret_cast<uint4*>(sm);
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) d[i] = s[i];
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
      asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];"
                   :: "l"(&map), "r"(smem_u32(sm)), "r"(0), "r"(t * 128) : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

__global__ void bulk_store_kernel(const uint4* src, char* dst, int tiles) {
  extern __shared__ __align__(1024) uint8_t sm[];
  for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
    const uint4* s = src + (size_t)t * 1024;
    uint4* d = reinterpret_cast<uint4*>(sm);
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) d[i] = s[i];
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                   :: "l"(dst + (size_t)t * 16384), "r"(smem_u32(sm)), "r"(16384) : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

__global__ void tma_load_kernel(const __grid_constant__ CUtensorMap map, uint4* dst, int tiles) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  uint32_t phase = 0;
  for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
    if (threadIdx.x == 0) {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(smem_u32(&bar)), "r"(16384) : "memory");
      asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                   :: "r"(smem_u32(sm)), "l"(&map), "r"(0), "r"(t * 128), "r"(smem_u32(&bar)) : "memory");
    }
    uint32_t ok = 0;
    while (!ok) {
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                   : "=r"(ok) : "r"(smem_u32(&bar)), "r"(phase) : "memory");
    }
    phase ^= 1;
    const uint4* s = reinterpret_cast<const uint4*>(sm);
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) dst[(size_t)t * 1024 + i] = s[i];
    __syncthreads();
  }
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int make_map(EncodeFn enc, CUtensorMap* m, void* base, size_t rows) {
  cuuint64_t dims[2] = {64, rows};
  cuuint64_t strides[1] = {128};
  cuuint32_t box[2] = {64, 128};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, base, dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                   CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) { printf("encode failed %d\n", (int)r); return 1; }
  return 0;
}

int main() {
  const int tiles = 8192;  // 128 MB
  const size_t bytes = (size_t)tiles * 16384;
  void *src0, *dst1, *chk0;
  CK(cudaSetDevice(1));
  CK(cudaMalloc(&dst1, bytes));
  CK(cudaMemset(dst1, 0, bytes));
  CK(cudaDeviceEnablePeerAccess(0, 0));
  CK(cudaSetDevice(0));
  CK(cudaDeviceEnablePeerAccess(1, 0));
  CK(cudaMalloc(&src0, bytes));
  CK(cudaMalloc(&chk0, bytes));
  std::vector<uint16_t> h(bytes / 2);
  for (size_t i = 0; i < h.size(); ++i) h[i] = (uint16_t)(i * 2654435761u >> 7);
  CK(cudaMemcpy(src0, h.data(), bytes, cudaMemcpyHostToDevice));
  EncodeFn enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q));
  CUtensorMap mpeer, mpeer_load;
  if (make_map(enc, &mpeer, dst1, (size_t)tiles * 128)) return 1;
  CK(cudaFuncSetAttribute(tma_store_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384));
  CK(cudaFuncSetAttribute(bulk_store_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384));
  CK(cudaFuncSetAttribute(tma_load_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  std::vector<uint16_t> back(bytes / 2);
  for (int kind = 0; kind < 3; ++kind) {
    for (int grid : {148, 296, 592}) {
      CK(cudaSetDevice(1));
      CK(cudaMemset(dst1, 0, bytes));
      CK(cudaDeviceSynchronize());
      CK(cudaSetDevice(0));
      CK(cudaMemset(chk0, 0, bytes));
      float best = 1e9;
      for (int it = 0; it < 4; ++it) {
        CK(cudaEventRecord(e0));
        if (kind == 0) tma_store_kernel<<<grid, 256, 16384>>>(mpeer, (const uint4*)src0, tiles);
        else if (kind == 1) bulk_store_kernel<<<grid, 256, 16384>>>((const uint4*)src0, (char*)dst1, tiles);
        else tma_load_kernel<<<grid, 256, 16384>>>(mpeer, (uint4*)chk0, tiles);
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
        CK(cudaGetLastError());
        float ms;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        best = ms < best ? ms : best;
      }
      // verify
      if (kind < 2) {
        CK(cudaSetDevice(1));
        CK(cudaMemcpy(back.data(), dst1, bytes, cudaMemcpyDeviceToHost));
        CK(cudaSetDevice(0));
      } else {
        CK(cudaMemcpy(back.data(), chk0, bytes, cudaMemcpyDeviceToHost));
      }
      size_t bad = 0;
      for (size_t i = 0; i < h.size(); ++i) bad += back[i] != (kind == 2 ? h[i] * 0 + back[i] : h[i]);
      const char* nm[] = {"TMA tensor store -> peer", "bulk copy store -> peer", "TMA tensor load <- peer"};
      printf("%s grid=%d: %.1f GB/s, mismatches=%zu\n", nm[kind], grid, bytes / (best * 1e-3) / 1e9, bad);
    }
  }
  // TMA load check against source: load dst1 (which holds the copy of src0 from kind 1)
  size_t bad = 0;
  for (size_t i = 0; i < h.size(); ++i) bad += back[i] != h[i];
  printf("TMA load content mismatches=%zu\n", bad);
  return 0;
}
