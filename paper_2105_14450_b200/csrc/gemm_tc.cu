// sm_100a tcgen05 GEMM: bf16 operands staged by TMA into 128B-swizzled shared
// memory, fp32 accumulators in TMEM, fused epilogue from TMEM to global.
//
// This is the B200 replacement of the reference's local product
// `multiply_accumulate` (cube3d/matrix.hpp:68-92): the NN / NT / TN forms map to
// K-major or MN-major UMMA operand descriptors instead of strided CPU loops.
//
// Structure (one CTA per SM, persistent over output tiles):
//   warp 0      TMA producer (one elected lane)           smem ring: full/empty mbarriers
//   warp 1      TMEM allocator + UMMA issuer (one lane)   TMEM ring: 2 accumulators
//   warps 2..5  epilogue: tcgen05.ld -> registers -> epilogue math -> st.global
// Tile: 128 x BN (UMMA M=128, N=BN, K=16), K-block 64 per pipeline stage.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <stdexcept>
#include <string>

#include "gemm.hpp"
#include "gemm_tc.hpp"
#include "epi.cuh"
#include "ptx.cuh"

namespace c3d {

namespace {

constexpr int kBM = 128;
constexpr int kBK = 64;
constexpr int kThreads = 192;
constexpr int kSmemBudget = 227 * 1024;

struct TcOperand {
  int mn_major = 0;  // 1: the r (M/N) index is contiguous
  int split = 0;     // 0 none, 1 split on r, 2 split on c (K)
  int split_n = 0;
  int b_lo_n = 1;
};

struct TcArgs {
  int M, N, K, batch;
  int m_tiles, n_tiles, k_blocks;
  int num_tiles;
  int stages;
  int vec_ok;
  TcOperand a, b;
  Epilogue epi;
};

__device__ __forceinline__ void load_operand(const CUtensorMap* map, const TcOperand& op,
                                             void* dst, uint64_t* bar, int r0, int rows,
                                             int k0, int b) {
  const int c3 = b % op.b_lo_n, c4 = b / op.b_lo_n;
  if (!op.mn_major) {
    const int c0 = op.split == 2 ? k0 % op.split_n : k0;
    const int c1 = op.split == 1 ? r0 % op.split_n : r0;
    const int c2 = op.split == 1 ? r0 / op.split_n : (op.split == 2 ? k0 / op.split_n : 0);
    ptx::tma_load_5d(dst, map, bar, c0, c1, c2, c3, c4);
  } else {
    // [64 K rows][64 MN] chunks, 8 KB each
    for (int j = 0; j < rows / 64; ++j) {
      const int r = r0 + 64 * j;
      const int c0 = op.split == 1 ? r % op.split_n : r;
      const int c1 = op.split == 2 ? k0 % op.split_n : k0;
      const int c2 = op.split == 1 ? r / op.split_n : (op.split == 2 ? k0 / op.split_n : 0);
      ptx::tma_load_5d(static_cast<char*>(dst) + j * 8192, map, bar, c0, c1, c2, c3, c4);
    }
  }
}

// Applies the epilogue to one row segment of 32 columns held in v[].
__device__ __forceinline__ void epilogue_row32(const TcArgs& args, int b, int m, int n0,
                                               float (&v)[32]) {
  const Epilogue& e = args.epi;
  const long long row_off = view_offset(e.out, b, m, n0) - n0;
  const int nvalid = min(32, args.N - n0);
#pragma unroll
  for (int j = 0; j < 32; ++j) {
    float x = v[j] * e.alpha;
    if (e.bias != nullptr && j < nvalid) x += __ldg(e.bias + n0 + j);
    v[j] = x;
  }
  if (e.pre_act != nullptr) {
    if (e.pre_dtype == kF32) {
      float* p = static_cast<float*>(e.pre_act) + row_off + n0;
      if (args.vec_ok && nvalid == 32) {
#pragma unroll
        for (int j = 0; j < 32; j += 4)
          *reinterpret_cast<float4*>(p + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
      } else {
        for (int j = 0; j < nvalid; ++j) p[j] = v[j];
      }
    } else {
      __nv_bfloat16* p = static_cast<__nv_bfloat16*>(e.pre_act) + row_off + n0;
      if (args.vec_ok && nvalid == 32) {
#pragma unroll
        for (int j = 0; j < 32; j += 8) {
          uint4 pk;
          __nv_bfloat162 h0 = __floats2bfloat162_rn(v[j], v[j + 1]);
          __nv_bfloat162 h1 = __floats2bfloat162_rn(v[j + 2], v[j + 3]);
          __nv_bfloat162 h2 = __floats2bfloat162_rn(v[j + 4], v[j + 5]);
          __nv_bfloat162 h3 = __floats2bfloat162_rn(v[j + 6], v[j + 7]);
          pk.x = *reinterpret_cast<uint32_t*>(&h0);
          pk.y = *reinterpret_cast<uint32_t*>(&h1);
          pk.z = *reinterpret_cast<uint32_t*>(&h2);
          pk.w = *reinterpret_cast<uint32_t*>(&h3);
          *reinterpret_cast<uint4*>(p + j) = pk;
        }
      } else {
        for (int j = 0; j < nvalid; ++j) p[j] = __float2bfloat16_rn(v[j]);
      }
    }
  }
  if (e.act == kActGelu) {
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] = gelu_f(v[j]);
  } else if (e.act == kActGeluGrad) {
    for (int j = 0; j < nvalid; ++j) v[j] *= gelu_grad_f(ld_any(e.aux, e.aux_dtype, row_off + n0 + j));
  }
  if (e.resid != nullptr) {
    for (int j = 0; j < nvalid; ++j) v[j] += ld_any(e.resid, e.resid_dtype, row_off + n0 + j);
  }
  if (e.accumulate) {
    for (int j = 0; j < nvalid; ++j) v[j] += ld_any(e.out.base, e.out.dtype, row_off + n0 + j);
  }
  if (e.out.dtype == kF32) {
    float* p = static_cast<float*>(e.out.base) + row_off + n0;
    if (args.vec_ok && nvalid == 32) {
#pragma unroll
      for (int j = 0; j < 32; j += 4)
        *reinterpret_cast<float4*>(p + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
    } else {
      for (int j = 0; j < nvalid; ++j) p[j] = v[j];
    }
  } else {
    __nv_bfloat16* p = static_cast<__nv_bfloat16*>(e.out.base) + row_off + n0;
    if (args.vec_ok && nvalid == 32) {
#pragma unroll
      for (int j = 0; j < 32; j += 8) {
        uint4 pk;
        __nv_bfloat162 h0 = __floats2bfloat162_rn(v[j], v[j + 1]);
        __nv_bfloat162 h1 = __floats2bfloat162_rn(v[j + 2], v[j + 3]);
        __nv_bfloat162 h2 = __floats2bfloat162_rn(v[j + 4], v[j + 5]);
        __nv_bfloat162 h3 = __floats2bfloat162_rn(v[j + 6], v[j + 7]);
        pk.x = *reinterpret_cast<uint32_t*>(&h0);
        pk.y = *reinterpret_cast<uint32_t*>(&h1);
        pk.z = *reinterpret_cast<uint32_t*>(&h2);
        pk.w = *reinterpret_cast<uint32_t*>(&h3);
        *reinterpret_cast<uint4*>(p + j) = pk;
      }
    } else {
      for (int j = 0; j < nvalid; ++j) p[j] = __float2bfloat16_rn(v[j]);
    }
  }
}

template <int BN, bool A_MN, bool B_MN>
__global__ void __launch_bounds__(kThreads, 1)
    tc_gemm_kernel(const __grid_constant__ CUtensorMap tmA,
                   const __grid_constant__ CUtensorMap tmB, const TcArgs args) {
  constexpr int kABytes = kBM * kBK * 2;  // 16 KB
  constexpr int kBBytes = BN * kBK * 2;
  constexpr int kStageBytes = kABytes + kBBytes;
  constexpr uint32_t kTmemCols = 2 * BN < 32 ? 32 : 2 * BN;
  constexpr uint32_t kIdesc = ptx::idesc_bf16_f32(kBM, BN, A_MN, B_MN);

  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1024-B alignment for the 128B swizzle atoms
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  const int S = args.stages;
  uint8_t* smem_a = smem;
  uint8_t* smem_b = smem + S * kABytes;
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + S * kStageBytes);
  uint64_t* empty_bar = full_bar + S;
  uint64_t* tfull_bar = empty_bar + S;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + 2);

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;

  if (warp == 0 && lane == 0) {
    ptx::prefetch_tmap(&tmA);
    ptx::prefetch_tmap(&tmB);
    for (int s = 0; s < S; ++s) {
      ptx::mbar_init(&full_bar[s], 1);
      ptx::mbar_init(&empty_bar[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      ptx::mbar_init(&tfull_bar[s], 1);
      ptx::mbar_init(&tempty_bar[s], 4);
    }
    ptx::fence_barrier_init();
  }
  if (warp == 1) ptx::tmem_alloc<kTmemCols>(tmem_slot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  const int tiles_per_batch = args.m_tiles * args.n_tiles;

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer
      int it = 0;
      for (int t = blockIdx.x; t < args.num_tiles; t += gridDim.x) {
        const int b = t / tiles_per_batch;
        const int rem = t % tiles_per_batch;
        const int m0 = (rem / args.n_tiles) * kBM;
        const int n0 = (rem % args.n_tiles) * BN;
        for (int kb = 0; kb < args.k_blocks; ++kb, ++it) {
          const int s = it % S;
          const uint32_t ph = (it / S) & 1;
          ptx::mbar_wait(&empty_bar[s], ph ^ 1);
          ptx::mbar_arrive_expect_tx(&full_bar[s], kStageBytes);
          load_operand(&tmA, args.a, smem_a + s * kABytes, &full_bar[s], m0, kBM, kb * kBK, b);
          load_operand(&tmB, args.b, smem_b + s * kBBytes, &full_bar[s], n0, BN, kb * kBK, b);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---------------- UMMA issuer
      int it = 0, tc = 0;
      for (int t = blockIdx.x; t < args.num_tiles; t += gridDim.x, ++tc) {
        const int acc = tc & 1;
        const uint32_t aph = (tc >> 1) & 1;
        ptx::mbar_wait(&tempty_bar[acc], aph ^ 1);
        ptx::tc_fence_after();
        const uint32_t tmem_d = tmem_base + acc * BN;
        for (int kb = 0; kb < args.k_blocks; ++kb, ++it) {
          const int s = it % S;
          const uint32_t ph = (it / S) & 1;
          ptx::mbar_wait(&full_bar[s], ph);
          ptx::tc_fence_after();
          const uint32_t a_addr = ptx::smem_u32(smem_a + s * kABytes);
          const uint32_t b_addr = ptx::smem_u32(smem_b + s * kBBytes);
#pragma unroll
          for (int k = 0; k < kBK / 16; ++k) {
            const uint64_t ad = A_MN ? ptx::smem_desc_sw128(a_addr + k * 2048, 8192, 1024)
                                     : ptx::smem_desc_sw128(a_addr + k * 32, 16, 1024);
            const uint64_t bd = B_MN ? ptx::smem_desc_sw128(b_addr + k * 2048, 8192, 1024)
                                     : ptx::smem_desc_sw128(b_addr + k * 32, 16, 1024);
            ptx::umma_bf16(tmem_d, ad, bd, kIdesc, (kb > 0 || k > 0) ? 1u : 0u);
          }
          ptx::umma_commit(&empty_bar[s]);
        }
        ptx::umma_commit(&tfull_bar[acc]);
      }
    }
  } else {
    // ---------------- epilogue warps 2..5 (TMEM lane quarter = warp % 4)
    const int quarter = warp & 3;
    int tc = 0;
    for (int t = blockIdx.x; t < args.num_tiles; t += gridDim.x, ++tc) {
      const int acc = tc & 1;
      const uint32_t aph = (tc >> 1) & 1;
      const int b = t / tiles_per_batch;
      const int rem = t % tiles_per_batch;
      const int m0 = (rem / args.n_tiles) * kBM;
      const int n0 = (rem % args.n_tiles) * BN;
      ptx::mbar_wait(&tfull_bar[acc], aph);
      ptx::tc_fence_after();
      const int m = m0 + quarter * 32 + lane;
      const uint32_t row_taddr = tmem_base + acc * BN + (static_cast<uint32_t>(quarter * 32) << 16);
#pragma unroll 1
      for (int c = 0; c < BN / 32; ++c) {
        float v[32];
        ptx::tmem_ld32(row_taddr + c * 32, v);
        const int nc = n0 + c * 32;
        if (m < args.M && nc < args.N) epilogue_row32(args, b, m, nc, v);
      }
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&tempty_bar[acc]);
    }
  }

  __syncthreads();
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<kTmemCols>(tmem_base);
  }
}

// ------------------------------------------------------------------ host side

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  if (!fn) throw std::runtime_error("cuTensorMapEncodeTiled unavailable");
  return fn;
}

// Builds the 5-D tensor map of one operand view (rows = logical r extent, cols = K).
CUtensorMap make_operand_map(const View& v, long long rows, long long cols, int batch,
                             int box_rows, TcOperand* op) {
  op->mn_major = (v.sr == 1 && v.sc != 1) ? 1 : 0;
  op->split = v.rsplit ? 1 : (v.csplit ? 2 : 0);
  op->split_n = static_cast<int>(v.rsplit ? v.rsplit : v.csplit);
  op->b_lo_n = v.b_lo_n;
  const long long rlo = v.rsplit ? v.rsplit : rows;
  const long long clo = v.csplit ? v.csplit : cols;
  const long long nhi = v.rsplit ? (rows + v.rsplit - 1) / v.rsplit
                                 : (v.csplit ? (cols + v.csplit - 1) / v.csplit : 1);
  const long long bhi = (batch + v.b_lo_n - 1) / v.b_lo_n;
  cuuint64_t dims[5];
  cuuint64_t strides[4];  // bytes, dims 1..4
  cuuint32_t box[5] = {64, 64, 1, 1, 1};
  cuuint32_t estr[5] = {1, 1, 1, 1, 1};
  auto safe = [](long long s, long long fallback) {
    long long b = (s > 0 ? s : fallback) * 2;
    return static_cast<cuuint64_t>(b);
  };
  if (!op->mn_major) {
    dims[0] = clo;
    dims[1] = rlo;
    strides[0] = safe(v.sr, clo);
    box[1] = box_rows;
  } else {
    dims[0] = rlo;
    dims[1] = clo;
    strides[0] = safe(v.sc, rlo);
    box[1] = 64;
  }
  dims[2] = nhi;
  dims[3] = v.b_lo_n;
  dims[4] = bhi;
  const long long base_extent = (op->mn_major ? v.sc : v.sr) * (op->mn_major ? clo : rlo);
  strides[1] = safe(v.s_hi, base_extent > 0 ? base_extent : 8);
  strides[2] = safe(v.sb_lo, base_extent > 0 ? base_extent : 8);
  strides[3] = safe(v.sb_hi, base_extent > 0 ? base_extent : 8);
  CUtensorMap map;
  std::memset(&map, 0, sizeof(map));
  CUresult r = encode_fn()(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5, v.base, dims, strides, box,
                           estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    char buf[512];
    std::snprintf(buf, sizeof(buf),
                  "cuTensorMapEncodeTiled failed (%d): dims %llu %llu %llu %llu %llu strides "
                  "%llu %llu %llu %llu box %u %u",
                  static_cast<int>(r), (unsigned long long)dims[0], (unsigned long long)dims[1],
                  (unsigned long long)dims[2], (unsigned long long)dims[3],
                  (unsigned long long)dims[4], (unsigned long long)strides[0],
                  (unsigned long long)strides[1], (unsigned long long)strides[2],
                  (unsigned long long)strides[3], box[0], box[1]);
    throw std::runtime_error(buf);
  }
  return map;
}

template <int BN, bool A_MN, bool B_MN>
void launch_tc(const CUtensorMap& ma, const CUtensorMap& mb, TcArgs& args, int num_sms,
               cudaStream_t stream) {
  constexpr int kStageBytes = (kBM + BN) * kBK * 2;
  int stages = (kSmemBudget - 1024 - 256) / kStageBytes;
  stages = std::min(stages, 8);
  args.stages = stages;
  const int smem = 1024 + stages * kStageBytes + (2 * stages + 4) * 8 + 16;
  auto kern = tc_gemm_kernel<BN, A_MN, B_MN>;
  static bool attr_set = false;  // per instantiation
  if (!attr_set) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBudget);
    attr_set = true;
  }
  const int grid = std::min(args.num_tiles, num_sms);
  kern<<<grid, kThreads, smem, stream>>>(ma, mb, args);
}

template <int BN>
void launch_bn(const CUtensorMap& ma, const CUtensorMap& mb, TcArgs& args, int num_sms,
               cudaStream_t stream) {
  const bool am = args.a.mn_major, bm = args.b.mn_major;
  if (!am && !bm) launch_tc<BN, false, false>(ma, mb, args, num_sms, stream);
  else if (!am && bm) launch_tc<BN, false, true>(ma, mb, args, num_sms, stream);
  else if (am && !bm) launch_tc<BN, true, false>(ma, mb, args, num_sms, stream);
  else launch_tc<BN, true, true>(ma, mb, args, num_sms, stream);
}

bool operand_ok(const View& v, long long rows, long long cols, int tile_rows) {
  if (v.dtype != kBF16) return false;
  if (!(v.sc == 1 || v.sr == 1)) return false;
  if (v.rsplit && v.csplit) return false;
  if (reinterpret_cast<uintptr_t>(v.base) % 16) return false;
  const bool mn = (v.sr == 1 && v.sc != 1);
  const long long outer_stride = mn ? v.sc : v.sr;
  if (rows > 1 || cols > 1) {
    if (outer_stride % 8) return false;
  }
  for (long long s : {v.s_hi, v.sb_lo, v.sb_hi})
    if (s % 8) return false;
  if (v.rsplit) {
    if (v.rsplit % (mn ? 64 : tile_rows)) return false;
  }
  if (v.csplit && v.csplit % 64) return false;
  // MN-major tiles are loaded in 64-wide chunks: the r extent must cover whole chunks of
  // the tile or be padded by TMA out-of-bounds fill, which is fine.
  return true;
}

}  // namespace

int tc_pick_bn(long long M, long long N, int batch, int num_sms) {
  if (N <= 64) return 64;
  if (N <= 128) return 128;
  const long long mt = (M + kBM - 1) / kBM;
  const long long tiles256 = mt * ((N + 255) / 256) * batch;
  if (N % 256 == 0 && tiles256 >= num_sms) return 256;
  return 128;
}

bool tc_gemm_supported(const GemmProblem& p, int bn) {
  if (p.M <= 0 || p.N <= 0 || p.K <= 0) return false;
  if (p.K % 8) return false;
  if (!operand_ok(p.a, p.M, p.K, kBM)) return false;
  if (!operand_ok(p.b, p.N, p.K, bn)) return false;
  if (p.epi.out.sc != 1 || (p.epi.out.csplit && p.epi.out.csplit % 32)) return false;
  return true;
}

void tc_gemm_launch(const GemmProblem& p, int bn, int num_sms, cudaStream_t stream) {
  TcArgs args;
  std::memset(&args, 0, sizeof(args));
  args.M = static_cast<int>(p.M);
  args.N = static_cast<int>(p.N);
  args.K = static_cast<int>(p.K);
  args.batch = p.batch;
  args.m_tiles = static_cast<int>((p.M + kBM - 1) / kBM);
  args.n_tiles = static_cast<int>((p.N + bn - 1) / bn);
  args.k_blocks = static_cast<int>((p.K + kBK - 1) / kBK);
  args.num_tiles = args.m_tiles * args.n_tiles * p.batch;
  args.epi = p.epi;
  // vector stores need 16-B aligned rows
  const int esz = p.epi.out.dtype == kF32 ? 4 : 2;
  bool vec = reinterpret_cast<uintptr_t>(p.epi.out.base) % 16 == 0 &&
             (p.epi.out.sr * esz) % 16 == 0 && (p.epi.out.s_hi * esz) % 16 == 0 &&
             (p.epi.out.sb_lo * esz) % 16 == 0 && (p.epi.out.sb_hi * esz) % 16 == 0;
  if (p.epi.pre_act) {
    const int pz = p.epi.pre_dtype == kF32 ? 4 : 2;
    vec = vec && reinterpret_cast<uintptr_t>(p.epi.pre_act) % 16 == 0 &&
          (p.epi.out.sr * pz) % 16 == 0;
  }
  args.vec_ok = vec ? 1 : 0;
  CUtensorMap ma = make_operand_map(p.a, p.M, p.K, p.batch, kBM, &args.a);
  CUtensorMap mb = make_operand_map(p.b, p.N, p.K, p.batch, bn, &args.b);
  switch (bn) {
    case 64: launch_bn<64>(ma, mb, args, num_sms, stream); break;
    case 128: launch_bn<128>(ma, mb, args, num_sms, stream); break;
    case 256: launch_bn<256>(ma, mb, args, num_sms, stream); break;
    default: throw std::runtime_error("tc_gemm: unsupported BN");
  }
}

}  // namespace c3d
