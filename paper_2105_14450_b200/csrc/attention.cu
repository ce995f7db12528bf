// Fused attention core for one rank whose slices hold the whole key range (the seq
// axis of the cube has extent 1): per (slice, 128-query tile) CTA
//
//   S = Q K^T                 tcgen05, Q/K staged by TMA, S (128 x keys fp32) in TMEM
//   P = softmax(scale * S)    epilogue warps, one query row per thread, fp32
//   P -> shared (bf16, UMMA K-major 128B-swizzled) -> global probs (TMA store, saved
//        for the backward exactly as the unfused path saves them)
//   O = P V                   tcgen05 with P from shared memory, V staged MN-major
//   O -> ctx (bf16)
//
// It replaces, for that case, the scores GEMM with its fp32 score buffer, the softmax
// kernel and the P V GEMM of attention_fwd (cube3d/attention.hpp:95-127): the scores
// never leave the SM. Limits: head dim 64, keys a multiple of 256 up to 512 (TMEM
// holds one full score row block: 512 fp32 columns), queries a multiple of 128.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstring>
#include <type_traits>

#include "common.hpp"
#include "gemm.hpp"
#include "gemm_tc.hpp"
#include "kernels.hpp"
#include "ptx.cuh"

namespace c3d {

namespace {

constexpr int kQ = 128;   // queries per CTA (UMMA M)
constexpr int kDh = 64;   // head dim (one 128-B K block)
constexpr int kSoftWarps = 16;     // 4 TMEM lane quarters x 4 column groups
constexpr int kThreadsAttn = 64 + 32 * kSoftWarps;  // warp 0 TMA, warp 1 MMA, softmax warps

// Modes: 0 whole softmax on this rank; with the key range split along the seq axis
// (distributed softmax, cube3d/attention.hpp:106-126): 1 local row max of S -> stat_max,
// 2 sum exp(scale (S - M)) with the all-reduced max M -> stat_sum, 3 P = exp(.) / L
// with both all-reduced, stored, and the partial context P V.
struct AttnArgs {
  int S, keys, H;
  float scale_log2;  // scale * log2(e)
  int q_split;       // rows per gathered query block (0: not split)
  __nv_bfloat16* ctx;
  long long ctx_sr, ctx_sb_lo, ctx_sb_hi;  // element strides of the context view
  long long ctx_split, ctx_s_hi;           // split rows of the (partial) context view
  float* stat_max;   // [slice][S]
  float* stat_sum;
};

__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}

template <int KEYS, int MODE>
__global__ void __launch_bounds__(kThreadsAttn, 1)
    attn_fwd_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                    const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmP,
                    const AttnArgs args) {
  constexpr int kQBytes = kQ * kDh * 2;              // 16 KB
  constexpr int kKBytes = KEYS * kDh * 2;            // keys x 128 B
  constexpr int kPBytes = KEYS / 64 * kQ * 128;      // 64-key chunks of [128 rows][128 B]
  constexpr int kVOff = (kQBytes + kKBytes > kPBytes ? kQBytes + kKBytes : kPBytes);
  constexpr int kVBytes = KEYS * kDh * 2;
  constexpr uint32_t kIdescS = ptx::idesc_bf16_f32(kQ, 256, false, false);
  constexpr uint32_t kIdescO = ptx::idesc_bf16_f32(kQ, kDh, false, true);

  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  uint8_t* sQ = smem;
  uint8_t* sK = smem + kQBytes;
  uint8_t* sP = smem;  // overwrites Q and K once S is in TMEM
  uint8_t* sV = smem + kVOff;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kVOff + kVBytes);
  uint64_t* bar_qk = bars;
  uint64_t* bar_v = bars + 1;
  uint64_t* bar_s = bars + 2;
  uint64_t* bar_p = bars + 3;
  uint64_t* bar_o = bars + 4;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 5);
  float* red = reinterpret_cast<float*>(bars + 8);  // [2][4 groups][128 rows] row partials

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int q0 = blockIdx.x * kQ;
  const int b = blockIdx.y;
  const int c3 = b % args.H, c4 = b / args.H;

  if (warp == 0 && lane == 0) {
    ptx::mbar_init(bar_qk, 1);
    ptx::mbar_init(bar_v, 1);
    ptx::mbar_init(bar_s, 1);
    ptx::mbar_init(bar_p, 32 * kSoftWarps);
    ptx::mbar_init(bar_o, 1);
    ptx::fence_barrier_init();
  }
  if (warp == 1) ptx::tmem_alloc<512>(tmem_slot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      ptx::mbar_arrive_expect_tx(bar_qk, kQBytes + kKBytes);
      const int qr = args.q_split ? q0 % args.q_split : q0;
      const int qh = args.q_split ? q0 / args.q_split : 0;
      ptx::tma_load_5d(sQ, &tmQ, bar_qk, 0, qr, qh, c3, c4);
#pragma unroll
      for (int h = 0; h < KEYS / 256; ++h)
        ptx::tma_load_5d(sK + h * 256 * 128, &tmK, bar_qk, 0, h * 256, 0, c3, c4);
      if (MODE == 0 || MODE == 3) {
        ptx::mbar_arrive_expect_tx(bar_v, kVBytes);
#pragma unroll
        for (int kb = 0; kb < KEYS / 64; ++kb)
          ptx::tma_load_5d(sV + kb * 8192, &tmV, bar_v, 0, kb * 64, 0, c3, c4);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      ptx::mbar_wait(bar_qk, 0);
      ptx::tc_fence_after();
      const uint32_t qa = ptx::smem_u32(sQ), ka = ptx::smem_u32(sK);
#pragma unroll
      for (int h = 0; h < KEYS / 256; ++h)
#pragma unroll
        for (int k = 0; k < kDh / 16; ++k)
          ptx::umma_bf16(tmem + h * 256, ptx::smem_desc_sw128(qa + 32 * k, 16, 1024),
                         ptx::smem_desc_sw128(ka + h * 256 * 128 + 32 * k, 16, 1024), kIdescS,
                         k > 0 ? 1u : 0u);
      ptx::umma_commit(bar_s);
      if (MODE == 0 || MODE == 3) {  // modes 1, 2: statistics only, no O
      // O = P V once the softmax warps have written P and released the S columns
      ptx::mbar_wait(bar_p, 0);
      ptx::mbar_wait(bar_v, 0);
      ptx::tc_fence_after();
      const uint32_t pa = ptx::smem_u32(sP), va = ptx::smem_u32(sV);
#pragma unroll
      for (int kb = 0; kb < KEYS / 64; ++kb)
#pragma unroll
        for (int k = 0; k < 4; ++k)
          ptx::umma_bf16(tmem, ptx::smem_desc_sw128(pa + kb * 16384 + 32 * k, 16, 1024),
                         ptx::smem_desc_sw128(va + kb * 8192 + 2048 * k, 8192, 1024), kIdescO,
                         (kb > 0 || k > 0) ? 1u : 0u);
      ptx::umma_commit(bar_o);
      }
    }
  } else {
    // ---------------- softmax: warp w owns TMEM lanes 32*(w % 4) .. +32 and column group
    // (w - 2) / 4 (a quarter of the keys); row max / sum combine through shared memory
    constexpr int kGroupCols = KEYS / 4;
    const int quarter = warp & 3;
    const int group = (warp - 2) >> 2;
    const int row = quarter * 32 + lane;
    const uint32_t trow = tmem + (static_cast<uint32_t>(quarter * 32) << 16);
    const int c0 = group * kGroupCols;
    ptx::mbar_wait(bar_s, 0);
    ptx::tc_fence_after();
    const long long srow = static_cast<long long>(b) * args.S + q0 + row;  // [slice][S]
    float m = -INFINITY;
    if (MODE == 2 || MODE == 3) {
      m = __ldg(args.stat_max + srow);  // all-reduced along the seq axis
    } else {
#pragma unroll 1
      for (int c = c0; c < c0 + kGroupCols; c += 32) {
        float v[32];
        ptx::tmem_ld32(trow + c, v);
#pragma unroll
        for (int j = 0; j < 32; ++j) m = fmaxf(m, v[j]);
      }
      red[group * kQ + row] = m;
      asm volatile("bar.sync 1, %0;" ::"n"(32 * kSoftWarps) : "memory");
      m = fmaxf(fmaxf(red[row], red[kQ + row]), fmaxf(red[2 * kQ + row], red[3 * kQ + row]));
      if (MODE == 1) {
        if (group == 0) args.stat_max[srow] = m;
      }
    }
    const float ms = m * args.scale_log2;
    float sum = 0.f;
    if (MODE == 3) {
      sum = __ldg(args.stat_sum + srow);
    } else if (MODE != 1) {
#pragma unroll 1
      for (int c = c0; c < c0 + kGroupCols; c += 32) {
        float v[32];
        ptx::tmem_ld32(trow + c, v);
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          v[j] = exp2f(fmaf(v[j], args.scale_log2, -ms));
          sum += v[j];
        }
        // keep exp(s - m) in TMEM: the normalising pass only scales it
        if (MODE == 0) ptx::tmem_st32(trow + c, v);
      }
      red[4 * kQ + group * kQ + row] = sum;
      asm volatile("bar.sync 1, %0;" ::"n"(32 * kSoftWarps) : "memory");
      sum = (red[4 * kQ + row] + red[5 * kQ + row]) + (red[6 * kQ + row] + red[7 * kQ + row]);
      if (MODE == 2 && group == 0) args.stat_sum[srow] = sum;
    }
    if (MODE == 0 || MODE == 3) {
    const float inv = 1.f / sum;
#pragma unroll 1
    for (int c = c0; c < c0 + kGroupCols; c += 32) {
      float v[32];
      ptx::tmem_ld32(trow + c, v);
      if (MODE != 0) {  // mode 0 left exp(s - m) in TMEM
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = exp2f(fmaf(v[j], args.scale_log2, -ms));
      }
      uint8_t* chunk_row = sP + (c >> 6) * 16384 + row * 128;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        uint4 pk;
        pk.x = pack_bf16(v[8 * j + 0] * inv, v[8 * j + 1] * inv);
        pk.y = pack_bf16(v[8 * j + 2] * inv, v[8 * j + 3] * inv);
        pk.z = pack_bf16(v[8 * j + 4] * inv, v[8 * j + 5] * inv);
        pk.w = pack_bf16(v[8 * j + 6] * inv, v[8 * j + 7] * inv);
        const int chunk = ((c >> 5) & 1) * 4 + j;
        *reinterpret_cast<uint4*>(chunk_row + ((chunk ^ (row & 7)) << 4)) = pk;
      }
    }
    // P visible to the tensor core (async proxy); S columns free for O
    ptx::fence_async_smem();
    ptx::tc_fence_before();
    ptx::mbar_arrive(bar_p);
    // probabilities to global (saved for the backward): one TMA store per 64-key chunk
    asm volatile("bar.sync 1, %0;" ::"n"(32 * kSoftWarps) : "memory");
    if (warp == 2 && lane == 0) {
#pragma unroll
      for (int kb = 0; kb < KEYS / 64; ++kb)
        ptx::tma_store_5d(&tmP, sP + kb * 16384, kb * 64, q0, 0, c3, c4);
      ptx::bulk_commit();
    }
    // context row: O (fp32 in TMEM columns 0..63) -> bf16, 32 columns per group 0 / 1
    if (group < 2) {
      ptx::mbar_wait(bar_o, 0);
      ptx::tc_fence_after();
      float o[32];
      ptx::tmem_ld32(trow + group * 32, o);
      const long long q = q0 + row;
      const long long qoff = args.ctx_split ? (q % args.ctx_split) * args.ctx_sr +
                                                  (q / args.ctx_split) * args.ctx_s_hi
                                            : q * args.ctx_sr;
      __nv_bfloat16* dst = args.ctx + c3 * args.ctx_sb_lo + c4 * args.ctx_sb_hi + qoff + group * 32;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        uint4 pk;
        pk.x = pack_bf16(o[8 * j + 0], o[8 * j + 1]);
        pk.y = pack_bf16(o[8 * j + 2], o[8 * j + 3]);
        pk.z = pack_bf16(o[8 * j + 4], o[8 * j + 5]);
        pk.w = pack_bf16(o[8 * j + 6], o[8 * j + 7]);
        reinterpret_cast<uint4*>(dst)[j] = pk;
      }
    }
    if (warp == 2 && lane == 0) ptx::bulk_wait_all();
    }  // MODE 0 / 3
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<512>(tmem);
  }
}

template <int KEYS, int MODE>
void launch_attn(const CUtensorMap& q, const CUtensorMap& k, const CUtensorMap& v,
                 const CUtensorMap& p, const AttnArgs& a, int nslices, cudaStream_t s) {
  constexpr int kQBytes = kQ * kDh * 2, kKBytes = KEYS * kDh * 2;
  constexpr int kPBytes = KEYS / 64 * kQ * 128;
  constexpr int kVOff = (kQBytes + kKBytes > kPBytes ? kQBytes + kKBytes : kPBytes);
  constexpr int smem = 1024 + kVOff + KEYS * kDh * 2 + 64 + 8 * kQ * 4;
  auto kern = attn_fwd_kernel<KEYS, MODE>;
  static bool attr = false;
  if (!attr) {
    C3D_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    attr = true;
  }
  kern<<<dim3(a.S / kQ, nslices), kThreadsAttn, smem, s>>>(q, k, v, p, a);
}


// ---------------------------------------------------------------- backward (dS, dQ)
// Per (slice, 128-query tile): dP = dO V^T in TMEM (keys fp32 columns); the saved P
// tile arrives by TMA into shared memory (UMMA K-major layout); 16 warps form
// dS = P * (dP - D) * scale in place (D = sum_j P dP = rowsum(dO * O), precomputed),
// dS goes to HBM (TMA store, for dK = dS^T Q) and stays in shared memory as the A
// operand of dQ = dS K (K staged MN-major into the buffer V used). Replaces the dS
// GEMM (with its fused softmax-backward epilogue) and the dQ GEMM of attention_bwd.
struct AttnBwdArgs {
  int S, keys, H;
  float scale;
  int o_split;          // rows per gathered dO block (0: not split)
  const float* rowdot;  // D per (slice, query): [slice][S], or [S / rd_split][slices][rd_split]
  long long rd_split, rd_slices;
  __nv_bfloat16* dq;    // dQ, or its partial [p][rows][hd] when the seq axis is split
  long long dq_sr, dq_sb_lo, dq_sb_hi, dq_split, dq_s_hi;
};

template <int KEYS>
__global__ void __launch_bounds__(kThreadsAttn, 1)
    attn_bwd_kernel(const __grid_constant__ CUtensorMap tmDO, const __grid_constant__ CUtensorMap tmV,
                    const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmP,
                    const __grid_constant__ CUtensorMap tmDS, const AttnBwdArgs args) {
  constexpr int kOBytes = kQ * kDh * 2;          // dO tile, 16 KB
  constexpr int kVBytes = KEYS * kDh * 2;        // V (then K), keys x 128 B
  constexpr int kPBytes = KEYS / 64 * kQ * 128;  // P / dS chunks
  constexpr uint32_t kIdescP = ptx::idesc_bf16_f32(kQ, 256, false, false);
  constexpr uint32_t kIdescQ = ptx::idesc_bf16_f32(kQ, kDh, false, true);

  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  uint8_t* sO = smem;
  uint8_t* sV = smem + kOBytes;  // V, then K (MN-major)
  uint8_t* sP = smem + kOBytes + kVBytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sP + kPBytes);
  uint64_t* bar_a = bars;      // dO + V
  uint64_t* bar_p = bars + 1;  // P
  uint64_t* bar_s = bars + 2;  // dP in TMEM
  uint64_t* bar_k = bars + 3;  // K
  uint64_t* bar_ds = bars + 4; // dS in shared memory
  uint64_t* bar_o = bars + 5;  // dQ in TMEM
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 6);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int q0 = blockIdx.x * kQ;
  const int b = blockIdx.y;
  const int c3 = b % args.H, c4 = b / args.H;

  if (warp == 0 && lane == 0) {
    for (int i = 0; i < 6; ++i) ptx::mbar_init(bars + i, i == 4 ? 32 * kSoftWarps : 1);
    ptx::fence_barrier_init();
  }
  if (warp == 1) ptx::tmem_alloc<512>(tmem_slot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      ptx::mbar_arrive_expect_tx(bar_a, kOBytes + kVBytes);
      ptx::tma_load_5d(sO, &tmDO, bar_a, 0, args.o_split ? q0 % args.o_split : q0,
                       args.o_split ? q0 / args.o_split : 0, c3, c4);
#pragma unroll
      for (int h = 0; h < KEYS / 256; ++h)
        ptx::tma_load_5d(sV + h * 256 * 128, &tmV, bar_a, 0, h * 256, 0, c3, c4);
      ptx::mbar_arrive_expect_tx(bar_p, kPBytes);
#pragma unroll
      for (int kb = 0; kb < KEYS / 64; ++kb)
        ptx::tma_load_5d(sP + kb * 16384, &tmP, bar_p, kb * 64, q0, 0, c3, c4);
      // K replaces V once the dP product has consumed it
      ptx::mbar_wait(bar_s, 0);
      ptx::mbar_arrive_expect_tx(bar_k, kVBytes);
#pragma unroll
      for (int kb = 0; kb < KEYS / 64; ++kb)
        ptx::tma_load_5d(sV + kb * 8192, &tmK, bar_k, 0, kb * 64, 0, c3, c4);
    }
  } else if (warp == 1) {
    if (lane == 0) {
      ptx::mbar_wait(bar_a, 0);
      ptx::tc_fence_after();
      const uint32_t oa = ptx::smem_u32(sO), va = ptx::smem_u32(sV);
#pragma unroll
      for (int h = 0; h < KEYS / 256; ++h)
#pragma unroll
        for (int k = 0; k < kDh / 16; ++k)
          ptx::umma_bf16(tmem + h * 256, ptx::smem_desc_sw128(oa + 32 * k, 16, 1024),
                         ptx::smem_desc_sw128(va + h * 256 * 128 + 32 * k, 16, 1024), kIdescP,
                         k > 0 ? 1u : 0u);
      ptx::umma_commit(bar_s);
      ptx::mbar_wait(bar_ds, 0);
      ptx::mbar_wait(bar_k, 0);
      ptx::tc_fence_after();
      const uint32_t pa = ptx::smem_u32(sP), ka = ptx::smem_u32(sV);
#pragma unroll
      for (int kb = 0; kb < KEYS / 64; ++kb)
#pragma unroll
        for (int k = 0; k < 4; ++k)
          ptx::umma_bf16(tmem, ptx::smem_desc_sw128(pa + kb * 16384 + 32 * k, 16, 1024),
                         ptx::smem_desc_sw128(ka + kb * 8192 + 2048 * k, 8192, 1024), kIdescQ,
                         (kb > 0 || k > 0) ? 1u : 0u);
      ptx::umma_commit(bar_o);
    }
  } else {
    constexpr int kGroupCols = KEYS / 4;
    const int quarter = warp & 3;
    const int group = (warp - 2) >> 2;
    const int row = quarter * 32 + lane;
    const uint32_t trow = tmem + (static_cast<uint32_t>(quarter * 32) << 16);
    const int c0 = group * kGroupCols;
    const long long q = q0 + row;
    const long long ri = args.rd_split ? (q / args.rd_split) * (args.rd_slices * args.rd_split) +
                                             b * args.rd_split + q % args.rd_split
                                       : static_cast<long long>(b) * args.S + q;
    const float sd = args.scale * __ldg(args.rowdot + ri);
    ptx::mbar_wait(bar_p, 0);
    ptx::mbar_wait(bar_s, 0);
    ptx::tc_fence_after();
#pragma unroll 1
    for (int c = c0; c < c0 + kGroupCols; c += 32) {
      float v[32];
      ptx::tmem_ld32(trow + c, v);
      uint8_t* chunk_row = sP + (c >> 6) * 16384 + row * 128;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int chunk = ((c >> 5) & 1) * 4 + j;
        uint4* ptr = reinterpret_cast<uint4*>(chunk_row + ((chunk ^ (row & 7)) << 4));
        uint4 pk = *ptr;
        __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&pk);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const float2 pp = __bfloat1622float2(h[i]);
          h[i] = __floats2bfloat162_rn(pp.x * fmaf(v[8 * j + 2 * i], args.scale, -sd),
                                       pp.y * fmaf(v[8 * j + 2 * i + 1], args.scale, -sd));
        }
        *ptr = pk;
      }
    }
    // dS visible to the tensor core; dP columns free for dQ
    ptx::fence_async_smem();
    ptx::tc_fence_before();
    ptx::mbar_arrive(bar_ds);
    asm volatile("bar.sync 1, %0;" ::"n"(32 * kSoftWarps) : "memory");
    if (warp == 2 && lane == 0) {
#pragma unroll
      for (int kb = 0; kb < KEYS / 64; ++kb)
        ptx::tma_store_5d(&tmDS, sP + kb * 16384, kb * 64, q0, 0, c3, c4);
      ptx::bulk_commit();
    }
    if (group < 2) {
      ptx::mbar_wait(bar_o, 0);
      ptx::tc_fence_after();
      float o[32];
      ptx::tmem_ld32(trow + group * 32, o);
      const long long qoff = args.dq_split ? (q % args.dq_split) * args.dq_sr +
                                                 (q / args.dq_split) * args.dq_s_hi
                                           : q * args.dq_sr;
      __nv_bfloat16* dst = args.dq + c3 * args.dq_sb_lo + c4 * args.dq_sb_hi + qoff + group * 32;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        uint4 pk;
        pk.x = pack_bf16(o[8 * j + 0], o[8 * j + 1]);
        pk.y = pack_bf16(o[8 * j + 2], o[8 * j + 3]);
        pk.z = pack_bf16(o[8 * j + 4], o[8 * j + 5]);
        pk.w = pack_bf16(o[8 * j + 6], o[8 * j + 7]);
        reinterpret_cast<uint4*>(dst)[j] = pk;
      }
    }
    if (warp == 2 && lane == 0) ptx::bulk_wait_all();
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<512>(tmem);
  }
}

template <int KEYS>
void launch_attn_bwd(const CUtensorMap& o, const CUtensorMap& v, const CUtensorMap& k,
                     const CUtensorMap& p, const CUtensorMap& ds, const AttnBwdArgs& a, int nslices,
                     cudaStream_t s) {
  constexpr int smem = 1024 + kQ * kDh * 2 + KEYS * kDh * 2 + KEYS / 64 * kQ * 128 + 64;
  auto kern = attn_bwd_kernel<KEYS>;
  static bool attr = false;
  if (!attr) {
    C3D_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    attr = true;
  }
  kern<<<dim3(a.S / kQ, nslices), kThreadsAttn, smem, s>>>(o, v, k, p, ds, a);
}

}  // namespace

bool attn_fwd_fused(const View& q, const View& k, const View& v, const View& probs, const View& ctx,
                    int64_t S, int64_t keys, int64_t dh, int64_t H, int nslices, float scale,
                    cudaStream_t s, int mode, float* stat_max, float* stat_sum) {
  if (std::getenv("C3D_NO_FUSED_ATTN")) return false;
  if (dh != kDh || S % kQ || (keys != 256 && keys != 512) || H <= 0) return false;
  if (mode < 0 || mode > 3 || (mode > 0 && (!stat_max || !stat_sum))) return false;
  for (const View* w : {&q, &k, &v, &probs, &ctx})
    if (w->dtype != kBF16 || reinterpret_cast<uintptr_t>(w->base) % 16) return false;
  if (q.csplit || (q.rsplit && q.rsplit % kQ) || k.rsplit || k.csplit || v.rsplit || v.csplit ||
      probs.rsplit || probs.csplit || ctx.csplit || (ctx.rsplit && ctx.rsplit % kQ))
    return false;
  if (ctx.sc != 1 || (ctx.sr * 2) % 16 || (ctx.sb_lo * 2) % 16 || (ctx.sb_hi * 2) % 16 ||
      (ctx.s_hi * 2) % 16)
    return false;
  if (ctx.b_lo_n != H || q.b_lo_n != H || k.b_lo_n != H || v.b_lo_n != H || probs.b_lo_n != H)
    return false;
  int mn = 0;
  const CUtensorMap mq = tc_operand_map(q, S, dh, nslices, kQ, &mn);
  if (mn) return false;
  const CUtensorMap mk = tc_operand_map(k, keys, dh, nslices, 256, &mn);
  if (mn) return false;
  const CUtensorMap mv = tc_operand_map(v, dh, keys, nslices, 64, &mn);
  if (!mn) return false;
  CUtensorMap mp;
  if (!tc_store_map(probs, S, keys, nslices, 64, kQ, &mp)) return false;
  AttnArgs a{};
  a.S = static_cast<int>(S);
  a.keys = static_cast<int>(keys);
  a.H = static_cast<int>(H);
  a.scale_log2 = scale * 1.4426950408889634f;
  a.q_split = static_cast<int>(q.rsplit);
  a.ctx = static_cast<__nv_bfloat16*>(ctx.base);
  a.ctx_sr = ctx.sr;
  a.ctx_sb_lo = ctx.sb_lo;
  a.ctx_sb_hi = ctx.sb_hi;
  a.ctx_split = ctx.rsplit;
  a.ctx_s_hi = ctx.s_hi;
  a.stat_max = stat_max;
  a.stat_sum = stat_sum;
  auto go = [&](auto kk) {
    constexpr int K = decltype(kk)::value;
    switch (mode) {
      case 0: launch_attn<K, 0>(mq, mk, mv, mp, a, nslices, s); break;
      case 1: launch_attn<K, 1>(mq, mk, mv, mp, a, nslices, s); break;
      case 2: launch_attn<K, 2>(mq, mk, mv, mp, a, nslices, s); break;
      default: launch_attn<K, 3>(mq, mk, mv, mp, a, nslices, s); break;
    }
  };
  if (keys == 512) go(std::integral_constant<int, 512>{});
  else go(std::integral_constant<int, 256>{});
  check_launch("attn_fwd_fused");
  return true;
}

}  // namespace c3d

namespace c3d {

bool attn_bwd_fused(const View& d_o, const View& v, const View& k_mn, const View& probs,
                    const View& ds, const View& dq, const float* rowdot, int64_t S, int64_t keys,
                    int64_t dh, int64_t H, int nslices, float scale, cudaStream_t s,
                    int64_t rd_split) {
  if (std::getenv("C3D_NO_FUSED_ATTN") || std::getenv("C3D_NO_FUSED_ATTN_BWD")) return false;
  if (dh != kDh || S % kQ || (keys != 256 && keys != 512) || H <= 0 || !rowdot) return false;
  for (const View* w : {&d_o, &v, &k_mn, &probs, &ds, &dq}) {
    if (w->dtype != kBF16 || reinterpret_cast<uintptr_t>(w->base) % 16) return false;
    if (w->csplit || w->b_lo_n != H) return false;
  }
  if (v.rsplit || k_mn.rsplit || probs.rsplit || ds.rsplit) return false;
  if ((d_o.rsplit && d_o.rsplit % kQ) || (dq.rsplit && dq.rsplit % kQ)) return false;
  if (dq.sc != 1 || (dq.sr * 2) % 16 || (dq.sb_lo * 2) % 16 || (dq.sb_hi * 2) % 16 ||
      (dq.s_hi * 2) % 16)
    return false;
  int mn = 0;
  const CUtensorMap mo = tc_operand_map(d_o, S, dh, nslices, kQ, &mn);
  if (mn) return false;
  const CUtensorMap mv = tc_operand_map(v, keys, dh, nslices, 256, &mn);
  if (mn) return false;
  const CUtensorMap mk = tc_operand_map(k_mn, dh, keys, nslices, 64, &mn);
  if (!mn) return false;
  CUtensorMap mp, mds;
  if (!tc_store_map(probs, S, keys, nslices, 64, kQ, &mp)) return false;
  if (!tc_store_map(ds, S, keys, nslices, 64, kQ, &mds)) return false;
  AttnBwdArgs a{};
  a.S = static_cast<int>(S);
  a.keys = static_cast<int>(keys);
  a.H = static_cast<int>(H);
  a.scale = scale;
  a.o_split = static_cast<int>(d_o.rsplit);
  a.rowdot = rowdot;
  a.rd_split = rd_split;
  a.rd_slices = nslices;
  a.dq = static_cast<__nv_bfloat16*>(dq.base);
  a.dq_sr = dq.sr;
  a.dq_sb_lo = dq.sb_lo;
  a.dq_sb_hi = dq.sb_hi;
  a.dq_split = dq.rsplit;
  a.dq_s_hi = dq.s_hi;
  if (keys == 512) launch_attn_bwd<512>(mo, mv, mk, mp, mds, a, nslices, s);
  else launch_attn_bwd<256>(mo, mv, mk, mp, mds, a, nslices, s);
  check_launch("attn_bwd_fused");
  return true;
}

}  // namespace c3d
