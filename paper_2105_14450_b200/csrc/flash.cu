// Flash-style attention core (tcgen05 + TMEM + TMA), forward and backward, for the
// 3-D attention of cube3d/attention.hpp:78-189 on one rank's (batch, head) slices.
//
// Forward, per CTA: one slice, two 128-query tiles processed ping-pong (the tensor
// core computes one tile's S = Q K^T while the other tile's softmax runs), key blocks
// of BK streamed through a TMA ring. Online softmax with a conditional rescale: the
// running row max only moves (and the TMEM accumulator O is rescaled) when a block
// raises it by more than 2^8, so exp2 arguments stay <= 8 and fp32 O never overflows.
// P goes registers -> shared memory (bf16, UMMA K-major SW128) -> O += P V. Output: the
// context (bf16, normalised) and the row log-sum-exp in log2 units (fp32). Neither the
// scores nor the probabilities reach HBM (the reference materialises both,
// attention.hpp:95-127).
//
// Backward, per CTA: one slice; key blocks j of 128 outer, query blocks i of 128 inner:
//   S^T = K Q^T, dP^T = V dO^T              (TMEM, keys on the lanes; the next iteration's
//                                            products are issued as soon as the elementwise
//                                            warps have pulled the current ones into registers)
//   P^T = exp2(S^T c - lse), dS^T = P^T (dP^T - D)   (elementwise warps -> smem, bf16)
//   dV += P^T dO, dK += dS^T Q               (TMEM accumulators over i, read out per j)
//   dQ_i (+)= dS K_j                          (double-buffered in TMEM; drained by four
//                                            warps into an fp32 workspace owned by the CTA,
//                                            column-major per query block so the
//                                            read-modify-write over j is coalesced; bf16
//                                            rows TMA-stored at the last j)
// The softmax scale is applied to dQ and dK where they leave TMEM. D = rowsum(dO * O) comes
// precomputed (k_attn_rowdot); P and dS never reach HBM.
//
// Shapes: head dim 64 (key blocks of 128) or 128 (key blocks of 64 in the forward);
// queries and keys multiples of 128.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <vector>

#include "common.hpp"
#include "gemm.hpp"
#include "gemm_tc.hpp"
#include "ops.hpp"
#include "ptx.cuh"

namespace c3d {

namespace {

__device__ __forceinline__ float fast_exp2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ uint32_t pack_bf16x2(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}

// Row r, 16-B piece p of a [rows][128 B] SW128 chunk.
__device__ __forceinline__ uint32_t sw128_off(int r, int p) {
  return static_cast<uint32_t>(r * 128 + ((p ^ (r & 7)) << 4));
}

// Output addressing of a [slice][rows][dh] view (possibly row-split: gathered / partial).
struct OutView {
  __nv_bfloat16* base;
  long long sr, sb_lo, sb_hi, split, s_hi;
  int b_lo_n;
  __device__ __forceinline__ __nv_bfloat16* row(int b, long long r) const {
    const long long off = (b % b_lo_n) * sb_lo + (b / b_lo_n) * sb_hi +
                          (split ? (r % split) * sr + (r / split) * s_hi : r * sr);
    return base + off;
  }
};

OutView out_view(const View& v) {
  OutView o;
  o.base = static_cast<__nv_bfloat16*>(v.base);
  o.sr = v.sr;
  o.sb_lo = v.sb_lo;
  o.sb_hi = v.sb_hi;
  o.split = v.rsplit;
  o.s_hi = v.s_hi;
  o.b_lo_n = v.b_lo_n;
  return o;
}

bool out_ok(const View& v, int H) {
  if (v.dtype != kBF16 || v.sc != 1 || v.csplit || v.b_lo_n != H) return false;
  if (reinterpret_cast<uintptr_t>(v.base) % 16) return false;
  for (long long s : {v.sr, v.sb_lo, v.sb_hi, v.s_hi})
    if ((s * 2) % 16) return false;
  return !(v.rsplit && v.rsplit % 128);
}

// =============================================================================== forward

template <int DH, int BK>
struct FwdCfg {
  static constexpr int kQ = 128;
  static constexpr int kStages = DH == 64 ? 2 : 3;
  static constexpr int kQBytes = kQ * DH * 2;
  static constexpr int kKBytes = BK * DH * 2;
  static constexpr int kStageBytes = 2 * kKBytes;  // K block + V block
  static constexpr int kPBytes = kQ * BK * 2;
  static constexpr int kOffStage = 2 * kQBytes;
  static constexpr int kOffP = kOffStage + kStages * kStageBytes;
  static constexpr int kOffBar = kOffP + 2 * kPBytes;
  static constexpr int kSmem = 1024 + kOffBar + 256;
  static constexpr int kColO = 2 * BK;  // S0 [0,BK), S1 [BK,2BK), O0, O1 after
  static constexpr int kThreads = 64 + 256;
  // TMEM columns (a power of two): with <= 256 two CTAs share an SM, so one CTA's
  // prologue (Q load, first S) and epilogue (O readout) overlap the other's key loop
  static constexpr int kTmemNeed = 2 * BK + 2 * DH;
  static constexpr int kTmemCols = kTmemNeed <= 128 ? 128 : (kTmemNeed <= 256 ? 256 : 512);
  static constexpr int kMinBlocks = (kTmemCols <= 256 && kSmem <= 112 * 1024) ? 2 : 1;
};

struct FwdArgs {
  int S, keys, H;
  float scale_log2;
  int q_split;  // rows per gathered query block (0: not split)
  OutView ctx;
  float* lse;   // [slice][S], log2 units
};

template <int DH, int BK>
__global__ void __launch_bounds__(FwdCfg<DH, BK>::kThreads, FwdCfg<DH, BK>::kMinBlocks)
    flash_fwd_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                     const __grid_constant__ CUtensorMap tmV, const FwdArgs args) {
  using C = FwdCfg<DH, BK>;
  constexpr int kST = C::kStages;
  constexpr uint32_t kIdescS = ptx::idesc_bf16_f32(128, BK, false, false);
  constexpr uint32_t kIdescO = ptx::idesc_bf16_f32(128, DH, false, true);

  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::kOffBar);
  uint64_t* bar_q = bars;                 // 1
  uint64_t* k_full = bars + 1;            // kST
  uint64_t* v_full = k_full + kST;        // kST
  uint64_t* kv_empty = v_full + kST;      // kST
  uint64_t* s_full = kv_empty + kST;      // 2
  uint64_t* p_full = s_full + 2;          // 2
  uint64_t* o_full = p_full + 2;          // 2
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_full + 2);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int b = blockIdx.y;
  const int c3 = b % args.H, c4 = b / args.H;
  const int q0 = blockIdx.x * 256;
  const bool two = q0 + 128 < args.S;
  const int nt = two ? 2 : 1;
  const int nb = args.keys / BK;

  if (warp == 0 && lane == 0) {
    ptx::mbar_init(bar_q, 1);
    for (int i = 0; i < kST; ++i) {
      ptx::mbar_init(k_full + i, 1);
      ptx::mbar_init(v_full + i, 1);
      ptx::mbar_init(kv_empty + i, 1);
    }
    for (int t = 0; t < 2; ++t) {
      ptx::mbar_init(s_full + t, 1);
      ptx::mbar_init(p_full + t, 128);
      ptx::mbar_init(o_full + t, 1);
    }
    ptx::fence_barrier_init();
  }
  if (warp == 1) ptx::tmem_alloc<C::kTmemCols>(tmem_slot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      ptx::mbar_arrive_expect_tx(bar_q, nt * C::kQBytes);
      for (int t = 0; t < nt; ++t) {
        const int q = q0 + 128 * t;
        const int qr = args.q_split ? q % args.q_split : q;
        const int qh = args.q_split ? q / args.q_split : 0;
#pragma unroll
        for (int c = 0; c < DH / 64; ++c)
          ptx::tma_load_5d(smem + t * C::kQBytes + c * 128 * 128, &tmQ, bar_q, 64 * c, qr, qh, c3, c4);
      }
      for (int j = 0; j < nb; ++j) {
        const int st = j % kST;
        if (j >= kST) ptx::mbar_wait(kv_empty + st, ((j / kST) - 1) & 1);
        uint8_t* sk = smem + C::kOffStage + st * C::kStageBytes;
        uint8_t* sv = sk + C::kKBytes;
        ptx::mbar_arrive_expect_tx(k_full + st, C::kKBytes);
#pragma unroll
        for (int c = 0; c < DH / 64; ++c)
          ptx::tma_load_5d(sk + c * BK * 128, &tmK, k_full + st, 64 * c, j * BK, 0, c3, c4);
        ptx::mbar_arrive_expect_tx(v_full + st, C::kKBytes);
#pragma unroll
        for (int c = 0; c < DH / 64; ++c)
#pragma unroll
          for (int kb = 0; kb < BK / 64; ++kb)
            ptx::tma_load_5d(sv + c * BK * 128 + kb * 64 * 128, &tmV, v_full + st, 64 * c,
                             j * BK + 64 * kb, 0, c3, c4);
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      const uint32_t sq = ptx::smem_u32(smem);
      const uint32_t sp = ptx::smem_u32(smem + C::kOffP);
      auto issue_s = [&](int t, int j) {
        const uint32_t sk = ptx::smem_u32(smem + C::kOffStage + (j % kST) * C::kStageBytes);
#pragma unroll
        for (int k = 0; k < DH / 16; ++k) {
          const uint32_t off = (k % 4) * 32;
          ptx::umma_bf16(tmem + t * BK,
                         ptx::smem_desc_sw128(sq + t * C::kQBytes + (k / 4) * 128 * 128 + off, 16, 1024),
                         ptx::smem_desc_sw128(sk + (k / 4) * BK * 128 + off, 16, 1024), kIdescS,
                         k > 0 ? 1u : 0u);
        }
        ptx::umma_commit(s_full + t);
      };
      ptx::mbar_wait(bar_q, 0);
      ptx::mbar_wait(k_full, 0);
      ptx::tc_fence_after();
      for (int t = 0; t < nt; ++t) issue_s(t, 0);
      for (int j = 0; j < nb; ++j) {
        const int st = j % kST;
        const uint32_t sv = ptx::smem_u32(smem + C::kOffStage + st * C::kStageBytes + C::kKBytes);
        for (int t = 0; t < nt; ++t) {
          ptx::mbar_wait(p_full + t, j & 1);  // S_t(j) consumed, P_t(j) in smem, O_t rescaled
          if (j + 1 < nb) {
            if (t == 0) ptx::mbar_wait(k_full + (j + 1) % kST, ((j + 1) / kST) & 1);
            ptx::tc_fence_after();
            issue_s(t, j + 1);
          }
          if (t == 0) ptx::mbar_wait(v_full + st, (j / kST) & 1);
          ptx::tc_fence_after();
#pragma unroll
          for (int k = 0; k < BK / 16; ++k)
            ptx::umma_bf16(tmem + C::kColO + t * DH,
                           ptx::smem_desc_sw128(sp + t * C::kPBytes + (k / 4) * 128 * 128 + (k % 4) * 32,
                                                16, 1024),
                           ptx::smem_desc_sw128(sv + 2048 * k, BK * 128, 1024), kIdescO,
                           (j > 0 || k > 0) ? 1u : 0u);
          ptx::umma_commit(o_full + t);
        }
        ptx::umma_commit(kv_empty + st);
      }
    }
  } else {
    // ------------------------------------------------------------ softmax warpgroups
    const int t = (warp - 2) / 4;
    if (t < nt) {
      const int quarter = warp & 3;
      const int r = quarter * 32 + lane;
      const uint32_t lane_base = static_cast<uint32_t>(quarter * 32) << 16;
      const uint32_t ts = tmem + lane_base + t * BK;
      const uint32_t to = tmem + lane_base + C::kColO + t * DH;
      uint8_t* sp = smem + C::kOffP + t * C::kPBytes;
      const float c = args.scale_log2;
      float m = -INFINITY, l = 0.f;
      for (int j = 0; j < nb; ++j) {
        ptx::mbar_wait(s_full + t, j & 1);
        ptx::tc_fence_after();
        // pass 1: row max of this block
        float mx = -INFINITY;
#pragma unroll
        for (int k = 0; k < BK / 32; ++k) {
          float v[32];
          ptx::tmem_ld32(ts + 32 * k, v);
#pragma unroll
          for (int i = 0; i < 32; ++i) mx = fmaxf(mx, v[i]);
        }
        mx *= c;
        float alpha = 1.f;
        const bool bump = j == 0 || mx > m + 8.f;
        if (bump) {
          alpha = fast_exp2(m - mx);  // 0 when m = -inf
          m = mx;
        }
        if (j > 0) {
          // PV_t(j-1) complete: O_t final for the blocks so far, P_t buffer free
          ptx::mbar_wait(o_full + t, (j - 1) & 1);
          ptx::tc_fence_after();
          if (__any_sync(0xffffffffu, bump)) {
#pragma unroll
            for (int k = 0; k < DH / 32; ++k) {
              float o[32];
              ptx::tmem_ld32(to + 32 * k, o);
#pragma unroll
              for (int i = 0; i < 32; ++i) o[i] *= alpha;
              ptx::tmem_st32(to + 32 * k, o);
            }
          }
        }
        // pass 2: P = exp2(s c - m) -> bf16 -> shared (UMMA K-major SW128), row sum
        float sum = 0.f;
#pragma unroll
        for (int k = 0; k < BK / 32; ++k) {
          float v[32];
          ptx::tmem_ld32(ts + 32 * k, v);
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            v[i] = fast_exp2(fmaf(v[i], c, -m));
            sum += v[i];
          }
          uint8_t* row = sp + (k / 2) * 128 * 128;
#pragma unroll
          for (int p = 0; p < 4; ++p) {
            uint4 pk;
            pk.x = pack_bf16x2(v[8 * p + 0], v[8 * p + 1]);
            pk.y = pack_bf16x2(v[8 * p + 2], v[8 * p + 3]);
            pk.z = pack_bf16x2(v[8 * p + 4], v[8 * p + 5]);
            pk.w = pack_bf16x2(v[8 * p + 6], v[8 * p + 7]);
            *reinterpret_cast<uint4*>(row + sw128_off(r, (k % 2) * 4 + p)) = pk;
          }
        }
        l = l * alpha + sum;
        ptx::fence_async_smem();
        ptx::tc_fence_before();
        ptx::mbar_arrive(p_full + t);
      }
      ptx::mbar_wait(o_full + t, (nb - 1) & 1);
      ptx::tc_fence_after();
      const float inv = 1.f / l;
      const int q = q0 + 128 * t + r;
      __nv_bfloat16* dst = args.ctx.row(b, q);
#pragma unroll
      for (int k = 0; k < DH / 32; ++k) {
        float o[32];
        ptx::tmem_ld32(to + 32 * k, o);
#pragma unroll
        for (int p = 0; p < 4; ++p) {
          uint4 pk;
          pk.x = pack_bf16x2(o[8 * p + 0] * inv, o[8 * p + 1] * inv);
          pk.y = pack_bf16x2(o[8 * p + 2] * inv, o[8 * p + 3] * inv);
          pk.z = pack_bf16x2(o[8 * p + 4] * inv, o[8 * p + 5] * inv);
          pk.w = pack_bf16x2(o[8 * p + 6] * inv, o[8 * p + 7] * inv);
          reinterpret_cast<uint4*>(dst + 32 * k)[p] = pk;
        }
      }
      args.lse[static_cast<long long>(b) * args.S + q] = m + __log2f(l);
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<C::kTmemCols>(tmem);
  }
}

template <int DH, int BK>
void launch_fwd(const CUtensorMap& q, const CUtensorMap& k, const CUtensorMap& v, const FwdArgs& a,
                int nslices, cudaStream_t s) {
  using C = FwdCfg<DH, BK>;
  auto kern = flash_fwd_kernel<DH, BK>;
  static bool attr = false;
  if (!attr) {
    C3D_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem));
    attr = true;
  }
  kern<<<dim3((a.S + 255) / 256, nslices), C::kThreads, C::kSmem, s>>>(q, k, v, a);
}

// ============================================================================== backward
//
// One CTA per slice: key blocks j outer, query blocks i inner. dK_j, dV_j accumulate in
// TMEM over i; the dQ_i partial of each (i, j) is drained by four dedicated warps into
// an fp32 workspace row that the same thread owns for every j (store at j = 0, add
// after, bf16 output at the last j) -- no atomics, no fences, no zeroing.

template <int DH>
struct BwdCfg {
  static constexpr bool kAlias = DH == 128;  // dQ shares the S^T columns (TMEM budget)
  static constexpr int kQStages = DH == 64 ? 2 : 1;
  static constexpr int kKVStages = DH == 64 ? 2 : 1;
  static constexpr int kTileBytes = 128 * DH * 2;            // Q_i, dO_i, K_j or V_j
  static constexpr int kKVBytes = 2 * kTileBytes;             // K_j + V_j
  static constexpr int kStageBytes = 2 * kTileBytes + 1024;   // Q_i, dO_i, lse_i, D_i
  static constexpr int kOffStage = kKVStages * kKVBytes;
  static constexpr int kOffP = kOffStage + kQStages * kStageBytes;
  static constexpr int kOffDS = kOffP + 128 * 128 * 2;
  static constexpr int kOffStg = kOffDS + 128 * 128 * 2;
  // staging for the bf16 dQ / dK / dV TMA stores: one [128 rows][64 cols] SW128 chunk
  static constexpr int kStgBytes = 128 * 128;
  static constexpr int kOffBar = kOffStg + kStgBytes;
  static constexpr int kSmem = 1024 + kOffBar + 256;
  static constexpr int kColS = 0, kColDP = 128, kColDV = 256, kColDK = 256 + DH;
  // dQ: double-buffered after dK (DH = 64), or in the S^T columns (DH = 128)
  static constexpr int kColDQ = kAlias ? 0 : 256 + 2 * DH;
  static constexpr int kDQBufs = kAlias ? 1 : 2;
  static constexpr int kEw = 8;                     // elementwise warps: 2 per TMEM lane quarter
  static constexpr int kCgPerWarp = 16 / kEw;       // 32-query column groups per warp
  static constexpr int kThreads = 64 + 32 * kEw + 128;  // producer, MMA, elementwise, 4 drain
};

struct BwdArgs {
  int S, keys, H, nslices;
  float scale, scale_log2;
  int q_split;                      // rows per gathered Q / dO block (0: not split)
  int q_split_dq;                   // rows per block of a split dQ partial (0: not split)
  const float* lse;                 // [slice][S]
  const float* rowdot;              // [slice][S] or [S / rd_split][slices][rd_split]
  long long rd_split;
  OutView dq, dk, dv;
  float* dq_ws;                     // [slice][S/128][DH][128] fp32 scratch
  // head dim 64, unsplit outputs: column sums of the stored dQ / dK / dV (the QKV bias
  // gradient), per (batch, drain warp): [batch][4][H][3 * 64], q | k | v per head
  float* bias_part;
};

template <int DH>
__global__ void __launch_bounds__(BwdCfg<DH>::kThreads, 1)
    flash_bwd_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmDO,
                     const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmV,
                     const __grid_constant__ CUtensorMap tmDQ, const __grid_constant__ CUtensorMap tmDK,
                     const __grid_constant__ CUtensorMap tmDV, const BwdArgs args) {
  using C = BwdCfg<DH>;
  constexpr int kQS = C::kQStages, kKS = C::kKVStages;
  constexpr uint32_t kIdescSP = ptx::idesc_bf16_f32(128, 128, false, false);
  constexpr uint32_t kIdescAcc = ptx::idesc_bf16_f32(128, DH, false, true);
  constexpr uint32_t kIdescDQ = ptx::idesc_bf16_f32(128, DH, true, true);

  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::kOffBar);
  uint64_t* kv_full = bars;               // kKS
  uint64_t* kv_empty = kv_full + kKS;     // kKS
  uint64_t* q_full = kv_empty + kKS;      // kQS
  uint64_t* q_empty = q_full + kQS;       // kQS
  uint64_t* s_full = q_empty + kQS;
  uint64_t* dp_full = s_full + 1;
  uint64_t* p_full = dp_full + 1;
  uint64_t* ds_full = p_full + 1;
  uint64_t* p_free = ds_full + 1;         // dV(it) done: the P buffer may be rewritten
  uint64_t* ds_free = p_free + 1;         // dK(it), dQ(it) done: the dS buffer likewise
  uint64_t* dq_full = ds_free + 1;        // 2 (per dQ buffer)
  uint64_t* dq_empty = dq_full + 2;       // 2
  uint64_t* acc_full = dq_empty + 2;
  uint64_t* acc_empty = acc_full + 1;
  uint64_t* s_cons = acc_empty + 1;       // S^T(it) / dP^T(it) in registers: columns free
  uint64_t* dp_cons = s_cons + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(dp_cons + 1);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int b = blockIdx.x;
  const int c3 = b % args.H, c4 = b / args.H;
  const int nq = args.S / 128;
  const int nkb = args.keys / 128;
  const int total = nq * nkb;

  if (warp == 0 && lane == 0) {
    for (int i = 0; i < kKS; ++i) {
      ptx::mbar_init(kv_full + i, 1);
      ptx::mbar_init(kv_empty + i, 1);
    }
    for (int i = 0; i < kQS; ++i) {
      ptx::mbar_init(q_full + i, 1);
      ptx::mbar_init(q_empty + i, 1);
    }
    ptx::mbar_init(s_full, 1);
    ptx::mbar_init(dp_full, 1);
    ptx::mbar_init(p_full, 32 * C::kEw);
    ptx::mbar_init(ds_full, 32 * C::kEw);
    ptx::mbar_init(p_free, 1);
    ptx::mbar_init(ds_free, 1);
    for (int k = 0; k < 2; ++k) {
      ptx::mbar_init(dq_full + k, 1);
      ptx::mbar_init(dq_empty + k, 128);
    }
    ptx::mbar_init(acc_full, 1);
    ptx::mbar_init(acc_empty, 128);
    ptx::mbar_init(s_cons, 32 * C::kEw);
    ptx::mbar_init(dp_cons, 32 * C::kEw);
    ptx::fence_barrier_init();
  }
  if (warp == 1) ptx::tmem_alloc<512>(tmem_slot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      for (int it = 0; it < total; ++it) {
        const int j = it / nq, i = it % nq;
        if (i == 0) {
          const int ks = j % kKS;
          if (j >= kKS) ptx::mbar_wait(kv_empty + ks, ((j / kKS) - 1) & 1);
          uint8_t* sk = smem + ks * C::kKVBytes;
          ptx::mbar_arrive_expect_tx(kv_full + ks, C::kKVBytes);
#pragma unroll
          for (int c = 0; c < DH / 64; ++c) {
            ptx::tma_load_5d(sk + c * 128 * 128, &tmK, kv_full + ks, 64 * c, j * 128, 0, c3, c4);
            ptx::tma_load_5d(sk + C::kTileBytes + c * 128 * 128, &tmV, kv_full + ks, 64 * c,
                             j * 128, 0, c3, c4);
          }
        }
        const int st = it % kQS;
        if (it >= kQS) ptx::mbar_wait(q_empty + st, ((it / kQS) - 1) & 1);
        uint8_t* sq = smem + C::kOffStage + st * C::kStageBytes;
        uint8_t* sdo = sq + C::kTileBytes;
        float* sl = reinterpret_cast<float*>(sdo + C::kTileBytes);
        const int q = i * 128;
        const int qr = args.q_split ? q % args.q_split : q;
        const int qh = args.q_split ? q / args.q_split : 0;
        ptx::mbar_arrive_expect_tx(q_full + st, 2 * C::kTileBytes + 1024);
#pragma unroll
        for (int c = 0; c < DH / 64; ++c) {
          ptx::tma_load_5d(sq + c * 128 * 128, &tmQ, q_full + st, 64 * c, qr, qh, c3, c4);
          ptx::tma_load_5d(sdo + c * 128 * 128, &tmDO, q_full + st, 64 * c, qr, qh, c3, c4);
        }
        ptx::bulk_load(sl, args.lse + static_cast<long long>(b) * args.S + q, 512, q_full + st);
        const float* rd = args.rd_split
                              ? args.rowdot + (q / args.rd_split) * (args.nslices * args.rd_split) +
                                    static_cast<long long>(b) * args.rd_split + q % args.rd_split
                              : args.rowdot + static_cast<long long>(b) * args.S + q;
        ptx::bulk_load(sl + 128, rd, 512, q_full + st);
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      const uint32_t sp = ptx::smem_u32(smem + C::kOffP), sds = ptx::smem_u32(smem + C::kOffDS);
      auto stage_q = [&](int it) {
        return ptx::smem_u32(smem + C::kOffStage + (it % kQS) * C::kStageBytes);
      };
      auto stage_k = [&](int it) { return ptx::smem_u32(smem + ((it / nq) % kKS) * C::kKVBytes); };
      // waits for the operands of iteration `it`, then S^T = K Q^T / dP^T = V dO^T
      auto issue_s = [&](int it, bool dp) {
        if (!dp) {
          if (it % nq == 0) ptx::mbar_wait(kv_full + (it / nq) % kKS, ((it / nq) / kKS) & 1);
          ptx::mbar_wait(q_full + it % kQS, (it / kQS) & 1);
        }
        ptx::tc_fence_after();
        const uint32_t sq = stage_q(it), sk = stage_k(it);
        const uint32_t a = dp ? sk + C::kTileBytes : sk, bb = dp ? sq + C::kTileBytes : sq;
#pragma unroll
        for (int k = 0; k < DH / 16; ++k) {
          const uint32_t off = (k / 4) * 128 * 128 + (k % 4) * 32;
          ptx::umma_bf16(tmem + (dp ? C::kColDP : C::kColS), ptx::smem_desc_sw128(a + off, 16, 1024),
                         ptx::smem_desc_sw128(bb + off, 16, 1024), kIdescSP, k > 0 ? 1u : 0u);
        }
        ptx::umma_commit(dp ? dp_full : s_full);
      };
      // acc[M = keys][N = DH] (+)= X^T[keys][queries] Y[queries][DH]  (X^T = P^T or dS^T)
      auto issue_acc = [&](uint32_t col, uint32_t xt, uint32_t y, bool acc) {
#pragma unroll
        for (int k = 0; k < 8; ++k)
          ptx::umma_bf16(tmem + col,
                         ptx::smem_desc_sw128(xt + (k / 4) * 128 * 128 + (k % 4) * 32, 16, 1024),
                         ptx::smem_desc_sw128(y + 2048 * k, 128 * 128, 1024), kIdescAcc,
                         (acc || k > 0) ? 1u : 0u);
      };
      issue_s(0, false);
      issue_s(0, true);
      for (int it = 0; it < total; ++it) {
        const int j = it / nq, i = it % nq;
        const uint32_t sq = stage_q(it), sdo = sq + C::kTileBytes, sk = stage_k(it);
        const int qb = it % C::kDQBufs;
        if (!C::kAlias && it + 1 < total) {
          ptx::mbar_wait(s_cons, it & 1);  // S^T(it) in registers
          issue_s(it + 1, false);
        }
        ptx::mbar_wait(p_full, it & 1);
        if (i == 0 && j > 0) ptx::mbar_wait(acc_empty, (j - 1) & 1);  // dK, dV read out
        ptx::tc_fence_after();
        issue_acc(C::kColDV, sp, sdo, i > 0);
        ptx::umma_commit(p_free);
        if (!C::kAlias && it + 1 < total) {
          ptx::mbar_wait(dp_cons, it & 1);
          issue_s(it + 1, true);
        }
        ptx::mbar_wait(ds_full, it & 1);
        ptx::tc_fence_after();
        issue_acc(C::kColDK, sds, sq, i > 0);
        if (i == nq - 1) ptx::umma_commit(acc_full);
        if (it >= C::kDQBufs) {
          ptx::mbar_wait(dq_empty + qb, ((it - C::kDQBufs) / C::kDQBufs) & 1);
          ptx::tc_fence_after();
        }
        // dQ_i[M = queries][N = DH] = dS[queries][keys] K[keys][DH]  (dS^T read MN-major)
#pragma unroll
        for (int k = 0; k < 8; ++k)
          ptx::umma_bf16(tmem + C::kColDQ + qb * DH, ptx::smem_desc_sw128(sds + 2048 * k, 128 * 128, 1024),
                         ptx::smem_desc_sw128(sk + 2048 * k, 128 * 128, 1024), kIdescDQ,
                         k > 0 ? 1u : 0u);
        ptx::umma_commit(dq_full + qb);
        ptx::umma_commit(ds_free);
        ptx::umma_commit(q_empty + it % kQS);
        if (i == nq - 1) ptx::umma_commit(kv_empty + j % kKS);
        if (C::kAlias && it + 1 < total) {
          ptx::mbar_wait(dq_empty, it & 1);  // dQ drained out of the S^T columns
          issue_s(it + 1, false);
          issue_s(it + 1, true);
        }
      }
    }
  } else if (warp < 2 + C::kEw) {
    // ------------------------------------------------------------ elementwise warps
    // warp -> TMEM lane quarter (key rows) and kCgPerWarp groups of 32 query columns
    constexpr int G = C::kCgPerWarp;
    const int quarter = warp & 3;
    const int cg0 = ((warp - 2) >> 2) * G;
    const int r = quarter * 32 + lane;
    const uint32_t lb = static_cast<uint32_t>(quarter * 32) << 16;
    const float c = args.scale_log2;
    for (int it = 0; it < total; ++it) {
      const float* sl = reinterpret_cast<const float*>(smem + C::kOffStage +
                                                       (it % kQS) * C::kStageBytes +
                                                       2 * C::kTileBytes);
      ptx::mbar_wait(q_full + it % kQS, (it / kQS) & 1);
      ptx::mbar_wait(s_full, it & 1);
      ptx::tc_fence_after();
      uint32_t pk[16 * G];  // P^T (this thread's key, 32 G queries) as bf16 pairs
#pragma unroll
      for (int g = 0; g < G; ++g) {
        float v[32];
        ptx::tmem_ld32(tmem + lb + C::kColS + 32 * (cg0 + g), v);
        if (g == G - 1) {
          ptx::tc_fence_before();
          ptx::mbar_arrive(s_cons);
        }
        const float4* l4p = reinterpret_cast<const float4*>(sl + 32 * (cg0 + g));
#pragma unroll
        for (int q4 = 0; q4 < 8; ++q4) {
          const float4 l4 = l4p[q4];
          pk[16 * g + 2 * q4] = pack_bf16x2(fast_exp2(fmaf(v[4 * q4], c, -l4.x)),
                                            fast_exp2(fmaf(v[4 * q4 + 1], c, -l4.y)));
          pk[16 * g + 2 * q4 + 1] = pack_bf16x2(fast_exp2(fmaf(v[4 * q4 + 2], c, -l4.z)),
                                                fast_exp2(fmaf(v[4 * q4 + 3], c, -l4.w)));
        }
      }
      if (it > 0) ptx::mbar_wait(p_free, (it - 1) & 1);  // dV of it-1 done with P
#pragma unroll
      for (int g = 0; g < G; ++g) {
        const int cg = cg0 + g;
        uint8_t* sp = smem + C::kOffP + (cg >> 1) * 128 * 128;
#pragma unroll
        for (int q8 = 0; q8 < 4; ++q8)
          *reinterpret_cast<uint4*>(sp + sw128_off(r, (cg & 1) * 4 + q8)) =
              make_uint4(pk[16 * g + 4 * q8], pk[16 * g + 4 * q8 + 1], pk[16 * g + 4 * q8 + 2],
                         pk[16 * g + 4 * q8 + 3]);
      }
      ptx::fence_async_smem();
      ptx::mbar_arrive(p_full);
      ptx::mbar_wait(dp_full, it & 1);
      ptx::tc_fence_after();
      if (it > 0) ptx::mbar_wait(ds_free, (it - 1) & 1);  // dK / dQ of it-1 done with dS
      {
        // dS^T = P^T (dP^T - D), unscaled: the softmax scale is applied to dK / dQ where
        // they leave TMEM (DH x fewer multiplies)
#pragma unroll
        for (int g = 0; g < G; ++g) {
          const int cg = cg0 + g;
          float v[32];
          ptx::tmem_ld32(tmem + lb + C::kColDP + 32 * cg, v);
          if (g == G - 1) {
            ptx::tc_fence_before();
            ptx::mbar_arrive(dp_cons);
          }
          const float4* d4p = reinterpret_cast<const float4*>(sl + 128 + 32 * cg);
#pragma unroll
          for (int q4 = 0; q4 < 8; ++q4) {
            const float4 d4 = d4p[q4];
            const float2 a0 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&pk[16 * g + 2 * q4]));
            const float2 a1 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&pk[16 * g + 2 * q4 + 1]));
            pk[16 * g + 2 * q4] = pack_bf16x2(a0.x * (v[4 * q4] - d4.x), a0.y * (v[4 * q4 + 1] - d4.y));
            pk[16 * g + 2 * q4 + 1] = pack_bf16x2(a1.x * (v[4 * q4 + 2] - d4.z), a1.y * (v[4 * q4 + 3] - d4.w));
          }
          uint8_t* sds = smem + C::kOffDS + (cg >> 1) * 128 * 128;
#pragma unroll
          for (int q8 = 0; q8 < 4; ++q8)
            *reinterpret_cast<uint4*>(sds + sw128_off(r, (cg & 1) * 4 + q8)) =
                make_uint4(pk[16 * g + 4 * q8], pk[16 * g + 4 * q8 + 1], pk[16 * g + 4 * q8 + 2],
                           pk[16 * g + 4 * q8 + 3]);
        }
      }
      ptx::fence_async_smem();
      ptx::tc_fence_before();
      ptx::mbar_arrive(ds_full);
    }
  } else {
    // ------------------------------------------------------------ dQ drain warps
    // dQ_i partial (TMEM, one query row per thread). The fp32 workspace is column-major
    // inside each 128-query block ([slice][block][col][128]), so for every column a warp's
    // 32 rows are 128 contiguous bytes: the read-modify-write over j is fully coalesced and
    // owned by this CTA (no atomics). At the last j the bf16 rows are staged (SW128) and
    // TMA-stored into the dQ view.
    const int quarter = warp & 3;
    const int r = quarter * 32 + lane;
    const int dt = threadIdx.x - (64 + 32 * C::kEw);  // 0..127
    const uint32_t lb = static_cast<uint32_t>(quarter * 32) << 16;
    uint8_t* stg = smem + C::kOffStg;
    auto stage_store = [&](const CUtensorMap* map, int col0, int row0, int qsplit) {
      ptx::fence_async_smem();
      ptx::named_bar(2, 128);
      if (dt == 0) {
        const int rr = qsplit ? row0 % qsplit : row0, rh = qsplit ? row0 / qsplit : 0;
        ptx::tma_store_5d(map, stg, col0, rr, rh, c3, c4);
        ptx::bulk_commit();
        ptx::bulk_wait_read();
      }
      ptx::named_bar(2, 128);
    };
    auto stage_row = [&](const float (&v)[32], int half) {
#pragma unroll
      for (int p = 0; p < 4; ++p)
        *reinterpret_cast<uint4*>(stg + sw128_off(r, 4 * half + p)) =
            make_uint4(pack_bf16x2(v[8 * p + 0], v[8 * p + 1]), pack_bf16x2(v[8 * p + 2], v[8 * p + 3]),
                       pack_bf16x2(v[8 * p + 4], v[8 * p + 5]), pack_bf16x2(v[8 * p + 6], v[8 * p + 7]));
    };
    // QKV bias gradient (head dim 64): column sums of every staged bf16 tile over this
    // warp's 32 rows -- lane L owns columns 2L, 2L + 1 (one pair per row, conflict-free)
    float bs[3][2] = {{0.f, 0.f}, {0.f, 0.f}, {0.f, 0.f}};  // q, k, v
    auto sum_staged = [&](float (&acc)[2]) {
      __syncwarp();
#pragma unroll 8
      for (int rr = 0; rr < 32; ++rr) {
        const int R = quarter * 32 + rr;
        const uint32_t u = *reinterpret_cast<const uint32_t*>(
            stg + R * 128 + (((lane >> 2) ^ (R & 7)) << 4) + (lane & 3) * 4);
        acc[0] += __uint_as_float(u << 16);
        acc[1] += __uint_as_float(u & 0xffff0000u);
      }
    };
    const bool want_bias = DH == 64 && args.bias_part != nullptr;
    for (int it = 0; it < total; ++it) {
      const int j = it / nq, i = it % nq;
      if (i == nq - 1) {
        // dV_j, dK_j final (their commit precedes dQ's): thread = key row
        ptx::mbar_wait(acc_full, j & 1);
        ptx::tc_fence_after();
#pragma unroll 1
        for (int t = 0; t < 2 * (DH / 64); ++t) {
          const int which = t / (DH / 64), ch = t % (DH / 64);
          const uint32_t col = (which == 0 ? C::kColDV : C::kColDK) + 64 * ch;
#pragma unroll
          for (int half = 0; half < 2; ++half) {
            float v[32];
            ptx::tmem_ld32(tmem + lb + col + 32 * half, v);
            if (which == 1)
#pragma unroll
              for (int e = 0; e < 32; ++e) v[e] *= args.scale;  // dK = scale dS^T Q
            stage_row(v, half);
          }
          if (t == 2 * (DH / 64) - 1) {
            ptx::tc_fence_before();
            ptx::mbar_arrive(acc_empty);
          }
          if (want_bias) sum_staged(bs[which == 0 ? 2 : 1]);
          stage_store(which == 0 ? &tmDV : &tmDK, 64 * ch, j * 128, 0);
        }
      }
      const int qb = it % C::kDQBufs;
      ptx::mbar_wait(dq_full + qb, (it / C::kDQBufs) & 1);
      ptx::tc_fence_after();
      float* ws = args.dq_ws + (static_cast<long long>(b) * nq + i) * DH * 128 + r;
      const bool last = j + 1 == nkb;
#pragma unroll 1
      for (int ch = 0; ch < DH / 64; ++ch) {
#pragma unroll
        for (int half = 0; half < 2; ++half) {
          const int c0 = 64 * ch + 32 * half;
          float v[32];
          ptx::tmem_ld32(tmem + lb + C::kColDQ + qb * DH + c0, v);
          if (ch == DH / 64 - 1 && half == 1) {  // every column of dQ_i is out of TMEM
            ptx::tc_fence_before();
            ptx::mbar_arrive(dq_empty + qb);
          }
#pragma unroll
          for (int c = 0; c < 32; ++c) v[c] *= args.scale;  // dQ = scale dS K
          if (j > 0) {
#pragma unroll
            for (int c = 0; c < 32; ++c) v[c] += __ldcg(ws + (c0 + c) * 128);
          }
          if (!last) {
#pragma unroll
            for (int c = 0; c < 32; ++c) __stcg(ws + (c0 + c) * 128, v[c]);
          } else {
            stage_row(v, half);
          }
        }
        if (last) {
          if (want_bias) sum_staged(bs[0]);
          stage_store(&tmDQ, 64 * ch, i * 128, args.q_split_dq);
        }
      }
    }
    if (want_bias) {
      // [batch][drain warp][head][q | k | v][64]
      float* p = args.bias_part +
                 ((static_cast<long long>(c4) * 4 + quarter) * args.H + c3) * (3 * 64) + 2 * lane;
#pragma unroll
      for (int part = 0; part < 3; ++part)
        *reinterpret_cast<float2*>(p + 64 * part) = make_float2(bs[part][0], bs[part][1]);
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<512>(tmem);
  }
}

template <int DH>
void launch_bwd(const CUtensorMap& q, const CUtensorMap& d_o, const CUtensorMap& k,
                const CUtensorMap& v, const CUtensorMap& dq, const CUtensorMap& dk,
                const CUtensorMap& dv, const BwdArgs& a, cudaStream_t s) {
  using C = BwdCfg<DH>;
  auto kern = flash_bwd_kernel<DH>;
  static bool attr = false;
  if (!attr) {
    C3D_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem));
    attr = true;
  }
  kern<<<a.nslices, C::kThreads, C::kSmem, s>>>(q, d_o, k, v, dq, dk, dv, a);
}

}  // namespace

bool flash_supported(int64_t S, int64_t keys, int64_t dh) {
  if (std::getenv("C3D_NO_FLASH") || std::getenv("C3D_NO_FUSED_ATTN")) return false;
  if (dh != 64 && dh != 128) return false;
  return S > 0 && keys > 0 && S % 128 == 0 && keys % 128 == 0;
}

bool flash_fwd(const View& q, const View& k, const View& v, const View& ctx, float* lse, int64_t S,
               int64_t keys, int64_t dh, int64_t H, int nslices, float scale, cudaStream_t s) {
  if (!flash_supported(S, keys, dh) || H <= 0 || !lse) return false;
  for (const View* w : {&q, &k, &v}) {
    if (w->dtype != kBF16 || reinterpret_cast<uintptr_t>(w->base) % 16) return false;
    if (w->csplit || w->b_lo_n != H) return false;
  }
  if (k.rsplit || v.rsplit || (q.rsplit && q.rsplit % 128) || !out_ok(ctx, static_cast<int>(H)))
    return false;
  // dh 64: key blocks of 64 (256 TMEM columns, two CTAs per SM); C3D_FWD_BK128 keeps
  // the one-CTA-per-SM variant with key blocks of 128
  static const bool bk128 = std::getenv("C3D_FWD_BK128") != nullptr;
  const int bk = dh == 64 && bk128 ? 128 : 64;
  int mn = 0;
  const CUtensorMap mq = tc_operand_map(q, S, dh, nslices, 128, &mn);
  if (mn) return false;
  const CUtensorMap mk = tc_operand_map(k, keys, dh, nslices, bk, &mn);
  if (mn) return false;
  const CUtensorMap mv = tc_operand_map(v, dh, keys, nslices, 64, &mn);
  if (!mn) return false;
  FwdArgs a{};
  a.S = static_cast<int>(S);
  a.keys = static_cast<int>(keys);
  a.H = static_cast<int>(H);
  a.scale_log2 = scale * 1.4426950408889634f;
  a.q_split = static_cast<int>(q.rsplit);
  a.ctx = out_view(ctx);
  a.lse = lse;
  if (dh == 64 && bk == 128) launch_fwd<64, 128>(mq, mk, mv, a, nslices, s);
  else if (dh == 64) launch_fwd<64, 64>(mq, mk, mv, a, nslices, s);
  else launch_fwd<128, 64>(mq, mk, mv, a, nslices, s);
  check_launch("flash_fwd");
  return true;
}

}  // namespace c3d

namespace c3d {

size_t flash_bwd_workspace_bytes(int64_t S, int64_t dh, int nslices) {
  return static_cast<size_t>(nslices) * S * dh * sizeof(float);
}

bool flash_bwd(const View& q, const View& k, const View& v, const View& d_o, const float* lse,
               const float* rowdot, int64_t rd_split, const View& dq, const View& dk, const View& dv,
               void* ws, int64_t S, int64_t keys, int64_t dh, int64_t H, int nslices, float scale,
               cudaStream_t s, float* bias_part) {
  if (!flash_supported(S, keys, dh) || H <= 0 || !lse || !rowdot || !ws) return false;
  if (bias_part && (dh != 64 || q.rsplit || dq.rsplit)) return false;
  for (const View* w : {&q, &k, &v, &d_o}) {
    if (w->dtype != kBF16 || reinterpret_cast<uintptr_t>(w->base) % 16) return false;
    if (w->csplit || w->b_lo_n != H || w->sc != 1) return false;
  }
  if (k.rsplit || v.rsplit || (q.rsplit && q.rsplit % 128) || d_o.rsplit != q.rsplit) return false;
  if (q.rsplit && (d_o.s_hi == 0 || q.s_hi == 0)) return false;
  if (rd_split && rd_split % 128) return false;
  const int Hi = static_cast<int>(H);
  if (!out_ok(dq, Hi) || !out_ok(dk, Hi) || !out_ok(dv, Hi) || dk.rsplit || dv.rsplit) return false;
  if (reinterpret_cast<uintptr_t>(ws) % 16 || reinterpret_cast<uintptr_t>(lse) % 16 ||
      reinterpret_cast<uintptr_t>(rowdot) % 16)
    return false;
  int mn = 0;
  const CUtensorMap mq = tc_operand_map(q, S, dh, nslices, 128, &mn);
  if (mn) return false;
  const CUtensorMap mo = tc_operand_map(d_o, S, dh, nslices, 128, &mn);
  if (mn) return false;
  const CUtensorMap mk = tc_operand_map(k, keys, dh, nslices, 128, &mn);
  if (mn) return false;
  const CUtensorMap mv = tc_operand_map(v, keys, dh, nslices, 128, &mn);
  if (mn) return false;
  BwdArgs a{};
  a.S = static_cast<int>(S);
  a.keys = static_cast<int>(keys);
  a.H = Hi;
  a.nslices = nslices;
  a.scale = scale;
  a.scale_log2 = scale * 1.4426950408889634f;
  a.q_split = static_cast<int>(q.rsplit);
  a.lse = lse;
  a.rowdot = rowdot;
  a.rd_split = rd_split;
  a.dq = out_view(dq);
  a.dk = out_view(dk);
  a.dv = out_view(dv);
  a.dq_ws = static_cast<float*>(ws);
  a.bias_part = bias_part;
  CUtensorMap mdq, mdk, mdv;
  if (!tc_store_map(dq, S, dh, nslices, 64, 128, &mdq) ||
      !tc_store_map(dk, keys, dh, nslices, 64, 128, &mdk) ||
      !tc_store_map(dv, keys, dh, nslices, 64, 128, &mdv))
    return false;
  a.q_split_dq = static_cast<int>(dq.rsplit);
  if (dh == 64) launch_bwd<64>(mq, mo, mk, mv, mdq, mdk, mdv, a, s);
  else launch_bwd<128>(mq, mo, mk, mv, mdq, mdk, mdv, a, s);
  check_launch("flash_bwd");
  return true;
}

}  // namespace c3d

namespace c3d {

namespace {

__global__ void lse_weights_kernel(const float* lr, const float* mx, float* w, int64_t n) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i < n) w[i] = exp2f(lr[i] - mx[i]);
}

// One warp per (slice, query) row: scale this rank's partial context row by its share
// exp2(lse_r - M) / W of the global normaliser, and turn M into the global lse.
__global__ void combine_kernel(OutView pv, const float* lr, float* lse, const float* W, int S,
                               int dh, int64_t rows) {
  const int64_t row = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) / 32;
  const int lane = threadIdx.x % 32;
  if (row >= rows) return;
  const int b = static_cast<int>(row / S), q = static_cast<int>(row % S);
  const float m = lse[row], w = W[row];
  const float f = exp2f(lr[row] - m) / w;
  __nv_bfloat16* p = pv.row(b, q);
  for (int d = 2 * lane; d < dh; d += 64) {
    __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(p + d);
    const float2 v = __bfloat1622float2(*h);
    *h = __floats2bfloat162_rn(v.x * f, v.y * f);
  }
  __syncwarp();
  if (lane == 0) lse[row] = m + log2f(w);
}

}  // namespace

void k_flash_lse_weights(const float* lr, const float* mx, float* w, int64_t n, cudaStream_t s) {
  if (n == 0) return;
  lse_weights_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, s>>>(lr, mx, w, n);
  check_launch("flash_lse_weights");
}

void k_flash_combine(const View& partial, const float* lr, float* lse_io, const float* W, int64_t S,
                     int64_t dh, int64_t H, int nslices, cudaStream_t s) {
  const int64_t rows = static_cast<int64_t>(nslices) * S;
  if (rows == 0) return;
  (void)H;
  combine_kernel<<<static_cast<unsigned>((rows * 32 + 255) / 256), 256, 0, s>>>(
      out_view(partial), lr, lse_io, W, static_cast<int>(S), static_cast<int>(dh), rows);
  check_launch("flash_combine");
}

}  // namespace c3d
