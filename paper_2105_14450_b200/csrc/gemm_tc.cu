// sm_100a tcgen05 GEMM: bf16 operands staged by TMA into 128B-swizzled shared
// memory, fp32 accumulators in TMEM, fused epilogue from TMEM to global.
//
// This is the B200 replacement of the reference's local product
// `multiply_accumulate` (cube3d/matrix.hpp:68-92): the NN / NT / TN forms map to
// K-major or MN-major UMMA operand descriptors instead of strided CPU loops.
//
// Structure (one CTA per SM, persistent over work units = output tiles x K splits):
//   warp 0      TMA producer (one lane)                  smem ring: full/empty mbarriers
//   warp 1      TMEM allocator + UMMA issuer (one lane)  TMEM ring: 2 accumulators
//   warps 2..9  epilogue: tcgen05.ld (32-column halves) -> registers -> epilogue math ->
//               128B-swizzled smem staging -> TMA bulk-tensor store (two warps per
//               TMEM lane quarter, each owning half of the columns); aux operands
//               arrive by TMA into a second per-warp buffer; row-wise st.global
//               fallback when the output view is not TMA-addressable
// Tile: 128 x BN (UMMA M=128, N=BN, K=16), K-block 64 per pipeline stage. The
// producer and issuer loops carry their stage/phase and TMA coordinates
// incrementally: no integer division on the per-K-block path.
// Split-K (batch 1 only): each split writes fp32 partials to a workspace and a
// deterministic reduction kernel applies the epilogue.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <stdexcept>
#include <string>

#include "common.hpp"
#include "epi.cuh"
#include "gemm.hpp"
#include "gemm_tc.hpp"
#include "ptx.cuh"

namespace c3d {

namespace {

constexpr int kBM = 128;
constexpr int kBK = 64;
constexpr int kEpiWarps = 8;
constexpr int kThreads = 64 + 32 * kEpiWarps;
constexpr int kSmemBudget = 227 * 1024;

struct TcOperand {
  int mn_major = 0;  // 1: the r (M/N) index is contiguous
  int split = 0;     // 0 none, 1 split on r, 2 split on c (K)
  int split_n = 0;
  int b_lo_n = 1;
};

struct TcArgs {
  int M, N, K, batch;
  int cg;  // CTAs per tile (2: cta_group::2 pair, M = 256)
  // k-segmented tiles (CTA pairs): each tile's K range is cut into sk segments, units
  // run segment-major (the pairs of a wave share k windows in L2); the last segment of
  // a tile to arrive (sk_count) finishes it, adding the others' fp32 partials (sk_ws,
  // raised by sk_flag) in k order -- no separate reduction pass
  int sk;               // segments per tile (0: off)
  float* sk_ws;         // [tile][segment][rank][BN][128] (column-major partial tiles)
  uint32_t* sk_flag;    // [tile][segment][rank]
  uint32_t* sk_count;   // [tile][rank]
  int m_tiles, n_tiles, k_blocks;
  int group_m;  // tile rows per rasterisation band (1: plain m-major order)
  int num_tiles;  // output tiles (batch * m_tiles * n_tiles)
  int ksplit, kb_per_split;
  int stages;
  int vec_ok;
  float* ws;  // split-K partials [ksplit][M][N] fp32
  // TMA-store epilogue: output tile chunks [32 rows][128 B] staged in swizzled smem
  int tma_store;             // 1: stores go through tmC / tmP
  int cw;                    // columns per store chunk (32 fp32, 64 bf16)
  int st_rsplit, st_csplit;  // split of the stored view (rows / cols)
  int st_blo;                // batch-lo extent of the stored view
  int x_tma;                 // 1: aux (2: residual) tile chunks arrive by TMA (tmP) into
                             //    a second per-warp buffer (same view geometry as the output)
  int pre_tma;               // 1: the pre-activation output is staged in that second
                             //    buffer and TMA-stored through tmP
  TcOperand a, b;
  Epilogue epi;
  // fused reduce-scatter (rs_P > 1): block k of the rows goes through rsm.m[k]
  int rs_P, rs_me, rs_block_rows, rs_block0, rs_done_offset;
  const uint32_t* rs_entered[kRsMax];
  ptx::Fault rs_fault;
  uint32_t* rs_done[kRsMax];
  const uint32_t* rs_epoch;
};

struct RsMaps {
  CUtensorMap m[kRsMax];
};

// Writes one 16-B chunk j (8 bf16 or 4 fp32 values) of row `lane` of the swizzled
// staging tile.
template <int CW>
__device__ __forceinline__ void stage_chunk(uint8_t* buf, int lane, int j, const float* v) {
  uint8_t* dst = buf + lane * 128 + ((j ^ (lane & 7)) << 4);
  if (CW == 32) {
    *reinterpret_cast<float4*>(dst) = make_float4(v[0], v[1], v[2], v[3]);
  } else {
    uint4 pk;
    __nv_bfloat162 h0 = __floats2bfloat162_rn(v[0], v[1]);
    __nv_bfloat162 h1 = __floats2bfloat162_rn(v[2], v[3]);
    __nv_bfloat162 h2 = __floats2bfloat162_rn(v[4], v[5]);
    __nv_bfloat162 h3 = __floats2bfloat162_rn(v[6], v[7]);
    pk.x = *reinterpret_cast<uint32_t*>(&h0);
    pk.y = *reinterpret_cast<uint32_t*>(&h1);
    pk.z = *reinterpret_cast<uint32_t*>(&h2);
    pk.w = *reinterpret_cast<uint32_t*>(&h3);
    *reinterpret_cast<uint4*>(dst) = pk;
  }
}

// Makes the staged tile visible to the async proxy and issues its TMA store.
__device__ __forceinline__ void store_staged(const CUtensorMap* map, const uint8_t* buf, int lane,
                                             int c0, int c1, int c2, int c3, int c4) {
  ptx::fence_async_smem();
  __syncwarp();
  if (lane == 0) {
    ptx::tma_store_5d(map, buf, c0, c1, c2, c3, c4);
    ptx::bulk_commit();
  }
}

// Waits until this warp's staging buffer may be rewritten.
__device__ __forceinline__ void staging_acquire(int lane) {
  if (lane == 0) ptx::bulk_wait_read();
  __syncwarp();
}

// TMA coordinates of one operand for the current tile, advanced per K-block.
struct OpPos {
  int r_lo[4];
  int r_hi[4];
  int k_lo, k_hi;
  int c3, c4;
};

__device__ __forceinline__ void op_init(const TcOperand& op, OpPos& p, int r0, int nchunks, int k0,
                                        int b) {
  p.c3 = b % op.b_lo_n;
  p.c4 = b / op.b_lo_n;
  for (int j = 0; j < nchunks; ++j) {
    const int r = r0 + 64 * j;
    p.r_lo[j] = op.split == 1 ? r % op.split_n : r;
    p.r_hi[j] = op.split == 1 ? r / op.split_n : 0;
  }
  p.k_lo = op.split == 2 ? k0 % op.split_n : k0;
  p.k_hi = op.split == 2 ? k0 / op.split_n : 0;
}

__device__ __forceinline__ void op_advance(const TcOperand& op, OpPos& p) {
  p.k_lo += kBK;
  if (op.split == 2 && p.k_lo == op.split_n) {
    p.k_lo = 0;
    ++p.k_hi;
  }
}

template <int ROWS>
__device__ __forceinline__ void op_issue(const CUtensorMap* map, const TcOperand& op,
                                         const OpPos& p, uint8_t* dst, uint64_t* bar) {
  if (!op.mn_major) {
    ptx::tma_load_5d(dst, map, bar, p.k_lo, p.r_lo[0], p.r_hi[0] + p.k_hi, p.c3, p.c4);
  } else {
#pragma unroll
    for (int j = 0; j < ROWS / 64; ++j)
      ptx::tma_load_5d(dst + j * 8192, map, bar, p.r_lo[j], p.k_lo, p.r_hi[j] + p.k_hi, p.c3, p.c4);
  }
}

// Same for a CTA pair: the load lands in this CTA's shared memory and completes on the
// leader's full barrier (shared::cluster address `bar`).
template <int ROWS>
__device__ __forceinline__ void op_issue_pair(const CUtensorMap* map, const TcOperand& op,
                                              const OpPos& p, uint8_t* dst, uint32_t bar) {
  if (!op.mn_major) {
    ptx::tma_load_5d_pair(dst, map, bar, p.k_lo, p.r_lo[0], p.r_hi[0] + p.k_hi, p.c3, p.c4);
  } else {
#pragma unroll
    for (int j = 0; j < ROWS / 64; ++j)
      ptx::tma_load_5d_pair(dst + j * 8192, map, bar, p.r_lo[j], p.k_lo, p.r_hi[j] + p.k_hi, p.c3,
                            p.c4);
  }
}

struct Unit {
  int b, m0, n0, kb0, kb1, ks;
  int tile;   // tile index; sk_seg: -1 whole tile, else the k segment of a split tile
  int sk_seg;
};

// CTA pairs (cg = 2): m tiles are 256-row pair tiles; CTA `rank` owns rows
// [m0 + 128 rank, +128) of its pair's tile.
__device__ __forceinline__ Unit decode_tile(const TcArgs& a, int tile, int bn, int rank) {
  Unit u;
  u.ks = 0;
  u.tile = tile;
  u.sk_seg = -1;
  const int per_batch = a.m_tiles * a.n_tiles;
  u.b = tile / per_batch;
  const int rem = tile - u.b * per_batch;
  // grouped rasterisation: a wave of CTAs covers a group_m-row band of tiles, so the A
  // and B panels of one wave stay resident in L2 even when B alone is larger than L2
  // (m-major order re-streams all of B for every tile row: 442 GB at M=N=K=32768)
  const int group = rem / (a.group_m * a.n_tiles);
  const int first_m = group * a.group_m;
  const int gsize = min(a.m_tiles - first_m, a.group_m);
  const int within = rem - group * (a.group_m * a.n_tiles);
  const int nt = within / gsize;
  const int mt = first_m + (within - nt * gsize);
  u.m0 = mt * kBM * a.cg + rank * kBM;
  u.n0 = nt * bn;
  u.kb0 = 0;
  u.kb1 = a.k_blocks;
  return u;
}

__device__ __forceinline__ Unit decode_unit(const TcArgs& a, int t, int bn, int rank = 0) {
  // split-major order: the persistent CTAs sweep K window by window together, so each
  // window's operand footprint stays resident in L2 (no drift-induced thrash).
  const int ks = t / a.num_tiles;
  Unit u = decode_tile(a, t - ks * a.num_tiles, bn, rank);
  u.ks = ks;
  u.kb0 = ks * a.kb_per_split;
  u.kb1 = min(a.k_blocks, u.kb0 + a.kb_per_split);
  return u;
}

// The units of CTA (pair) `id` of `stride`, round-robin: tiles, split-K windows, or
// (tile, k segment) pairs in segment-major order.
struct UnitIter {
  int t, stride;
  __device__ __forceinline__ UnitIter(const TcArgs&, int id, int stride_) : t(id), stride(stride_) {}
  __device__ __forceinline__ bool next(const TcArgs& a, int bn, int rank, Unit& u) {
    if (!a.sk) {
      if (t >= a.num_tiles * a.ksplit) return false;
      u = decode_unit(a, t, bn, rank);
      t += stride;
      return true;
    }
    if (t >= a.num_tiles * a.sk) return false;
    const int seg = t / a.num_tiles;
    u = decode_tile(a, t - seg * a.num_tiles, bn, rank);
    u.kb0 = seg * a.k_blocks / a.sk;
    u.kb1 = (seg + 1) * a.k_blocks / a.sk;
    u.sk_seg = seg;
    t += stride;
    return true;
  }
};
__device__ __forceinline__ void load8(const void* base, int dtype, long long off, float* out) {
  if (dtype == kF32) {
    const float4 x = *reinterpret_cast<const float4*>(static_cast<const float*>(base) + off);
    const float4 y = *reinterpret_cast<const float4*>(static_cast<const float*>(base) + off + 4);
    out[0] = x.x; out[1] = x.y; out[2] = x.z; out[3] = x.w;
    out[4] = y.x; out[5] = y.y; out[6] = y.z; out[7] = y.w;
  } else {
    const uint4 q = *reinterpret_cast<const uint4*>(static_cast<const __nv_bfloat16*>(base) + off);
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&q);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float2 f = __bfloat1622float2(h[i]);
      out[2 * i] = f.x;
      out[2 * i + 1] = f.y;
    }
  }
}

__device__ __forceinline__ void store8(void* base, int dtype, long long off, const float* v) {
  if (dtype == kF32) {
    float* p = static_cast<float*>(base) + off;
    *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
    *reinterpret_cast<float4*>(p + 4) = make_float4(v[4], v[5], v[6], v[7]);
  } else {
    uint4 pk;
    __nv_bfloat162 h0 = __floats2bfloat162_rn(v[0], v[1]);
    __nv_bfloat162 h1 = __floats2bfloat162_rn(v[2], v[3]);
    __nv_bfloat162 h2 = __floats2bfloat162_rn(v[4], v[5]);
    __nv_bfloat162 h3 = __floats2bfloat162_rn(v[6], v[7]);
    pk.x = *reinterpret_cast<uint32_t*>(&h0);
    pk.y = *reinterpret_cast<uint32_t*>(&h1);
    pk.z = *reinterpret_cast<uint32_t*>(&h2);
    pk.w = *reinterpret_cast<uint32_t*>(&h3);
    *reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(base) + off) = pk;
  }
}

// Applies the epilogue to one row segment of 32 columns (v[]) whose first element
// sits at output offset `off` (column n0).
__device__ __forceinline__ void epilogue_row32(const TcArgs& args, long long off, int n0,
                                               float (&v)[32]) {
  const Epilogue& e = args.epi;
  const int nvalid = min(32, args.N - n0);
  if (args.vec_ok && nvalid == 32) {
    if (e.alpha != 1.f) {
#pragma unroll
      for (int j = 0; j < 32; ++j) v[j] *= e.alpha;
    }
    if (e.bias != nullptr) {
#pragma unroll
      for (int j = 0; j < 32; j += 4) {
        const float4 bb = __ldg(reinterpret_cast<const float4*>(e.bias + n0 + j));
        v[j] += bb.x; v[j + 1] += bb.y; v[j + 2] += bb.z; v[j + 3] += bb.w;
      }
    }
    if (e.act == kActGeluSave) {
#pragma unroll
      for (int j = 0; j < 32; j += 8) {
        float gd[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) gelu_both(v[j + i], v[j + i], gd[i]);
        if (e.pre_act != nullptr) store8(e.pre_act, e.pre_dtype, off + j, gd);
      }
    } else if (e.pre_act != nullptr) {
#pragma unroll
      for (int j = 0; j < 32; j += 8) store8(e.pre_act, e.pre_dtype, off + j, v + j);
    }
    if (e.act == kActGelu) {
#pragma unroll
      for (int j = 0; j < 32; ++j) v[j] = gelu_f(v[j]);
    } else if (e.act == kActGeluGrad || e.act == kActMulAux || e.act == kActSoftmaxBwd) {
      const float rv = e.act == kActSoftmaxBwd ? e.alpha * e.rowvec[off / e.rv_div] : 0.f;
      float g[32];
#pragma unroll
      for (int j = 0; j < 32; j += 8) load8(e.aux, e.aux_dtype, off + j, g + j);
      if (e.act == kActMulAux) {
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] *= g[j];
      } else if (e.act == kActSoftmaxBwd) {
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = g[j] * (v[j] - rv);
      } else {
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] *= gelu_grad_f(g[j]);
      }
    }
    if (e.resid != nullptr) {
#pragma unroll
      for (int j = 0; j < 32; j += 8) {
        float r[8];
        load8(e.resid, e.resid_dtype, off + j, r);
#pragma unroll
        for (int i = 0; i < 8; ++i) v[j + i] += r[i];
      }
    }
    if (e.accumulate) {
#pragma unroll
      for (int j = 0; j < 32; j += 8) {
        float r[8];
        load8(e.out.base, e.out.dtype, off + j, r);
#pragma unroll
        for (int i = 0; i < 8; ++i) v[j + i] += r[i];
      }
    }
#pragma unroll
    for (int j = 0; j < 32; j += 8) store8(e.out.base, e.out.dtype, off + j, v + j);
  } else {
#pragma unroll
    for (int j = 0; j < 32; ++j)
      if (j < nvalid) epi_scalar(e, off + j, n0 + j, v[j]);
  }
}

// Element j (0..CW) of row `lane` of a swizzled [32][128 B] chunk buffer.
template <int CW>
__device__ __forceinline__ float smem_at(const uint8_t* xbuf, int lane, int j) {
  constexpr int VPC = CW == 32 ? 4 : 8;
  const uint8_t* p = xbuf + lane * 128 + (((j / VPC) ^ (lane & 7)) << 4);
  if (CW == 32) return reinterpret_cast<const float*>(p)[j % VPC];
  const uint16_t u = reinterpret_cast<const uint16_t*>(p)[j % VPC];
  return __uint_as_float(static_cast<uint32_t>(u) << 16);
}

// Epilogue math on 32 values of one output row starting at column n0 (half h of a CW-wide
// chunk); `off` is the element offset of (m, n0) (valid when row_ok). `xbuf`: the chunk's
// aux (x_tma 1) or residual (x_tma 2) values, TMA-loaded into shared memory. `rv`: the
// row's kActSoftmaxBwd value, alpha * rowvec[row]. A pre-activation output is written
// with direct 16-B stores (the staging buffer carries the main output only).
// Bias values of columns [n0, n0 + 32) (zero past N).
__device__ __forceinline__ void load_bias32(const float* bias, int n0, int N, int vec_ok,
                                            float (&bb)[32]) {
  if (n0 + 32 <= N && vec_ok) {
#pragma unroll
    for (int j = 0; j < 32; j += 4) {
      const float4 b4 = __ldg(reinterpret_cast<const float4*>(bias + n0 + j));
      bb[j] = b4.x; bb[j + 1] = b4.y; bb[j + 2] = b4.z; bb[j + 3] = b4.w;
    }
  } else {
#pragma unroll
    for (int j = 0; j < 32; ++j) bb[j] = n0 + j < N ? bias[n0 + j] : 0.f;
  }
}

template <int CW>
__device__ __forceinline__ void epi_math32(const TcArgs& args, long long off, int n0, float (&v)[32],
                                           bool row_ok, bool vec, uint8_t* xbuf, int lane,
                                           int h, float rv, bool applied = false) {
  const Epilogue& e = args.epi;
  const int nvalid = min(32, args.N - n0);
  // applied: v already holds alpha * acc + bias (and gelu of it for kActGeluSave), the
  // pre-activation value having been staged by epi_tile_tma
  if (e.alpha != 1.f && !applied) {
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] *= e.alpha;
  }
  if (e.bias != nullptr && !applied) {
    if (vec) {
#pragma unroll
      for (int j = 0; j < 32; j += 4) {
        const float4 bb = __ldg(reinterpret_cast<const float4*>(e.bias + n0 + j));
        v[j] += bb.x; v[j + 1] += bb.y; v[j + 2] += bb.z; v[j + 3] += bb.w;
      }
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j)
        if (j < nvalid) v[j] += e.bias[n0 + j];
    }
  }
  if (e.pre_act != nullptr && args.pre_tma) {
    // staged and stored by epi_tile_tma
  } else if (e.pre_act != nullptr && row_ok) {
    if (e.act == kActGeluSave) {
#pragma unroll
      for (int j = 0; j < 32; j += 8) {
        float gd[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) gelu_both(v[j + i], v[j + i], gd[i]);
        if (vec) {
          store8(e.pre_act, e.pre_dtype, off + j, gd);
        } else {
#pragma unroll
          for (int i = 0; i < 8; ++i)
            if (j + i < nvalid) st_any(e.pre_act, e.pre_dtype, off + j + i, gd[i]);
        }
      }
    } else if (vec) {
#pragma unroll
      for (int j = 0; j < 32; j += 8) store8(e.pre_act, e.pre_dtype, off + j, v + j);
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j)
        if (j < nvalid) st_any(e.pre_act, e.pre_dtype, off + j, v[j]);
    }
  } else if (e.act == kActGeluSave) {
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] = gelu_f(v[j]);
  }
  if (e.act == kActGelu) {
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] = gelu_f(v[j]);
  } else if ((e.act == kActGeluGrad || e.act == kActMulAux || e.act == kActSoftmaxBwd) && row_ok) {
    float g[32];
    if (args.x_tma == 1) {
#pragma unroll
      for (int j = 0; j < 32; ++j) g[j] = smem_at<CW>(xbuf, lane, 32 * h + j);
    } else if (vec) {
#pragma unroll
      for (int j = 0; j < 32; j += 8) load8(e.aux, e.aux_dtype, off + j, g + j);
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j) g[j] = j < nvalid ? ld_any(e.aux, e.aux_dtype, off + j) : 0.f;
    }
    if (e.act == kActMulAux) {
#pragma unroll
      for (int j = 0; j < 32; ++j) v[j] *= g[j];
    } else if (e.act == kActSoftmaxBwd) {
#pragma unroll
      for (int j = 0; j < 32; ++j) v[j] = g[j] * (v[j] - rv);
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j) v[j] *= gelu_grad_f(g[j]);
    }
  }
  if (e.resid != nullptr && row_ok) {
    if (args.x_tma == 2) {  // the residual chunk arrived by TMA into xbuf
#pragma unroll
      for (int j = 0; j < 32; ++j) v[j] += smem_at<CW>(xbuf, lane, 32 * h + j);
    } else if (vec) {
#pragma unroll
      for (int j = 0; j < 32; j += 8) {
        float r[8];
        load8(e.resid, e.resid_dtype, off + j, r);
#pragma unroll
        for (int i = 0; i < 8; ++i) v[j + i] += r[i];
      }
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j)
        if (j < nvalid) v[j] += ld_any(e.resid, e.resid_dtype, off + j);
    }
  }
  if (e.accumulate && row_ok) {
#pragma unroll
    for (int j = 0; j < 32; ++j)
      if (j < nvalid) v[j] += ld_any(e.out.base, e.out.dtype, off + j);
  }
}

// Stream-K fix-up of a finishing segment: the other segments' fp32 partial rows (this
// lane's row, the warp's column base) in k order; `self` is this segment's position.
struct SkFix {
  int n = -1;                   // segments - 1
  int self = 0;                 // this segment's position
  const float* base = nullptr;  // the tile's segment 0 partial (+ rank / lane / column offset)
  size_t seg_stride = 0;        // elements between consecutive segments' partials
  __device__ __forceinline__ const float* part(const TcArgs&, int q) const {
    return base + static_cast<size_t>(q) * seg_stride;
  }
};

// Replaces this warp's accumulator columns in TMEM by the sum of all segments of the
// split tile, in k order (this segment's accumulator at its position): the regular
// epilogue then runs unchanged.
template <int COLS>
__device__ __forceinline__ void sk_fixup(const TcArgs& a, const SkFix& fx, uint32_t row_taddr) {
#pragma unroll 1
  for (int c = 0; c < COLS / 32; ++c) {
    float v[32];
    ptx::tmem_ld32(row_taddr + 32 * c, v);
#pragma unroll
    for (int j0 = 0; j0 < 32; j0 += 8) {
      float t8[8];
#pragma unroll 1
      for (int q = 0; q <= fx.n; ++q) {
        float pv[8];
        if (q == fx.self) {
#pragma unroll
          for (int i = 0; i < 8; ++i) pv[i] = v[j0 + i];
        } else {
          const float* src = fx.part(a, q) + (32 * c + j0) * kBM;  // column-major partial
#pragma unroll
          for (int i = 0; i < 8; ++i) pv[i] = __ldcg(src + i * kBM);
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) t8[i] = q == 0 ? pv[i] : t8[i] + pv[i];
      }
#pragma unroll
      for (int i = 0; i < 8; ++i) v[j0 + i] = t8[i];
    }
    ptx::tmem_st32(row_taddr + 32 * c, v);
  }
}

template <int CW, int COLS>
__device__ __forceinline__ void epi_tile_tma(const TcArgs& args, const CUtensorMap* tmC,
                                             const CUtensorMap* tmX, uint8_t* buf, uint8_t* xbuf,
                                             uint64_t* xbar, uint32_t& xph, int lane,
                                             uint32_t row_taddr, int ncol0, long long row_off,
                                             bool row_ok, int c1, int c2r, int c3, int c4) {
  const Epilogue& e = args.epi;
  constexpr int VPC = CW == 32 ? 4 : 8;  // values per 16-B staging chunk
  // per-row softmax-backward value (contiguous rows: row = offset / row length)
  const float rv = (e.act == kActSoftmaxBwd && row_ok && args.ksplit == 1)
                       ? e.alpha * __ldg(e.rowvec + row_off / e.rv_div)
                       : 0.f;
  auto coords = [&](int n, int& c0, int& c2) {
    c0 = args.st_csplit ? n % args.st_csplit : n;
    c2 = c2r + (args.st_csplit ? n / args.st_csplit : 0);
  };
  // the first chunk's operand load overlaps the first TMEM read
  if (args.x_tma && ncol0 < args.N && lane == 0) {
    int c0, c2;
    coords(ncol0, c0, c2);
    ptx::mbar_arrive_expect_tx(xbar, 4096);
    ptx::tma_load_5d(xbuf, tmX, xbar, c0, c1, c2, c3, c4);
  }
#pragma unroll 1
  for (int cc = 0; cc < COLS / CW; ++cc) {
    const int n = ncol0 + cc * CW;
    const bool live = n < args.N;  // warp-uniform
    const long long off =
        row_off + (e.out.csplit ? (n % e.out.csplit) + (n / e.out.csplit) * e.out.s_hi : n);
    const bool vec = live && args.ksplit == 1 && row_ok && args.vec_ok && n + CW <= args.N;
    if (args.pre_tma && live && args.ksplit == 1) {
      // one pass: alpha * acc + bias, the pre-activation value (gelu'(x) for kActGeluSave)
      // staged in xbuf, the output in buf, two TMA stores
      staging_acquire(lane);
#pragma unroll
      for (int h = 0; h < CW / 32; ++h) {
        float v[32], pre[32];
        const int nh = n + 32 * h;
        ptx::tmem_ld32(row_taddr + cc * CW + 32 * h, v);
        if (e.alpha != 1.f) {
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] *= e.alpha;
        }
        if (e.bias != nullptr) {
          float bb[32];
          load_bias32(e.bias, nh, args.N, args.vec_ok, bb);
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] += bb[j];
        }
        if (e.act == kActGeluSave) {
#pragma unroll
          for (int j = 0; j < 32; j += 2) {
            float2 g2, d2;
            gelu_both2(make_float2(v[j], v[j + 1]), g2, d2);
            v[j] = g2.x;
            v[j + 1] = g2.y;
            pre[j] = d2.x;
            pre[j + 1] = d2.y;
          }
        } else {
#pragma unroll
          for (int j = 0; j < 32; ++j) pre[j] = v[j];
        }
#pragma unroll
        for (int q = 0; q < 32 / VPC; ++q)
          stage_chunk<CW>(xbuf, lane, h * (32 / VPC) + q, pre + VPC * q);
        epi_math32<CW>(args, off + 32 * h, nh, v, row_ok, vec, xbuf, lane, h, rv, true);
#pragma unroll
        for (int q = 0; q < 32 / VPC; ++q) stage_chunk<CW>(buf, lane, h * (32 / VPC) + q, v + VPC * q);
      }
      int c0, c2;
      coords(n, c0, c2);
      store_staged(tmX, xbuf, lane, c0, c1, c2, c3, c4);
      store_staged(tmC, buf, lane, c0, c1, c2, c3, c4);
      continue;
    }
    staging_acquire(lane);
    if (args.x_tma && live) {
      ptx::mbar_wait(xbar, xph);
      xph ^= 1;
    }
#pragma unroll
    for (int h = 0; h < CW / 32; ++h) {
      float v[32];
      ptx::tmem_ld32(row_taddr + cc * CW + 32 * h, v);
      if (live && args.ksplit == 1)
        epi_math32<CW>(args, off + 32 * h, n + 32 * h, v, row_ok, vec, xbuf, lane, h, rv);
#pragma unroll
      for (int q = 0; q < 32 / VPC; ++q) stage_chunk<CW>(buf, lane, h * (32 / VPC) + q, v + VPC * q);
    }
    if (!live) continue;
    // every lane has read the operand chunk: fetch the next one during this store
    __syncwarp();
    const int nn = n + CW;
    if (args.x_tma && cc + 1 < COLS / CW && nn < args.N && lane == 0) {
      int c0n, c2n;
      coords(nn, c0n, c2n);
      ptx::mbar_arrive_expect_tx(xbar, 4096);
      ptx::tma_load_5d(xbuf, tmX, xbar, c0n, c1, c2n, c3, c4);
    }
    int c0, c2;
    coords(n, c0, c2);
    store_staged(tmC, buf, lane, c0, c1, c2, c3, c4);
  }
}

// CG = 2: a CTA pair (cluster of 2) computes a 256 x BN tile with tcgen05.mma.cta_group::2:
// each CTA stages its 128 rows of A and its BN/2 rows of B (half the operand bytes per SM),
// the leader's single thread issues the M = 256 MMAs and commits to both CTAs' barriers,
// and each CTA's epilogue drains its own 128 TMEM lanes.
template <int BN, bool A_MN, bool B_MN, int CG = 1>
__global__ void __launch_bounds__(kThreads, 1)
    tc_gemm_kernel(const __grid_constant__ CUtensorMap tmA,
                   const __grid_constant__ CUtensorMap tmB,
                   const __grid_constant__ CUtensorMap tmC,
                   const __grid_constant__ CUtensorMap tmP, const TcArgs args,
                   const __grid_constant__ RsMaps rsm) {
  constexpr int kABytes = kBM * kBK * 2;  // 16 KB
  constexpr int kBRows = BN / CG;         // B rows staged by this CTA
  constexpr int kBBytes = kBRows * kBK * 2;
  constexpr int kStageBytes = kABytes + kBBytes;
  constexpr uint32_t kTmemCols = 2 * BN < 32 ? 32 : 2 * BN;
  constexpr uint32_t kIdesc = ptx::idesc_bf16_f32(kBM * CG, BN, A_MN, B_MN);
  const int rank = CG == 2 ? static_cast<int>(ptx::cluster_rank()) : 0;
  const int cta_id = blockIdx.x / CG, cta_stride = gridDim.x / CG;
  constexpr int kColsPerWarp = BN / 2;  // two epilogue warps per lane quarter

  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  const int S = args.stages;
  uint8_t* smem_a = smem;
  uint8_t* smem_b = smem + S * kABytes;
  uint8_t* smem_stage = smem + S * kStageBytes;  // 8 epilogue warps x 4 KB, 1024-aligned
  uint8_t* smem_x = smem_stage + kEpiWarps * 4096;  // operand chunks (x_tma)
  const int staging = args.tma_store ? kEpiWarps * 4096 * ((args.x_tma || args.pre_tma) ? 2 : 1) : 0;
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + S * kStageBytes + staging);
  uint64_t* empty_bar = full_bar + S;
  uint64_t* tfull_bar = empty_bar + S;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint64_t* x_bar = tempty_bar + 2;  // one per epilogue warp
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(x_bar + kEpiWarps);
  uint32_t* sk_last = tmem_slot + 1;  // stream-K: this CTA finishes the current split tile

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const int units = args.num_tiles * args.ksplit;

  if (warp == 0 && lane == 0) {
    ptx::prefetch_tmap(&tmA);
    ptx::prefetch_tmap(&tmB);
    for (int s = 0; s < S; ++s) {
      ptx::mbar_init(&full_bar[s], 1);
      ptx::mbar_init(&empty_bar[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      ptx::mbar_init(&tfull_bar[s], 1);
      ptx::mbar_init(&tempty_bar[s], kEpiWarps * CG);  // both CTAs' epilogues (leader's)
    }
    for (int w = 0; w < kEpiWarps; ++w) ptx::mbar_init(&x_bar[w], 1);
    ptx::fence_barrier_init();
  }
  if (warp == 1) {
    if (CG == 2) ptx::tmem_alloc_pair<kTmemCols>(tmem_slot);
    else ptx::tmem_alloc<kTmemCols>(tmem_slot);
  }
  ptx::tc_fence_before();
  if (CG == 2) ptx::cluster_sync();  // the peer's barriers exist before any remote arrive
  else __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer
      int s = 0;
      uint32_t ph = 0;
      OpPos pa, pb;
      const uint32_t full_leader = CG == 2 ? ptx::mapa(ptx::smem_u32(full_bar), 0) : 0u;
      UnitIter ui(args, cta_id, cta_stride);
      Unit u;
      while (ui.next(args, BN, rank, u)) {
        op_init(args.a, pa, u.m0, A_MN ? kBM / 64 : 1, u.kb0 * kBK, u.b);
        op_init(args.b, pb, u.n0 + rank * kBRows, B_MN ? kBRows / 64 : 1, u.kb0 * kBK, u.b);
        for (int kb = u.kb0; kb < u.kb1; ++kb) {
          ptx::mbar_wait(&empty_bar[s], ph ^ 1);
          if (CG == 2) {
            // the leader expects both CTAs' bytes; the peer's loads only complete_tx on the
            // leader's barrier (a remote release-arrive would cost a membar per stage)
            const uint32_t fb = full_leader + s * 8;
            if (rank == 0) ptx::mbar_arrive_expect_tx(&full_bar[s], 2 * kStageBytes);
            op_issue_pair<kBM>(&tmA, args.a, pa, smem_a + s * kABytes, fb);
            op_issue_pair<kBRows>(&tmB, args.b, pb, smem_b + s * kBBytes, fb);
          } else {
            ptx::mbar_arrive_expect_tx(&full_bar[s], kStageBytes);
            op_issue<kBM>(&tmA, args.a, pa, smem_a + s * kABytes, &full_bar[s]);
            op_issue<BN>(&tmB, args.b, pb, smem_b + s * kBBytes, &full_bar[s]);
          }
          op_advance(args.a, pa);
          op_advance(args.b, pb);
          if (++s == S) {
            s = 0;
            ph ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && rank == 0) {
      // ---------------- UMMA issuer (the pair's leader for CG = 2)
      int s = 0;
      uint32_t ph = 0;
      int acc = 0;
      uint32_t aph = 0;
      const uint32_t a0 = ptx::smem_u32(smem_a), b0 = ptx::smem_u32(smem_b);
      UnitIter ui(args, cta_id, cta_stride);
      Unit u;
      while (ui.next(args, BN, 0, u)) {
        ptx::mbar_wait(&tempty_bar[acc], aph ^ 1);
        ptx::tc_fence_after();
        const uint32_t tmem_d = tmem_base + acc * BN;
        for (int kb = u.kb0; kb < u.kb1; ++kb) {
          ptx::mbar_wait(&full_bar[s], ph);
          ptx::tc_fence_after();
          const uint32_t a_addr = a0 + s * kABytes;
          const uint32_t b_addr = b0 + s * kBBytes;
#pragma unroll
          for (int k = 0; k < kBK / 16; ++k) {
            const uint64_t ad = A_MN ? ptx::smem_desc_sw128(a_addr + k * 2048, 8192, 1024)
                                     : ptx::smem_desc_sw128(a_addr + k * 32, 16, 1024);
            const uint64_t bd = B_MN ? ptx::smem_desc_sw128(b_addr + k * 2048, 8192, 1024)
                                     : ptx::smem_desc_sw128(b_addr + k * 32, 16, 1024);
            if (CG == 2) ptx::umma_bf16_pair(tmem_d, ad, bd, kIdesc, (kb > u.kb0 || k > 0) ? 1u : 0u);
            else ptx::umma_bf16(tmem_d, ad, bd, kIdesc, (kb > u.kb0 || k > 0) ? 1u : 0u);
          }
          if (CG == 2) ptx::umma_commit_pair(&empty_bar[s], 3);
          else ptx::umma_commit(&empty_bar[s]);
          if (++s == S) {
            s = 0;
            ph ^= 1;
          }
        }
        if (CG == 2) ptx::umma_commit_pair(&tfull_bar[acc], 3);
        else ptx::umma_commit(&tfull_bar[acc]);
        if (++acc == 2) {
          acc = 0;
          aph ^= 1;
        }
      }
    }
  } else {
    // ---------------- epilogue warps 2..9: lane quarter = warp % 4, column half = (warp-2)/4
    const int quarter = warp & 3;
    const int half = (warp - 2) >> 2;
    int acc = 0;
    uint32_t aph = 0;
    const Epilogue& e = args.epi;
    if (args.tma_store) {
      uint8_t* buf = smem_stage + (warp - 2) * 4096;
      uint8_t* xbuf = smem_x + (warp - 2) * 4096;
      uint64_t* xbar = &x_bar[warp - 2];
      uint32_t xph = 0;
      const bool need_off = args.ksplit == 1 && (e.aux != nullptr || e.resid != nullptr ||
                                                 e.accumulate || e.rowvec != nullptr ||
                                                 e.pre_act != nullptr);
      const uint32_t epoch = args.rs_P ? *args.rs_epoch : 0u;
      uint32_t entered_mask = 0;
      UnitIter ui(args, cta_id, cta_stride);
      Unit u;
      while (ui.next(args, BN, rank, u)) {
        const int mrow0 = u.m0 + quarter * 32;
        const int m = mrow0 + lane;
        const bool row_ok = m < args.M;
        const long long row_off = (need_off && row_ok) ? view_offset(e.out, u.b, m, 0) : 0;
        const int bidx = args.ksplit > 1 ? u.ks : u.b;
        const int c3 = bidx % args.st_blo, c4 = bidx / args.st_blo;
        int c1 = args.st_rsplit ? mrow0 % args.st_rsplit : mrow0;
        const int c2r = args.st_rsplit ? mrow0 / args.st_rsplit : 0;
        const CUtensorMap* cmap = &tmC;
        if (args.rs_P) {
          // whole tiles per block (block_rows % 128 == 0): pick the block's map
          const int kr = u.m0 / args.rs_block_rows;
          const int k = args.rs_block0 + kr;
          c1 = mrow0 - kr * args.rs_block_rows;
          cmap = &rsm.m[k];
          if (k != args.rs_me && !(entered_mask & (1u << k))) {
            if (lane == 0) ptx::wait_epoch(args.rs_entered[k], epoch, args.rs_fault, 0x600u | k);
            __syncwarp();
            entered_mask |= 1u << k;
          }
        }
        ptx::mbar_wait(&tfull_bar[acc], aph);
        ptx::tc_fence_after();
        const uint32_t row_taddr = tmem_base + acc * BN +
                                   (static_cast<uint32_t>(quarter * 32) << 16) + half * kColsPerWarp;
        const int ncol0 = u.n0 + half * kColsPerWarp;
        SkFix fx;
        bool finish = true;
        if (u.sk_seg >= 0) {
          // a k segment of a split tile: the last of its segments to arrive finishes it
          // partials are column-major per CTA tile ([BN][128]): for each column a warp's 32
          // rows are 128 contiguous bytes, so every store / load is one coalesced line
          const size_t lane_off = static_cast<size_t>(half * kColsPerWarp) * kBM + quarter * 32 + lane;
          const size_t slot_elems = static_cast<size_t>(kBM) * BN;
          const int S = args.sk;
          if (threadIdx.x == 64) {
            const uint32_t prev = atomicAdd(&args.sk_count[u.tile * 2 + rank], 1u);
            *sk_last = prev + 1 == static_cast<uint32_t>(S) ? 1u : 0u;
          }
          ptx::named_bar(1, 32 * kEpiWarps);
          finish = *sk_last != 0;
          ptx::named_bar(1, 32 * kEpiWarps);
          const size_t slot0 = static_cast<size_t>(u.tile) * S;
          if (!finish) {
            // raw fp32 partial into the segment's slot, then raise its flag
            float* w = args.sk_ws + ((slot0 + u.sk_seg) * 2 + rank) * slot_elems + lane_off;
#pragma unroll 1
            for (int c = 0; c < kColsPerWarp / 32; ++c) {
              float v[32];
              ptx::tmem_ld32(row_taddr + 32 * c, v);
#pragma unroll
              for (int j = 0; j < 32; ++j) __stcg(w + (32 * c + j) * kBM, v[j]);
            }
            __threadfence();
            ptx::named_bar(1, 32 * kEpiWarps);
            if (threadIdx.x == 64)
              ptx::st_release_gpu(&args.sk_flag[(slot0 + u.sk_seg) * 2 + rank], 1u);
          } else {
            // the other segments' partials (their flags: they have arrived, may still be
            // writing), summed with this one in k order
            if (lane == 0)
              for (int q = 0; q < S; ++q) {
                if (q == u.sk_seg) continue;
                while (ptx::ld_acquire_gpu(&args.sk_flag[(slot0 + q) * 2 + rank]) == 0) {
                }
              }
            __syncwarp();
            fx.n = S - 1;
            fx.self = u.sk_seg;
            fx.base = args.sk_ws + (slot0 * 2 + rank) * slot_elems + lane_off;
            fx.seg_stride = 2 * slot_elems;
            sk_fixup<kColsPerWarp>(args, fx, row_taddr);
          }
        }
        if (finish) {
          if (args.cw == 32)
            epi_tile_tma<32, kColsPerWarp>(args, cmap, &tmP, buf, xbuf, xbar, xph, lane, row_taddr,
                                           ncol0, row_off, row_ok, c1, c2r, c3, c4);
          else
            epi_tile_tma<(kColsPerWarp >= 64 ? 64 : 32), kColsPerWarp>(
                args, cmap, &tmP, buf, xbuf, xbar, xph, lane, row_taddr, ncol0, row_off, row_ok, c1,
                c2r, c3, c4);
        }
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if (CG == 2) ptx::mbar_arrive_cluster(ptx::mapa(ptx::smem_u32(&tempty_bar[acc]), 0));
          else ptx::mbar_arrive(&tempty_bar[acc]);
        }
        if (++acc == 2) {
          acc = 0;
          aph ^= 1;
        }
      }
      if (lane == 0) {
        ptx::bulk_wait_all();
        if (args.rs_P) {
          // this warp's peer-bound tile stores are complete: order them before the
          // done flag raised below (system scope: the reader is another GPU)
          ptx::fence_proxy_async_global();
          __threadfence_system();
        }
      }
    } else
    for (int t = cta_id; t < units; t += cta_stride) {  // (no stream-K without TMA stores)
      const Unit u = decode_unit(args, t, BN, rank);
      const int m = u.m0 + quarter * 32 + lane;
      // row offset once per unit (the only divisions on the epilogue path)
      long long row_off = 0;
      if (args.ksplit > 1) row_off = (static_cast<long long>(u.ks) * args.M + m) * args.N;
      else if (m < args.M) row_off = view_offset(e.out, u.b, m, 0);
      ptx::mbar_wait(&tfull_bar[acc], aph);
      ptx::tc_fence_after();
      const uint32_t row_taddr =
          tmem_base + acc * BN + (static_cast<uint32_t>(quarter * 32) << 16) + half * kColsPerWarp;
#pragma unroll 1
      for (int c = 0; c < kColsPerWarp / 32; ++c) {
        float v[32];
        ptx::tmem_ld32(row_taddr + c * 32, v);
        const int nc = u.n0 + half * kColsPerWarp + c * 32;
        if (m < args.M && nc < args.N) {
          if (args.ksplit > 1) {
            float* p = args.ws + row_off + nc;
            const int nvalid = min(32, args.N - nc);
            if (nvalid == 32 && args.vec_ok) {
#pragma unroll
              for (int j = 0; j < 32; j += 8) store8(p, kF32, j, v + j);
            } else {
#pragma unroll
              for (int j = 0; j < 32; ++j)
                if (j < nvalid) p[j] = v[j];
            }
          } else {
            long long off = row_off + nc;
            if (e.out.csplit) off = row_off + (nc % e.out.csplit) + (nc / e.out.csplit) * e.out.s_hi;
            epilogue_row32(args, off, nc, v);
          }
        }
      }
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (CG == 2) ptx::mbar_arrive_cluster(ptx::mapa(ptx::smem_u32(&tempty_bar[acc]), 0));
        else ptx::mbar_arrive(&tempty_bar[acc]);
      }
      if (++acc == 2) {
        acc = 0;
        aph ^= 1;
      }
    }
  }

  ptx::tc_fence_before();
  if (CG == 2) ptx::cluster_sync();  // no remote arrive or multicast commit still in flight
  else __syncthreads();
  if (warp == 1) {
    ptx::tc_fence_after();
    if (CG == 2) ptx::tmem_dealloc_pair<kTmemCols>(tmem_base);
    else ptx::tmem_dealloc<kTmemCols>(tmem_base);
  }
  if (args.rs_P && threadIdx.x == 0) {
    const uint32_t epoch = *args.rs_epoch;
    __threadfence_system();
    for (int k = 0; k < args.rs_P; ++k)
      if (k != args.rs_me)
        ptx::st_release_sys(args.rs_done[k] + args.rs_done_offset + blockIdx.x, epoch);
  }
}

// Split-K reduction, plain epilogue into a contiguous output: 4 columns per thread, all
// splits' loads in flight (the weight-gradient case).
__global__ void splitk_reduce4_kernel(const float* ws, int ksplit, long long total4, void* out,
                                      int out_dtype) {
  for (long long t = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; t < total4;
       t += static_cast<long long>(gridDim.x) * blockDim.x) {
    float4 acc = __ldcs(reinterpret_cast<const float4*>(ws) + t);
    for (int k = 1; k < ksplit; ++k) {
      const float4 x = __ldcs(reinterpret_cast<const float4*>(ws) + k * total4 + t);
      acc.x += x.x; acc.y += x.y; acc.z += x.z; acc.w += x.w;
    }
    if (out_dtype == kF32) {
      reinterpret_cast<float4*>(out)[t] = acc;
    } else {
      __nv_bfloat162 lo = __floats2bfloat162_rn(acc.x, acc.y), hi = __floats2bfloat162_rn(acc.z, acc.w);
      uint2 u;
      u.x = *reinterpret_cast<uint32_t*>(&lo);
      u.y = *reinterpret_cast<uint32_t*>(&hi);
      reinterpret_cast<uint2*>(out)[t] = u;
    }
  }
}

// Split-K reduction: out = epilogue(sum_k ws[k][m][n]) in ascending split order.
__global__ void splitk_reduce_kernel(const float* ws, int ksplit, int M, int N, Epilogue e) {
  const long long total = static_cast<long long>(M) * N;
  for (long long t = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; t < total;
       t += static_cast<long long>(gridDim.x) * blockDim.x) {
    float acc = 0.f;
    for (int k = 0; k < ksplit; ++k) acc += ws[k * total + t];
    const long long m = t / N, n = t - (t / N) * N;
    epi_scalar(e, view_offset(e.out, 0, m, n), n, acc);
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

// Output store map: 5-D view of the stored tensor (cols, rows, split-hi, batch-lo,
// batch-hi), box [32 rows][128 B], 128B swizzle. Returns false when the view is not
// TMA-addressable (the kernel then stores directly from registers).
bool make_store_map(const View& v, long long rows, long long cols, int batch, int cw,
                    CUtensorMap* map, int box_rows = 32) {
  const long long es = v.dtype == kF32 ? 4 : 2;
  if (v.sc != 1 || reinterpret_cast<uintptr_t>(v.base) % 16) return false;
  if (v.rsplit && v.csplit) return false;
  if (v.rsplit && v.rsplit % box_rows) return false;
  if (v.csplit && v.csplit % cw) return false;
  for (long long s : {v.sr, v.s_hi, v.sb_lo, v.sb_hi})
    if ((s * es) % 16) return false;
  const long long rlo = v.rsplit ? v.rsplit : rows;
  const long long clo = v.csplit ? v.csplit : cols;
  const long long nhi = v.rsplit ? (rows + v.rsplit - 1) / v.rsplit
                                 : (v.csplit ? (cols + v.csplit - 1) / v.csplit : 1);
  const long long bhi = (batch + v.b_lo_n - 1) / v.b_lo_n;
  cuuint64_t dims[5] = {static_cast<cuuint64_t>(clo), static_cast<cuuint64_t>(rlo),
                        static_cast<cuuint64_t>(nhi), static_cast<cuuint64_t>(v.b_lo_n),
                        static_cast<cuuint64_t>(bhi)};
  const long long fb = std::max<long long>(16, v.sr * es * rlo);
  cuuint64_t strides[4] = {static_cast<cuuint64_t>(v.sr * es),
                           static_cast<cuuint64_t>(v.s_hi ? v.s_hi * es : fb),
                           static_cast<cuuint64_t>(v.sb_lo ? v.sb_lo * es : fb),
                           static_cast<cuuint64_t>(v.sb_hi ? v.sb_hi * es : fb)};
  if (rows == 1 || rlo == 1) strides[0] = std::max<cuuint64_t>(strides[0], 16);
  cuuint32_t box[5] = {static_cast<cuuint32_t>(cw), static_cast<cuuint32_t>(box_rows), 1, 1, 1};
  cuuint32_t estr[5] = {1, 1, 1, 1, 1};
  std::memset(map, 0, sizeof(*map));
  const CUresult r = encode_fn()(
      map, v.dtype == kF32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5,
      v.base, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
      CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

template <int BN, bool A_MN, bool B_MN, int CG = 1>
void launch_tc(const CUtensorMap& ma, const CUtensorMap& mb, const CUtensorMap& mc,
               const CUtensorMap& mp, TcArgs& args, const RsMaps& rsm, int num_sms,
               cudaStream_t stream) {
  constexpr int kStageBytes = (kBM + BN / CG) * kBK * 2;
  const int staging = args.tma_store ? kEpiWarps * 4096 * ((args.x_tma || args.pre_tma) ? 2 : 1) : 0;
  int stages = (kSmemBudget - 1024 - 256 - staging) / kStageBytes;
  stages = std::min(stages, 8);
  args.stages = stages;
  const int smem = 1024 + stages * kStageBytes + staging + (2 * stages + 4 + kEpiWarps) * 8 + 16;
  auto kern = tc_gemm_kernel<BN, A_MN, B_MN, CG>;
  static bool attr_set = false;  // per instantiation
  if (!attr_set) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBudget);
    if (CG == 2) cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 0);
    attr_set = true;
  }
  const int units = args.num_tiles * args.ksplit;
  if (CG == 1) {
    const int grid = std::min(units, num_sms);
    kern<<<grid, kThreads, smem, stream>>>(ma, mb, mc, mp, args, rsm);
    return;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = static_cast<size_t>(smem);
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  // A persistent grid must be co-resident: the GPCs' SM counts need not be even, so the
  // number of resident pairs can be below num_sms / 2 (a second wave would double the time).
  static int max_pairs = 0;  // per instantiation (smem is fixed per instantiation)
  if (max_pairs == 0) {
    cfg.gridDim = dim3(static_cast<unsigned>(num_sms & ~1));
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, kern, &cfg) != cudaSuccess || n <= 0) {
      (void)cudaGetLastError();
      n = num_sms / 2;
    }
    max_pairs = std::min(n, num_sms / 2);
    if (std::getenv("C3D_GEMM_VERBOSE"))
      std::fprintf(stderr, "tc_gemm pair kernel: %d resident pairs\n", max_pairs);
  }
  char* skbuf = nullptr;
  if (args.sk) {
    const size_t ws = static_cast<size_t>(args.num_tiles) * args.sk * 2 * kBM * BN * sizeof(float);
    const size_t flags = static_cast<size_t>(args.num_tiles) * args.sk * 2 * sizeof(uint32_t);
    const size_t counts = static_cast<size_t>(args.num_tiles) * 2 * sizeof(uint32_t);
    C3D_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&skbuf), ws + flags + counts, stream));
    C3D_CUDA(cudaMemsetAsync(skbuf + ws, 0, flags + counts, stream));
    args.sk_ws = reinterpret_cast<float*>(skbuf);
    args.sk_flag = reinterpret_cast<uint32_t*>(skbuf + ws);
    args.sk_count = reinterpret_cast<uint32_t*>(skbuf + ws + flags);
    cfg.gridDim = dim3(static_cast<unsigned>(2 * std::min(args.num_tiles * args.sk, max_pairs)));
  } else if (args.rs_P) {
    // fused reduce-scatter: the grid must be the one tc_gemm_grid reported (done flags);
    // its CTAs wait only on other GPUs, never on each other, so co-residency is not needed
    cfg.gridDim = dim3(static_cast<unsigned>(2 * std::min(units, num_sms / 2)));
  } else {
    cfg.gridDim = dim3(static_cast<unsigned>(2 * std::min(units, max_pairs)));
  }
  C3D_CUDA(cudaLaunchKernelEx(&cfg, kern, ma, mb, mc, mp, args, rsm));
  if (skbuf) C3D_CUDA(cudaFreeAsync(skbuf, stream));
}

template <int BN>
void launch_bn(const CUtensorMap& ma, const CUtensorMap& mb, const CUtensorMap& mc,
               const CUtensorMap& mp, TcArgs& args, const RsMaps& rsm, int num_sms,
               cudaStream_t stream) {
  const bool am = args.a.mn_major, bm = args.b.mn_major;
  if constexpr (BN == 256) {
    if (args.cg == 2) {
    if (!am && !bm) launch_tc<BN, false, false, 2>(ma, mb, mc, mp, args, rsm, num_sms, stream);
    else if (!am && bm) launch_tc<BN, false, true, 2>(ma, mb, mc, mp, args, rsm, num_sms, stream);
    else if (am && !bm) launch_tc<BN, true, false, 2>(ma, mb, mc, mp, args, rsm, num_sms, stream);
    else launch_tc<BN, true, true, 2>(ma, mb, mc, mp, args, rsm, num_sms, stream);
    return;
    }
  }
  if (!am && !bm) launch_tc<BN, false, false>(ma, mb, mc, mp, args, rsm, num_sms, stream);
  else if (!am && bm) launch_tc<BN, false, true>(ma, mb, mc, mp, args, rsm, num_sms, stream);
  else if (am && !bm) launch_tc<BN, true, false>(ma, mb, mc, mp, args, rsm, num_sms, stream);
  else launch_tc<BN, true, true>(ma, mb, mc, mp, args, rsm, num_sms, stream);
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
  return true;
}

// Picks the number of K splits for a batch-1 problem with few output tiles: only
// when fewer than half the SMs would get a tile, maximising wave efficiency
// (units / (waves * SMs)) with >= 16 K-blocks per split (measured on B200: splitting
// a 128-tile GEMM loses to the extra partial-sum traffic; a 32-tile one gains 2x).
int pick_ksplit(long long M, long long N, int tiles, int k_blocks, int batch, int num_sms, int bn) {
  (void)M;
  (void)N;
  (void)bn;
  if (const char* env = std::getenv("C3D_KSPLIT")) {  // experiments only
    const int ks = std::atoi(env);
    if (ks >= 1 && batch == 1) return std::min(ks, std::max(1, k_blocks / 4));
  }
  // measured: with >= num_sms / 2 tiles the partial-sum traffic costs more than the
  // idle SMs (e.g. 96 tiles of 1024 x 3072 x 16384: 112 us unsplit, 118 us at 3 splits)
  if (batch != 1 || 2 * tiles > num_sms) return 1;
  int best = 1;
  double best_eff = static_cast<double>(tiles) / num_sms;
  for (int ks = 2; ks <= 8; ++ks) {
    if (k_blocks / ks < 16) break;
    const int units = tiles * ks;
    const int waves = (units + num_sms - 1) / num_sms;
    const double eff = static_cast<double>(units) / (waves * num_sms) - 0.01 * ks;
    if (eff > best_eff + 0.02) {
      best_eff = eff;
      best = ks;
    }
  }
  return best;
}

}  // namespace

CUtensorMap tc_operand_map(const View& v, long long rows, long long cols, int batch, int box_rows,
                           int* mn_major) {
  TcOperand op;
  CUtensorMap m = make_operand_map(v, rows, cols, batch, box_rows, &op);
  if (mn_major) *mn_major = op.mn_major;
  return m;
}

bool tc_store_map(const View& v, long long rows, long long cols, int batch, int box_cols,
                  int box_rows, CUtensorMap* map) {
  return make_store_map(v, rows, cols, batch, box_cols, map, box_rows);
}

int tc_pick_bn(long long M, long long N, int batch, int num_sms) {
  if (const char* e = std::getenv("C3D_BN")) {  // experiments only
    const int bn = std::atoi(e);
    if (bn == 64 || bn == 128 || bn == 256) return bn;
  }
  if (N <= 64) return 64;
  if (N <= 128) return 128;
  // 256-wide tiles whenever N allows: measured on B200 they beat 128-wide tiles by
  // ~1.4x per tile, more than any wave-quantisation loss at these sizes
  (void)M;
  (void)batch;
  (void)num_sms;
  return N % 256 == 0 ? 256 : 128;
}

bool tc_gemm_rs_supported(const GemmProblem& p, int bn) {
  const RsOut& r = p.rs;
  if (r.P < 2 || r.P > kRsMax || p.batch != 1) return false;
  if (r.block_rows <= 0 || r.block_rows % kBM || p.M % r.block_rows) return false;
  if (r.block0 < 0 || r.block0 + p.M / r.block_rows > r.P) return false;
  const int cw = p.epi.out.dtype == kF32 ? 32 : 64;
  if (cw > bn / 2 || std::getenv("C3D_NO_TMA_STORE")) return false;
  const Epilogue& e = p.epi;
  if (e.bias || e.act != kActNone || e.pre_act || e.resid || e.accumulate || e.alpha != 1.f)
    return false;
  for (int k = r.block0; k < r.block0 + p.M / r.block_rows; ++k) {
    View v;
    v.base = r.dst[k];
    v.dtype = e.out.dtype;
    v.sr = p.N;
    CUtensorMap m;
    if (!make_store_map(v, r.block_rows, p.N, 1, cw, &m)) return false;
  }
  return true;
}

// CTA pairs for 256-wide tiles (the decision tc_gemm_launch takes for unsplit products).
static bool use_pairs(const GemmProblem& p, int bn, int ksplit) {
  // with a fused reduce-scatter every CTA's 128 rows must fall inside the blocks
  return bn == 256 && ksplit == 1 && !std::getenv("C3D_NO_CG2") && (p.M + kBM - 1) / kBM >= 2 &&
         (p.rs.P <= 1 || p.M % (2 * kBM) == 0);
}

int tc_gemm_grid(const GemmProblem& p, int bn, int num_sms) {
  // the fused reduce-scatter (ksplit 1) sizes its done flags by this grid
  if (use_pairs(p, bn, 1)) {
    const long long ptiles = ((p.M + 2 * kBM - 1) / (2 * kBM)) * ((p.N + bn - 1) / bn) * p.batch;
    return static_cast<int>(2 * std::min<long long>(ptiles, num_sms / 2));
  }
  const long long tiles = ((p.M + kBM - 1) / kBM) * ((p.N + bn - 1) / bn) * p.batch;
  return static_cast<int>(std::min<long long>(tiles, num_sms));
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
  args.cg = 1;
  args.m_tiles = static_cast<int>((p.M + kBM - 1) / kBM);
  args.n_tiles = static_cast<int>((p.N + bn - 1) / bn);
  args.k_blocks = static_cast<int>((p.K + kBK - 1) / kBK);
  args.num_tiles = args.m_tiles * args.n_tiles * p.batch;
  // bands of 16 tile rows once the B operand outgrows a comfortable share of L2
  args.group_m = (p.N * p.K * 2 > (48ll << 20)) ? std::min(16, args.m_tiles) : 1;
  if (const char* e = std::getenv("C3D_GROUP_M")) args.group_m = std::max(1, std::min(std::atoi(e), args.m_tiles));
  // stream-K on CTA pairs when 256 x 256 pair tiles leave a poor last wave and K is long
  // (the weight-gradient products: 48 tiles of 1024 x 3072 x 16384 on 74 pairs)
  int sk = 0;
  if (bn == 256 && p.rs.P <= 1 && p.batch == 1 && !p.epi.pre_act && args.m_tiles >= 2 &&
      !std::getenv("C3D_NO_SK") && !std::getenv("C3D_NO_CG2")) {
    // segments per tile: the best wave fill, each extra segment charged 3% (its fp32
    // partial round trip), and only for a clear gain. Measured on B200: a segment must keep
    // >= 64 k-blocks of main loop, or its partial / fix-up epilogue outweighs the better
    // wave fill (1024 x 3072 x 16384 in 3 segments: 99.8 us vs 102.8; 16384 x 1024 x 4096
    // in 2: 137.6 vs 104.9); tile counts that suit single-CTA split-K keep that path
    // (1024 x 1024 x 16384: 53.7 us split-K vs 60.9 in 4 segments)
    const int pairs = num_sms / 2;
    const int ptiles = static_cast<int>((p.M + 2 * kBM - 1) / (2 * kBM)) * args.n_tiles;
    auto eff = [&](int S) {
      const int units = ptiles * S;
      const int waves = (units + pairs - 1) / pairs;
      return static_cast<double>(units) / (static_cast<double>(waves) * pairs) - 0.03 * (S - 1);
    };
    double best = eff(1);
    const bool splitk = pick_ksplit(p.M, p.N, args.num_tiles, args.k_blocks, p.batch, num_sms, bn) > 1;
    for (int S = 2; S <= 8 && args.k_blocks / S >= 64 && !splitk; ++S)
      if (eff(S) > best + 0.15) {
        best = eff(S);
        sk = S;
      }
    if (const char* e = std::getenv("C3D_SK")) sk = std::max(0, std::atoi(e));  // experiments
  }
  args.ksplit = (p.rs.P > 1 || sk) ? 1
                                    : pick_ksplit(p.M, p.N, args.num_tiles, args.k_blocks, p.batch,
                                                  num_sms, bn);
  args.kb_per_split = (args.k_blocks + args.ksplit - 1) / args.ksplit;
  args.ksplit = (args.k_blocks + args.kb_per_split - 1) / args.kb_per_split;
  // CTA pairs (cta_group::2, 256 x 256 tiles) for plain 256-wide tiles
  if (use_pairs(p, bn, args.ksplit)) {
    args.cg = 2;
    args.m_tiles = static_cast<int>((p.M + 2 * kBM - 1) / (2 * kBM));
    args.num_tiles = args.m_tiles * args.n_tiles * p.batch;
    args.group_m = std::min(args.group_m, args.m_tiles);
    args.sk = sk > 1 ? sk : 0;
  }
  args.epi = p.epi;
  // vector loads/stores need 16-B aligned rows and 32-column chunks
  const int esz = p.epi.out.dtype == kF32 ? 4 : 2;
  auto al = [](const void* q) { return reinterpret_cast<uintptr_t>(q) % 16 == 0; };
  bool vec = al(p.epi.out.base) && (p.epi.out.sr * esz) % 16 == 0 &&
             (p.epi.out.s_hi * esz) % 16 == 0 && (p.epi.out.sb_lo * esz) % 16 == 0 &&
             (p.epi.out.sb_hi * esz) % 16 == 0 && (p.epi.out.csplit % 32) == 0;
  const int sizes[3] = {p.epi.pre_dtype == kF32 ? 4 : 2, p.epi.aux_dtype == kF32 ? 4 : 2,
                        p.epi.resid_dtype == kF32 ? 4 : 2};
  const void* ptrs[3] = {p.epi.pre_act, p.epi.aux, p.epi.resid};
  for (int i = 0; i < 3; ++i)
    if (ptrs[i]) vec = vec && al(ptrs[i]) && (p.epi.out.sr * sizes[i]) % 16 == 0;
  if (p.epi.bias) vec = vec && al(p.epi.bias);
  if (args.ksplit > 1) vec = vec && (p.N % 4 == 0);
  args.vec_ok = vec ? 1 : 0;
  CUtensorMap ma = make_operand_map(p.a, p.M, p.K, p.batch, kBM, &args.a);
  CUtensorMap mb = make_operand_map(p.b, p.N, p.K, p.batch, bn / args.cg, &args.b);
  float* ws = nullptr;
  if (args.ksplit > 1) {
    C3D_CUDA(cudaMallocAsync(&ws, sizeof(float) * args.ksplit * p.M * p.N, stream));
    args.ws = ws;
  }
  // TMA-store epilogue when the stored view (output, or the split-K workspace) and the
  // optional pre-activation output are TMA-addressable.
  CUtensorMap mc, mp;
  std::memset(&mc, 0, sizeof(mc));
  std::memset(&mp, 0, sizeof(mp));
  View sv = p.epi.out;
  int sbatch = p.batch;
  if (args.ksplit > 1) {
    sv = View();
    sv.base = ws;
    sv.dtype = kF32;
    sv.sr = p.N;
    sv.sb_lo = p.M * p.N;
    sv.b_lo_n = args.ksplit;
    sbatch = args.ksplit;
  }
  args.cw = sv.dtype == kF32 ? 32 : 64;
  bool tma = !std::getenv("C3D_NO_TMA_STORE") && args.cw <= bn / 2 &&
             make_store_map(sv, p.M, p.N, sbatch, args.cw, &mc);
  // epilogue operand (aux or residual, same layout as the output) by TMA when the output
  // goes out by TMA; the pre-activation output is written directly
  if (tma && args.ksplit == 1 && !std::getenv("C3D_NO_X_TMA")) {
    View xv = p.epi.out;
    if (p.epi.pre_act && p.epi.pre_dtype == p.epi.out.dtype) {
      xv.base = p.epi.pre_act;
      if (make_store_map(xv, p.M, p.N, p.batch, args.cw, &mp)) args.pre_tma = 1;
    } else if (p.epi.aux && p.epi.aux_dtype == p.epi.out.dtype) {
      xv.base = const_cast<void*>(p.epi.aux);
      if (make_store_map(xv, p.M, p.N, p.batch, args.cw, &mp)) args.x_tma = 1;
    } else if (p.epi.resid && !p.epi.aux && p.epi.resid_dtype == p.epi.out.dtype &&
               args.k_blocks <= 16) {
      // short K: the residual read dominates the epilogue, worth a pipeline stage of smem
      xv.base = const_cast<void*>(p.epi.resid);
      if (make_store_map(xv, p.M, p.N, p.batch, args.cw, &mp)) args.x_tma = 2;
    }
  }
  RsMaps rsm;
  std::memset(&rsm, 0, sizeof(rsm));
  if (p.rs.P > 1) {
    if (!tc_gemm_rs_supported(p, bn)) throw std::runtime_error("tc_gemm: fused reduce-scatter unsupported");
    for (int k = 0; k < p.rs.P; ++k) {
      args.rs_entered[k] = p.rs.entered[k];
      args.rs_fault = p.rs.fault;
      args.rs_done[k] = p.rs.done[k];
      if (k < p.rs.block0 || k >= p.rs.block0 + p.M / p.rs.block_rows) continue;
      View v;
      v.base = p.rs.dst[k];
      v.dtype = p.epi.out.dtype;
      v.sr = p.N;
      make_store_map(v, p.rs.block_rows, p.N, 1, args.cw, &rsm.m[k]);
    }
    mc = rsm.m[p.rs.block0];
    tma = true;
    args.rs_P = p.rs.P;
    args.rs_me = p.rs.me;
    args.rs_block_rows = static_cast<int>(p.rs.block_rows);
    args.rs_block0 = p.rs.block0;
    args.rs_done_offset = p.rs.done_offset;
    args.rs_epoch = p.rs.epoch;
    sv = View();
  }
  args.tma_store = tma ? 1 : 0;
  if (!tma) args.sk = 0;  // the split-tile fix-up lives in the TMA-store epilogue
  args.st_rsplit = static_cast<int>(sv.rsplit);
  args.st_csplit = static_cast<int>(sv.csplit);
  args.st_blo = sv.b_lo_n;
  switch (bn) {
    case 64: launch_bn<64>(ma, mb, mc, mp, args, rsm, num_sms, stream); break;
    case 128: launch_bn<128>(ma, mb, mc, mp, args, rsm, num_sms, stream); break;
    case 256: launch_bn<256>(ma, mb, mc, mp, args, rsm, num_sms, stream); break;
    default: throw std::runtime_error("tc_gemm: unsupported BN");
  }
  if (args.ksplit > 1) {
    check_launch("tc_gemm(split-k)");
    const long long total = p.M * p.N;
    const int blocks = static_cast<int>(std::min<long long>((total + 255) / 256, 148LL * 8));
    const Epilogue& e = p.epi;
    const bool plain = !e.bias && e.act == kActNone && !e.pre_act && !e.aux && !e.resid &&
                       !e.accumulate && e.alpha == 1.f && !e.rowvec;
    const bool contig = e.out.sr == p.N && e.out.sc == 1 && !e.out.rsplit && !e.out.csplit &&
                        p.batch == 1 && p.N % 4 == 0 &&
                        reinterpret_cast<uintptr_t>(e.out.base) % 16 == 0;
    if (plain && contig) {
      const long long total4 = total / 4;
      const int b4 = static_cast<int>(std::min<long long>((total4 + 255) / 256, 148LL * 8));
      splitk_reduce4_kernel<<<b4, 256, 0, stream>>>(ws, args.ksplit, total4, e.out.base,
                                                    e.out.dtype);
    } else {
      splitk_reduce_kernel<<<blocks, 256, 0, stream>>>(ws, args.ksplit, args.M, args.N, p.epi);
    }
    C3D_CUDA(cudaFreeAsync(ws, stream));
  }
}

}  // namespace c3d
