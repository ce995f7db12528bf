// Local GEMM interface shared by the tcgen05 kernel, the SIMT fp32 kernel and
// the host dispatcher.
//
// Every local product of the reference (`multiply_accumulate`,
// cube3d/matrix.hpp:68-92, in its NN / NT / TN forms) becomes one call of
//
//     C[b][m][n] (op)= epilogue( alpha * sum_k A[b][m][k] * B[b][n][k] )
//
// where A and B are *views*: strided, optionally batched, optionally split
// logical matrices over device memory. The split lets one operand span the p
// buffers an all-gather produced (`gather_cols`, cube3d/ops3d.hpp:55-67) or a
// row block stack (`gather_rows`, :48-53) without a reorder copy: the split
// coordinate becomes a TMA dimension.
#pragma once

#include <cstdint>

#include "ptx_fault.hpp"

namespace c3d {

enum DType : int { kF32 = 0, kBF16 = 1 };

// Logical X[b][r][c] at
//   base + (b % b_lo_n)*sb_lo + (b / b_lo_n)*sb_hi + R(r) + C(c)
// with R(r) = (r % rsplit)*sr + (r / rsplit)*s_hi if rsplit else r*sr, and C
// likewise with csplit. At most one of rsplit/csplit is non-zero. Strides are
// in elements. For GEMM operands r is the M (or N) index and c the K index.
struct View {
  void* base = nullptr;
  int dtype = kBF16;
  long long sr = 0, sc = 1;
  long long s_hi = 0;
  long long rsplit = 0, csplit = 0;
  long long sb_lo = 0, sb_hi = 0;
  int b_lo_n = 1;
};

__host__ __device__ inline long long view_offset(const View& v, long long b, long long r,
                                                 long long c) {
  long long off = (b % v.b_lo_n) * v.sb_lo + (b / v.b_lo_n) * v.sb_hi;
  if (v.rsplit) off += (r % v.rsplit) * v.sr + (r / v.rsplit) * v.s_hi;
  else off += r * v.sr;
  if (v.csplit) off += (c % v.csplit) * v.sc + (c / v.csplit) * v.s_hi;
  else off += c * v.sc;
  return off;
}

// kActGeluSave: gelu, and the pre-activation output receives gelu'(x) instead of x (the
//   backward then only multiplies: kActMulAux).
// kActSoftmaxBwd: v = aux * (v - alpha * rowvec[off / rv_div]) (softmax backward with the
//   row dot product precomputed; alpha already applied to v).
enum ActKind : int {
  kActNone = 0,
  kActGelu = 1,
  kActGeluGrad = 2,
  kActGeluSave = 3,
  kActMulAux = 4,
  kActSoftmaxBwd = 5
};

// Fused epilogue, applied per output element in this order:
//   v = alpha*acc; v += bias[n]; pre = v (stored if pre_act);
//   v = gelu(v) | v * gelu'(aux[m][n]) | v;  v += resid[m][n];
//   v += C_old[m][n] (if accumulate); C = v.
// `out`, `pre_act`, `aux` and `resid` share the output addressing (base pointer and
// dtype of their own, strides from `out`).
struct Epilogue {
  View out;
  float alpha = 1.f;
  const float* bias = nullptr;
  int act = kActNone;
  void* pre_act = nullptr;
  int pre_dtype = kBF16;
  const void* aux = nullptr;
  int aux_dtype = kBF16;
  const void* resid = nullptr;
  int resid_dtype = kBF16;
  int accumulate = 0;
  const float* rowvec = nullptr;  // kActSoftmaxBwd
  long long rv_div = 1;
};

// Reduce-scatter fused into the tcgen05 GEMM epilogue: C's rows form P blocks of
// block_rows; block k is TMA-stored to dst[k] ([block_rows][N] row-major), which for
// k != me is this rank's slot in rank k's symmetric receive buffer over NVLink. Before
// its first store to block k a CTA waits for k's entry flag; after its last store it
// raises done[k][blockIdx.x] to the epoch (release, system scope).
constexpr int kRsMax = 4;
struct RsOut {
  int P = 0;  // 0: plain GEMM
  int me = 0;
  int block0 = 0;       // block index of the GEMM's first row (row-split launches)
  int done_offset = 0;  // first done-flag slot of this launch
  long long block_rows = 0;
  void* dst[kRsMax] = {};
  const uint32_t* entered[kRsMax] = {};
  uint32_t* done[kRsMax] = {};
  const uint32_t* epoch = nullptr;
  Fault fault;  // where a peer that never enters is reported
};

struct GemmProblem {
  long long M = 0, N = 0, K = 0;
  int batch = 1;
  View a, b;  // a: [batch][M][K], b: [batch][N][K]
  Epilogue epi;
  RsOut rs;
};

}  // namespace c3d
