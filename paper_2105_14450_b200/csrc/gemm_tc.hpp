#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include "gemm.hpp"

namespace c3d {

// tcgen05 path (bf16 operands, fp32 accumulate). `tc_gemm_supported` checks the
// TMA constraints (16-B aligned bases and strides, split sizes that tiles do not
// straddle); callers fall back to the SIMT kernel otherwise.
int tc_pick_bn(long long M, long long N, int batch, int num_sms);
bool tc_gemm_supported(const GemmProblem& p, int bn);
void tc_gemm_launch(const GemmProblem& p, int bn, int num_sms, cudaStream_t stream);
// Fused reduce-scatter epilogue (p.rs.P > 1): supported when every destination block
// is TMA-storable with whole tiles; `tc_gemm_grid` is the CTA count (one done flag each).
bool tc_gemm_rs_supported(const GemmProblem& p, int bn);
int tc_gemm_grid(const GemmProblem& p, int bn, int num_sms);

// TMA maps for the other tcgen05 kernels (flash.cu): a 5-D operand map (box
// 64 K-columns x box_rows rows, 128B swizzle; MN-major views get 64 x 64 boxes) and a
// store/load map with an explicit box (128B swizzle).
CUtensorMap tc_operand_map(const View& v, long long rows, long long cols, int batch, int box_rows,
                           int* mn_major);
bool tc_store_map(const View& v, long long rows, long long cols, int batch, int box_cols,
                  int box_rows, CUtensorMap* map);

// SIMT fp32 path: any view, fp32 or bf16 operands, fp32 FMA in ascending k.
void simt_gemm_launch(const GemmProblem& p, cudaStream_t stream);

}  // namespace c3d
