#pragma once

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

// SIMT fp32 path: any view, fp32 or bf16 operands, fp32 FMA in ascending k.
void simt_gemm_launch(const GemmProblem& p, cudaStream_t stream);

}  // namespace c3d
