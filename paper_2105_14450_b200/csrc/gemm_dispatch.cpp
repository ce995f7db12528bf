// Chooses the tcgen05 or SIMT kernel for one local product.
#include <string>

#include "common.hpp"
#include "gemm_tc.hpp"
#include "ops.hpp"

namespace c3d {

void run_gemm(const GemmProblem& p, int mode, int num_sms, cudaStream_t s) {
  if (p.M == 0 || p.N == 0 || p.batch == 0) return;
  const bool bf16_ops = p.a.dtype == kBF16 && p.b.dtype == kBF16;
  if (mode != C3D_MODE_F32 && bf16_ops && p.K > 0) {
    const int bn = tc_pick_bn(p.M, p.N, p.batch, num_sms);
    if (tc_gemm_supported(p, bn)) {
      tc_gemm_launch(p, bn, num_sms, s);
      check_launch("tc_gemm");
      return;
    }
    if (mode == C3D_MODE_TC)
      fail(C3D_ERR_SHAPE_MISMATCH,
           "operands are not TMA-addressable for the tcgen05 path (M=" + std::to_string(p.M) +
               " N=" + std::to_string(p.N) + " K=" + std::to_string(p.K) + ")");
  } else if (mode == C3D_MODE_TC) {
    fail(C3D_ERR_SHAPE_MISMATCH, "tcgen05 mode needs bf16 operands");
  }
  simt_gemm_launch(p, s);
  check_launch("simt_gemm");
}

}  // namespace c3d
