// Chooses the tcgen05 or SIMT kernel for one local product, and (when enabled)
// brackets every tcgen05 launch with CUDA events on its stream so bench.py can
// report the dominant kernel's achieved TFLOP/s from the live run.
#include <mutex>
#include <string>
#include <vector>

#include "common.hpp"
#include "gemm_tc.hpp"
#include "ops.hpp"

namespace c3d {

namespace {

struct ProfRec {
  cudaEvent_t start, stop;
  double flops;
};

struct Profiler {
  std::mutex mu;
  bool enabled = false;
  std::vector<cudaEvent_t> pool;
  size_t next = 0;
  std::vector<ProfRec> recs;

  cudaEvent_t take() {
    if (next == pool.size()) {
      cudaEvent_t e;
      C3D_CUDA(cudaEventCreate(&e));
      pool.push_back(e);
    }
    return pool[next++];
  }
};

Profiler& prof() {
  static Profiler p;
  return p;
}

}  // namespace

void prof_enable(bool on) {
  std::lock_guard<std::mutex> g(prof().mu);
  prof().enabled = on;
  prof().recs.clear();
  prof().next = 0;
}

// Returns (sum of per-launch ms, sum of flops, launches) and resets the log.
void prof_read(double* ms, double* flops, long long* launches) {
  std::lock_guard<std::mutex> g(prof().mu);
  double t = 0, f = 0;
  for (auto& r : prof().recs) {
    C3D_CUDA(cudaEventSynchronize(r.stop));
    float x = 0;
    C3D_CUDA(cudaEventElapsedTime(&x, r.start, r.stop));
    t += x;
    f += r.flops;
  }
  *ms = t;
  *flops = f;
  *launches = static_cast<long long>(prof().recs.size());
  prof().recs.clear();
  prof().next = 0;
}

void run_gemm(const GemmProblem& p, int mode, int num_sms, cudaStream_t s) {
  if (p.M == 0 || p.N == 0 || p.batch == 0) return;
  const bool bf16_ops = p.a.dtype == kBF16 && p.b.dtype == kBF16;
  if (mode != C3D_MODE_F32 && bf16_ops && p.K > 0) {
    const int bn = tc_pick_bn(p.M, p.N, p.batch, num_sms);
    if (tc_gemm_supported(p, bn)) {
      Profiler& pr = prof();
      ProfRec rec{};
      const bool on = pr.enabled;
      if (on) {
        std::lock_guard<std::mutex> g(pr.mu);
        rec.start = pr.take();
        rec.stop = pr.take();
        rec.flops = 2.0 * p.M * p.N * p.K * p.batch;
        C3D_CUDA(cudaEventRecord(rec.start, s));
      }
      tc_gemm_launch(p, bn, num_sms, s);
      check_launch("tc_gemm");
      if (on) {
        std::lock_guard<std::mutex> g(pr.mu);
        C3D_CUDA(cudaEventRecord(rec.stop, s));
        pr.recs.push_back(rec);
      }
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
