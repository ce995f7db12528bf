// Chooses the tcgen05 or SIMT kernel for one local product, and (when enabled)
// brackets every tcgen05 launch with CUDA events on its stream so bench.py can
// report the dominant kernel's achieved TFLOP/s from the live run.
#include <cstdio>
#include <cstdlib>
#include <cstdint>
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
  double flops;  // GEMM flops, or collective payload bytes
  int kind;      // 0 = tcgen05 GEMM, 1 = collective
  int tag;       // collective kind (C3D_BROADCAST ...)
  long long M, N, K;
  int batch, bn, amn, bmn, outdt;
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

// Inside stream capture an event must be recorded as an external event node to stay
// a real (timed) event in the graph.
void record(cudaEvent_t e, cudaStream_t s) {
  cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
  C3D_CUDA(cudaStreamIsCapturing(s, &st));
  if (st == cudaStreamCaptureStatusActive)
    C3D_CUDA(cudaEventRecordWithFlags(e, s, cudaEventRecordExternal));
  else
    C3D_CUDA(cudaEventRecord(e, s));
}

}  // namespace

void prof_enable(bool on) {
  std::lock_guard<std::mutex> g(prof().mu);
  prof().enabled = on;
  prof().recs.clear();
  prof().next = 0;
}

namespace {
// Sums the records of one kind and drops them (the event pool is recycled once the log
// is empty). C3D_PROF_DUMP prints every collective record.
void read_kind(int kind, double* ms, double* amount, long long* count) {
  Profiler& pr = prof();
  std::lock_guard<std::mutex> g(pr.mu);
  static const bool dump = std::getenv("C3D_PROF_DUMP") != nullptr;
  double t = 0, f = 0;
  long long n = 0;
  std::vector<ProfRec> rest;
  for (auto& r : pr.recs) {
    if (r.kind != kind) {
      rest.push_back(r);
      continue;
    }
    float x = 0;
    if (cudaEventSynchronize(r.stop) != cudaSuccess ||
        cudaEventElapsedTime(&x, r.start, r.stop) != cudaSuccess) {
      cudaGetLastError();
      continue;  // unreadable (e.g. never replayed): dropped
    }
    if (dump && kind == 1)
      std::fprintf(stderr, "[c3d prof] coll kind=%d bytes=%.0f us=%.1f GB/s=%.1f\n", r.tag, r.flops,
                   1e3 * x, x > 0 ? r.flops / (x * 1e6) : 0.0);
    if (dump && kind == 0)
      std::fprintf(stderr,
                   "[c3d prof] gemm M=%lld N=%lld K=%lld batch=%d bn=%d a_mn=%d b_mn=%d out=%s "
                   "us=%.1f TF/s=%.1f\n",
                   r.M, r.N, r.K, r.batch, r.bn, r.amn, r.bmn, r.outdt == kF32 ? "f32" : "bf16",
                   1e3 * x, x > 0 ? r.flops / (x * 1e9) : 0.0);
    if (kind == 1 && r.tag >= 5) continue;  // fused-operator spans: dumped, not summed
    t += x;
    f += r.flops;
    ++n;
  }
  *ms = t;
  *amount = f;
  *count = n;
  pr.recs.swap(rest);
  if (pr.recs.empty()) pr.next = 0;
}
}  // namespace

// Returns (sum of per-launch ms, sum of flops, launches) of the tcgen05 GEMMs.
void prof_read(double* ms, double* flops, long long* launches) {
  read_kind(0, ms, flops, launches);
}

// Returns (sum of per-call ms, sum of payload bytes, calls) of the collectives.
void prof_read_comm(double* ms, double* bytes, long long* calls) {
  read_kind(1, ms, bytes, calls);
}

bool prof_on() { return prof().enabled; }

void prof_begin(cudaStream_t s, void** token) {
  Profiler& pr = prof();
  std::lock_guard<std::mutex> g(pr.mu);
  cudaEvent_t e = pr.take();
  record(e, s);
  *token = e;
}

void prof_end(cudaStream_t s, void* token, int tag, double bytes) {
  Profiler& pr = prof();
  std::lock_guard<std::mutex> g(pr.mu);
  ProfRec rec{};
  rec.start = static_cast<cudaEvent_t>(token);
  rec.stop = pr.take();
  rec.flops = bytes;
  rec.kind = 1;
  rec.tag = tag;
  record(rec.stop, s);
  pr.recs.push_back(rec);
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
        rec.kind = 0;
        rec.M = p.M;
        rec.N = p.N;
        rec.K = p.K;
        rec.batch = p.batch;
        rec.bn = bn;
        rec.amn = p.a.sr == 1 && p.a.sc != 1;
        rec.bmn = p.b.sr == 1 && p.b.sc != 1;
        rec.outdt = p.epi.out.dtype;
        record(rec.start, s);
      }
      tc_gemm_launch(p, bn, num_sms, s);
      check_launch("tc_gemm");
      if (on) {
        std::lock_guard<std::mutex> g(pr.mu);
        record(rec.stop, s);
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
