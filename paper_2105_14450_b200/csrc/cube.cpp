#include "cube.hpp"

#include <cstdint>
#include <cstdio>
#include <cstdlib>

namespace c3d {

size_t dtype_size(int dtype) { return dtype == kF32 ? 4 : 2; }

namespace {

ncclDataType_t nccl_type(int dtype) { return dtype == kF32 ? ncclFloat32 : ncclBfloat16; }

void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess)
    fail(C3D_ERR_NCCL, std::string(what) + ": " + ncclGetErrorString(r));
}

// Brackets one collective with profiler events when profiling is on. `bytes` is the
// full (gathered / pre-scatter) payload.
struct Timed {
  cudaStream_t s;
  void* tok = nullptr;
  int tag;
  double bytes;
  Timed(cudaStream_t st, int kind, double b) : s(st), tag(kind), bytes(b) {
    if (prof_on()) prof_begin(s, &tok);
  }
  ~Timed() {
    if (tok) prof_end(s, tok, tag, bytes);
  }
};

}  // namespace

Cube::Cube(const int dims[3], int rank, int device, const unsigned char* uid)
    : grid_(dims), rank_(rank), device_(device) {
  coords_ = grid_.coords_of(rank);
  C3D_CUDA(cudaSetDevice(device));
  C3D_CUDA(cudaDeviceGetAttribute(&num_sms_, cudaDevAttrMultiProcessorCount, device));
  // Keep pooled scratch resident: collectives and kernels reuse it every step.
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
    uint64_t threshold = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &threshold);
  }
  if (grid_.size() > 1) {
    if (uid == nullptr) fail(C3D_ERR_CONFIG_INVALID, "multi-rank grid needs an NCCL unique id");
    ncclUniqueId id;
    std::memcpy(&id, uid, sizeof(id));
    nccl_check(ncclCommInitRank(&world_, grid_.size(), id, rank), "ncclCommInitRank");
    for (int a = 0; a < 3; ++a) {
      if (grid_.dims[a] == 1) continue;  // uniform across ranks: all skip together
      const int color = grid_.line_index(coords_, a);
      nccl_check(ncclCommSplit(world_, color, coords_[a], &axis_comm_[a], nullptr),
                 "ncclCommSplit");
    }
    if (std::getenv("C3D_NCCL_COLL") == nullptr) {
      const char* mb = std::getenv("C3D_MAILBOX_MB");
      const size_t bytes = static_cast<size_t>(mb ? std::atol(mb) : 256) << 20;
      const char* ab = std::getenv("C3D_ARENA_MB");
      const size_t arena = static_cast<size_t>(ab ? std::atol(ab) : 512) << 20;
      symm_ = std::make_unique<SymmHeap>(world_, grid_.size(), rank, bytes, arena, nullptr);
    }
  }
  for (int a = 0; a < 3; ++a) line_[a] = grid_.axis_group(coords_, a);
}

Cube::~Cube() {
  symm_.reset();
  for (auto& c : axis_comm_)
    if (c) ncclCommDestroy(c);
  if (world_) ncclCommDestroy(world_);
}

void Cube::check_fault() {
  if (poisoned_.empty() && symm_) poisoned_ = symm_->fault_message();
  if (!poisoned_.empty()) fail(C3D_ERR_DESYNC, "rank " + std::to_string(rank_) + ": " + poisoned_);
}

ncclComm_t Cube::comm(int axis) const {
  if (axis < 0 || axis > 2 || !axis_comm_[axis])
    fail(C3D_ERR_INTERNAL, "no communicator for axis " + std::to_string(axis));
  return axis_comm_[axis];
}

namespace {
bool trace_on() {
  static const bool on = std::getenv("C3D_TRACE") != nullptr;
  return on;
}
}  // namespace

void Cube::charge(int kind, uint64_t sent, uint64_t received) {
  if (trace_on()) {
    static const char* names[] = {"broadcast", "all_gather", "reduce_scatter", "all_reduce",
                                  "barrier"};
    std::fprintf(stderr, "[c3d rank %d] #%llu %s sent=%llu recv=%llu\n", rank_,
                 static_cast<unsigned long long>(counters_.calls_by_kind[0] +
                                                 counters_.calls_by_kind[1] +
                                                 counters_.calls_by_kind[2] +
                                                 counters_.calls_by_kind[3]),
                 names[kind], static_cast<unsigned long long>(sent),
                 static_cast<unsigned long long>(received));
    std::fflush(stderr);
  }
  counters_.elements_sent += sent;
  counters_.elements_received += received;
  counters_.sent_by_kind[kind] += sent;
  counters_.received_by_kind[kind] += received;
  counters_.calls_by_kind[kind] += 1;
}

void Cube::all_gather(int axis, const void* send, void* recv, size_t count, int dtype,
                      cudaStream_t s) {
  const int p = extent(axis);
  if (p == 1) {
    if (send != recv)
      C3D_CUDA(cudaMemcpyAsync(recv, send, count * dtype_size(dtype), cudaMemcpyDeviceToDevice, s));
    return;
  }
  Timed t(s, C3D_ALL_GATHER, static_cast<double>(p) * count * dtype_size(dtype));
  if (symm_)
    symm_->collective(kCollAllGather, line_[axis], coords_[axis], send, recv, count, dtype, 0,
                      false, num_sms_, s);
  else
    nccl_check(ncclAllGather(send, recv, count, nccl_type(dtype), comm(axis), s), "ncclAllGather");
  charge(C3D_ALL_GATHER, static_cast<uint64_t>(p - 1) * count, static_cast<uint64_t>(p - 1) * count);
}

void Cube::all_gather_sym(int axis, const void* send, const SymBuf& recv, size_t count, int dtype,
                          cudaStream_t s) {
  const int p = extent(axis);
  if (p == 1 || !symm_) fail(C3D_ERR_INTERNAL, "all_gather_sym needs the peer transport");
  Timed t(s, C3D_ALL_GATHER, static_cast<double>(p) * count * dtype_size(dtype));
  symm_->all_gather_direct(line_[axis], coords_[axis], send, recv.offset(), count, dtype, num_sms_,
                           s);
  charge(C3D_ALL_GATHER, static_cast<uint64_t>(p - 1) * count, static_cast<uint64_t>(p - 1) * count);
}

void Cube::reduce_scatter(int axis, const void* send, void* recv, size_t count, int dtype,
                          cudaStream_t s) {
  const int p = extent(axis);
  if (p == 1) {
    if (send != recv)
      C3D_CUDA(cudaMemcpyAsync(recv, send, count * dtype_size(dtype), cudaMemcpyDeviceToDevice, s));
    return;
  }
  Timed t(s, C3D_REDUCE_SCATTER, static_cast<double>(p) * count * dtype_size(dtype));
  if (symm_)
    symm_->collective(kCollReduceScatter, line_[axis], coords_[axis], send, recv, count, dtype, 0,
                      false, num_sms_, s);
  else
    nccl_check(ncclReduceScatter(send, recv, count, nccl_type(dtype), ncclSum, comm(axis), s),
               "ncclReduceScatter");
  charge(C3D_REDUCE_SCATTER, static_cast<uint64_t>(p - 1) * count,
         static_cast<uint64_t>(p - 1) * count);
}

void Cube::all_reduce(int axis, void* buf, size_t count, int dtype, bool is_max, cudaStream_t s) {
  const int p = extent(axis);
  if (p == 1) return;
  Timed t(s, C3D_ALL_REDUCE, static_cast<double>(count) * dtype_size(dtype));
  if (symm_)
    symm_->collective(kCollAllReduce, line_[axis], coords_[axis], buf, buf, count, dtype, 0,
                      is_max, num_sms_, s);
  else
    nccl_check(ncclAllReduce(buf, buf, count, nccl_type(dtype), is_max ? ncclMax : ncclSum,
                             comm(axis), s),
               "ncclAllReduce");
  charge(C3D_ALL_REDUCE, static_cast<uint64_t>(p - 1) * count, static_cast<uint64_t>(p - 1) * count);
}

void Cube::broadcast(int axis, int root_position, void* buf, size_t count, int dtype,
                     cudaStream_t s) {
  const int p = extent(axis);
  if (root_position < 0 || root_position >= p)
    fail(C3D_ERR_OUT_OF_RANGE, "broadcast root position " + std::to_string(root_position));
  if (p == 1) return;
  Timed t(s, C3D_BROADCAST, static_cast<double>(count) * dtype_size(dtype));
  if (symm_)
    symm_->collective(kCollBroadcast, line_[axis], coords_[axis], buf, buf, count, dtype,
                      root_position, false, num_sms_, s);
  else
    nccl_check(ncclBroadcast(buf, buf, count, nccl_type(dtype), root_position, comm(axis), s),
               "ncclBroadcast");
  if (coords_[axis] == root_position)
    charge(C3D_BROADCAST, static_cast<uint64_t>(p - 1) * count, 0);
  else
    charge(C3D_BROADCAST, 0, count);
}

void Cube::barrier(cudaStream_t s) {
  if (grid_.size() == 1) return;
  // A zero-payload all-reduce over the world communicator orders all ranks.
  DevBuf one(sizeof(float), s);
  C3D_CUDA(cudaMemsetAsync(one.get(), 0, sizeof(float), s));
  nccl_check(ncclAllReduce(one.get(), one.get(), 1, ncclFloat32, ncclSum, world_, s),
             "ncclAllReduce(barrier)");
  counters_.calls_by_kind[C3D_BARRIER] += 1;
}

}  // namespace c3d
