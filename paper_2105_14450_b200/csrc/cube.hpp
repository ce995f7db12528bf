// One rank's handle on the processor grid: topology, NCCL communicators over
// NVLink, traffic counters and stream-ordered device scratch.
//
// Replaces the reference's in-process Transport/Endpoint (cube3d/transport.hpp:
// 89-398): the per-axis rendezvous slots become one NCCL communicator per axis
// line (ncclCommSplit of the world communicator, color = line index, key = the
// axis coordinate, so NCCL rank order is the reference's ascending group
// position). Every collective charges CostCounters exactly as
// Endpoint::{broadcast, all_gather, reduce_scatter, all_reduce} do
// (cube3d/transport.hpp:160-257; convention cube3d/counters.hpp:32-36).
#pragma once

#include <cuda_runtime.h>
#include <nccl.h>

#include <array>
#include <cstddef>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "common.hpp"
#include "gemm.hpp"
#include "grid.hpp"
#include "symm.hpp"

namespace c3d {

size_t dtype_size(int dtype);

// Event brackets for collectives (profiler in gemm_dispatch.cpp; no-ops when disabled).
bool prof_on();
void prof_begin(cudaStream_t s, void** token);
void prof_end(cudaStream_t s, void* token, int tag, double bytes);

// Stream-ordered scratch buffer (cudaMallocAsync / cudaFreeAsync).
class DevBuf {
 public:
  DevBuf() = default;
  DevBuf(size_t bytes, cudaStream_t s) : bytes_(bytes), s_(s) {
    if (bytes) C3D_CUDA(cudaMallocAsync(&p_, bytes, s));
  }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept { *this = std::move(o); }
  DevBuf& operator=(DevBuf&& o) noexcept {
    if (this != &o) {
      release();
      p_ = o.p_;
      bytes_ = o.bytes_;
      s_ = o.s_;
      o.p_ = nullptr;
      o.bytes_ = 0;
    }
    return *this;
  }
  ~DevBuf() { release(); }
  void* get() const { return p_; }
  template <typename T>
  T* as() const {
    return static_cast<T*>(p_);
  }
  size_t bytes() const { return bytes_; }
  // Re-homes the free onto another stream (ownership moves with saved state).
  void set_stream(cudaStream_t s) { s_ = s; }

 private:
  void release() {
    if (p_) cudaFreeAsync(p_, s_);
    p_ = nullptr;
  }
  void* p_ = nullptr;
  size_t bytes_ = 0;
  cudaStream_t s_ = nullptr;
};

class Cube {
 public:
  Cube(const int dims[3], int rank, int device, const unsigned char* uid);
  ~Cube();

  const Grid& grid() const { return grid_; }
  int rank() const { return rank_; }
  const std::array<int, 3>& coords() const { return coords_; }
  int coord(int axis) const { return coords_[axis]; }
  int extent(int axis) const { return grid_.dims[axis]; }
  int device() const { return device_; }
  int num_sms() const { return num_sms_; }
  // Peer-memory transport, or null when collectives go through NCCL (C3D_NCCL_COLL=1).
  SymmHeap* symm() const { return symm_.get(); }
  const std::vector<int>& line(int axis) const { return line_[axis]; }

  // Collectives along one axis line. Counts are in elements.
  void all_gather(int axis, const void* send, void* recv, size_t count, int dtype,
                  cudaStream_t s);
  // Same into a symmetric arena buffer (peer-memory transport only).
  void all_gather_sym(int axis, const void* send, const SymBuf& recv, size_t count, int dtype,
                      cudaStream_t s);
  // send holds extent(axis)*count elements; recv receives this rank's count-slice of the sum.
  void reduce_scatter(int axis, const void* send, void* recv, size_t count, int dtype,
                      cudaStream_t s);
  void all_reduce(int axis, void* buf, size_t count, int dtype, bool is_max, cudaStream_t s);
  void broadcast(int axis, int root_position, void* buf, size_t count, int dtype, cudaStream_t s);
  void barrier(cudaStream_t s);

  // Charges a transfer done outside the collectives above (fused operators).
  void account(int kind, uint64_t sent, uint64_t received) { charge(kind, sent, received); }
  c3d_counters& counters() { return counters_; }
  const c3d_counters& counters() const { return counters_; }
  void add_madds(uint64_t n) { counters_.multiply_adds += n; }

  // Fails with C3D_ERR_DESYNC when a peer-memory wait of an earlier (completed) kernel
  // timed out or saw a mismatched collective header; the cube then stays poisoned, as
  // the reference poisons a group whose collective failed (cube3d/transport.hpp:67-78).
  void check_fault();

  void reset_counters() { std::memset(&counters_, 0, sizeof(counters_)); }

 private:
  void charge(int kind, uint64_t sent, uint64_t received);
  ncclComm_t comm(int axis) const;

  Grid grid_;
  int rank_ = 0;
  std::array<int, 3> coords_{0, 0, 0};
  int device_ = 0;
  int num_sms_ = 148;
  ncclComm_t world_ = nullptr;
  ncclComm_t axis_comm_[3] = {nullptr, nullptr, nullptr};
  std::unique_ptr<SymmHeap> symm_;  // peer-memory transport (null: NCCL for everything)
  std::vector<int> line_[3];        // world ranks of this rank's axis lines, by position
  c3d_counters counters_{};
  std::string poisoned_;
};

}  // namespace c3d
