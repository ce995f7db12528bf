// Peer-memory transport over NVLink / NVSwitch: one symmetric heap per rank
// (cudaMalloc, mapped into every other rank with CUDA IPC) holding per-block
// handshake flags and a receive mailbox. Collectives along an axis line are
// single push kernels: every CTA announces entry to its peers, stores its
// piece of the payload straight into the peers' mailboxes with SM stores over
// NVLink, raises a per-CTA "done" flag with release semantics, waits for the
// peers' pieces and finishes the gather / reduction locally.
//
// This replaces the NCCL calls of Cube::{all_gather, reduce_scatter,
// all_reduce, broadcast} (cube3d/transport.hpp:160-257 semantics: positions
// ascend along the axis, reduce-scatter and all-reduce sum in ascending
// position order) and is what the GEMM epilogues push into directly.
#pragma once

#include <cuda_runtime.h>
#include <nccl.h>

#include "ptx_fault.hpp"

#include <cstddef>
#include <cstdint>
#include <string>
#include <utility>
#include <vector>

namespace c3d {

constexpr int kSymmMaxBlocks = 512;
constexpr int kSymmMaxRanks = 64;
constexpr int kSymmMaxLine = 8;

enum CollOp { kCollAllGather = 0, kCollReduceScatter = 1, kCollAllReduce = 2, kCollBroadcast = 3 };

// One rank's view of every rank's heap.
class SymmHeap {
 public:
  // Collective over `world` (NCCL, used once to exchange the IPC handles).
  SymmHeap(ncclComm_t world, int world_size, int rank, size_t mailbox_bytes, size_t arena_bytes,
           cudaStream_t s);
  ~SymmHeap();
  SymmHeap(const SymmHeap&) = delete;
  SymmHeap& operator=(const SymmHeap&) = delete;

  size_t mailbox_bytes() const { return mailbox_bytes_; }
  int world_size() const { return world_; }
  int rank() const { return rank_; }

  // `line`: world ranks of the axis line in position order; `pos`: this rank's position.
  // Counts in elements (NCCL conventions: AG `count` = per-rank shard, RS `count` = per-rank
  // result; AR / BC `count` = buffer length). Payloads larger than the mailbox are chunked.
  void collective(CollOp op, const std::vector<int>& line, int pos, const void* send, void* recv,
                  size_t count, int dtype, int root_pos, bool is_max, int num_sms,
                  cudaStream_t s);

  // All-gather into a symmetric arena buffer (offset recv_off on every rank): each rank
  // writes its shard straight into the peers' buffers -- no mailbox, no copy-out.
  void all_gather_direct(const std::vector<int>& line, int pos, const void* send, size_t recv_off,
                         size_t count, int dtype, int num_sms, cudaStream_t s);

  // Mailbox of rank `r` as mapped in this process (own heap for r == rank()).
  char* mailbox(int r) const { return mbox_[r]; }
  uint32_t* entered(int r) const { return entered_[r]; }
  uint32_t* done(int r) const { return done_[r]; }
  uint32_t* seq() const { return seq_; }

  // Fused-operator handshake (see fused.cu): one entry flag per source rank, one done
  // flag per (source rank, producer CTA), and this rank's fused-op epoch counter.
  uint32_t* op_entered(int r) const { return op_entered_[r]; }
  uint32_t* op_done(int r) const { return op_done_[r]; }
  uint32_t* op_ag(int r) const { return op_ag_[r]; }  // gathered-operand arrival, [src][cta]
  uint32_t* op_seq() const { return seq_ + kSymmMaxRanks * kSymmMaxBlocks; }

  // Device-visible fault record of this rank's peer waits (Fault), and its description
  // ("" while no wait failed).
  const Fault& fault() const { return fault_; }
  std::string fault_message() const;

  // Symmetric arena: every rank performs the same allocation sequence, so an allocation
  // sits at the same offset in every rank's heap and peers can address it directly.
  // First fit over an address-ordered free list (deterministic). Returns false when full.
  bool arena_alloc(size_t bytes, size_t* off);
  void arena_free(size_t off);
  char* arena(int r) const { return arena_[r]; }

 private:
  int world_ = 1, rank_ = 0;
  size_t mailbox_bytes_ = 0;
  size_t flags_bytes_ = 0;
  void* heap_ = nullptr;    // own heap
  uint32_t* seq_ = nullptr;  // own per-(peer, block) epoch counters (not shared)
  std::vector<void*> base_;  // mapped heaps (own at rank_)
  std::vector<char*> mbox_;
  std::vector<uint32_t*> entered_, done_, op_entered_, op_done_, op_ag_, hdr_;
  uint32_t* fault_host_ = nullptr;
  Fault fault_;
  std::vector<char*> arena_;
  size_t arena_bytes_ = 0;
  std::vector<std::pair<size_t, size_t>> free_;  // (offset, size), address order
  std::vector<std::pair<size_t, size_t>> used_;  // (offset, size)
};

// Stream-ordered symmetric allocation (returned to the arena on destruction; the
// single-stream discipline makes immediate reuse safe, peers write only after the
// owner's entry handshake for the op using it).
class SymBuf {
 public:
  SymBuf() = default;
  SymBuf(SymmHeap* h, size_t bytes) : h_(h), bytes_(bytes) {
    if (h_ && !h_->arena_alloc(bytes, &off_)) h_ = nullptr;
  }
  SymBuf(const SymBuf&) = delete;
  SymBuf& operator=(const SymBuf&) = delete;
  ~SymBuf() {
    if (h_) h_->arena_free(off_);
  }
  bool ok() const { return h_ != nullptr; }
  size_t offset() const { return off_; }
  char* local() const { return h_->arena(h_->rank()) + off_; }
  char* at(int r) const { return h_->arena(r) + off_; }

 private:
  SymmHeap* h_ = nullptr;
  size_t off_ = 0, bytes_ = 0;
};

}  // namespace c3d
