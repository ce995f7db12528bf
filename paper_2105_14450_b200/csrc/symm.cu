// Peer-memory collectives (see symm.hpp). One launch per collective (per mailbox-sized
// chunk); CTA b of every rank on the line handles the same element piece, so the
// handshake is pairwise per CTA and needs no grid-wide synchronisation.
#include "symm.hpp"

#include <cuda_bf16.h>

#include <algorithm>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <string>

#include "common.hpp"
#include "gemm.hpp"
#include "ptx.cuh"

namespace c3d {

size_t dtype_size(int dtype);

namespace {

struct SymmArgs {
  int op, P, me, root, is_max, rank, G;
  int line[kSymmMaxLine];
  char* mbox[kSymmMaxLine];         // mailbox of each line position (mapped here)
  uint32_t* entered[kSymmMaxLine];  // flag arrays of each position's rank, [src][block]
  uint32_t* done[kSymmMaxLine];
  uint32_t* my_entered;
  uint32_t* my_done;
  uint32_t* my_seq;
  uint32_t* hdr[kSymmMaxLine];      // header arrays of each position's rank, [src][block]
  const uint32_t* my_hdr;
  uint32_t header;                  // (kind, root, op, dtype, count) of this call
  ptx::Fault fault;
  const char* send;
  char* recv;
  long long count, c0, n, slot_bytes;
  int direct;  // all-gather straight into the peers' symmetric receive buffers (mbox = recv)
};

using ptx::ld_acquire_sys;
using ptx::st_release_sys;

// Fault sites: 0x100 | peer position (entry), 0x200 | peer position (done), 0x300 | peer
// position (header mismatch).
__device__ __forceinline__ bool wait_epoch(const SymmArgs& a, const uint32_t* f, uint32_t e,
                                           uint32_t site) {
  return ptx::wait_epoch(f, e, a.fault, site);
}

// 16-byte vector (or scalar) lanes of dtype DT converted to fp32 for reductions.
template <int DT, bool VEC>
struct Lane {
  static constexpr int kElem = DT == kF32 ? 4 : 2;
  static constexpr int kBytes = VEC ? 16 : kElem;
  static constexpr int kN = kBytes / kElem;
  using Raw = typename std::conditional<VEC, uint4,
                                        typename std::conditional<DT == kF32, float,
                                                                  __nv_bfloat16>::type>::type;
  static __device__ __forceinline__ Raw ld(const char* p) { return *reinterpret_cast<const Raw*>(p); }
  static __device__ __forceinline__ Raw ld_cg(const char* p) {
    if constexpr (VEC) {
      return __ldcg(reinterpret_cast<const uint4*>(p));
    } else if constexpr (DT == kF32) {
      return __ldcg(reinterpret_cast<const float*>(p));
    } else {
      unsigned short u = __ldcg(reinterpret_cast<const unsigned short*>(p));
      return __ushort_as_bfloat16(u);
    }
  }
  static __device__ __forceinline__ void st(char* p, const Raw& v) {
    *reinterpret_cast<Raw*>(p) = v;
  }
  static __device__ __forceinline__ void to_f(const Raw& r, float (&f)[kN]) {
    if constexpr (DT == kF32) {
      const float* s = reinterpret_cast<const float*>(&r);
#pragma unroll
      for (int i = 0; i < kN; ++i) f[i] = s[i];
    } else {
      const __nv_bfloat16* s = reinterpret_cast<const __nv_bfloat16*>(&r);
#pragma unroll
      for (int i = 0; i < kN; ++i) f[i] = __bfloat162float(s[i]);
    }
  }
  static __device__ __forceinline__ Raw from_f(const float (&f)[kN]) {
    Raw r;
    if constexpr (DT == kF32) {
      float* d = reinterpret_cast<float*>(&r);
#pragma unroll
      for (int i = 0; i < kN; ++i) d[i] = f[i];
    } else {
      __nv_bfloat16* d = reinterpret_cast<__nv_bfloat16*>(&r);
#pragma unroll
      for (int i = 0; i < kN; ++i) d[i] = __float2bfloat16_rn(f[i]);
    }
    return r;
  }
};

template <int DT, bool VEC>
__global__ void __launch_bounds__(1024) symm_coll_kernel(const SymmArgs a) {
  using L = Lane<DT, VEC>;
  constexpr int B = L::kBytes;
  const int b = blockIdx.x;
  const int t = threadIdx.x;
  const long long nv = a.n / L::kN;
  const long long lo = nv * b / a.G, hi = nv * (b + 1) / a.G;
  __shared__ uint32_t ep[kSymmMaxLine];

  // entry: the peer has started this collective, so it no longer reads its mailbox
  if (t < a.P && t != a.me) {
    const int q = a.line[t];
    const uint32_t e = a.my_seq[q * kSymmMaxBlocks + b] + 1;
    ep[t] = e;
    st_release_sys(a.entered[t] + a.rank * kSymmMaxBlocks + b, e);
    wait_epoch(a, a.my_entered + q * kSymmMaxBlocks + b, e, 0x100u | static_cast<uint32_t>(t));
  }
  __syncthreads();

  const long long es = L::kBytes / L::kN;
  const char* send = a.send;
  // push this block's piece into every peer's mailbox slot `me` (4 loads in flight
  // per thread before the stores go out over NVLink)
  constexpr int U = 4;
  const long long step = static_cast<long long>(blockDim.x) * U;
  if (a.op == kCollReduceScatter) {
    for (int q = 0; q < a.P; ++q) {
      if (q == a.me) continue;
      const char* src = send + (q * a.count + a.c0) * es;
      char* dst = a.mbox[q] + a.me * a.slot_bytes;
      for (long long i0 = lo + t; i0 < hi; i0 += step) {
        typename L::Raw v[U];
#pragma unroll
        for (int u = 0; u < U; ++u)
          if (i0 + u * blockDim.x < hi) v[u] = L::ld(src + (i0 + u * blockDim.x) * B);
#pragma unroll
        for (int u = 0; u < U; ++u)
          if (i0 + u * blockDim.x < hi) L::st(dst + (i0 + u * blockDim.x) * B, v[u]);
      }
    }
  } else if (a.op != kCollBroadcast || a.me == a.root) {
    const char* src = send + a.c0 * es;
    for (long long i0 = lo + t; i0 < hi; i0 += step) {
      typename L::Raw v[U];
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (i0 + u * blockDim.x < hi) v[u] = L::ld(src + (i0 + u * blockDim.x) * B);
      for (int q = 0; q < a.P; ++q) {
        if (q == a.me) continue;
        char* dst = a.mbox[q] + a.me * a.slot_bytes;
#pragma unroll
        for (int u = 0; u < U; ++u)
          if (i0 + u * blockDim.x < hi) L::st(dst + (i0 + u * blockDim.x) * B, v[u]);
      }
    }
  }
  // own slot of a gather does not depend on the peers: copy it while the stores drain
  if (a.op == kCollAllGather) {
    const char* src = send + a.c0 * es;
    char* dst = a.recv + (a.me * a.count + a.c0) * es;
    if (src != dst)
      for (long long i = lo + t; i < hi; i += blockDim.x) L::st(dst + i * B, L::ld(src + i * B));
  }
  __syncthreads();

  // done: release this block's stores, then wait for the peers' pieces
  if (t < a.P && t != a.me) {
    const int q = a.line[t];
    // the call's header travels with the done flag (the reference's RoundHeader of kind,
    // op, length, root and sequence, cube3d/transport.hpp:32-40, 305-319): a peer in a
    // different collective is a desync, not a silent mix of payloads
    a.hdr[t][a.rank * kSymmMaxBlocks + b] = a.header;
    __threadfence_system();
    st_release_sys(a.done[t] + a.rank * kSymmMaxBlocks + b, ep[t]);
    if (wait_epoch(a, a.my_done + q * kSymmMaxBlocks + b, ep[t], 0x200u | static_cast<uint32_t>(t))) {
      const uint32_t ph = ld_acquire_sys(a.my_hdr + q * kSymmMaxBlocks + b);
      if (ph != a.header) ptx::record_fault(a.fault, 2u, 0x300u | static_cast<uint32_t>(t), a.header, ph);
    }
    a.my_seq[q * kSymmMaxBlocks + b] = ep[t];
  }
  __syncthreads();

  const char* mine = a.mbox[a.me];
  if (a.op == kCollAllGather && a.direct) {
    // the peers wrote their slots of recv directly; the own slot was copied above
  } else if (a.op == kCollAllGather) {
    for (int p = 0; p < a.P; ++p) {
      if (p == a.me) continue;
      const char* src = mine + p * a.slot_bytes;
      char* dst = a.recv + (p * a.count + a.c0) * es;
      for (long long i = lo + t; i < hi; i += blockDim.x) L::st(dst + i * B, L::ld_cg(src + i * B));
    }
  } else if (a.op == kCollBroadcast) {
    if (a.me != a.root || send != a.recv) {
      const char* src = a.me == a.root ? send + a.c0 * es : mine + a.root * a.slot_bytes;
      char* dst = a.recv + a.c0 * es;
      for (long long i = lo + t; i < hi; i += blockDim.x)
        L::st(dst + i * B, a.me == a.root ? L::ld(src + i * B) : L::ld_cg(src + i * B));
    }
  } else {
    // reduce in ascending position order (cube3d/transport.hpp:208-257)
    const char* own = send + ((a.op == kCollReduceScatter ? a.me * a.count : 0) + a.c0) * es;
    char* dst = a.recv + a.c0 * es;
    for (long long i = lo + t; i < hi; i += blockDim.x) {
      float acc[L::kN];
      for (int p = 0; p < a.P; ++p) {
        float v[L::kN];
        L::to_f(p == a.me ? L::ld(own + i * B) : L::ld_cg(mine + p * a.slot_bytes + i * B), v);
#pragma unroll
        for (int k = 0; k < L::kN; ++k)
          acc[k] = p == 0 ? v[k] : (a.is_max ? fmaxf(acc[k], v[k]) : acc[k] + v[k]);
      }
      L::st(dst + i * B, L::from_f(acc));
    }
  }
}

template <int DT, bool VEC>
void launch(const SymmArgs& a, cudaStream_t s) {
  static const int threads = [] {
    const char* e = std::getenv("C3D_SYMM_THREADS");
    return e ? std::atoi(e) : 1024;  // sweep (tools/symm_sweep.sh): 1024 x 1 per SM best
  }();
  symm_coll_kernel<DT, VEC><<<a.G, threads, 0, s>>>(a);
}

// (kind 2 b | root 4 b | max 1 b | dtype 1 b | count 24 b): what every member of the line
// must agree on for one collective.
uint32_t coll_header(int op, int root, bool is_max, int dtype, size_t count) {
  return (static_cast<uint32_t>(op & 3) << 30) | (static_cast<uint32_t>(root & 15) << 26) |
         (static_cast<uint32_t>(is_max ? 1 : 0) << 25) | (static_cast<uint32_t>(dtype & 1) << 24) |
         static_cast<uint32_t>(count & 0xFFFFFFu);
}

}  // namespace

std::string SymmHeap::fault_message() const {
  if (!fault_host_) return "";
  volatile uint32_t* w = fault_host_;
  if (w[0] == 0u) return "";
  static const char* kinds[] = {"all_gather", "reduce_scatter", "all_reduce", "broadcast"};
  char buf[256];
  if (w[0] == 1u) {
    std::snprintf(buf, sizeof(buf),
                  "peer did not arrive within the timeout (site 0x%x: expected epoch %u, saw %u)",
                  w[1], w[2], w[3]);
  } else {
    std::snprintf(buf, sizeof(buf),
                  "collective header mismatch with line position %u: this rank %s count %u, peer "
                  "%s count %u",
                  w[1] & 0xFFu, kinds[w[2] >> 30], w[2] & 0xFFFFFFu, kinds[w[3] >> 30],
                  w[3] & 0xFFFFFFu);
  }
  return buf;
}

SymmHeap::SymmHeap(ncclComm_t world, int world_size, int rank, size_t mailbox_bytes,
                   size_t arena_bytes, cudaStream_t s)
    : world_(world_size), rank_(rank) {
  if (world_size > kSymmMaxRanks)
    fail(C3D_ERR_CONFIG_INVALID, "peer transport supports at most 64 ranks");
  mailbox_bytes_ = (mailbox_bytes + 4095) / 4096 * 4096;
  arena_bytes_ = (arena_bytes + 4095) / 4096 * 4096;
  constexpr size_t RB = static_cast<size_t>(kSymmMaxRanks) * kSymmMaxBlocks;
  // [entered RB][done RB][op_entered R][op_done RB][op_ag RB][hdr RB]
  flags_bytes_ = ((5 * RB + kSymmMaxRanks) * sizeof(uint32_t) + 4095) / 4096 * 4096;
  C3D_CUDA(cudaMalloc(&heap_, flags_bytes_ + mailbox_bytes_ + arena_bytes_));
  C3D_CUDA(cudaMemset(heap_, 0, flags_bytes_));
  C3D_CUDA(cudaMalloc(&seq_, (RB + 32) * sizeof(uint32_t)));
  C3D_CUDA(cudaMemset(seq_, 0, (RB + 32) * sizeof(uint32_t)));
  if (arena_bytes_) free_.push_back({0, arena_bytes_});
  C3D_CUDA(cudaHostAlloc(&fault_host_, 8 * sizeof(uint32_t), cudaHostAllocMapped));
  std::memset(fault_host_, 0, 8 * sizeof(uint32_t));
  C3D_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&fault_.word), fault_host_, 0));
  if (const char* e = std::getenv("C3D_PEER_TIMEOUT_MS"))
    fault_.timeout_ns = static_cast<unsigned long long>(std::atoll(e)) * 1000000ull;
  C3D_CUDA(cudaDeviceSynchronize());

  // exchange IPC handles over the world communicator (the flags are zeroed everywhere
  // before any rank can see a peer's heap: the gather completes only after all ranks
  // reached it)
  cudaIpcMemHandle_t mine;
  C3D_CUDA(cudaIpcGetMemHandle(&mine, heap_));
  const size_t hs = sizeof(cudaIpcMemHandle_t);
  void* dev = nullptr;
  C3D_CUDA(cudaMalloc(&dev, hs * (world_size + 1)));
  C3D_CUDA(cudaMemcpy(static_cast<char*>(dev) + hs * world_size, &mine, hs, cudaMemcpyHostToDevice));
  ncclResult_t r = ncclAllGather(static_cast<char*>(dev) + hs * world_size, dev, hs, ncclUint8,
                                 world, s);
  if (r != ncclSuccess) fail(C3D_ERR_NCCL, std::string("ncclAllGather(ipc): ") + ncclGetErrorString(r));
  C3D_CUDA(cudaStreamSynchronize(s));
  std::vector<cudaIpcMemHandle_t> all(world_size);
  C3D_CUDA(cudaMemcpy(all.data(), dev, hs * world_size, cudaMemcpyDeviceToHost));
  C3D_CUDA(cudaFree(dev));

  base_.assign(world_size, nullptr);
  for (int q = 0; q < world_size; ++q) {
    if (q == rank) {
      base_[q] = heap_;
    } else {
      C3D_CUDA(cudaIpcOpenMemHandle(&base_[q], all[q], cudaIpcMemLazyEnablePeerAccess));
    }
  }
  for (int q = 0; q < world_size; ++q) {
    char* b = static_cast<char*>(base_[q]);
    uint32_t* f = reinterpret_cast<uint32_t*>(b);
    entered_.push_back(f);
    done_.push_back(f + RB);
    op_entered_.push_back(f + 2 * RB);
    op_done_.push_back(f + 2 * RB + kSymmMaxRanks);
    op_ag_.push_back(f + 3 * RB + kSymmMaxRanks);
    hdr_.push_back(f + 4 * RB + kSymmMaxRanks);
    mbox_.push_back(b + flags_bytes_);
    arena_.push_back(b + flags_bytes_ + mailbox_bytes_);
  }
}

SymmHeap::~SymmHeap() {
  for (int q = 0; q < world_; ++q)
    if (q != rank_ && q < static_cast<int>(base_.size()) && base_[q]) cudaIpcCloseMemHandle(base_[q]);
  if (heap_) cudaFree(heap_);
  if (seq_) cudaFree(seq_);
  if (fault_host_) cudaFreeHost(fault_host_);
}

bool SymmHeap::arena_alloc(size_t bytes, size_t* off) {
  bytes = (bytes + 1023) / 1024 * 1024;
  for (size_t i = 0; i < free_.size(); ++i) {
    if (free_[i].second < bytes) continue;
    *off = free_[i].first;
    free_[i].first += bytes;
    free_[i].second -= bytes;
    if (free_[i].second == 0) free_.erase(free_.begin() + i);
    used_.push_back({*off, bytes});
    return true;
  }
  return false;
}

void SymmHeap::arena_free(size_t off) {
  size_t bytes = 0;
  for (size_t i = 0; i < used_.size(); ++i) {
    if (used_[i].first == off) {
      bytes = used_[i].second;
      used_.erase(used_.begin() + i);
      break;
    }
  }
  if (!bytes) return;
  auto it = free_.begin();
  while (it != free_.end() && it->first < off) ++it;
  it = free_.insert(it, {off, bytes});
  // coalesce with the next and previous ranges
  auto nx = it + 1;
  if (nx != free_.end() && it->first + it->second == nx->first) {
    it->second += nx->second;
    free_.erase(nx);
  }
  if (it != free_.begin()) {
    auto pv = it - 1;
    if (pv->first + pv->second == it->first) {
      pv->second += it->second;
      free_.erase(it);
    }
  }
}

void SymmHeap::all_gather_direct(const std::vector<int>& line, int pos, const void* send,
                                 size_t recv_off, size_t count, int dtype, int num_sms,
                                 cudaStream_t s) {
  const int P = static_cast<int>(line.size());
  if (P > kSymmMaxLine) fail(C3D_ERR_CONFIG_INVALID, "axis line longer than 8 ranks");
  if (P == 1 || count == 0) return;
  const size_t es = dtype_size(dtype);
  SymmArgs a{};
  a.op = kCollAllGather;
  a.P = P;
  a.me = pos;
  a.rank = rank_;
  a.direct = 1;
  for (int p = 0; p < P; ++p) {
    a.line[p] = line[p];
    a.mbox[p] = arena_[line[p]] + recv_off;  // slot `me` of the peer's buffer: + me * count
    a.entered[p] = entered_[line[p]];
    a.done[p] = done_[line[p]];
  }
  a.my_entered = entered_[rank_];
  a.my_done = done_[rank_];
  a.my_seq = seq_;
  for (int p = 0; p < P; ++p) a.hdr[p] = hdr_[line[p]];
  a.my_hdr = hdr_[rank_];
  a.header = coll_header(kCollAllGather, 0, false, dtype, count);
  a.fault = fault_;
  a.send = static_cast<const char*>(send);
  a.recv = arena_[rank_] + recv_off;
  a.count = static_cast<long long>(count);
  a.slot_bytes = static_cast<long long>(count * es);
  a.c0 = 0;
  a.n = static_cast<long long>(count);
  static const size_t chunk = [] {
    const char* e = std::getenv("C3D_SYMM_CHUNK_KB");
    return static_cast<size_t>(e ? std::atoi(e) : 32) << 10;
  }();
  static const int per_sm = [] {
    const char* e = std::getenv("C3D_SYMM_PER_SM");
    return e ? std::atoi(e) : 1;
  }();
  const size_t blocks = (count * es + chunk - 1) / chunk;
  a.G = static_cast<int>(std::max<size_t>(
      1, std::min<size_t>(blocks, std::min(per_sm * num_sms, kSymmMaxBlocks))));
  const bool vec_ok = reinterpret_cast<uintptr_t>(send) % 16 == 0 && recv_off % 16 == 0 &&
                      count % (16 / es) == 0;
  if (dtype == kF32) {
    if (vec_ok) launch<kF32, true>(a, s); else launch<kF32, false>(a, s);
  } else {
    if (vec_ok) launch<kBF16, true>(a, s); else launch<kBF16, false>(a, s);
  }
  check_launch("symm_all_gather_direct");
}

void SymmHeap::collective(CollOp op, const std::vector<int>& line, int pos, const void* send,
                          void* recv, size_t count, int dtype, int root_pos, bool is_max,
                          int num_sms, cudaStream_t s) {
  const int P = static_cast<int>(line.size());
  if (P > kSymmMaxLine) fail(C3D_ERR_CONFIG_INVALID, "axis line longer than 8 ranks");
  if (P == 1 || count == 0) return;
  const size_t es = dtype_size(dtype);
  const size_t slot_bytes = mailbox_bytes_ / P / 256 * 256;
  const size_t cap = slot_bytes / es / 8 * 8;  // elements per chunk and slot
  if (cap == 0) fail(C3D_ERR_INTERNAL, "peer mailbox too small");

  SymmArgs a{};
  a.op = op;
  a.P = P;
  a.me = pos;
  a.root = root_pos;
  a.is_max = is_max ? 1 : 0;
  a.rank = rank_;
  for (int p = 0; p < P; ++p) {
    a.line[p] = line[p];
    a.mbox[p] = mbox_[line[p]];
    a.entered[p] = entered_[line[p]];
    a.done[p] = done_[line[p]];
  }
  a.my_entered = entered_[rank_];
  a.my_done = done_[rank_];
  a.my_seq = seq_;
  for (int p = 0; p < P; ++p) a.hdr[p] = hdr_[line[p]];
  a.my_hdr = hdr_[rank_];
  a.header = coll_header(op, root_pos, is_max, dtype, count);
  a.fault = fault_;
  a.send = static_cast<const char*>(send);
  a.recv = static_cast<char*>(recv);
  a.count = static_cast<long long>(count);
  a.slot_bytes = static_cast<long long>(slot_bytes);

  const size_t vec = 16 / es;
  const bool vec_ok = reinterpret_cast<uintptr_t>(send) % 16 == 0 &&
                      reinterpret_cast<uintptr_t>(recv) % 16 == 0 && count % vec == 0;
  for (size_t c0 = 0; c0 < count; c0 += cap) {
    const size_t n = std::min(cap, count - c0);
    a.c0 = static_cast<long long>(c0);
    a.n = static_cast<long long>(n);
    // one block per `chunk` bytes of payload, at most `per_sm` per SM (all co-resident)
    static const size_t chunk = [] {
      const char* e = std::getenv("C3D_SYMM_CHUNK_KB");
      return static_cast<size_t>(e ? std::atoi(e) : 32) << 10;
    }();
    static const int per_sm = [] {
      const char* e = std::getenv("C3D_SYMM_PER_SM");
      return e ? std::atoi(e) : 1;
    }();
    const size_t blocks = (n * es + chunk - 1) / chunk;
    a.G = static_cast<int>(std::max<size_t>(
        1, std::min<size_t>(blocks, std::min(per_sm * num_sms, kSymmMaxBlocks))));
    if (dtype == kF32) {
      if (vec_ok) launch<kF32, true>(a, s); else launch<kF32, false>(a, s);
    } else {
      if (vec_ok) launch<kBF16, true>(a, s); else launch<kBF16, false>(a, s);
    }
    check_launch("symm_collective");
  }
}

}  // namespace c3d
