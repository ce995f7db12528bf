// GEMM -> reduce-scatter as one overlapped operator over NVLink peer memory.
//
// The reference's matmul forward / backward end with `scatter_rows` (the
// reduce_scatter of the local partial product along the output axis,
// cube3d/ops3d.hpp:70-76, 129, 163). Here the tcgen05 GEMM's epilogue TMA-stores
// each output tile straight into the rank that owns its row block: its own block
// into the local slot, the others into this rank's slot of the owner's symmetric
// receive buffer (SymBuf) through the NVLink mapping, so the transfer overlaps the
// MMAs tile by tile. A short finishing kernel then waits for the peers' producer
// CTAs, sums the P slots in ascending position order (cube3d/transport.hpp:208-232)
// and applies the deferred epilogue (bias, pre-activation, GELU / GELU', residual).
//
// Handshake (all flags in the symmetric heap, epochs from a per-rank fused-op counter
// that every rank advances in lockstep -- the SPMD call sequence is identical):
//   enter kernel:  epoch = ++op_seq; raise op_entered[me] on every peer of the line
//                  (all of this rank's earlier stream work has finished, so peers may
//                  now write its receive buffer);
//   GEMM CTA:      waits for op_entered[k] before its first store into block k;
//                  raises op_done[me][cta] on k after its last store;
//   finish kernel: waits op_done[k][cta] for all peers and CTAs, then reduces.
#include <cuda.h>
#include <cuda_bf16.h>

#include <algorithm>

#include "common.hpp"
#include "epi.cuh"
#include "gemm_tc.hpp"
#include "kernels.hpp"
#include "ops.hpp"
#include "ptx.cuh"

namespace c3d {

namespace {

struct EnterArgs {
  int n, rank, wait;
  uint32_t* peer_entered[2 * kRsMax];    // each peer's op_entered array (mapped)
  const uint32_t* my_entered[2 * kRsMax];  // this rank's flag raised by that peer
  uint32_t* seq;
  ptx::Fault fault;
};

// Advances the fused-op epoch and announces this rank's entry to its peers; with
// `wait`, also waits for theirs (then every peer has finished its earlier work and
// its symmetric buffers of this op may be written).
__global__ void enter_kernel(EnterArgs a) {
  if (threadIdx.x != 0) return;
  const uint32_t e = *a.seq + 1;
  *a.seq = e;
  __threadfence_system();
  for (int k = 0; k < a.n; ++k) ptx::st_release_sys(a.peer_entered[k] + a.rank, e);
  if (a.wait)
    for (int k = 0; k < a.n; ++k) ptx::wait_epoch(a.my_entered[k], e, a.fault, 0x400u | k);
}

struct FinishArgs {
  int P, me, grid, done_offset;
  const uint32_t* done[kRsMax];  // this rank's op_done row for source line[k]
  const uint32_t* seq;
  ptx::Fault fault;
  const char* slots;  // [P][rows*cols] partials (own slot written locally)
  long long slot_elems;
  long long rows, cols;
  int dtype;
  int vec;
  Epilogue e;  // out = contiguous [rows][cols]
};

template <int DT>
__device__ __forceinline__ void load8(const char* p, float (&v)[8], bool cg) {
  if (DT == kF32) {
    const float4* q = reinterpret_cast<const float4*>(p);
    const float4 x = cg ? __ldcg(q) : q[0];
    const float4 y = cg ? __ldcg(q + 1) : q[1];
    v[0] = x.x; v[1] = x.y; v[2] = x.z; v[3] = x.w;
    v[4] = y.x; v[5] = y.y; v[6] = y.z; v[7] = y.w;
  } else {
    const uint4* q = reinterpret_cast<const uint4*>(p);
    const uint4 r = cg ? __ldcg(q) : q[0];
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&r);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float2 f = __bfloat1622float2(h[i]);
      v[2 * i] = f.x;
      v[2 * i + 1] = f.y;
    }
  }
}

template <int DT>
__device__ __forceinline__ void store8(char* p, const float (&v)[8]) {
  if (DT == kF32) {
    float4* q = reinterpret_cast<float4*>(p);
    q[0] = make_float4(v[0], v[1], v[2], v[3]);
    q[1] = make_float4(v[4], v[5], v[6], v[7]);
  } else {
    uint4 r;
    __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&r);
#pragma unroll
    for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(v[2 * i], v[2 * i + 1]);
    *reinterpret_cast<uint4*>(p) = r;
  }
}

template <int DT>
__global__ void __launch_bounds__(256) rs_finish_kernel(const FinishArgs a) {
  const uint32_t epoch = *a.seq;
  for (int i = threadIdx.x; i < (a.P - 1) * a.grid; i += blockDim.x) {
    int k = i / a.grid;
    const int cta = i - k * a.grid;
    if (k >= a.me) ++k;
    ptx::wait_epoch(a.done[k] + a.done_offset + cta, epoch, a.fault, 0x500u | k);
  }
  __syncthreads();
  const Epilogue& e = a.e;
  constexpr long long es = DT == kF32 ? 4 : 2;
  const long long total = a.rows * a.cols;
  if (a.vec) {
    const long long nv = total / 8;
    for (long long v8 = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; v8 < nv;
         v8 += static_cast<long long>(gridDim.x) * blockDim.x) {
      const long long off = v8 * 8;
      const long long n = off % a.cols;
      float acc[8];
      for (int p = 0; p < a.P; ++p) {
        float x[8];
        load8<DT>(a.slots + (p * a.slot_elems + off) * es, x, p != a.me);
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[j] = p == 0 ? x[j] : acc[j] + x[j];
      }
      if (e.bias) {
        const float4 b0 = __ldg(reinterpret_cast<const float4*>(e.bias + n));
        const float4 b1 = __ldg(reinterpret_cast<const float4*>(e.bias + n + 4));
        acc[0] += b0.x; acc[1] += b0.y; acc[2] += b0.z; acc[3] += b0.w;
        acc[4] += b1.x; acc[5] += b1.y; acc[6] += b1.z; acc[7] += b1.w;
      }
      if (e.act == kActGeluSave) {
        float gd[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) gelu_both(acc[j], acc[j], gd[j]);
        if (e.pre_act) store8<DT>(static_cast<char*>(e.pre_act) + off * es, gd);
      } else if (e.pre_act) {
        store8<DT>(static_cast<char*>(e.pre_act) + off * es, acc);
      }
      if (e.act == kActGelu) {
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[j] = gelu_f(acc[j]);
      } else if (e.act == kActGeluGrad || e.act == kActMulAux) {
        float g[8];
        load8<DT>(static_cast<const char*>(e.aux) + off * es, g, false);
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[j] *= e.act == kActMulAux ? g[j] : gelu_grad_f(g[j]);
      }
      if (e.resid) {
        float r[8];
        load8<DT>(static_cast<const char*>(e.resid) + off * es, r, false);
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[j] += r[j];
      }
      store8<DT>(static_cast<char*>(e.out.base) + off * es, acc);
    }
  } else {
    for (long long off = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
         off < total; off += static_cast<long long>(gridDim.x) * blockDim.x) {
      float acc = 0.f;
      for (int p = 0; p < a.P; ++p) {
        const float x = ld_any(a.slots, DT, p * a.slot_elems + off);
        acc = p == 0 ? x : acc + x;
      }
      epi_scalar(e, off, off % a.cols, acc);
    }
  }
}

void launch_finish(Cube& cube, SymmHeap* h, int axis, int grid, int done_offset,
                   const char* slots, long long slot_elems, long long rows, long long cols,
                   const Epilogue& post, cudaStream_t s) {
  const int P = cube.extent(axis);
  const std::vector<int>& line = cube.line(axis);
  FinishArgs fa{};
  fa.P = P;
  fa.me = cube.coord(axis);
  fa.grid = grid;
  fa.done_offset = done_offset;
  fa.seq = h->op_seq();
  fa.fault = h->fault();
  for (int k = 0; k < P; ++k)
    fa.done[k] = h->op_done(cube.rank()) + static_cast<size_t>(line[k]) * kSymmMaxBlocks;
  fa.slots = slots;
  fa.slot_elems = slot_elems;
  fa.rows = rows;
  fa.cols = cols;
  const int dtype = post.out.dtype;
  fa.dtype = dtype;
  fa.e = post;
  auto al = [](const void* q) { return reinterpret_cast<uintptr_t>(q) % 16 == 0; };
  bool vec = cols % 8 == 0 && al(post.out.base) && post.out.sr == cols && post.alpha == 1.f &&
             !post.accumulate && (!post.bias || al(post.bias)) && post.act != kActSoftmaxBwd;
  for (const void* q : {static_cast<const void*>(post.pre_act), post.aux, post.resid})
    vec = vec && (!q || al(q));
  vec = vec && (!post.pre_act || post.pre_dtype == dtype) &&
        (!post.aux || post.aux_dtype == dtype) && (!post.resid || post.resid_dtype == dtype);
  fa.vec = vec ? 1 : 0;
  const long long work = vec ? slot_elems / 8 : slot_elems;
  const int blocks = static_cast<int>(std::max<long long>(
      1, std::min<long long>((work + 255) / 256, static_cast<long long>(cube.num_sms()) * 4)));
  if (dtype == kF32) rs_finish_kernel<kF32><<<blocks, 256, 0, s>>>(fa);
  else rs_finish_kernel<kBF16><<<blocks, 256, 0, s>>>(fa);
  check_launch("fused_rs_finish");
}

// Fills the reduce-scatter destinations of one GEMM launch covering row blocks
// [block0, block0 + M / block_rows) of the P blocks along `axis`.
void fill_rs(Cube& cube, SymmHeap* h, int axis, const SymBuf& recv, long long block_rows,
             long long slot_bytes, int block0, int done_offset, RsOut* rs) {
  const int P = cube.extent(axis);
  const int me = cube.coord(axis);
  const std::vector<int>& line = cube.line(axis);
  rs->P = P;
  rs->me = me;
  rs->block0 = block0;
  rs->done_offset = done_offset;
  rs->block_rows = block_rows;
  rs->epoch = h->op_seq();
  rs->fault = h->fault();
  for (int k = 0; k < P; ++k) {
    rs->dst[k] = (k == me ? recv.local() : recv.at(line[k])) + me * slot_bytes;
    rs->entered[k] = h->op_entered(cube.rank()) + line[k];
    rs->done[k] = h->op_done(line[k]) + static_cast<size_t>(cube.rank()) * kSymmMaxBlocks;
  }
}

void launch_enter(Cube& cube, SymmHeap* h, const std::vector<int>& peers, bool wait,
                  cudaStream_t s) {
  EnterArgs ea{};
  ea.n = static_cast<int>(peers.size());
  ea.rank = cube.rank();
  ea.wait = wait ? 1 : 0;
  ea.seq = h->op_seq();
  ea.fault = h->fault();
  for (int k = 0; k < ea.n; ++k) {
    ea.peer_entered[k] = h->op_entered(peers[k]);
    ea.my_entered[k] = h->op_entered(cube.rank()) + peers[k];
  }
  enter_kernel<<<1, 32, 0, s>>>(ea);
  check_launch("fused_enter");
}

// Profiler brackets (C3D_PROF_DUMP): tags 5 enter, 6 GEMM+RS, 7 AG+GEMM+RS, 8 finish.
struct Span {
  cudaStream_t s;
  void* tok = nullptr;
  int tag;
  double bytes;
  Span(cudaStream_t st, int t, double b) : s(st), tag(t), bytes(b) {
    if (prof_on()) prof_begin(s, &tok);
  }
  ~Span() {
    if (tok) prof_end(s, tok, tag, bytes);
  }
};

View kview(const void* p, int dtype, long long ld) {
  View v;
  v.base = const_cast<void*>(p);
  v.dtype = dtype;
  v.sr = ld;
  v.sc = 1;
  return v;
}

}  // namespace

bool gemm_reduce_scatter(Cube& cube, int mode, int axis, int64_t M, int64_t N, int64_t K,
                         const View& a, const View& b, const Epilogue& post, cudaStream_t s) {
  SymmHeap* h = cube.symm();
  const int P = cube.extent(axis);
  if (!h || P < 2 || P > kRsMax || mode == C3D_MODE_F32) return false;
  if (a.dtype != kBF16 || b.dtype != kBF16 || M % P) return false;
  if (std::getenv("C3D_NO_FUSED_RS")) return false;
  // the finishing pass addresses the output (and residual / aux / pre-activation, which
  // share its layout) as contiguous [rows][N] blocks
  if (post.out.sr != N || post.out.sc != 1 || post.out.csplit || post.out.rsplit) return false;
  const int dtype = post.out.dtype;
  const long long es = dtype == kF32 ? 4 : 2;
  const long long block_rows = M / P;
  const long long slot_elems = block_rows * N;
  SymBuf recv(h, static_cast<size_t>(P * slot_elems * es));
  if (!recv.ok()) return false;

  GemmProblem p;
  p.M = M;
  p.N = N;
  p.K = K;
  p.a = a;
  p.b = b;
  p.epi.out = kview(recv.local(), dtype, N);
  fill_rs(cube, h, axis, recv, block_rows, slot_elems * es, 0, 0, &p.rs);
  const int bn = tc_pick_bn(M, N, 1, cube.num_sms());
  if (!tc_gemm_supported(p, bn) || !tc_gemm_rs_supported(p, bn)) return false;
  const int grid = tc_gemm_grid(p, bn, cube.num_sms());
  if (grid > kSymmMaxBlocks) return false;

  std::vector<int> peers;
  for (int k = 0; k < P; ++k)
    if (k != cube.coord(axis)) peers.push_back(cube.line(axis)[k]);
  launch_enter(cube, h, peers, false, s);
  {
    Span sp(s, 6, static_cast<double>(P * slot_elems * es));
    run_gemm(p, C3D_MODE_TC, cube.num_sms(), s);
  }
  cube.add_madds(static_cast<uint64_t>(M) * N * K);
  {
    Span sp(s, 8, static_cast<double>(P * slot_elems * es));
    launch_finish(cube, h, axis, grid, 0, recv.local(), slot_elems, block_rows, N, post, s);
  }
  cube.account(C3D_REDUCE_SCATTER, static_cast<uint64_t>(P - 1) * slot_elems,
               static_cast<uint64_t>(P - 1) * slot_elems);
  return true;
}

}  // namespace c3d
