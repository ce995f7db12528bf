// cube3d_b200.hpp -- C++ drop-in over the C ABI (c3d.h) that restores the reference's
// operator shapes (namespace cube3d, /root/reference/proj/include/cube3d/):
//
//   reference                                           here (namespace cube3d_b200)
//   Endpoint<T>& ep                                      Endpoint& ep (one per GPU / rank)
//   ShardedMatrix<T>{global_rows, global_cols, layout,   ShardedMatrix (device shard, RAII)
//                    dirs, shard}  (sharding.hpp:18-34)
//   DiagonalVector<T>  (sharding.hpp:38-47)              DiagonalVector
//   Activation3D<T>    (activation.hpp:41-62)            Activation3D
//   GroupState         (activation.hpp:20-35)            GroupState
//   matmul_ab_fwd(ep, a, b)          ops3d.hpp:114-132   matmul_ab_fwd(ep, a, b)
//   matmul_ab_bwd(ep, dc, a, b)      ops3d.hpp:137-168   matmul_ab_bwd(ep, dc, a, b)
//   linear3d_fwd(ep, x, p, gs, saved*)    nn.hpp:81-97   linear3d_fwd(ep, x, p, gs, saved*)
//   linear3d_bwd(ep, dy, saved, p)       nn.hpp:99-112   linear3d_bwd(ep, dy, saved, p)
//   layernorm3d_fwd/bwd                 nn.hpp:140-222   layernorm3d_fwd/bwd
//   transformer_layer_fwd(ep, x, p, cfg, gs, saved*)     transformer_layer_fwd(...)
//   transformer_layer_bwd(ep, dy, saved, p, cfg)         transformer_layer_bwd(...)
//                                 transformer.hpp:115-148
//   cube3d::Error subclasses (errors.hpp:12-37)          Error{code, "Name: detail"}
//
// Results are returned by value as in the reference; their device storage is owned by
// the returned objects (stream-ordered allocations on the endpoint's stream). Host
// transfer helpers (to_device / to_host) stand in for the reference's host matrices.
// The element type is chosen at runtime (C3D_F32 or C3D_BF16) instead of a template T.
#ifndef CUBE3D_B200_HPP_
#define CUBE3D_B200_HPP_

#include <cuda_runtime.h>

#include <array>
#include <cstdint>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "c3d.h"

namespace cube3d_b200 {

// --------------------------------------------------------------------- errors
class Error : public std::runtime_error {
 public:
  Error(int code, const std::string& what) : std::runtime_error(what), code_(code) {}
  int code() const { return code_; }

 private:
  int code_;
};

inline void check(int rc) {
  if (rc != C3D_OK) throw Error(rc, c3d_last_error());
}
inline void check_cuda(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw Error(C3D_ERR_CUDA, std::string("CudaError: ") + what + ": " +
                                                      cudaGetErrorString(e));
}

inline size_t dtype_bytes(int dtype) { return dtype == C3D_BF16 ? 2 : 4; }

// ------------------------------------------------------------- device memory
// Stream-ordered device buffer (freed on the stream it was allocated on).
class DeviceBuffer {
 public:
  DeviceBuffer() = default;
  DeviceBuffer(size_t bytes, cudaStream_t s) : bytes_(bytes), s_(s) {
    if (bytes) check_cuda(cudaMallocAsync(&p_, bytes, s), "cudaMallocAsync");
  }
  DeviceBuffer(const DeviceBuffer&) = delete;
  DeviceBuffer& operator=(const DeviceBuffer&) = delete;
  DeviceBuffer(DeviceBuffer&& o) noexcept { swap(o); }
  DeviceBuffer& operator=(DeviceBuffer&& o) noexcept {
    if (this != &o) {
      reset();
      swap(o);
    }
    return *this;
  }
  ~DeviceBuffer() { reset(); }
  void* get() const { return p_; }
  size_t bytes() const { return bytes_; }

 private:
  void swap(DeviceBuffer& o) {
    std::swap(p_, o.p_);
    std::swap(bytes_, o.bytes_);
    std::swap(s_, o.s_);
  }
  void reset() {
    if (p_) cudaFreeAsync(p_, s_);
    p_ = nullptr;
    bytes_ = 0;
  }
  void* p_ = nullptr;
  size_t bytes_ = 0;
  cudaStream_t s_ = nullptr;
};

// --------------------------------------------------------------- topology
struct DirectionTriple {  // cube3d/layout.hpp:44-61
  int input = C3D_AXIS_Y, weight = C3D_AXIS_X, output = C3D_AXIS_Z;
  DirectionTriple swapped() const { return {output, weight, input}; }
};
inline DirectionTriple triple_for_group(int g) {  // activation.hpp:28-35
  return g == 0 ? DirectionTriple{C3D_AXIS_Y, C3D_AXIS_X, C3D_AXIS_Z}
                : DirectionTriple{C3D_AXIS_Z, C3D_AXIS_X, C3D_AXIS_Y};
}
inline DirectionTriple default_directions(int layout) {  // layout.hpp:67-69
  DirectionTriple d;
  return layout == C3D_OUTPUT ? d.swapped() : d;
}

struct GroupState {  // activation.hpp:20-27
  int input_group = 0;
};

// One rank of the px x py x pz grid: the reference's Endpoint (transport.hpp:138-149).
class Endpoint {
 public:
  // Single-process, single-GPU p = 1 cube.
  explicit Endpoint(int device = 0, cudaStream_t stream = nullptr)
      : Endpoint(std::array<int, 3>{1, 1, 1}, 0, device, nullptr, stream) {}
  // One rank of a multi-GPU grid; `uid` is the 128-byte NCCL id from c3d_unique_id on
  // rank 0, shared by the caller's launcher.
  Endpoint(std::array<int, 3> dims, int rank, int device, const unsigned char* uid,
           cudaStream_t stream = nullptr)
      : dims_(dims), stream_(stream) {
    check_cuda(cudaSetDevice(device), "cudaSetDevice");
    c3d_cube* h = nullptr;
    check(c3d_cube_create(dims_.data(), rank, device, uid, &h));
    h_.reset(h);
    check(c3d_cube_info(h, &rank_, coords_.data(), nullptr));
  }
  c3d_cube* handle() const { return h_.get(); }
  cudaStream_t stream() const { return stream_; }
  int rank() const { return rank_; }
  const std::array<int, 3>& coords() const { return coords_; }
  const std::array<int, 3>& dims() const { return dims_; }
  int p(int axis) const { return dims_[axis]; }
  void barrier() { check(c3d_cube_barrier(h_.get(), stream_)); }
  void synchronize() { check(c3d_cube_check(h_.get(), stream_)); }
  c3d_counters counters() const {
    c3d_counters c;
    check(c3d_counters_get(h_.get(), &c));
    return c;
  }
  void reset_counters() { check(c3d_counters_reset(h_.get())); }

 private:
  struct Del {
    void operator()(c3d_cube* c) const { c3d_cube_destroy(c); }
  };
  std::array<int, 3> dims_{1, 1, 1};
  std::array<int, 3> coords_{0, 0, 0};
  int rank_ = 0;
  cudaStream_t stream_ = nullptr;
  std::unique_ptr<c3d_cube, Del> h_;
};

// ----------------------------------------------------------------- tensors
struct ShardedMatrix {  // sharding.hpp:18-34
  int64_t global_rows = 0, global_cols = 0;
  int layout = C3D_INPUT;
  DirectionTriple dirs;
  int dtype = C3D_F32;
  int64_t rows = 0, cols = 0;  // local shard
  std::shared_ptr<DeviceBuffer> shard;

  c3d_matrix c() const {
    c3d_matrix m;
    m.data = shard ? shard->get() : nullptr;
    m.dtype = dtype;
    m.global_rows = global_rows;
    m.global_cols = global_cols;
    m.layout = layout;
    m.dirs[0] = dirs.input;
    m.dirs[1] = dirs.weight;
    m.dirs[2] = dirs.output;
    return m;
  }
};

struct DiagonalVector {  // sharding.hpp:38-47
  int64_t global_len = 0;
  int dtype = C3D_F32;
  int64_t len = 0;  // local slice (0 off the diagonal)
  std::shared_ptr<DeviceBuffer> slice;
  c3d_vector c() const {
    c3d_vector v;
    v.data = slice ? slice->get() : nullptr;
    v.dtype = dtype;
    v.global_len = global_len;
    return v;
  }
};

struct Activation3D {  // activation.hpp:41-62
  int64_t batch = 0, seq = 0, hidden = 0;
  int group = 0;
  int dtype = C3D_F32;
  int64_t rows = 0, cols = 0;  // local [(b/px)(s/p_in)][h/p_out]
  std::shared_ptr<DeviceBuffer> local;
  c3d_activation c() const {
    c3d_activation a;
    a.data = local ? local->get() : nullptr;
    a.dtype = dtype;
    a.batch = batch;
    a.seq = seq;
    a.hidden = hidden;
    a.group = group;
    return a;
  }
};

inline std::array<int64_t, 4> bounds(const Endpoint& ep, int layout, int64_t rows, int64_t cols,
                                     const DirectionTriple& d) {
  std::array<int64_t, 4> b{};
  const int dirs[3] = {d.input, d.weight, d.output};
  check(c3d_shard_bounds(layout, ep.dims().data(), ep.coords().data(), rows, cols, dirs, b.data()));
  return b;
}

inline ShardedMatrix empty_matrix(const Endpoint& ep, int64_t rows, int64_t cols, int layout,
                                  const DirectionTriple& d, int dtype) {
  const auto b = bounds(ep, layout, rows, cols, d);
  ShardedMatrix m;
  m.global_rows = rows;
  m.global_cols = cols;
  m.layout = layout;
  m.dirs = d;
  m.dtype = dtype;
  m.rows = b[1] - b[0];
  m.cols = b[3] - b[2];
  m.shard = std::make_shared<DeviceBuffer>(m.rows * m.cols * dtype_bytes(dtype), ep.stream());
  return m;
}

inline DiagonalVector empty_vector(const Endpoint& ep, int64_t n, int dtype = C3D_F32) {
  int holds = 0;
  int64_t r[2] = {0, 0};
  check(c3d_diagonal_slice(ep.dims().data(), ep.coords().data(), n, &holds, r));
  DiagonalVector v;
  v.global_len = n;
  v.dtype = dtype;
  v.len = holds ? r[1] - r[0] : 0;
  v.slice = std::make_shared<DeviceBuffer>(v.len * dtype_bytes(dtype), ep.stream());
  return v;
}

inline Activation3D empty_activation(const Endpoint& ep, int64_t batch, int64_t seq, int64_t hidden,
                                     int group, int dtype) {
  const int in = group == 0 ? C3D_AXIS_Y : C3D_AXIS_Z, out = group == 0 ? C3D_AXIS_Z : C3D_AXIS_Y;
  Activation3D a;
  a.batch = batch;
  a.seq = seq;
  a.hidden = hidden;
  a.group = group;
  a.dtype = dtype;
  a.rows = (batch / ep.p(C3D_AXIS_X)) * (seq / ep.p(in));
  a.cols = hidden / ep.p(out);
  a.local = std::make_shared<DeviceBuffer>(a.rows * a.cols * dtype_bytes(dtype), ep.stream());
  return a;
}

// Host <-> device of a local buffer (fp32 host data, converted on the host for bf16).
inline uint16_t to_bf16(float f) {
  uint32_t u;
  std::memcpy(&u, &f, 4);
  u += 0x7FFFu + ((u >> 16) & 1u);  // round to nearest even
  return static_cast<uint16_t>(u >> 16);
}
inline float from_bf16(uint16_t h) {
  const uint32_t u = static_cast<uint32_t>(h) << 16;
  float f;
  std::memcpy(&f, &u, 4);
  return f;
}
inline void to_device(const Endpoint& ep, const std::vector<float>& host, DeviceBuffer& dst,
                      int dtype) {
  if (dtype == C3D_F32) {
    check_cuda(cudaMemcpyAsync(dst.get(), host.data(), host.size() * 4, cudaMemcpyHostToDevice,
                               ep.stream()),
               "cudaMemcpyAsync");
  } else {
    std::vector<uint16_t> h(host.size());
    for (size_t i = 0; i < host.size(); ++i) h[i] = to_bf16(host[i]);
    check_cuda(cudaMemcpyAsync(dst.get(), h.data(), h.size() * 2, cudaMemcpyHostToDevice,
                               ep.stream()),
               "cudaMemcpyAsync");
  }
  check_cuda(cudaStreamSynchronize(ep.stream()), "cudaStreamSynchronize");
}
inline std::vector<float> to_host(const Endpoint& ep, const DeviceBuffer& src, size_t n, int dtype) {
  std::vector<float> out(n);
  if (dtype == C3D_F32) {
    check_cuda(cudaMemcpyAsync(out.data(), src.get(), n * 4, cudaMemcpyDeviceToHost, ep.stream()),
               "cudaMemcpyAsync");
    check_cuda(cudaStreamSynchronize(ep.stream()), "cudaStreamSynchronize");
  } else {
    std::vector<uint16_t> h(n);
    check_cuda(cudaMemcpyAsync(h.data(), src.get(), n * 2, cudaMemcpyDeviceToHost, ep.stream()),
               "cudaMemcpyAsync");
    check_cuda(cudaStreamSynchronize(ep.stream()), "cudaStreamSynchronize");
    for (size_t i = 0; i < n; ++i) out[i] = from_bf16(h[i]);
  }
  return out;
}

// ----------------------------------------------------------- 3-D matmuls
struct MatmulGrads {  // ops3d.hpp:134-136
  ShardedMatrix da, db;
};

// `out_dtype` < 0: the operands' type (bf16 operands accumulate in fp32 either way).
inline ShardedMatrix matmul_ab_fwd(Endpoint& ep, const ShardedMatrix& a, const ShardedMatrix& b,
                                   int mode = C3D_MODE_AUTO, int out_dtype = -1) {
  ShardedMatrix c = empty_matrix(ep, a.global_rows, b.global_cols, C3D_OUTPUT, a.dirs.swapped(),
                                 out_dtype < 0 ? a.dtype : out_dtype);
  c3d_matrix ca = a.c(), cb = b.c(), cc = c.c();
  check(c3d_matmul_ab_fwd(ep.handle(), mode, &ca, &cb, &cc, ep.stream()));
  return c;
}

inline MatmulGrads matmul_ab_bwd(Endpoint& ep, const ShardedMatrix& dc, const ShardedMatrix& a,
                                 const ShardedMatrix& b, int mode = C3D_MODE_AUTO,
                                 int out_dtype = -1) {
  const int odt = out_dtype < 0 ? a.dtype : out_dtype;
  MatmulGrads g{empty_matrix(ep, a.global_rows, a.global_cols, a.layout, a.dirs, odt),
                empty_matrix(ep, b.global_rows, b.global_cols, C3D_WEIGHT, b.dirs, odt)};
  c3d_matrix cdc = dc.c(), ca = a.c(), cb = b.c(), cda = g.da.c(), cdb = g.db.c();
  check(c3d_matmul_ab_bwd(ep.handle(), mode, &cdc, &ca, &cb, &cda, &cdb, ep.stream()));
  return g;
}

// ------------------------------------------------------------ NN blocks
struct TransformerConfig {  // nn.hpp:16-41
  int64_t batch = 0, seq = 0, heads = 0, hidden = 0;
  double eps = 1e-5;
  c3d_config c() const { return {batch, seq, heads, hidden, eps}; }
};

// Saved-for-backward state (reference: caller-owned structs filled through Saved*).
class Saved {
 public:
  c3d_saved** out() { return &h_; }
  const c3d_saved* get() const { return h_; }
  Saved() = default;
  Saved(const Saved&) = delete;
  Saved& operator=(const Saved&) = delete;
  ~Saved() {
    if (h_) c3d_saved_free(h_);
  }

 private:
  c3d_saved* h_ = nullptr;
};
using LinearSaved = Saved;
using LayerNormSaved = Saved;
using LayerSaved = Saved;

struct LinearParams {  // nn.hpp:62-67
  ShardedMatrix weight;
  DiagonalVector bias;
  int input_group = 0;
  c3d_linear_params c() const { return {weight.c(), bias.c(), input_group}; }
};
struct LinearGrads {  // nn.hpp:74-78
  Activation3D dx;
  ShardedMatrix dweight;
  DiagonalVector dbias;
};

inline Activation3D linear3d_fwd(Endpoint& ep, const Activation3D& x, const LinearParams& p,
                                 GroupState& gs, LinearSaved* saved = nullptr,
                                 int mode = C3D_MODE_AUTO) {
  Activation3D y = empty_activation(ep, x.batch, x.seq, p.weight.global_cols, 1 - x.group, x.dtype);
  c3d_activation cx = x.c(), cy = y.c();
  c3d_linear_params cp = p.c();
  Saved local;
  check(c3d_linear_fwd(ep.handle(), mode, &cx, &cp, &gs.input_group, &cy,
                       saved ? saved->out() : local.out(), ep.stream()));
  return y;
}

inline LinearGrads linear3d_bwd(Endpoint& ep, const Activation3D& dy, const LinearSaved& saved,
                                const LinearParams& p, int mode = C3D_MODE_AUTO) {
  LinearGrads g{empty_activation(ep, dy.batch, dy.seq, p.weight.global_rows, p.input_group, dy.dtype),
                empty_matrix(ep, p.weight.global_rows, p.weight.global_cols, C3D_WEIGHT,
                             p.weight.dirs, C3D_F32),
                empty_vector(ep, p.weight.global_cols)};
  c3d_activation cdy = dy.c(), cdx = g.dx.c();
  c3d_linear_params cp = p.c();
  c3d_matrix cdw = g.dweight.c();
  c3d_vector cdb = g.dbias.c();
  check(c3d_linear_bwd(ep.handle(), mode, &cdy, saved.get(), &cp, &cdx, &cdw, &cdb, ep.stream()));
  return g;
}

struct LayerNormParams {  // nn.hpp:119-124
  DiagonalVector gamma, beta;
  double eps = 1e-5;
};
struct LayerNormGrads {  // nn.hpp:131-135
  Activation3D dx;
  DiagonalVector dgamma, dbeta;
};

inline Activation3D layernorm3d_fwd(Endpoint& ep, const Activation3D& x, const LayerNormParams& p,
                                    LayerNormSaved* saved = nullptr) {
  Activation3D y = empty_activation(ep, x.batch, x.seq, x.hidden, x.group, x.dtype);
  c3d_activation cx = x.c(), cy = y.c();
  c3d_layernorm_params cp{p.gamma.c(), p.beta.c(), p.eps};
  Saved local;
  check(c3d_layernorm_fwd(ep.handle(), &cx, &cp, &cy, saved ? saved->out() : local.out(),
                          ep.stream()));
  return y;
}

inline LayerNormGrads layernorm3d_bwd(Endpoint& ep, const Activation3D& dy,
                                      const LayerNormSaved& saved) {
  LayerNormGrads g{empty_activation(ep, dy.batch, dy.seq, dy.hidden, dy.group, dy.dtype),
                   empty_vector(ep, dy.hidden), empty_vector(ep, dy.hidden)};
  c3d_activation cdy = dy.c(), cdx = g.dx.c();
  c3d_vector cg = g.dgamma.c(), cb = g.dbeta.c();
  check(c3d_layernorm_bwd(ep.handle(), &cdy, saved.get(), &cdx, &cg, &cb, ep.stream()));
  return g;
}

// LayerParams / LayerGrads (transformer.hpp:78-101).
struct LayerParams {
  DiagonalVector ln1_gamma, ln1_beta;
  ShardedMatrix w_qkv;
  DiagonalVector b_qkv;
  ShardedMatrix w_out;
  DiagonalVector b_out;
  DiagonalVector ln2_gamma, ln2_beta;
  ShardedMatrix w_fc1;
  DiagonalVector b_fc1;
  ShardedMatrix w_fc2;
  DiagonalVector b_fc2;
  c3d_layer_params c() const {
    return {ln1_gamma.c(), ln1_beta.c(), w_qkv.c(), b_qkv.c(), w_out.c(), b_out.c(),
            ln2_gamma.c(), ln2_beta.c(), w_fc1.c(), b_fc1.c(), w_fc2.c(), b_fc2.c()};
  }
};
struct LayerGrads {
  Activation3D dx;
  LayerParams dparams;  // same shapes as the parameters, fp32
};

// Parameters of one layer for this rank from global host matrices (partition_layer_params,
// transformer.hpp:223-254): QKV and FC1 under the input group's triple, OUT and FC2 under
// the swapped one, vectors on the diagonal.
inline LayerParams empty_layer_params(const Endpoint& ep, int64_t hidden, int input_group,
                                      int dtype) {
  const DirectionTriple din = triple_for_group(input_group), dsw = triple_for_group(1 - input_group);
  const int64_t h = hidden;
  LayerParams p;
  p.ln1_gamma = empty_vector(ep, h);
  p.ln1_beta = empty_vector(ep, h);
  p.w_qkv = empty_matrix(ep, h, 3 * h, C3D_WEIGHT, din, dtype);
  p.b_qkv = empty_vector(ep, 3 * h);
  p.w_out = empty_matrix(ep, h, h, C3D_WEIGHT, dsw, dtype);
  p.b_out = empty_vector(ep, h);
  p.ln2_gamma = empty_vector(ep, h);
  p.ln2_beta = empty_vector(ep, h);
  p.w_fc1 = empty_matrix(ep, h, 4 * h, C3D_WEIGHT, din, dtype);
  p.b_fc1 = empty_vector(ep, 4 * h);
  p.w_fc2 = empty_matrix(ep, 4 * h, h, C3D_WEIGHT, dsw, dtype);
  p.b_fc2 = empty_vector(ep, h);
  return p;
}

inline Activation3D transformer_layer_fwd(Endpoint& ep, const Activation3D& x, const LayerParams& p,
                                          const TransformerConfig& cfg, GroupState& gs,
                                          LayerSaved* saved = nullptr, int mode = C3D_MODE_AUTO) {
  Activation3D y = empty_activation(ep, x.batch, x.seq, x.hidden, x.group, x.dtype);
  c3d_activation cx = x.c(), cy = y.c();
  c3d_layer_params cp = p.c();
  c3d_config cc = cfg.c();
  Saved local;
  check(c3d_layer_fwd(ep.handle(), mode, &cc, &cx, &cp, &gs.input_group, &cy,
                      saved ? saved->out() : local.out(), ep.stream()));
  return y;
}

inline LayerGrads transformer_layer_bwd(Endpoint& ep, const Activation3D& dy, const LayerSaved& saved,
                                        const LayerParams& p, const TransformerConfig& cfg,
                                        int mode = C3D_MODE_AUTO) {
  LayerGrads g{empty_activation(ep, dy.batch, dy.seq, dy.hidden, dy.group, dy.dtype),
               empty_layer_params(ep, cfg.hidden, p.w_qkv.dirs.input == C3D_AXIS_Y ? 0 : 1, C3D_F32)};
  c3d_activation cdy = dy.c(), cdx = g.dx.c();
  c3d_layer_params cp = p.c(), cg = g.dparams.c();
  c3d_config cc = cfg.c();
  check(c3d_layer_bwd(ep.handle(), mode, &cc, &cdy, saved.get(), &cp, &cdx, &cg, ep.stream()));
  return g;
}

}  // namespace cube3d_b200

#endif  // CUBE3D_B200_HPP_
