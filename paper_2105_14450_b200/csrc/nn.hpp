// 3-D Transformer blocks (cube3d/nn.hpp, cube3d/attention.hpp, cube3d/transformer.hpp).
#pragma once

#include <cuda_runtime.h>

#include <deque>
#include <memory>
#include <vector>

#include "ops.hpp"

namespace c3d {

// Activation3D (cube3d/activation.hpp:41-62) with resolved local dims.
struct Act {
  void* data = nullptr;
  int dtype = kBF16;
  int64_t batch = 0, seq = 0, hidden = 0;
  int group = 0;
  int64_t rows = 0, cols = 0;
  size_t elems() const { return static_cast<size_t>(rows * cols); }
};
Act make_act(const Cube& cube, void* data, int dtype, int64_t batch, int64_t seq, int64_t hidden,
             int group);
Mat flatten(const Cube& cube, const Act& a);

struct Config {
  int64_t batch = 0, seq = 0, heads = 0, hidden = 0;
  double eps = 1e-5;
};
void validate_config(const Cube& cube, const Config& cfg);

struct LinearP {
  Mat w;
  Vec b;
  int input_group = 0;
};

// Saved-for-backward state: owns its device buffers.
struct Saved {
  virtual ~Saved() = default;
  std::deque<DevBuf> bufs;  // deque: references stay valid as buffers are added
  DevBuf& keep(DevBuf&& b) {
    bufs.push_back(std::move(b));
    return bufs.back();
  }
};

struct LinearSaved : Saved {
  Mat x;           // flattened forward input (LinearSaved::x_flat, cube3d/nn.hpp:69-72)
  Gathered a_full;  // the input as gathered by the forward (reused by the dW product)
};

// Layer-level precomputation handed to one linear: its bias already expanded and its
// weight already gathered along x (one packed collective per layer for all of them).
struct LinearPre {
  const float* bias = nullptr;
  Operand wg;
};
// Backward destinations for packed, deferred reductions: the bias column sums and the
// un-reduced weight-gradient partial (reduced once per layer).
struct LinearSinks {
  float* bias_colsum = nullptr;
  bool bias_elsewhere = false;  // the bias gradient is summed by another pass (LN backward)
  DwSink dw;
};
struct LNSaved : Saved {
  void* xhat = nullptr;
  int dtype = kBF16;
  float* inv_std = nullptr;
  float* gamma_block = nullptr;
  int group = 0;
  int64_t hidden = 0;
};
struct AttnSaved : Saved {
  LinearSaved qkv_lin, out_lin;
  Act qkv;                 // (b/px)(s/p_s) x 3h/p_h, head-major [head][q|k|v][dim]
  void* q_full = nullptr;  // gathered queries [p_s][rows][H*dh] (p_s > 1)
  void* probs = nullptr;   // [b_loc*H][s][s_loc] (unfused paths)
  float* lse = nullptr;    // [b_loc*H][s] row log-sum-exp, log2 units (flash path)
};
struct MlpSaved : Saved {
  LinearSaved fc1_lin, fc2_lin;
  void* pre_act = nullptr;
};
struct LayerSaved : Saved {
  LNSaved ln1, ln2;
  AttnSaved attn;
  MlpSaved mlp;
  // expanded vectors (group-g triple: ln1 g/b, b_out, ln2 g/b, b_fc2; other triple:
  // b_qkv, b_fc1) and the packed x-gathered weights, shared by forward and backward
  std::vector<const float*> vec0, vec1;
  Operand wg[4];  // qkv, out, fc1, fc2
};

// 3-D cross-entropy (loss.cu): logits kept in fp32 with their row statistics.
struct LossSaved : Saved {
  LinearSaved lin;
  Act logits;  // fp32
  float* mx = nullptr;
  float* st = nullptr;  // [sum exp | target logit], all-reduced along the vocabulary axis
  const int32_t* targets = nullptr;
  int64_t col0 = 0, tokens = 0;
  int64_t map_w = 0, map_a = 0;
};

struct LayerP {
  Vec ln1_g, ln1_b;
  LinearP qkv, out;
  Vec ln2_g, ln2_b;
  LinearP fc1, fc2;
};
struct LayerG {  // gradients (outputs), same shapes as LayerP
  Vec ln1_g, ln1_b;
  Mat w_qkv;
  Vec b_qkv;
  Mat w_out;
  Vec b_out;
  Vec ln2_g, ln2_b;
  Mat w_fc1;
  Vec b_fc1;
  Mat w_fc2;
  Vec b_fc2;
};

// `own_input`: copy x into the saved state (standalone API); otherwise keep a view
// (the caller guarantees x outlives backward, as inside a layer).
void linear_fwd(Cube& cube, int mode, const Act& x, const LinearP& p, int& group, Act& y,
                LinearSaved* saved, bool own_input, const LinearEpi& extra, cudaStream_t s,
                const LinearPre* pre = nullptr);
void linear_bwd(Cube& cube, int mode, const Act& dy, const LinearSaved& saved, const LinearP& p,
                Act* dx, Mat* dw, const Vec* db, const void* dx_gelu_aux, cudaStream_t s,  // aux: gelu'(x) values (kActMulAux)
                const Operand* wg = nullptr, const LinearSinks* sinks = nullptr);

// `gblock`/`bblock`: gamma/beta already expanded (layer-level); `colsum_sink`: write
// [dgamma block | dbeta block] column sums there instead of reducing them here.
void layernorm_fwd(Cube& cube, const Act& x, const Vec& gamma, const Vec& beta, double eps,
                   Act& y, LNSaved* saved, cudaStream_t s, const float* gblock = nullptr,
                   const float* bblock = nullptr);
// `colsum_sink`: dgamma | dbeta column sums land there (the caller reduces them);
// `resid_sink`: also the residual's column sum (bias gradient of the linear whose output
// gradient the residual is), from the same pass when the fused kernel applies.
void layernorm_bwd(Cube& cube, const Act& dy, const LNSaved& saved, Act& dx, const Vec* dgamma,
                   const Vec* dbeta, const void* resid, cudaStream_t s,
                   float* colsum_sink = nullptr, float* resid_sink = nullptr);

void attention_fwd(Cube& cube, int mode, const Config& cfg, const Act& x, const LinearP& qkv,
                   const LinearP& out, int& group, Act& y, AttnSaved* saved, bool own_input,
                   const void* resid, cudaStream_t s, const LinearPre* qkv_pre = nullptr,
                   const LinearPre* out_pre = nullptr);
void attention_bwd(Cube& cube, int mode, const Config& cfg, const Act& dy, const AttnSaved& sv,
                   const LinearP& qkv, const LinearP& out, Act& dx, LayerG& g, cudaStream_t s,
                   const Operand* qkv_wg = nullptr, const Operand* out_wg = nullptr,
                   const LinearSinks* qkv_sinks = nullptr, const LinearSinks* out_sinks = nullptr);

void mlp_fwd(Cube& cube, int mode, const Config& cfg, const Act& x, const LinearP& fc1,
             const LinearP& fc2, int& group, Act& y, MlpSaved* saved, bool own_input,
             const void* resid, cudaStream_t s, const LinearPre* fc1_pre = nullptr,
             const LinearPre* fc2_pre = nullptr);
void mlp_bwd(Cube& cube, int mode, const Config& cfg, const Act& dy, const MlpSaved& sv,
             const LinearP& fc1, const LinearP& fc2, Act& dx, LayerG& g, cudaStream_t s,
             const Operand* fc1_wg = nullptr, const Operand* fc2_wg = nullptr,
             const LinearSinks* fc1_sinks = nullptr, const LinearSinks* fc2_sinks = nullptr);

// transformer_stack_fwd/bwd (cube3d/transformer.hpp:150-176): the layer loop, the
// backward in reverse. Intermediate activations are owned by the saved state.
struct StackSaved : Saved {
  std::vector<std::unique_ptr<LayerSaved>> layers;
};
void stack_fwd(Cube& cube, int mode, const Config& cfg, const Act& x,
               const std::vector<LayerP>& ps, int& group, Act& y, StackSaved* saved,
               cudaStream_t s);
void stack_bwd(Cube& cube, int mode, const Config& cfg, const Act& dy, const StackSaved& sv,
               const std::vector<LayerP>& ps, Act& dx, std::vector<LayerG>& gs, cudaStream_t s);

// Mean cross-entropy of softmax(x W + b) against global token targets (int32 [batch *
// seq], device); `loss` is one device float (identical on every rank). `targets` must
// stay valid until loss_bwd.
void loss_fwd(Cube& cube, int mode, const Act& x, const LinearP& head, const int32_t* targets,
              int& group, float* loss, LossSaved* saved, cudaStream_t s);
void loss_bwd(Cube& cube, int mode, const LossSaved& sv, const LinearP& head, Act* dx, Mat* dw,
              const Vec* db, int grad_dtype, cudaStream_t s);

void layer_fwd(Cube& cube, int mode, const Config& cfg, const Act& x, const LayerP& p, int& group,
               Act& y, LayerSaved* saved, cudaStream_t s);
void layer_bwd(Cube& cube, int mode, const Config& cfg, const Act& dy, const LayerSaved& sv,
               const LayerP& p, Act& dx, LayerG& g, cudaStream_t s);

}  // namespace c3d
