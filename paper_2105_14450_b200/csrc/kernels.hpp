// HBM-bound row / column / elementwise kernels of the layer path. Each cites the
// reference loop it replaces.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "gemm.hpp"

namespace c3d {

// Generic elementwise epilogue over a contiguous rows x cols matrix `in`
// (same semantics as the GEMM epilogue with acc = in[m][n]); e.out may alias in.
// Covers add_vec_fwd (cube3d/ops3d.hpp:352-356), GELU (cube3d/transformer.hpp:51),
// GELU' (cube3d/transformer.hpp:60-61) and the residual add_into (:105-111).
void k_apply_epilogue(const void* in, int in_dtype, int64_t rows, int64_t cols,
                      const Epilogue& e, cudaStream_t s);

// out[c] = sum_r x[r][c] (* y[r][c] if y), fp32, deterministic order; with out_x also
// out_x[c] = sum_r x[r][c] from the same pass (LayerNorm dgamma and dbeta together).
// add_vec_bwd colsum (cube3d/ops3d.hpp:365-367), mul_vec_bwd (:408-413), LN dbeta/dgamma.
void k_colsum(const void* x, int xdt, const void* y, int ydt, int64_t rows, int64_t cols,
              float* out, cudaStream_t s, float* out_x = nullptr);

void k_convert(const void* src, int sdt, void* dst, int ddt, int64_t n, cudaStream_t s);
// Several conversions in one launch (grid.y = segment).
struct ConvSeg {
  const void* src;
  void* dst;
  int sdt, ddt;
  int64_t n;
};
struct ConvBatch {
  static constexpr int kMax = 8;
  ConvSeg seg[kMax];
};
void k_convert_batch(const ConvSeg* segs, int n, cudaStream_t s);
// out[j] = sum over p < parts of partial[p][j] (j < width), in part order.
void k_colsum_parts(const float* partial, int parts, int64_t width, float* out, cudaStream_t s);
// y = gelu(x), x <- gelu'(x) (n elements, in place on x).
void k_gelu_save(void* x, int xdt, void* y, int ydt, int64_t n, cudaStream_t s);

// c[r][col] = a[r][col] * b[col] (mul_vec_fwd, cube3d/ops3d.hpp:391-393).
void k_mul_cols(const void* a, int adt, const float* b, void* c, int cdt, int64_t rows,
                int64_t cols, cudaStream_t s);

// ---- LayerNorm (cube3d/nn.hpp:140-222) ----
// out[r] = sum_c x[r][c]               (mean == nullptr)
// out[r] = sum_c (x[r][c] - mean[r])^2 (mean given; `sum_is_total`: mean = out_sum*inv_h)
void k_row_sum(const void* x, int dt, int64_t rows, int64_t cols, const float* sums,
               float inv_h, float* out, cudaStream_t s);
// y = gamma * xhat + beta with xhat = (x - sum*inv_h) * rsqrt(sq*inv_h + eps).
void k_ln_apply(const void* x, int dt, int64_t rows, int64_t cols, const float* sums,
                const float* sq, float inv_h, float eps, const float* gamma, const float* beta,
                void* y, int ydt, void* xhat, int xhdt, float* inv_std, cudaStream_t s);
// Single-kernel forward when the hidden dimension is not partitioned.
void k_ln_fwd_fused(const void* x, int dt, int64_t rows, int64_t cols, float eps,
                    const float* gamma, const float* beta, void* y, int ydt, void* xhat,
                    int xhdt, float* inv_std, cudaStream_t s);
// row_sum[r] = sum_c dy*gamma, row_dot[r] = sum_c dy*gamma*xhat (into rs[0:rows], rs[rows:2rows]).
// Distributed LayerNorm statistics in one collective: local (mean, M2) per row, gathered
// along the output axis ([P][rows][2]) and merged (Chan et al.) into sums / centred sum of
// squares for k_ln_apply. k_row_moments returns false without a vectorised form.
bool k_row_moments(const void* x, int dt, int64_t rows, int64_t cols, float* st, cudaStream_t s);
void k_combine_moments(const float* st, int P, int64_t rows, int64_t n, float* sums, float* sq,
                       cudaStream_t s);
// p_out = 1 backward in one pass (row sums and dx); false when the shape has no
// vectorised form (the caller then runs k_ln_bwd_rows + k_ln_bwd_dx).
// LayerNorm backward of bf16 rows with its column sums in the same pass: dgamma = sum
// dy * xhat, dbeta = sum dy, and (resid given) dx += resid, dresid = sum resid. False (nothing
// launched) when the shape / dtypes / alignment do not fit; resid and dresid go together.
bool k_ln_bwd_sums(const void* dy, int dt, const void* xhat, int xdt, const float* gamma,
                   const float* inv_std, int64_t rows, int64_t cols, const void* resid, int rdt,
                   void* dx, int dxdt, float* dgamma, float* dbeta, float* dresid,
                   cudaStream_t s);
bool k_ln_bwd_fused(const void* dy, int dt, const void* xhat, int xdt, const float* gamma,
                    const float* inv_std, int64_t rows, int64_t cols, const void* resid, int rdt,
                    void* dx, int dxdt, cudaStream_t s);
void k_ln_bwd_rows(const void* dy, int dt, const void* xhat, int xdt, const float* gamma,
                   int64_t rows, int64_t cols, float* rs, cudaStream_t s);
// dx = inv_std*(dy*gamma - row_sum*inv_h - xhat*row_dot*inv_h) (+ resid).
void k_ln_bwd_dx(const void* dy, int dt, const void* xhat, int xdt, const float* gamma,
                 const float* inv_std, const float* rs, float inv_h, int64_t rows, int64_t cols,
                 const void* resid, int rdt, void* dx, int dxdt, cudaStream_t s);

// ---- attention softmax (cube3d/attention.hpp:106-126, 161-169) ----
// Scores / dP are fp32 (bf16 logits would distort exp after LayerNorm); the
// probabilities P and dS are written in the activation dtype for the GEMMs.
void k_softmax_rowmax(const float* sc, int64_t rows, int64_t cols, float* mx, cudaStream_t s);
void k_softmax_rowexpsum(const float* sc, int64_t rows, int64_t cols, const float* mx,
                         float* sum, cudaStream_t s);
void k_softmax_norm(const float* sc, int64_t rows, int64_t cols, const float* mx,
                    const float* sum, void* p, int pdt, cudaStream_t s);
void k_softmax_fused(const float* sc, int64_t rows, int64_t cols, void* p, int pdt,
                     cudaStream_t s);
void k_softmax_bwd_rowdot(const float* dp, const void* p, int pdt, int64_t rows, int64_t cols,
                          float* rowdot, cudaStream_t s);
void k_softmax_bwd_ds(const float* dp, const void* p, int pdt, int64_t rows, int64_t cols,
                      const float* rowdot, float scale, void* ds, int dsdt, cudaStream_t s);
// ---- cross-entropy (loss.cu): local logits row -> global token and vocabulary offset
struct LossMap {
  int64_t w = 0, a = 0;      // coordinates on x and on the logits' input axis
  int64_t bl = 0, sl = 0;    // local batch and sequence extents
  int64_t seq = 0;           // global sequence length
  int64_t col0 = 0;          // first vocabulary column of the local block
};
void k_loss_stats(const float* logits, int64_t rows, int64_t cols, const float* mx,
                  const int32_t* targets, const LossMap& map, float* st, cudaStream_t s);
void k_loss_reduce(const float* mx, const float* st, int64_t rows, float scale, float* out,
                   cudaStream_t s);
void k_loss_grad(const float* logits, int64_t rows, int64_t cols, const float* mx, const float* st,
                 const int32_t* targets, const LossMap& map, float scale, void* out, int dt,
                 cudaStream_t s);

// Row dot products sum_d dO*O of packed [bi][q][head][dh] buffers (softmax backward).
void k_attn_rowdot(const void* d_o, const void* o, int dt, int64_t nslices, int64_t S, int64_t H,
                   int64_t dh, int64_t sb_hi, float* out, cudaStream_t s);
void k_softmax_bwd_fused(const float* dp, const void* p, int pdt, int64_t rows, int64_t cols,
                         float scale, void* ds, int dsdt, cudaStream_t s);

// dst[r][h*dst_hs + t] = src[r][h*src_hs + t], t < dh (head-major column blocks).
void k_copy_heads(const void* src, int64_t src_ld, int64_t src_hs, void* dst, int64_t dst_ld,
                  int64_t dst_hs, int64_t rows, int64_t heads, int64_t dh, int dt,
                  cudaStream_t s);

}  // namespace c3d
