// 3-D parallel operators (cube3d/ops3d.hpp) over device-resident shards.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <memory>
#include <vector>

#include "cube.hpp"
#include "gemm.hpp"
#include "grid.hpp"

namespace c3d {

void run_gemm(const GemmProblem& p, int mode, int num_sms, cudaStream_t s);
void prof_enable(bool on);
void prof_read(double* ms, double* flops, long long* launches);
void prof_read_comm(double* ms, double* bytes, long long* calls);

// Flash attention core (flash.cu), bf16, head dim 64 or 128, queries and keys multiples
// of 128. Forward: ctx = softmax(scale q k^T) v per slice (normalised over this rank's
// keys) and lse[slice][S] = log2-domain log-sum-exp of (scale log2e) q k^T. Backward:
// dq, dk, dv from q, k, v, dO, lse and rowdot D = rowsum(dO * O); `ws` is an fp32
// scratch of flash_bwd_workspace_bytes() (no initialisation needed).
// `rd_split` > 0: rowdot is laid out [S / rd_split][slices][rd_split] (all-gathered along
// the seq axis); q / dO and dq may be row-split (gathered, partial). Both return false (nothing launched) outside the
// supported shapes / layouts.
bool flash_supported(int64_t S, int64_t keys, int64_t dh);
bool flash_fwd(const View& q, const View& k, const View& v_mn, const View& ctx, float* lse,
               int64_t S, int64_t keys, int64_t dh, int64_t H, int nslices, float scale,
               cudaStream_t s);
// Key range split along the seq axis: w = exp2(lse_r - M) (M the all-reduced max), then
// partial *= exp2(lse_r - M) / W (W the all-reduced sum of w) and lse_io: M -> M + log2 W.
void k_flash_lse_weights(const float* lr, const float* mx, float* w, int64_t n, cudaStream_t s);
void k_flash_combine(const View& partial, const float* lr, float* lse_io, const float* W, int64_t S,
                     int64_t dh, int64_t H, int nslices, cudaStream_t s);
size_t flash_bwd_workspace_bytes(int64_t S, int64_t dh, int nslices);
bool flash_bwd(const View& q, const View& k, const View& v, const View& d_o, const float* lse,
               const float* rowdot, int64_t rd_split, const View& dq, const View& dk, const View& dv,
               void* ws, int64_t S, int64_t keys, int64_t dh, int64_t H, int nslices, float scale,
               cudaStream_t s, float* bias_part = nullptr);

// One (batched) local GEMM on this rank, charging batch*M*N*K multiply-adds.
void gemm_views(Cube& cube, int mode, int64_t M, int64_t N, int64_t K, int batch, const View& a,
                const View& b, const Epilogue& e, cudaStream_t s);

// ShardedMatrix with its local shard dims resolved (cube3d/sharding.hpp:18-34).
struct Mat {
  void* data = nullptr;
  int dtype = kBF16;
  int64_t grows = 0, gcols = 0;
  int layout = kInput;
  Dirs dirs;
  int64_t rows = 0, cols = 0;  // local shard
  size_t elems() const { return static_cast<size_t>(rows * cols); }
};

Mat make_mat(const Cube& cube, void* data, int dtype, int64_t grows, int64_t gcols, int layout,
             const Dirs& dirs);
Mat from_c(const Cube& cube, const c3d_matrix& m);
void to_c(const Mat& m, c3d_matrix* out);

// DiagonalVector (cube3d/sharding.hpp:38-47).
struct Vec {
  void* data = nullptr;
  int dtype = kF32;
  int64_t len = 0;
};

// Device buffer holding the gathered operand, or the shard itself when the axis
// has extent 1.
struct Gathered {
  DevBuf buf;
  std::unique_ptr<SymBuf> sym;  // gathered in place in the symmetric arena (fused path)
  const void* ptr = nullptr;
};
Gathered gather(Cube& cube, int axis, const void* shard, size_t count, int dtype, cudaStream_t s);

// Local GEMM whose row blocks are reduce-scattered along `axis` inside its epilogue over
// NVLink peer memory (fused.cu); `post` (out = this rank's contiguous result block) is
// applied after the sum. Returns false (nothing launched) when the fused path does not
// apply -- the decision is identical on every rank -- and the caller falls back.
bool gemm_reduce_scatter(Cube& cube, int mode, int axis, int64_t M, int64_t N, int64_t K,
                         const View& a, const View& b, const Epilogue& post, cudaStream_t s);


// expand_diagonal (cube3d/ops3d.hpp:291-310): fp32 column block of length len/p_out
// for an operand with triple d. Returns a stream-ordered fp32 buffer.
DevBuf expand_diagonal(Cube& cube, const Dirs& d, const Vec& v, cudaStream_t s);
// Several vectors sharing triple d in one broadcast + one all-gather: the result holds
// their fp32 column blocks back to back; blocks[k] points at vector k's block.
DevBuf expand_diagonal_multi(Cube& cube, const Dirs& d, const std::vector<Vec>& vs,
                             std::vector<const float*>* blocks, cudaStream_t s);
// reduce_to_diagonal (cube3d/ops3d.hpp:315-336) of `nvec` packed fp32 column-sum vectors
// (each of length len/p_out) into the vectors out[0..nvec) on holder ranks.
void reduce_to_diagonal(Cube& cube, const Dirs& d, const float* colsums, int nvec,
                        const Vec* outs, cudaStream_t s);
// Same for vectors of different lengths: colsums holds their column-sum blocks
// (len_k / p_out each) back to back; one reduce-scatter + one all-reduce in total.
void reduce_to_diagonal_multi(Cube& cube, const Dirs& d, const float* colsums,
                              const std::vector<Vec>& outs, cudaStream_t s);

// An operand already gathered along its axis: [P][shard] blocks `s_hi` elements apart.
// Batch / sequence structure of an activation operand (Activation3D rows are [batch][seq]);
// needed by the linear on grids with py != pz, where the row blocks of a gather / scatter
// along the input and output axes interleave differently.
struct ActRows {
  int64_t bl = 0;   // local batch (b / px)
  int64_t seq = 0;  // global sequence length
};
struct Operand {
  const void* ptr = nullptr;
  long long s_hi = 0;
};
// Destination of an un-reduced weight-gradient partial inside a packed buffer that is
// reduce-scattered along x once for all weights: column-block-major, blocks s_hi apart.
struct DwSink {
  void* base = nullptr;
  long long s_hi = 0;
  int dtype = kF32;
};

void matmul_ab_fwd(Cube& cube, int mode, const Mat& a, const Mat& b, Mat& c, cudaStream_t s);
void matmul_ab_bwd(Cube& cube, int mode, const Mat& dc, const Mat& a, const Mat& b, Mat& da,
                   Mat& db, cudaStream_t s);
void matmul_abt_fwd(Cube& cube, int mode, const Mat& a, const Mat& b, Mat& c, cudaStream_t s);
void matmul_abt_bwd(Cube& cube, int mode, const Mat& dc, const Mat& a, const Mat& b, Mat& da,
                    Mat& db, cudaStream_t s);
void matmul_atb_fwd(Cube& cube, int mode, const Mat& a, const Mat& b, Mat& c, cudaStream_t s);
void matmul_atb_bwd(Cube& cube, int mode, const Mat& dc, const Mat& a, const Mat& b, Mat& da,
                    Mat& db, cudaStream_t s);

void add_vec_fwd(Cube& cube, const Mat& a, const Vec& b, Mat& c, cudaStream_t s);
void add_vec_bwd(Cube& cube, const Mat& dc, Mat& da, const Vec& db, cudaStream_t s);
void mul_vec_fwd(Cube& cube, const Mat& a, const Vec& b, Mat& c, cudaStream_t s);
void mul_vec_bwd(Cube& cube, const Mat& dc, const Mat& a, const Vec& b, Mat& da, const Vec& db,
                 cudaStream_t s);

// Linear-layer building block shared by matmul_ab_fwd and linear3d_fwd: C = A B with an
// optional fused epilogue (bias already expanded, activation, residual).
struct LinearEpi {
  const float* bias = nullptr;  // expanded column block (len = C local cols)
  int act = kActNone;
  void* pre_act = nullptr;      // stores pre-activation (C layout)
  const void* resid = nullptr;  // C layout, C dtype
};
// `bg`: B already gathered along x (skips the gather). `keep_a`: receives the gathered A
// (the caller keeps it for the backward instead of re-gathering, cube3d/ops3d.hpp:160).
void ab_forward(Cube& cube, int mode, const Mat& a, const Mat& b, Mat& c, const LinearEpi& epi,
                cudaStream_t s, const Operand* bg = nullptr, Gathered* keep_a = nullptr,
                const ActRows* ar = nullptr);
// dA = dC B^T (RS along d.in), dB = A^T dC (RS along x); either output may be skipped
// (data == nullptr). `da_epi_aux`: if set, dA *= gelu'(aux) is fused (aux in dA layout).
// `bg` / `ag`: pre-gathered B (along x) / A (along d.in). `dw`: write the dB partial into
// a packed sink instead of reduce-scattering it here.
void ab_backward(Cube& cube, int mode, const Mat& dc, const Mat& a, const Mat& b, Mat* da,
                 Mat* db, const void* da_gelu_aux, cudaStream_t s, const Operand* bg = nullptr,
                 const void* ag = nullptr, const DwSink* dw = nullptr, const ActRows* ar = nullptr);

}  // namespace c3d
