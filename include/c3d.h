/*
 * c3d.h -- C ABI of the B200-native 3-D parallel matmul / Transformer-layer
 * library (arXiv 2105.14450), a drop-in for the operator API of the reference
 * C++ library `cube3d` (/root/reference/proj/include/cube3d/).
 *
 * The reference has no C ABI or FFI: it is header-only C++ whose every op is
 *     R op(Endpoint<T>& ep, const In&..., [GroupState&], [Saved* = nullptr])
 * (SURVEY.md §8(b)). Each entry point below names the reference function it
 * replaces (file:line, relative to /root/reference/proj/include/). The mapping:
 *   Endpoint<T>&            -> c3d_cube*   (one per rank / GPU; NCCL + CUDA state)
 *   ShardedMatrix<T>        -> c3d_matrix  (device-resident local shard + metadata)
 *   DiagonalVector<T>       -> c3d_vector  (device-resident diagonal slice)
 *   Activation3D<T>         -> c3d_activation
 *   GroupState&             -> int* group  (in/out)
 *   Saved*                  -> c3d_saved** (opaque, library-allocated, freed by caller)
 *   cube3d::Error subclass  -> int status, one code per reference error name;
 *                              c3d_last_error() gives "Name: detail" (thread-local)
 * All ops are stream-ordered on the given cudaStream_t (passed as void*), and
 * SPMD like the reference: every rank issues the identical call sequence.
 * Shapes, layouts and directions are validated on the host before anything is
 * enqueued (cube3d/ops3d.hpp:117-124).
 *
 * Grids generalise the reference's p x p x p cube (cube3d/topology.hpp:57-118)
 * to px x py x pz; layer ops (and diagonal vectors) need py == pz -- the reference's
 * rule -- or one of py, pz equal to 1, e.g. the 2x2x1 sub-cube.
 */
#ifndef C3D_H_
#define C3D_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ------------------------------------------------------------------ status */
/* One code per reference error (cube3d/errors.hpp:24-37), same order. */
enum c3d_status {
  C3D_OK = 0,
  C3D_ERR_NOT_A_CUBE = 1,
  C3D_ERR_OUT_OF_RANGE = 2,
  C3D_ERR_LENGTH_MISMATCH = 3,
  C3D_ERR_DESYNC = 4,
  C3D_ERR_INDIVISIBLE_SHAPE = 5,
  C3D_ERR_INCONSISTENT_FAMILY = 6,
  C3D_ERR_SHAPE_MISMATCH = 7,
  C3D_ERR_DIRECTION_CLASH = 8,
  C3D_ERR_BATCH_MISMATCH = 9,
  C3D_ERR_GROUP_MISMATCH = 10,
  C3D_ERR_HEADS_INDIVISIBLE = 11,
  C3D_ERR_CONFIG_INVALID = 12,
  C3D_ERR_NON_FINITE = 13,
  C3D_ERR_IO = 14,
  C3D_ERR_CUDA = 100,
  C3D_ERR_NCCL = 101,
  C3D_ERR_INTERNAL = 102
};

/* Element types and compute modes. */
enum c3d_dtype { C3D_F32 = 0, C3D_BF16 = 1 };
enum c3d_mode {
  C3D_MODE_AUTO = 0, /* tcgen05 bf16 when operands are bf16 and TMA-addressable, else SIMT */
  C3D_MODE_TC = 1,   /* force tcgen05 bf16 x bf16 -> fp32 (error if not addressable) */
  C3D_MODE_F32 = 2   /* SIMT fp32 ("fp32-exact" oracle mode) */
};

/* Axes and layouts: cube3d/topology.hpp:15 (Axis) and cube3d/layout.hpp:29 (Layout). */
enum c3d_axis { C3D_AXIS_X = 0, C3D_AXIS_Y = 1, C3D_AXIS_Z = 2 };
enum c3d_layout {
  C3D_INPUT = 0,
  C3D_WEIGHT = 1,
  C3D_OUTPUT = 2,
  C3D_WEIGHT_OF_TRANSPOSE = 3
};

/* Collective kinds, cube3d/counters.hpp:11-17. */
enum c3d_collective {
  C3D_BROADCAST = 0,
  C3D_ALL_GATHER = 1,
  C3D_REDUCE_SCATTER = 2,
  C3D_ALL_REDUCE = 3,
  C3D_BARRIER = 4
};

const char* c3d_last_error(void);
const char* c3d_version(void);
/* Number of kernels this library has launched in this process. */
long long c3d_launch_count(void);
/* Live kernel timing: when enabled, every tcgen05 GEMM launch is bracketed by CUDA
 * events on its own stream; c3d_prof_read returns the summed per-launch time (ms),
 * summed algorithmic flops (2*M*N*K*batch) and launch count, then resets. */
int c3d_prof_enable(int on);
int c3d_prof_read(double* ms, double* flops, long long* launches);
/* Same for the collectives recorded since c3d_prof_enable: summed per-call time (ms),
 * summed payload bytes (full gathered / pre-scatter buffer) and call count. */
int c3d_prof_read_comm(double* ms, double* bytes, long long* calls);

/* ------------------------------------------------------ pure host: inputs */
/* Rng (cube3d/rng.hpp:17-34): mt19937_64 with the reference's explicit 53-bit
 * mapping, so seeded synthetic inputs are bit-identical to the reference's. */
typedef struct c3d_rng c3d_rng;
int c3d_rng_create(uint64_t seed, c3d_rng** out);
int c3d_rng_destroy(c3d_rng* rng);
int c3d_rng_next_u64(c3d_rng* rng, uint64_t* out, int64_t n);
/* random_matrix / random_vector (cube3d/rng.hpp:36-59): lo + (hi-lo)*unit, as double. */
int c3d_rng_uniform(c3d_rng* rng, double lo, double hi, double* out, int64_t n);
/* random_integer_matrix (cube3d/rng.hpp:46-52): next_u64() % bound. */
int c3d_rng_below(c3d_rng* rng, uint64_t bound, double* out, int64_t n);

/* --------------------------------------------------------- pure host: grid */
/* Row-major (i, j, l) linearisation: rank = (i*py + j)*pz + l.
 * Replaces CubeTopology::rank_of / coords_of (cube3d/topology.hpp:68-77). */
int c3d_grid_rank_of(const int dims[3], const int coords[3], int* rank);
int c3d_grid_coords_of(const int dims[3], int rank, int coords[3]);
/* Members of the axis line through `rank`, ascending along the axis
 * (CubeTopology::axis_group, cube3d/topology.hpp:79-95). members has dims[axis] slots. */
int c3d_grid_axis_group(const int dims[3], int rank, int axis, int* members, int* my_position);
/* CubeTopology::line_index, cube3d/topology.hpp:99-107. */
int c3d_grid_line_index(const int dims[3], int rank, int axis, int* line);
/* build_cube: perfect cubes only, else C3D_ERR_NOT_A_CUBE (cube3d/topology.hpp:121-127). */
int c3d_build_cube(int total_ranks, int* side);

/* ------------------------------------------------------- pure host: layout */
/* shard_bounds (cube3d/layout.hpp:93-123), generalised to px x py x pz.
 * out = {row_begin, row_end, col_begin, col_end}. dirs = {input, weight, output}. */
int c3d_shard_bounds(int layout, const int dims[3], const int coords[3], int64_t rows,
                     int64_t cols, const int dirs[3], int64_t out[4]);
/* diagonal_holder / diagonal_slice (cube3d/layout.hpp:134-142). out = {begin, end}.
 * On py != pz grids with min(py, pz) = 1 every rank holds a slice. */
int c3d_diagonal_slice(const int dims[3], const int coords[3], int64_t global_len,
                       int* holds, int64_t out[2]);
/* activation_from_global's index map (cube3d/activation.hpp:103-138): global row of
 * every local row of an activation in `group` (0: input axis y, 1: z), and the first
 * global column. rows_out has (batch/px)*(seq/p_in) slots. */
int c3d_activation_rows(const int dims[3], const int coords[3], int64_t batch, int64_t seq,
                        int64_t hidden, int group, int64_t* rows_out, int64_t* col_begin,
                        int64_t* local_cols);

/* -------------------------------------------------------------- the cube */
typedef struct c3d_cube c3d_cube;

/* Per-rank traffic / compute meters (CostCounters, cube3d/counters.hpp:37-68),
 * charged with the reference's ring-style convention. */
typedef struct {
  uint64_t elements_sent;
  uint64_t elements_received;
  uint64_t sent_by_kind[5];
  uint64_t received_by_kind[5];
  uint64_t calls_by_kind[5];
  uint64_t multiply_adds;
} c3d_counters;

/* NCCL unique id for the world communicator (rank 0 creates, all ranks receive). */
int c3d_unique_id(unsigned char uid[128]);
/* Creates this rank's cube handle on `device`: world NCCL communicator, one
 * ncclCommSplit communicator per axis (color = line index, key = axis coordinate,
 * so comm rank order equals the reference's ascending group position,
 * cube3d/transport.hpp:186-199). Replaces Transport + Endpoint
 * (cube3d/transport.hpp:89-149) and run_spmd's per-rank worker. */
int c3d_cube_create(const int dims[3], int rank, int device, const unsigned char uid[128],
                    c3d_cube** out);
int c3d_cube_destroy(c3d_cube* cube);
int c3d_cube_info(const c3d_cube* cube, int* rank, int coords[3], int dims[3]);
/* Endpoint::barrier (cube3d/transport.hpp:260-266), stream-ordered. */
int c3d_cube_barrier(c3d_cube* cube, void* stream);
int c3d_counters_get(const c3d_cube* cube, c3d_counters* out);
/* Synchronises `stream` and reports whether any peer-memory wait of this cube failed:
 * a peer that did not arrive within C3D_PEER_TIMEOUT_MS (default 30 s) or a collective
 * whose (kind, root, op, dtype, count) header differs between the members of a line
 * (the reference's RoundHeader check, cube3d/transport.hpp:32-40, 305-319). Then returns
 * C3D_ERR_DESYNC and the cube stays poisoned: every later operation on it fails with
 * C3D_ERR_DESYNC too (the reference poisons the group, transport.hpp:67-78). Operations
 * check the record at entry, so a failure is also reported by the next call. */
int c3d_cube_check(c3d_cube* cube, void* stream);
int c3d_counters_reset(c3d_cube* cube);

/* Endpoint collectives along one axis line (cube3d/transport.hpp:160-257), device
 * buffers, stream-ordered, charged to the counters like the reference. Counts are in
 * elements of `dtype`. Positions ascend along the axis; reductions sum (or max) in
 * ascending position order. Transport: peer-memory push kernels over NVLink
 * (NCCL when C3D_NCCL_COLL=1).
 *   broadcast:      buf[count] from the rank at `root_position`   (:160-184)
 *   all_gather:     send[count] -> recv[p][count]                 (:188-203)
 *   reduce_scatter: send[p][count] -> recv[count] (own position)  (:208-232)
 *   all_reduce:     buf[count] in place, op 0 = sum, 1 = max      (:236-257) */
int c3d_broadcast(c3d_cube* cube, int axis, int root_position, void* buf, size_t count,
                  int dtype, void* stream);
int c3d_all_gather(c3d_cube* cube, int axis, const void* send, void* recv, size_t count,
                   int dtype, void* stream);
int c3d_reduce_scatter(c3d_cube* cube, int axis, const void* send, void* recv, size_t count,
                       int dtype, void* stream);
int c3d_all_reduce(c3d_cube* cube, int axis, void* buf, size_t count, int dtype, int op,
                   void* stream);

/* ------------------------------------------------------------- tensors */
/* ShardedMatrix (cube3d/sharding.hpp:18-34): the local shard is a dense row-major
 * block of the bounds c3d_shard_bounds gives (ld = local cols). */
typedef struct {
  void* data;
  int dtype;
  int64_t global_rows, global_cols;
  int layout;
  int dirs[3];
} c3d_matrix;

/* DiagonalVector (cube3d/sharding.hpp:38-47): data holds the diagonal slice on
 * holder ranks and is ignored elsewhere. */
typedef struct {
  void* data;
  int dtype;
  int64_t global_len;
} c3d_vector;

/* Activation3D (cube3d/activation.hpp:41-62): local [(b/px)*(s/p_in), h/p_out]. */
typedef struct {
  void* data;
  int dtype;
  int64_t batch, seq, hidden;
  int group;
} c3d_activation;

/* ------------------------------------------------------------ local GEMM */
/* Strided, batched, optionally split logical matrix X[b][r][c] (see csrc/gemm.hpp). */
typedef struct {
  void* base;
  int dtype;
  int64_t sr, sc, s_hi, rsplit, csplit, sb_lo, sb_hi;
  int b_lo_n;
} c3d_view;
/* C[b][m][n] (+)= act(alpha * sum_k A[b][m][k] B[b][n][k] + bias[n]).
 * The per-rank product of multiply_accumulate (cube3d/matrix.hpp:68-92). */
int c3d_gemm(int64_t M, int64_t N, int64_t K, int batch, const c3d_view* a, const c3d_view* b,
             const c3d_view* out, float alpha, const float* bias, int act, int accumulate,
             int mode, void* stream);

/* ------------------------------------------------------------ 3-D matmuls */
/* C = A B: A Input family (M x N), B Weight (N x K) -> C Output (M x K), swapped triple.
 * matmul_ab_fwd (cube3d/ops3d.hpp:114-132). c->data must hold the output shard. */
int c3d_matmul_ab_fwd(c3d_cube* cube, int mode, const c3d_matrix* a, const c3d_matrix* b,
                      c3d_matrix* c, void* stream);
/* matmul_ab_bwd (cube3d/ops3d.hpp:137-168): dA = dC B^T, dB = A^T dC. */
int c3d_matmul_ab_bwd(c3d_cube* cube, int mode, const c3d_matrix* dc, const c3d_matrix* a,
                      const c3d_matrix* b, c3d_matrix* da, c3d_matrix* db, void* stream);
/* matmul_abt_fwd/bwd (cube3d/ops3d.hpp:174-223): B in WeightOfTranspose. */
int c3d_matmul_abt_fwd(c3d_cube* cube, int mode, const c3d_matrix* a, const c3d_matrix* b,
                       c3d_matrix* c, void* stream);
int c3d_matmul_abt_bwd(c3d_cube* cube, int mode, const c3d_matrix* dc, const c3d_matrix* a,
                       const c3d_matrix* b, c3d_matrix* da, c3d_matrix* db, void* stream);
/* matmul_atb_fwd/bwd (cube3d/ops3d.hpp:230-277): B Input family with A's swapped triple. */
int c3d_matmul_atb_fwd(c3d_cube* cube, int mode, const c3d_matrix* a, const c3d_matrix* b,
                       c3d_matrix* c, void* stream);
int c3d_matmul_atb_bwd(c3d_cube* cube, int mode, const c3d_matrix* dc, const c3d_matrix* a,
                       const c3d_matrix* b, c3d_matrix* da, c3d_matrix* db, void* stream);

/* Batched 3-D matmuls (cube3d/ops3d.hpp:418-494, BatchedShardedMatrix): `na` slices of A,
 * `nb` of B (and `ndc` of dC), one full 3-D product per slice in order -- the counters equal
 * the looped accounting. Different extents: C3D_ERR_BATCH_MISMATCH before any work. */
int c3d_batched_matmul_ab_fwd(c3d_cube* cube, int mode, int na, const c3d_matrix* a, int nb,
                              const c3d_matrix* b, c3d_matrix* c, void* stream);
int c3d_batched_matmul_abt_fwd(c3d_cube* cube, int mode, int na, const c3d_matrix* a, int nb,
                               const c3d_matrix* b, c3d_matrix* c, void* stream);
int c3d_batched_matmul_atb_fwd(c3d_cube* cube, int mode, int na, const c3d_matrix* a, int nb,
                               const c3d_matrix* b, c3d_matrix* c, void* stream);
int c3d_batched_matmul_ab_bwd(c3d_cube* cube, int mode, int ndc, const c3d_matrix* dc, int na,
                              const c3d_matrix* a, int nb, const c3d_matrix* b, c3d_matrix* da,
                              c3d_matrix* db, void* stream);
int c3d_batched_matmul_abt_bwd(c3d_cube* cube, int mode, int ndc, const c3d_matrix* dc, int na,
                               const c3d_matrix* a, int nb, const c3d_matrix* b, c3d_matrix* da,
                               c3d_matrix* db, void* stream);
int c3d_batched_matmul_atb_bwd(c3d_cube* cube, int mode, int ndc, const c3d_matrix* dc, int na,
                               const c3d_matrix* a, int nb, const c3d_matrix* b, c3d_matrix* da,
                               c3d_matrix* db, void* stream);

/* ---------------------------------------------------------- vector ops */
/* add_vec_fwd/bwd (cube3d/ops3d.hpp:347-372): C = A + b rowwise; db = colsum(dC)
 * reduced onto the diagonal ranks (reduce_to_diagonal, :315-336). */
int c3d_add_vec_fwd(c3d_cube* cube, const c3d_matrix* a, const c3d_vector* b, c3d_matrix* c,
                    void* stream);
int c3d_add_vec_bwd(c3d_cube* cube, const c3d_matrix* dc, c3d_matrix* da, c3d_vector* db,
                    void* stream);
/* mul_vec_fwd/bwd (cube3d/ops3d.hpp:382-416). */
int c3d_mul_vec_fwd(c3d_cube* cube, const c3d_matrix* a, const c3d_vector* b, c3d_matrix* c,
                    void* stream);
int c3d_mul_vec_bwd(c3d_cube* cube, const c3d_matrix* dc, const c3d_matrix* a,
                    const c3d_vector* b, c3d_matrix* da, c3d_vector* db, void* stream);

/* ------------------------------------------------------------ NN blocks */
/* TransformerConfig (cube3d/nn.hpp:16-41); validated with the reference's rules. */
typedef struct {
  int64_t batch, seq, heads, hidden;
  double eps;
} c3d_config;

typedef struct c3d_saved c3d_saved; /* opaque saved-for-backward state */
int c3d_saved_free(c3d_saved* saved);

/* LinearParams (cube3d/nn.hpp:62-67). */
typedef struct {
  c3d_matrix weight;
  c3d_vector bias;
  int input_group;
} c3d_linear_params;
/* linear3d_fwd/bwd (cube3d/nn.hpp:81-112). */
int c3d_linear_fwd(c3d_cube* cube, int mode, const c3d_activation* x,
                   const c3d_linear_params* p, int* group, c3d_activation* y, c3d_saved** saved,
                   void* stream);
int c3d_linear_bwd(c3d_cube* cube, int mode, const c3d_activation* dy, const c3d_saved* saved,
                   const c3d_linear_params* p, c3d_activation* dx, c3d_matrix* dweight,
                   c3d_vector* dbias, void* stream);

/* 3-D cross-entropy (not in the reference): logits = x W + b
 * through the 3-D linear (fp32 logits), loss = mean over the batch*seq tokens of
 * logsumexp(logits) - logits[target]. `targets`: int32 device array of the GLOBAL
 * token targets [batch * seq] (identical on every rank; must stay valid until
 * c3d_loss_bwd). `loss`: one device float, identical on every rank. The backward
 * returns dx, dW, db of the head in `grad_dtype` for dx (dW / db in their
 * descriptors' dtypes). */
int c3d_loss_fwd(c3d_cube* cube, int mode, const c3d_activation* x, const c3d_linear_params* head,
                 const int32_t* targets, int* group, float* loss, c3d_saved** saved, void* stream);
int c3d_loss_bwd(c3d_cube* cube, int mode, const c3d_saved* saved, const c3d_linear_params* head,
                 c3d_activation* dx, c3d_matrix* dweight, c3d_vector* dbias, void* stream);

/* LayerNormParams (cube3d/nn.hpp:119-124); layernorm3d_fwd/bwd (:140-222). */
typedef struct {
  c3d_vector gamma, beta;
  double eps;
} c3d_layernorm_params;
int c3d_layernorm_fwd(c3d_cube* cube, const c3d_activation* x, const c3d_layernorm_params* p,
                      c3d_activation* y, c3d_saved** saved, void* stream);
int c3d_layernorm_bwd(c3d_cube* cube, const c3d_activation* dy, const c3d_saved* saved,
                      c3d_activation* dx, c3d_vector* dgamma, c3d_vector* dbeta, void* stream);

/* Full layer parameters (LayerParams, cube3d/transformer.hpp:78-85); the same struct
 * carries gradients (LayerGrads, :94-101). */
typedef struct {
  c3d_vector ln1_gamma, ln1_beta;
  c3d_matrix w_qkv;
  c3d_vector b_qkv;
  c3d_matrix w_out;
  c3d_vector b_out;
  c3d_vector ln2_gamma, ln2_beta;
  c3d_matrix w_fc1;
  c3d_vector b_fc1;
  c3d_matrix w_fc2;
  c3d_vector b_fc2;
} c3d_layer_params;

/* attention_fwd/bwd (cube3d/attention.hpp:78-189), using the w_qkv/b_qkv/w_out/b_out
 * members of c3d_layer_params. */
int c3d_attention_fwd(c3d_cube* cube, int mode, const c3d_config* cfg, const c3d_activation* x,
                      const c3d_layer_params* p, int* group, c3d_activation* y,
                      c3d_saved** saved, void* stream);
int c3d_attention_bwd(c3d_cube* cube, int mode, const c3d_config* cfg, const c3d_activation* dy,
                      const c3d_saved* saved, const c3d_layer_params* p, c3d_activation* dx,
                      c3d_layer_params* grads, void* stream);
/* mlp_fwd/bwd (cube3d/transformer.hpp:44-70), using w_fc1/b_fc1/w_fc2/b_fc2. */
int c3d_mlp_fwd(c3d_cube* cube, int mode, const c3d_config* cfg, const c3d_activation* x,
                const c3d_layer_params* p, int* group, c3d_activation* y, c3d_saved** saved,
                void* stream);
int c3d_mlp_bwd(c3d_cube* cube, int mode, const c3d_config* cfg, const c3d_activation* dy,
                const c3d_saved* saved, const c3d_layer_params* p, c3d_activation* dx,
                c3d_layer_params* grads, void* stream);
/* transformer_layer_fwd/bwd (cube3d/transformer.hpp:115-148), pre-norm residual. */
int c3d_layer_fwd(c3d_cube* cube, int mode, const c3d_config* cfg, const c3d_activation* x,
                  const c3d_layer_params* p, int* group, c3d_activation* y, c3d_saved** saved,
                  void* stream);
int c3d_layer_bwd(c3d_cube* cube, int mode, const c3d_config* cfg, const c3d_activation* dy,
                  const c3d_saved* saved, const c3d_layer_params* p, c3d_activation* dx,
                  c3d_layer_params* grads, void* stream);

/* transformer_stack_fwd/bwd (cube3d/transformer.hpp:150-176): `n_layers` layers
 * applied in order (backward in reverse); `layers` / `grads` are arrays of n_layers. */
int c3d_stack_fwd(c3d_cube* cube, int mode, const c3d_config* cfg, const c3d_activation* x,
                  const c3d_layer_params* layers, int n_layers, int* group, c3d_activation* y,
                  c3d_saved** saved, void* stream);
int c3d_stack_bwd(c3d_cube* cube, int mode, const c3d_config* cfg, const c3d_activation* dy,
                  const c3d_saved* saved, const c3d_layer_params* layers, int n_layers,
                  c3d_activation* dx, c3d_layer_params* grads, void* stream);


#ifdef __cplusplus
}
#endif

#endif /* C3D_H_ */
