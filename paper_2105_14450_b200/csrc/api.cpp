// extern "C" entry points (include/c3d.h). Every call validates on the host,
// enqueues on the caller's stream, and maps exceptions to status codes with a
// thread-local "Name: detail" message (cube3d/errors.hpp:17-22).
#include <cuda_runtime.h>
#include <nccl.h>

#include <cstring>
#include <memory>
#include <random>
#include <string>

#include "../../include/c3d.h"
#include "common.hpp"
#include "cube.hpp"
#include "grid.hpp"
#include "kernels.hpp"
#include "nn.hpp"
#include "ops.hpp"

struct c3d_cube {
  std::unique_ptr<c3d::Cube> impl;
};

struct c3d_rng {
  std::mt19937_64 gen;
  explicit c3d_rng(uint64_t seed) : gen(seed) {}
};

struct c3d_saved {
  std::unique_ptr<c3d::Saved> impl;
  int kind = 0;  // 1 linear, 2 layernorm, 3 attention, 4 mlp, 5 layer, 6 loss, 7 stack
  int mode = 0;
};

namespace {

thread_local std::string g_last_error;

template <typename F>
int guard(F&& f) {
  try {
    f();
    g_last_error.clear();
    return C3D_OK;
  } catch (const c3d::Error& e) {
    g_last_error = e.what();
    return e.code();
  } catch (const std::exception& e) {
    g_last_error = std::string("InternalError: ") + e.what();
    return C3D_ERR_INTERNAL;
  } catch (...) {
    g_last_error = "InternalError: unknown exception";
    return C3D_ERR_INTERNAL;
  }
}

cudaStream_t as_stream(void* s) { return static_cast<cudaStream_t>(s); }

// Every operation entry checks the cube's fault record first (cheap host read): a peer
// wait that failed in an earlier kernel makes this and every later call fail with
// C3D_ERR_DESYNC.
c3d::Cube& peek(c3d_cube* c) {
  if (!c || !c->impl) c3d::fail(C3D_ERR_CONFIG_INVALID, "null cube handle");
  return *c->impl;
}
c3d::Cube& get(c3d_cube* c) {
  c3d::Cube& cube = peek(c);
  cube.check_fault();
  return cube;
}

void need(const void* p, const char* what) {
  if (!p) c3d::fail(C3D_ERR_CONFIG_INVALID, std::string("null ") + what);
}

std::array<int, 3> coords3(const int c[3]) { return {c[0], c[1], c[2]}; }

c3d::Vec vec_of(const c3d_vector& v) {
  c3d::Vec o;
  o.data = v.data;
  o.dtype = v.dtype;
  o.len = v.global_len;
  return o;
}

c3d::Act act_of(const c3d::Cube& cube, const c3d_activation& a) {
  return c3d::make_act(cube, a.data, a.dtype, a.batch, a.seq, a.hidden, a.group);
}

void act_out(const c3d::Act& a, c3d_activation* out) {
  out->data = a.data;
  out->dtype = a.dtype;
  out->batch = a.batch;
  out->seq = a.seq;
  out->hidden = a.hidden;
  out->group = a.group;
}

c3d::Act act_dest(const c3d_activation* y) {
  c3d::Act a;
  a.data = y->data;
  a.dtype = y->dtype;
  return a;
}

int group_of_dirs(const c3d::Mat& w) {
  if (w.dirs == c3d::triple_for_group(0)) return 0;
  if (w.dirs == c3d::triple_for_group(1)) return 1;
  c3d::fail(C3D_ERR_GROUP_MISMATCH, "weight directions do not match either activation group");
}

c3d::LinearP linear_of(const c3d::Cube& cube, const c3d_matrix& w, const c3d_vector& b) {
  c3d::LinearP p;
  p.w = c3d::from_c(cube, w);
  p.b = vec_of(b);
  p.input_group = group_of_dirs(p.w);
  return p;
}

c3d::LayerP layer_of(const c3d::Cube& cube, const c3d_layer_params& p) {
  c3d::LayerP o;
  o.ln1_g = vec_of(p.ln1_gamma);
  o.ln1_b = vec_of(p.ln1_beta);
  o.qkv = linear_of(cube, p.w_qkv, p.b_qkv);
  o.out = linear_of(cube, p.w_out, p.b_out);
  o.ln2_g = vec_of(p.ln2_gamma);
  o.ln2_b = vec_of(p.ln2_beta);
  o.fc1 = linear_of(cube, p.w_fc1, p.b_fc1);
  o.fc2 = linear_of(cube, p.w_fc2, p.b_fc2);
  return o;
}

c3d::Mat mat_dest(const c3d_matrix& m) {
  c3d::Mat o;
  o.data = m.data;
  o.dtype = m.dtype;
  return o;
}

c3d::LayerG grads_of(const c3d_layer_params& g) {
  c3d::LayerG o;
  o.ln1_g = vec_of(g.ln1_gamma);
  o.ln1_b = vec_of(g.ln1_beta);
  o.w_qkv = mat_dest(g.w_qkv);
  o.b_qkv = vec_of(g.b_qkv);
  o.w_out = mat_dest(g.w_out);
  o.b_out = vec_of(g.b_out);
  o.ln2_g = vec_of(g.ln2_gamma);
  o.ln2_b = vec_of(g.ln2_beta);
  o.w_fc1 = mat_dest(g.w_fc1);
  o.b_fc1 = vec_of(g.b_fc1);
  o.w_fc2 = mat_dest(g.w_fc2);
  o.b_fc2 = vec_of(g.b_fc2);
  return o;
}

void grads_out(const c3d::LayerG& g, c3d_layer_params* out) {
  if (g.w_qkv.data) c3d::to_c(g.w_qkv, &out->w_qkv);
  if (g.w_out.data) c3d::to_c(g.w_out, &out->w_out);
  if (g.w_fc1.data) c3d::to_c(g.w_fc1, &out->w_fc1);
  if (g.w_fc2.data) c3d::to_c(g.w_fc2, &out->w_fc2);
}

c3d::Config cfg_of(const c3d_config* c) {
  need(c, "config");
  c3d::Config o;
  o.batch = c->batch;
  o.seq = c->seq;
  o.heads = c->heads;
  o.hidden = c->hidden;
  o.eps = c->eps;
  return o;
}

template <typename T>
T& saved_as(const c3d_saved* s, int kind) {
  if (!s || !s->impl || s->kind != kind)
    c3d::fail(C3D_ERR_CONFIG_INVALID, "saved state is missing or from a different op");
  return *static_cast<T*>(s->impl.get());
}

}  // namespace

extern "C" {

const char* c3d_last_error(void) { return g_last_error.c_str(); }
const char* c3d_version(void) { return "c3d-b200 0.1 (sm_100a)"; }
long long c3d_launch_count(void) { return c3d::launch_counter().load(); }
int c3d_prof_enable(int on) {
  return guard([&] { c3d::prof_enable(on != 0); });
}
int c3d_prof_read(double* ms, double* flops, long long* launches) {
  return guard([&] { c3d::prof_read(ms, flops, launches); });
}
int c3d_prof_read_comm(double* ms, double* bytes, long long* calls) {
  return guard([&] { c3d::prof_read_comm(ms, bytes, calls); });
}

// ---------------------------------------------------------------- rng
int c3d_rng_create(uint64_t seed, c3d_rng** out) {
  return guard([&] { *out = new c3d_rng(seed); });
}
int c3d_rng_destroy(c3d_rng* rng) {
  return guard([&] { delete rng; });
}
int c3d_rng_next_u64(c3d_rng* rng, uint64_t* out, int64_t n) {
  return guard([&] {
    need(rng, "rng");
    for (int64_t i = 0; i < n; ++i) out[i] = rng->gen();
  });
}
int c3d_rng_uniform(c3d_rng* rng, double lo, double hi, double* out, int64_t n) {
  // Rng::next_unit / uniform (cube3d/rng.hpp:24-26)
  return guard([&] {
    need(rng, "rng");
    for (int64_t i = 0; i < n; ++i) {
      const double u = static_cast<double>(rng->gen() >> 11) * 0x1.0p-53;
      out[i] = lo + (hi - lo) * u;
    }
  });
}
int c3d_rng_below(c3d_rng* rng, uint64_t bound, double* out, int64_t n) {
  return guard([&] {
    need(rng, "rng");
    if (bound == 0) c3d::fail(C3D_ERR_CONFIG_INVALID, "bound must be positive");
    for (int64_t i = 0; i < n; ++i) out[i] = static_cast<double>(rng->gen() % bound);
  });
}

// ---------------------------------------------------------------- grid
int c3d_grid_rank_of(const int dims[3], const int coords[3], int* rank) {
  return guard([&] {
    need(rank, "rank");
    *rank = c3d::Grid(dims).rank_of(coords3(coords));
  });
}
int c3d_grid_coords_of(const int dims[3], int rank, int coords[3]) {
  return guard([&] {
    auto c = c3d::Grid(dims).coords_of(rank);
    for (int a = 0; a < 3; ++a) coords[a] = c[a];
  });
}
int c3d_grid_axis_group(const int dims[3], int rank, int axis, int* members, int* my_position) {
  return guard([&] {
    if (axis < 0 || axis > 2) c3d::fail(C3D_ERR_OUT_OF_RANGE, "axis " + std::to_string(axis));
    c3d::Grid g(dims);
    auto c = g.coords_of(rank);
    auto m = g.axis_group(c, axis);
    for (size_t q = 0; q < m.size(); ++q) members[q] = m[q];
    if (my_position) *my_position = c[axis];
  });
}
int c3d_grid_line_index(const int dims[3], int rank, int axis, int* line) {
  return guard([&] {
    if (axis < 0 || axis > 2) c3d::fail(C3D_ERR_OUT_OF_RANGE, "axis " + std::to_string(axis));
    c3d::Grid g(dims);
    *line = g.line_index(g.coords_of(rank), axis);
  });
}
int c3d_build_cube(int total_ranks, int* side) {
  // build_cube (cube3d/topology.hpp:121-127)
  return guard([&] {
    if (total_ranks < 1)
      c3d::fail(C3D_ERR_NOT_A_CUBE,
                "rank count must be positive, got " + std::to_string(total_ranks));
    for (int s = 1; s * s * s <= total_ranks; ++s)
      if (s * s * s == total_ranks) {
        *side = s;
        return;
      }
    c3d::fail(C3D_ERR_NOT_A_CUBE, std::to_string(total_ranks) + " has no integer cube root");
  });
}

// ---------------------------------------------------------------- layout
int c3d_shard_bounds(int layout, const int dims[3], const int coords[3], int64_t rows,
                     int64_t cols, const int dirs[3], int64_t out[4]) {
  return guard([&] {
    if (layout < 0 || layout > 3) c3d::fail(C3D_ERR_SHAPE_MISMATCH, "unknown layout");
    c3d::Dirs d{dirs[0], dirs[1], dirs[2]};
    auto b = c3d::shard_bounds(layout, c3d::Grid(dims), coords3(coords), rows, cols, d);
    out[0] = b.rows.begin;
    out[1] = b.rows.end;
    out[2] = b.cols.begin;
    out[3] = b.cols.end;
  });
}
int c3d_diagonal_slice(const int dims[3], const int coords[3], int64_t global_len, int* holds,
                       int64_t out[2]) {
  return guard([&] {
    c3d::Grid g(dims);
    auto c = coords3(coords);
    g.check(c);
    auto r = c3d::diagonal_slice(g, c, global_len);
    if (holds) *holds = c3d::diagonal_holder(g, c) ? 1 : 0;
    out[0] = r.begin;
    out[1] = r.end;
  });
}
int c3d_activation_rows(const int dims[3], const int coords[3], int64_t batch, int64_t seq,
                        int64_t hidden, int group, int64_t* rows_out, int64_t* col_begin,
                        int64_t* local_cols) {
  // activation_from_global (cube3d/activation.hpp:119-134): local row bi*(s/p_in)+si
  // <-> global row (w*b/px + bi)*s + a*s/p_in + si, col o*h/p_out + t.
  return guard([&] {
    c3d::Grid g(dims);
    auto c = coords3(coords);
    g.check(c);
    auto geo = c3d::act_geom(g, batch, seq, hidden, group);
    const int64_t w = c[c3d::kX], a = c[geo.in_axis], o = c[geo.out_axis];
    if (rows_out)
      for (int64_t bi = 0; bi < geo.bl; ++bi)
        for (int64_t si = 0; si < geo.sl; ++si)
          rows_out[bi * geo.sl + si] = (w * geo.bl + bi) * seq + a * geo.sl + si;
    if (col_begin) *col_begin = o * geo.hl;
    if (local_cols) *local_cols = geo.hl;
  });
}

// ---------------------------------------------------------------- cube
int c3d_unique_id(unsigned char uid[128]) {
  return guard([&] {
    ncclUniqueId id;
    ncclResult_t r = ncclGetUniqueId(&id);
    if (r != ncclSuccess)
      c3d::fail(C3D_ERR_NCCL, std::string("ncclGetUniqueId: ") + ncclGetErrorString(r));
    static_assert(sizeof(id) == 128, "NCCL unique id size");
    std::memcpy(uid, &id, sizeof(id));
  });
}
int c3d_cube_create(const int dims[3], int rank, int device, const unsigned char uid[128],
                    c3d_cube** out) {
  return guard([&] {
    need(out, "output handle");
    auto h = std::make_unique<c3d_cube>();
    h->impl = std::make_unique<c3d::Cube>(dims, rank, device, uid);
    *out = h.release();
  });
}
int c3d_cube_destroy(c3d_cube* cube) {
  return guard([&] { delete cube; });
}
int c3d_cube_info(const c3d_cube* cube, int* rank, int coords[3], int dims[3]) {
  return guard([&] {
    auto& c = peek(const_cast<c3d_cube*>(cube));
    if (rank) *rank = c.rank();
    for (int a = 0; a < 3; ++a) {
      if (coords) coords[a] = c.coords()[a];
      if (dims) dims[a] = c.grid().dims[a];
    }
  });
}
int c3d_cube_barrier(c3d_cube* cube, void* stream) {
  return guard([&] { get(cube).barrier(as_stream(stream)); });
}
int c3d_counters_get(const c3d_cube* cube, c3d_counters* out) {
  return guard([&] { *out = peek(const_cast<c3d_cube*>(cube)).counters(); });
}
int c3d_cube_check(c3d_cube* cube, void* stream) {
  return guard([&] {
    auto& c = peek(cube);
    C3D_CUDA(cudaStreamSynchronize(as_stream(stream)));
    c.check_fault();
  });
}
int c3d_counters_reset(c3d_cube* cube) {
  return guard([&] { get(cube).reset_counters(); });
}

namespace {
void check_axis_dtype(int axis, int dtype) {
  if (axis < 0 || axis > 2) c3d::fail(C3D_ERR_OUT_OF_RANGE, "axis " + std::to_string(axis));
  if (dtype != C3D_F32 && dtype != C3D_BF16)
    c3d::fail(C3D_ERR_CONFIG_INVALID, "dtype " + std::to_string(dtype));
}
}  // namespace

int c3d_broadcast(c3d_cube* cube, int axis, int root_position, void* buf, size_t count,
                  int dtype, void* stream) {
  return guard([&] {
    check_axis_dtype(axis, dtype);
    get(cube).broadcast(axis, root_position, buf, count, dtype, as_stream(stream));
  });
}
int c3d_all_gather(c3d_cube* cube, int axis, const void* send, void* recv, size_t count,
                   int dtype, void* stream) {
  return guard([&] {
    check_axis_dtype(axis, dtype);
    get(cube).all_gather(axis, send, recv, count, dtype, as_stream(stream));
  });
}
int c3d_reduce_scatter(c3d_cube* cube, int axis, const void* send, void* recv, size_t count,
                       int dtype, void* stream) {
  return guard([&] {
    check_axis_dtype(axis, dtype);
    get(cube).reduce_scatter(axis, send, recv, count, dtype, as_stream(stream));
  });
}
int c3d_all_reduce(c3d_cube* cube, int axis, void* buf, size_t count, int dtype, int op,
                   void* stream) {
  return guard([&] {
    check_axis_dtype(axis, dtype);
    if (op != 0 && op != 1) c3d::fail(C3D_ERR_CONFIG_INVALID, "all_reduce op must be 0 or 1");
    get(cube).all_reduce(axis, buf, count, dtype, op == 1, as_stream(stream));
  });
}

// ---------------------------------------------------------------- GEMM
int c3d_gemm(int64_t M, int64_t N, int64_t K, int batch, const c3d_view* a, const c3d_view* b,
             const c3d_view* out, float alpha, const float* bias, int act, int accumulate,
             int mode, void* stream) {
  return guard([&] {
    need(a, "A view");
    need(b, "B view");
    need(out, "output view");
    auto cv = [](const c3d_view* v) {
      c3d::View o;
      o.base = v->base;
      o.dtype = v->dtype;
      o.sr = v->sr;
      o.sc = v->sc;
      o.s_hi = v->s_hi;
      o.rsplit = v->rsplit;
      o.csplit = v->csplit;
      o.sb_lo = v->sb_lo;
      o.sb_hi = v->sb_hi;
      o.b_lo_n = v->b_lo_n < 1 ? 1 : v->b_lo_n;
      return o;
    };
    c3d::GemmProblem p;
    p.M = M;
    p.N = N;
    p.K = K;
    p.batch = batch;
    p.a = cv(a);
    p.b = cv(b);
    p.epi.out = cv(out);
    p.epi.alpha = alpha;
    p.epi.bias = bias;
    p.epi.act = act;
    p.epi.accumulate = accumulate;
    int dev = 0, sms = 148;
    C3D_CUDA(cudaGetDevice(&dev));
    C3D_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    c3d::run_gemm(p, mode, sms, as_stream(stream));
  });
}

// ---------------------------------------------------------------- 3-D matmuls
#define C3D_MATMUL_FWD(name)                                                                    \
  int c3d_##name(c3d_cube* cube, int mode, const c3d_matrix* a, const c3d_matrix* b,            \
                 c3d_matrix* c, void* stream) {                                                 \
    return guard([&] {                                                                          \
      need(a, "A");                                                                             \
      need(b, "B");                                                                             \
      need(c, "C");                                                                             \
      auto& cb = get(cube);                                                                     \
      c3d::Mat am = c3d::from_c(cb, *a), bm = c3d::from_c(cb, *b), cm = mat_dest(*c);           \
      c3d::name(cb, mode, am, bm, cm, as_stream(stream));                                       \
      c3d::to_c(cm, c);                                                                         \
    });                                                                                         \
  }
#define C3D_MATMUL_BWD(name)                                                                    \
  int c3d_##name(c3d_cube* cube, int mode, const c3d_matrix* dc, const c3d_matrix* a,           \
                 const c3d_matrix* b, c3d_matrix* da, c3d_matrix* db, void* stream) {           \
    return guard([&] {                                                                          \
      need(dc, "dC");                                                                           \
      need(a, "A");                                                                             \
      need(b, "B");                                                                             \
      need(da, "dA");                                                                           \
      need(db, "dB");                                                                           \
      auto& cb = get(cube);                                                                     \
      c3d::Mat dcm = c3d::from_c(cb, *dc), am = c3d::from_c(cb, *a), bm = c3d::from_c(cb, *b);  \
      c3d::Mat dam = mat_dest(*da), dbm = mat_dest(*db);                                        \
      c3d::name(cb, mode, dcm, am, bm, dam, dbm, as_stream(stream));                            \
      c3d::to_c(dam, da);                                                                       \
      c3d::to_c(dbm, db);                                                                       \
    });                                                                                         \
  }
C3D_MATMUL_FWD(matmul_ab_fwd)
C3D_MATMUL_FWD(matmul_abt_fwd)
C3D_MATMUL_FWD(matmul_atb_fwd)
C3D_MATMUL_BWD(matmul_ab_bwd)
C3D_MATMUL_BWD(matmul_abt_bwd)
C3D_MATMUL_BWD(matmul_atb_bwd)

// Batched variants (cube3d/ops3d.hpp:418-494): one full 3-D matmul per slice, in order,
// so the counters equal the looped accounting; extents that differ are BatchMismatch
// before anything is enqueued (ops3d.hpp:432-437).
namespace {
void require_same_batch(int na, int nb) {
  if (na != nb)
    c3d::fail(C3D_ERR_BATCH_MISMATCH,
              "batch extents differ: " + std::to_string(na) + " vs " + std::to_string(nb));
  if (na < 0) c3d::fail(C3D_ERR_CONFIG_INVALID, "negative batch extent");
}
}  // namespace
#define C3D_BATCHED_FWD(name)                                                                   \
  int c3d_batched_##name(c3d_cube* cube, int mode, int na, const c3d_matrix* a, int nb,         \
                         const c3d_matrix* b, c3d_matrix* c, void* stream) {                    \
    return guard([&] {                                                                          \
      require_same_batch(na, nb);                                                               \
      auto& cb = get(cube);                                                                     \
      for (int t = 0; t < na; ++t) {                                                            \
        c3d::Mat am = c3d::from_c(cb, a[t]), bm = c3d::from_c(cb, b[t]), cm = mat_dest(c[t]);   \
        c3d::name(cb, mode, am, bm, cm, as_stream(stream));                                     \
        c3d::to_c(cm, &c[t]);                                                                   \
      }                                                                                         \
    });                                                                                         \
  }
#define C3D_BATCHED_BWD(name)                                                                   \
  int c3d_batched_##name(c3d_cube* cube, int mode, int ndc, const c3d_matrix* dc, int na,       \
                         const c3d_matrix* a, int nb, const c3d_matrix* b, c3d_matrix* da,      \
                         c3d_matrix* db, void* stream) {                                        \
    return guard([&] {                                                                          \
      require_same_batch(na, nb);                                                               \
      require_same_batch(na, ndc);                                                              \
      auto& cb = get(cube);                                                                     \
      for (int t = 0; t < na; ++t) {                                                            \
        c3d::Mat dcm = c3d::from_c(cb, dc[t]), am = c3d::from_c(cb, a[t]),                      \
                 bm = c3d::from_c(cb, b[t]);                                                    \
        c3d::Mat dam = mat_dest(da[t]), dbm = mat_dest(db[t]);                                  \
        c3d::name(cb, mode, dcm, am, bm, dam, dbm, as_stream(stream));                          \
        c3d::to_c(dam, &da[t]);                                                                 \
        c3d::to_c(dbm, &db[t]);                                                                 \
      }                                                                                         \
    });                                                                                         \
  }
C3D_BATCHED_FWD(matmul_ab_fwd)
C3D_BATCHED_FWD(matmul_abt_fwd)
C3D_BATCHED_FWD(matmul_atb_fwd)
C3D_BATCHED_BWD(matmul_ab_bwd)
C3D_BATCHED_BWD(matmul_abt_bwd)
C3D_BATCHED_BWD(matmul_atb_bwd)

// ---------------------------------------------------------------- vector ops
int c3d_add_vec_fwd(c3d_cube* cube, const c3d_matrix* a, const c3d_vector* b, c3d_matrix* c,
                    void* stream) {
  return guard([&] {
    auto& cb = get(cube);
    c3d::Mat am = c3d::from_c(cb, *a), cm = mat_dest(*c);
    c3d::add_vec_fwd(cb, am, vec_of(*b), cm, as_stream(stream));
    c3d::to_c(cm, c);
  });
}
int c3d_add_vec_bwd(c3d_cube* cube, const c3d_matrix* dc, c3d_matrix* da, c3d_vector* db,
                    void* stream) {
  return guard([&] {
    auto& cb = get(cube);
    c3d::Mat dcm = c3d::from_c(cb, *dc), dam = mat_dest(*da);
    c3d::Vec dbv = vec_of(*db);
    c3d::add_vec_bwd(cb, dcm, dam, dbv, as_stream(stream));
    c3d::to_c(dam, da);
    db->global_len = dcm.gcols;
  });
}
int c3d_mul_vec_fwd(c3d_cube* cube, const c3d_matrix* a, const c3d_vector* b, c3d_matrix* c,
                    void* stream) {
  return guard([&] {
    auto& cb = get(cube);
    c3d::Mat am = c3d::from_c(cb, *a), cm = mat_dest(*c);
    c3d::mul_vec_fwd(cb, am, vec_of(*b), cm, as_stream(stream));
    c3d::to_c(cm, c);
  });
}
int c3d_mul_vec_bwd(c3d_cube* cube, const c3d_matrix* dc, const c3d_matrix* a,
                    const c3d_vector* b, c3d_matrix* da, c3d_vector* db, void* stream) {
  return guard([&] {
    auto& cb = get(cube);
    c3d::Mat dcm = c3d::from_c(cb, *dc), am = c3d::from_c(cb, *a), dam = mat_dest(*da);
    c3d::mul_vec_bwd(cb, dcm, am, vec_of(*b), dam, vec_of(*db), as_stream(stream));
    c3d::to_c(dam, da);
    db->global_len = dcm.gcols;
  });
}

// ---------------------------------------------------------------- NN blocks
int c3d_saved_free(c3d_saved* saved) {
  return guard([&] { delete saved; });
}

int c3d_linear_fwd(c3d_cube* cube, int mode, const c3d_activation* x, const c3d_linear_params* p,
                   int* group, c3d_activation* y, c3d_saved** saved, void* stream) {
  return guard([&] {
    need(x, "x");
    need(p, "params");
    need(group, "group");
    need(y, "y");
    auto& cb = get(cube);
    c3d::Act xa = act_of(cb, *x), ya = act_dest(y);
    c3d::LinearP lp;
    lp.w = c3d::from_c(cb, p->weight);
    lp.b = vec_of(p->bias);
    lp.input_group = p->input_group;
    std::unique_ptr<c3d::LinearSaved> sv;
    if (saved) sv = std::make_unique<c3d::LinearSaved>();
    c3d::linear_fwd(cb, mode, xa, lp, *group, ya, sv.get(), true, c3d::LinearEpi{},
                    as_stream(stream));
    act_out(ya, y);
    if (saved) {
      auto h = std::make_unique<c3d_saved>();
      h->kind = 1;
      h->impl = std::move(sv);
      *saved = h.release();
    }
  });
}
int c3d_linear_bwd(c3d_cube* cube, int mode, const c3d_activation* dy, const c3d_saved* saved,
                   const c3d_linear_params* p, c3d_activation* dx, c3d_matrix* dweight,
                   c3d_vector* dbias, void* stream) {
  return guard([&] {
    need(dy, "dy");
    need(p, "params");
    auto& cb = get(cube);
    auto& sv = saved_as<c3d::LinearSaved>(saved, 1);
    c3d::Act dya = act_of(cb, *dy);
    c3d::LinearP lp;
    lp.w = c3d::from_c(cb, p->weight);
    lp.b = vec_of(p->bias);
    lp.input_group = p->input_group;
    c3d::Act dxa;
    if (dx) dxa = act_dest(dx);
    c3d::Mat dw;
    if (dweight) dw = mat_dest(*dweight);
    c3d::Vec db;
    if (dbias) db = vec_of(*dbias);
    c3d::linear_bwd(cb, mode, dya, sv, lp, dx ? &dxa : nullptr, dweight ? &dw : nullptr,
                    dbias ? &db : nullptr, nullptr, as_stream(stream));
    if (dx) act_out(dxa, dx);
    if (dweight && dw.data) c3d::to_c(dw, dweight);
    if (dbias) dbias->global_len = lp.w.gcols;
  });
}

int c3d_loss_fwd(c3d_cube* cube, int mode, const c3d_activation* x, const c3d_linear_params* head,
                 const int32_t* targets, int* group, float* loss, c3d_saved** saved, void* stream) {
  return guard([&] {
    need(x, "x");
    need(head, "head");
    need(group, "group");
    need(saved, "saved");
    if (!targets || !loss) c3d::fail(C3D_ERR_CONFIG_INVALID, "loss needs targets and output");
    auto& cb = get(cube);
    c3d::Act xa = act_of(cb, *x);
    c3d::LinearP lp;
    lp.w = c3d::from_c(cb, head->weight);
    lp.b = vec_of(head->bias);
    lp.input_group = head->input_group;
    auto sv = std::make_unique<c3d::LossSaved>();
    c3d::loss_fwd(cb, mode, xa, lp, targets, *group, loss, sv.get(), as_stream(stream));
    auto h = std::make_unique<c3d_saved>();
    h->kind = 6;
    h->impl = std::move(sv);
    *saved = h.release();
  });
}
int c3d_loss_bwd(c3d_cube* cube, int mode, const c3d_saved* saved, const c3d_linear_params* head,
                 c3d_activation* dx, c3d_matrix* dweight, c3d_vector* dbias, void* stream) {
  return guard([&] {
    need(head, "head");
    auto& cb = get(cube);
    auto& sv = saved_as<c3d::LossSaved>(saved, 6);
    c3d::LinearP lp;
    lp.w = c3d::from_c(cb, head->weight);
    lp.b = vec_of(head->bias);
    lp.input_group = head->input_group;
    c3d::Act dxa;
    if (dx) dxa = act_dest(dx);
    c3d::Mat dw;
    if (dweight) dw = mat_dest(*dweight);
    c3d::Vec db;
    if (dbias) db = vec_of(*dbias);
    const int gdt = dx ? dx->dtype : sv.lin.x.dtype;
    c3d::loss_bwd(cb, mode, sv, lp, dx ? &dxa : nullptr, dweight ? &dw : nullptr,
                  dbias ? &db : nullptr, gdt, as_stream(stream));
    if (dx) act_out(dxa, dx);
    if (dweight && dw.data) c3d::to_c(dw, dweight);
    if (dbias) dbias->global_len = lp.w.gcols;
  });
}

int c3d_layernorm_fwd(c3d_cube* cube, const c3d_activation* x, const c3d_layernorm_params* p,
                      c3d_activation* y, c3d_saved** saved, void* stream) {
  return guard([&] {
    need(x, "x");
    need(p, "params");
    need(y, "y");
    auto& cb = get(cube);
    c3d::Act xa = act_of(cb, *x), ya = act_dest(y);
    auto sv = std::make_unique<c3d::LNSaved>();
    c3d::layernorm_fwd(cb, xa, vec_of(p->gamma), vec_of(p->beta), p->eps, ya, sv.get(),
                       as_stream(stream));
    act_out(ya, y);
    if (saved) {
      auto h = std::make_unique<c3d_saved>();
      h->kind = 2;
      h->impl = std::move(sv);
      *saved = h.release();
    }
  });
}
int c3d_layernorm_bwd(c3d_cube* cube, const c3d_activation* dy, const c3d_saved* saved,
                      c3d_activation* dx, c3d_vector* dgamma, c3d_vector* dbeta, void* stream) {
  return guard([&] {
    need(dy, "dy");
    need(dx, "dx");
    auto& cb = get(cube);
    auto& sv = saved_as<c3d::LNSaved>(saved, 2);
    c3d::Act dya = act_of(cb, *dy), dxa = act_dest(dx);
    c3d::Vec dg, dbv;
    if (dgamma) dg = vec_of(*dgamma);
    if (dbeta) dbv = vec_of(*dbeta);
    c3d::layernorm_bwd(cb, dya, sv, dxa, dgamma ? &dg : nullptr, dbeta ? &dbv : nullptr, nullptr,
                       as_stream(stream));
    act_out(dxa, dx);
    if (dgamma) dgamma->global_len = dya.hidden;
    if (dbeta) dbeta->global_len = dya.hidden;
  });
}

int c3d_attention_fwd(c3d_cube* cube, int mode, const c3d_config* cfg, const c3d_activation* x,
                      const c3d_layer_params* p, int* group, c3d_activation* y,
                      c3d_saved** saved, void* stream) {
  return guard([&] {
    need(x, "x");
    need(p, "params");
    need(group, "group");
    need(y, "y");
    auto& cb = get(cube);
    c3d::Act xa = act_of(cb, *x), ya = act_dest(y);
    c3d::LinearP qkv = linear_of(cb, p->w_qkv, p->b_qkv);
    c3d::LinearP out = linear_of(cb, p->w_out, p->b_out);
    auto sv = std::make_unique<c3d::AttnSaved>();
    c3d::attention_fwd(cb, mode, cfg_of(cfg), xa, qkv, out, *group, ya, sv.get(), true, nullptr,
                       as_stream(stream));
    act_out(ya, y);
    if (saved) {
      auto h = std::make_unique<c3d_saved>();
      h->kind = 3;
      h->impl = std::move(sv);
      *saved = h.release();
    }
  });
}
int c3d_attention_bwd(c3d_cube* cube, int mode, const c3d_config* cfg, const c3d_activation* dy,
                      const c3d_saved* saved, const c3d_layer_params* p, c3d_activation* dx,
                      c3d_layer_params* grads, void* stream) {
  return guard([&] {
    need(dy, "dy");
    need(p, "params");
    need(dx, "dx");
    need(grads, "grads");
    auto& cb = get(cube);
    auto& sv = saved_as<c3d::AttnSaved>(saved, 3);
    c3d::Act dya = act_of(cb, *dy), dxa = act_dest(dx);
    c3d::LinearP qkv = linear_of(cb, p->w_qkv, p->b_qkv);
    c3d::LinearP out = linear_of(cb, p->w_out, p->b_out);
    c3d::LayerG g = grads_of(*grads);
    c3d::attention_bwd(cb, mode, cfg_of(cfg), dya, sv, qkv, out, dxa, g, as_stream(stream));
    act_out(dxa, dx);
    grads_out(g, grads);
  });
}

int c3d_mlp_fwd(c3d_cube* cube, int mode, const c3d_config* cfg, const c3d_activation* x,
                const c3d_layer_params* p, int* group, c3d_activation* y, c3d_saved** saved,
                void* stream) {
  return guard([&] {
    need(x, "x");
    need(p, "params");
    need(group, "group");
    need(y, "y");
    auto& cb = get(cube);
    c3d::Act xa = act_of(cb, *x), ya = act_dest(y);
    c3d::LinearP fc1 = linear_of(cb, p->w_fc1, p->b_fc1);
    c3d::LinearP fc2 = linear_of(cb, p->w_fc2, p->b_fc2);
    auto sv = std::make_unique<c3d::MlpSaved>();
    c3d::mlp_fwd(cb, mode, cfg_of(cfg), xa, fc1, fc2, *group, ya, sv.get(), true, nullptr,
                 as_stream(stream));
    act_out(ya, y);
    if (saved) {
      auto h = std::make_unique<c3d_saved>();
      h->kind = 4;
      h->impl = std::move(sv);
      *saved = h.release();
    }
  });
}
int c3d_mlp_bwd(c3d_cube* cube, int mode, const c3d_config* cfg, const c3d_activation* dy,
                const c3d_saved* saved, const c3d_layer_params* p, c3d_activation* dx,
                c3d_layer_params* grads, void* stream) {
  return guard([&] {
    need(dy, "dy");
    need(p, "params");
    need(dx, "dx");
    need(grads, "grads");
    auto& cb = get(cube);
    auto& sv = saved_as<c3d::MlpSaved>(saved, 4);
    c3d::Act dya = act_of(cb, *dy), dxa = act_dest(dx);
    c3d::LinearP fc1 = linear_of(cb, p->w_fc1, p->b_fc1);
    c3d::LinearP fc2 = linear_of(cb, p->w_fc2, p->b_fc2);
    c3d::LayerG g = grads_of(*grads);
    c3d::mlp_bwd(cb, mode, cfg_of(cfg), dya, sv, fc1, fc2, dxa, g, as_stream(stream));
    act_out(dxa, dx);
    grads_out(g, grads);
  });
}

int c3d_layer_fwd(c3d_cube* cube, int mode, const c3d_config* cfg, const c3d_activation* x,
                  const c3d_layer_params* p, int* group, c3d_activation* y, c3d_saved** saved,
                  void* stream) {
  return guard([&] {
    need(x, "x");
    need(p, "params");
    need(group, "group");
    need(y, "y");
    auto& cb = get(cube);
    c3d::Act xa = act_of(cb, *x), ya = act_dest(y);
    c3d::LayerP lp = layer_of(cb, *p);
    auto sv = std::make_unique<c3d::LayerSaved>();
    c3d::layer_fwd(cb, mode, cfg_of(cfg), xa, lp, *group, ya, saved ? sv.get() : nullptr,
                   as_stream(stream));
    act_out(ya, y);
    if (saved) {
      auto h = std::make_unique<c3d_saved>();
      h->kind = 5;
      h->impl = std::move(sv);
      *saved = h.release();
    }
  });
}
int c3d_layer_bwd(c3d_cube* cube, int mode, const c3d_config* cfg, const c3d_activation* dy,
                  const c3d_saved* saved, const c3d_layer_params* p, c3d_activation* dx,
                  c3d_layer_params* grads, void* stream) {
  return guard([&] {
    need(dy, "dy");
    need(p, "params");
    need(dx, "dx");
    need(grads, "grads");
    auto& cb = get(cube);
    auto& sv = saved_as<c3d::LayerSaved>(saved, 5);
    c3d::Act dya = act_of(cb, *dy), dxa = act_dest(dx);
    c3d::LayerP lp = layer_of(cb, *p);
    c3d::LayerG g = grads_of(*grads);
    c3d::layer_bwd(cb, mode, cfg_of(cfg), dya, sv, lp, dxa, g, as_stream(stream));
    act_out(dxa, dx);
    grads_out(g, grads);
  });
}

int c3d_stack_fwd(c3d_cube* cube, int mode, const c3d_config* cfg, const c3d_activation* x,
                  const c3d_layer_params* layers, int n_layers, int* group, c3d_activation* y,
                  c3d_saved** saved, void* stream) {
  return guard([&] {
    need(x, "x");
    need(layers, "layers");
    need(group, "group");
    need(y, "y");
    need(saved, "saved");
    if (n_layers < 1) c3d::fail(C3D_ERR_CONFIG_INVALID, "n_layers must be >= 1");
    auto& cb = get(cube);
    c3d::Act xa = act_of(cb, *x), ya = act_dest(y);
    std::vector<c3d::LayerP> ps;
    for (int i = 0; i < n_layers; ++i) ps.push_back(layer_of(cb, layers[i]));
    auto sv = std::make_unique<c3d::StackSaved>();
    c3d::stack_fwd(cb, mode, cfg_of(cfg), xa, ps, *group, ya, sv.get(), as_stream(stream));
    act_out(ya, y);
    auto h = std::make_unique<c3d_saved>();
    h->kind = 7;
    h->impl = std::move(sv);
    *saved = h.release();
  });
}
int c3d_stack_bwd(c3d_cube* cube, int mode, const c3d_config* cfg, const c3d_activation* dy,
                  const c3d_saved* saved, const c3d_layer_params* layers, int n_layers,
                  c3d_activation* dx, c3d_layer_params* grads, void* stream) {
  return guard([&] {
    need(dy, "dy");
    need(layers, "layers");
    need(dx, "dx");
    need(grads, "grads");
    auto& cb = get(cube);
    auto& sv = saved_as<c3d::StackSaved>(saved, 7);
    c3d::Act dya = act_of(cb, *dy), dxa = act_dest(dx);
    std::vector<c3d::LayerP> ps;
    std::vector<c3d::LayerG> gs;
    for (int i = 0; i < n_layers; ++i) {
      ps.push_back(layer_of(cb, layers[i]));
      gs.push_back(grads_of(grads[i]));
    }
    c3d::stack_bwd(cb, mode, cfg_of(cfg), dya, sv, ps, dxa, gs, as_stream(stream));
    act_out(dxa, dx);
    for (int i = 0; i < n_layers; ++i) grads_out(gs[i], &grads[i]);
  });
}

}  // extern "C"
