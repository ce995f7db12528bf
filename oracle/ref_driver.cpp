// TEST INFRASTRUCTURE ONLY (the checker, never the product).
//
// extern "C" shim over the *unmodified* reference library: it #includes the
// reference headers where they lie (/root/reference/proj/include, passed with -I
// by oracle/Makefile) and exposes the reference's own drivers and serial oracle
// to ctypes. Built into oracle/_ref/libcube3d_ref.so with the reference's flags
// (-std=c++20 -O2 -ffp-contract=off -pthread, proj/CMakeLists.txt:3,8-14).
// Nothing here re-implements reference logic; it only marshals arrays.
#include <chrono>
#include <cstdint>
#include <cstring>
#include <sstream>
#include <string>
#include <vector>

#include "cube3d/cost_model.hpp"
#include "cube3d/matrix_io.hpp"
#include "cube3d/bench.hpp"
#include "cube3d/transformer.hpp"
#include "cube3d/reference.hpp"
#include "cube3d/rng.hpp"
#include "cube3d/verify.hpp"

using namespace cube3d;

namespace {

template <typename T>
Matrix<T> to_mat(const double* p, std::size_t r, std::size_t c) {
  Matrix<T> m(r, c);
  for (std::size_t i = 0; i < r * c; ++i) m.data[i] = static_cast<T>(p[i]);
  return m;
}
template <typename T>
std::vector<T> to_vec(const double* p, std::size_t n) {
  std::vector<T> v(n);
  for (std::size_t i = 0; i < n; ++i) v[i] = static_cast<T>(p[i]);
  return v;
}
template <typename T>
void put(const Matrix<T>& m, double* out) {
  for (std::size_t i = 0; i < m.data.size(); ++i) out[i] = static_cast<double>(m.data[i]);
}
template <typename T>
void put(const std::vector<T>& v, double* out) {
  for (std::size_t i = 0; i < v.size(); ++i) out[i] = static_cast<double>(v[i]);
}

thread_local std::string g_err;

template <typename F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

TransformerConfig make_cfg(int p, int64_t b, int64_t s, int64_t n, int64_t h) {
  TransformerConfig cfg;
  cfg.batch = b;
  cfg.seq = s;
  cfg.heads = n;
  cfg.hidden = h;
  cfg.p = p;
  cfg.layers = 1;
  cfg.eps = 1e-5;
  return cfg;
}

// params: 12 arrays in GlobalLayerParams order
template <typename T>
GlobalLayerParams<T> params_of(const TransformerConfig& cfg, const double* const* ps) {
  const std::size_t h = cfg.hidden;
  GlobalLayerParams<T> g;
  g.ln1_gamma = to_vec<T>(ps[0], h);
  g.ln1_beta = to_vec<T>(ps[1], h);
  g.w_qkv = to_mat<T>(ps[2], h, 3 * h);
  g.b_qkv = to_vec<T>(ps[3], 3 * h);
  g.w_out = to_mat<T>(ps[4], h, h);
  g.b_out = to_vec<T>(ps[5], h);
  g.ln2_gamma = to_vec<T>(ps[6], h);
  g.ln2_beta = to_vec<T>(ps[7], h);
  g.w_fc1 = to_mat<T>(ps[8], h, 4 * h);
  g.b_fc1 = to_vec<T>(ps[9], 4 * h);
  g.w_fc2 = to_mat<T>(ps[10], 4 * h, h);
  g.b_fc2 = to_vec<T>(ps[11], h);
  return g;
}

template <typename T>
void put_params(const GlobalLayerParams<T>& g, double* const* out) {
  put(g.ln1_gamma, out[0]);
  put(g.ln1_beta, out[1]);
  put(g.w_qkv, out[2]);
  put(g.b_qkv, out[3]);
  put(g.w_out, out[4]);
  put(g.b_out, out[5]);
  put(g.ln2_gamma, out[6]);
  put(g.ln2_beta, out[7]);
  put(g.w_fc1, out[8]);
  put(g.b_fc1, out[9]);
  put(g.w_fc2, out[10]);
  put(g.b_fc2, out[11]);
}

void put_counters(const std::vector<CostCounters>& cs, uint64_t* out) {
  // per rank: sent, received, madds
  for (std::size_t r = 0; r < cs.size(); ++r) {
    out[3 * r + 0] = cs[r].elements_sent;
    out[3 * r + 1] = cs[r].elements_received;
    out[3 * r + 2] = cs[r].multiply_adds;
  }
}

template <typename T>
void run_matmul_t(int p, int form, int64_t M, int64_t N, int64_t K, const double* a,
                  const double* b, const double* g, double* c, double* da, double* db,
                  uint64_t* counters) {
  MatmulForm f = form == 0 ? MatmulForm::AB : form == 1 ? MatmulForm::ABt : MatmulForm::AtB;
  // shapes per form: AB: A MxN, B NxK, G MxK; ABt: A MxN, B KxN, G MxK; AtB: A MxN, B MxK, G NxK
  Matrix<T> A = to_mat<T>(a, M, N);
  Matrix<T> B = f == MatmulForm::AB ? to_mat<T>(b, N, K)
                : f == MatmulForm::ABt ? to_mat<T>(b, K, N)
                                       : to_mat<T>(b, M, K);
  Matrix<T> G = f == MatmulForm::AtB ? to_mat<T>(g, N, K) : to_mat<T>(g, M, K);
  auto art = verify_detail::run_matmul<T>(p, A, B, G, f, Scheduler::threads);
  put(art.c, c);
  put(art.da, da);
  put(art.db, db);
  if (counters) put_counters(art.counters, counters);
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// ---- Rng (cube3d/rng.hpp)
int ref_rng_uniform(uint64_t seed, int64_t skip, double lo, double hi, int64_t n, double* out) {
  return guard([&] {
    Rng r(seed);
    for (int64_t i = 0; i < skip; ++i) r.next_u64();
    for (int64_t i = 0; i < n; ++i) out[i] = r.uniform(lo, hi);
  });
}
int ref_rng_u64(uint64_t seed, int64_t n, uint64_t* out) {
  return guard([&] {
    Rng r(seed);
    for (int64_t i = 0; i < n; ++i) out[i] = r.next_u64();
  });
}
int ref_random_integer_matrix(uint64_t seed, int64_t rows, int64_t cols, double* out) {
  return guard([&] {
    Rng r(seed);
    put(random_integer_matrix<double>(rows, cols, r), out);
  });
}
// init_layer_params (cube3d/transformer.hpp:198-218), float64
int ref_init_layer_params(int64_t hidden, uint64_t seed, double* const* out) {
  return guard([&] {
    TransformerConfig cfg = make_cfg(1, 1, 1, 1, hidden);
    put_params(init_layer_params<double>(cfg, seed), out);
  });
}

// ---- placement (cube3d/layout.hpp, activation.hpp)
int ref_shard_bounds(int layout, int p, int i, int j, int l, int64_t rows, int64_t cols,
                     int din, int dw, int dout, int64_t* out) {
  return guard([&] {
    DirectionTriple d{static_cast<Axis>(din), static_cast<Axis>(dw), static_cast<Axis>(dout)};
    ShardBounds b = shard_bounds(static_cast<Layout>(layout), Coords{i, j, l}, rows, cols, p, d);
    out[0] = b.rows.begin;
    out[1] = b.rows.end;
    out[2] = b.cols.begin;
    out[3] = b.cols.end;
  });
}
int ref_diagonal_slice(int p, int i, int j, int l, int64_t len, int* holds, int64_t* out) {
  return guard([&] {
    Coords c{i, j, l};
    *holds = diagonal_holder(c) ? 1 : 0;
    IndexRange r = diagonal_slice(c, len, p);
    out[0] = r.begin;
    out[1] = r.end;
  });
}
// activation_from_global of an iota matrix: out[rank][local] = global flat index
int ref_activation_map(int p, int64_t batch, int64_t seq, int64_t hidden, int group,
                       double* out) {
  return guard([&] {
    CubeTopology topo(p);
    Matrix<double> g(batch * seq, hidden);
    for (std::size_t t = 0; t < g.data.size(); ++t) g.data[t] = static_cast<double>(t);
    auto fam = activation_from_global(g, batch, seq, group, topo);
    std::size_t off = 0;
    for (const auto& a : fam) {
      put(a.local, out + off);
      off += a.local.data.size();
    }
  });
}

// ---- drivers (cube3d/verify.hpp:60-232) and the serial oracle (cube3d/reference.hpp)
int ref_run_matmul(int p, int form, int f32, int64_t M, int64_t N, int64_t K, const double* a,
                   const double* b, const double* g, double* c, double* da, double* db,
                   uint64_t* counters) {
  return guard([&] {
    if (f32) run_matmul_t<float>(p, form, M, N, K, a, b, g, c, da, db, counters);
    else run_matmul_t<double>(p, form, M, N, K, a, b, g, c, da, db, counters);
  });
}

int ref_serial_matmul(int form, int64_t M, int64_t N, int64_t K, const double* a,
                      const double* b, double* c) {
  return guard([&] {
    MatmulForm f = form == 0 ? MatmulForm::AB : form == 1 ? MatmulForm::ABt : MatmulForm::AtB;
    Matrix<double> A = f == MatmulForm::AtB ? to_mat<double>(a, K, M) : to_mat<double>(a, M, K);
    Matrix<double> B = f == MatmulForm::ABt ? to_mat<double>(b, N, K) : to_mat<double>(b, K, N);
    put(serial_matmul(A, B, f), c);
  });
}

// Full layer through the 3-D path (run_layer) at cube side p; params/x/dy given.
// outs: y, dx, then 12 parameter gradients. counters: 3 per rank.
int ref_run_layer(int p, int f32, int64_t b, int64_t s, int64_t n, int64_t h,
                  const double* const* params, const double* x, const double* dy, double* y,
                  double* dx, double* const* dparams, uint64_t* counters, double* seconds) {
  return guard([&] {
    TransformerConfig cfg = make_cfg(p, b, s, n, h);
    cfg.validate();
    auto t0 = std::chrono::steady_clock::now();
    if (f32) {
      auto gp = params_of<float>(cfg, params);
      auto art = verify_detail::run_layer<float>(cfg, gp, to_mat<float>(x, b * s, h),
                                                 to_mat<float>(dy, b * s, h), Scheduler::threads);
      put(art.y, y);
      put(art.dx, dx);
      put_params(art.dparams, dparams);
      if (counters) put_counters(art.counters, counters);
    } else {
      auto gp = params_of<double>(cfg, params);
      auto art = verify_detail::run_layer<double>(cfg, gp, to_mat<double>(x, b * s, h),
                                                  to_mat<double>(dy, b * s, h), Scheduler::threads);
      put(art.y, y);
      put(art.dx, dx);
      put_params(art.dparams, dparams);
      if (counters) put_counters(art.counters, counters);
    }
    if (seconds)
      *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  });
}

// The reference's own 3-D layer fwd and bwd (transformer_layer_fwd/bwd,
// cube3d/transformer.hpp:116-148) on run_spmd's rank threads, float, with an
// Endpoint barrier between the two so the forward and backward are timed
// separately (SURVEY.md §8(d) "time fwd and bwd separately with a barrier").
// Same partitioning as verify_detail::run_layer (cube3d/verify.hpp:182-202);
// outputs are discarded: this entry is the CPU baseline clock, run_layer above
// is the checker. seconds[0] = fwd, seconds[1] = bwd (rank 0's wall clock).
int ref_time_layer(int p, int64_t b, int64_t s, int64_t n, int64_t h,
                   const double* const* params, const double* x, const double* dy,
                   double* seconds) {
  return guard([&] {
    TransformerConfig cfg = make_cfg(p, b, s, n, h);
    cfg.validate();
    CubeTopology topo(cfg.p);
    auto gp = params_of<float>(cfg, params);
    auto ps = partition_layer_params(gp, cfg, topo, 0);
    auto xs = activation_from_global(to_mat<float>(x, b * s, h), cfg.batch, cfg.seq, 0, topo);
    auto dys = activation_from_global(to_mat<float>(dy, b * s, h), cfg.batch, cfg.seq, 0, topo);
    Transport<float> tr(topo, Scheduler::threads);
    double tf = 0, tb = 0;
    run_spmd(tr, [&](Endpoint<float>& ep) {
      const int r = ep.rank();
      GroupState gs{0};
      LayerSaved<float> saved;
      ep.barrier();
      auto t0 = std::chrono::steady_clock::now();
      auto y = transformer_layer_fwd(ep, xs[r], ps[r], cfg, gs, &saved);
      ep.barrier();
      auto t1 = std::chrono::steady_clock::now();
      auto g = transformer_layer_bwd(ep, dys[r], saved, ps[r], cfg);
      ep.barrier();
      auto t2 = std::chrono::steady_clock::now();
      if (r == 0) {
        tf = std::chrono::duration<double>(t1 - t0).count();
        tb = std::chrono::duration<double>(t2 - t1).count();
      }
      (void)y;
      (void)g;
    });
    seconds[0] = tf;
    seconds[1] = tb;
  });
}

// The reference's own matrix files (cube3d/matrix_io.hpp) and checkpoints
// (transformer.hpp:259-293), to pin the format of paper_2105_14450_b200/matrix_io.py.
int ref_write_matrix(const char* path, int64_t rows, int64_t cols, const double* data, int f32) {
  return guard([&] {
    if (f32) write_matrix_file(path, to_mat<float>(data, rows, cols));
    else write_matrix_file(path, to_mat<double>(data, rows, cols));
  });
}
int ref_read_matrix(const char* path, int f32, int64_t* rows, int64_t* cols, double* data,
                    int64_t cap) {
  return guard([&] {
    auto rd = [&](auto m) {
      *rows = static_cast<int64_t>(m.rows);
      *cols = static_cast<int64_t>(m.cols);
      if (data && static_cast<int64_t>(m.data.size()) <= cap) put(m, data);
    };
    if (f32) rd(read_matrix_file<float>(path));
    else rd(read_matrix_file<double>(path));
  });
}
int ref_save_layer_params(int64_t h, const double* const* params, const char* prefix) {
  return guard([&] {
    TransformerConfig cfg = make_cfg(1, 1, 1, 1, h);
    save_layer_params(params_of<double>(cfg, params), prefix);
  });
}
int ref_load_layer_params(int64_t h, const char* prefix, double* const* out) {
  return guard([&] {
    (void)h;
    put_params(load_layer_params<double>(prefix), out);
  });
}
// The bench subcommand's modeled scaling table (cube3d/bench.hpp), as CSV text.
int ref_scaling_csv(int weak, int64_t b, int64_t s, int64_t n, int64_t h, int64_t layers,
                    const int* p_list, int np, double lambda, char* buf, int64_t buflen) {
  return guard([&] {
    TransformerConfig base = make_cfg(1, b, s, n, h);
    base.layers = layers;
    std::vector<int> ps(p_list, p_list + np);
    auto rows = run_scaling(weak ? ScalingMode::weak : ScalingMode::strong, base, ps, lambda);
    std::ostringstream os;
    write_scaling_csv(os, rows);
    std::strncpy(buf, os.str().c_str(), static_cast<std::size_t>(buflen - 1));
    buf[buflen - 1] = 0;
  });
}

// Serial reference layer (ref_layer_fwd/bwd, cube3d/reference.hpp:301-354), float64.
int ref_layer_serial(int64_t b, int64_t s, int64_t n, int64_t h, const double* const* params,
                     const double* x, const double* dy, double* y, double* dx,
                     double* const* dparams) {
  return guard([&] {
    TransformerConfig cfg = make_cfg(1, b, s, n, h);
    auto gp = params_of<double>(cfg, params);
    RefLayerCache<double> cache;
    auto yy = ref_layer_fwd(cfg, to_mat<double>(x, b * s, h), gp, &cache);
    auto g = ref_layer_bwd(cfg, to_mat<double>(dy, b * s, h), cache, gp);
    put(yy, y);
    put(g.dx, dx);
    put_params(g.dparams, dparams);
  });
}

// Cost model (cube3d/cost_model.hpp): global traffic of a layer fwd / bwd, per-rank madds.
int ref_layer_costs(int p, int64_t b, int64_t s, int64_t n, int64_t h, uint64_t* out) {
  return guard([&] {
    TransformerConfig cfg = make_cfg(p, b, s, n, h);
    out[0] = traffic::transformer_layer_fwd(cfg);
    out[1] = traffic::transformer_layer_bwd(cfg);
    out[2] = madds::transformer_layer_fwd(cfg);
    out[3] = madds::transformer_layer_bwd(cfg);
  });
}
int ref_predict_costs(int64_t m, int64_t n, int64_t k, int p, uint64_t* out) {
  return guard([&] {
    CostPrediction c = predict_costs(m, n, k, p);
    out[0] = c.memory_elems;
    out[1] = c.multiply_adds;
    out[2] = c.comm_elems;
    out[3] = c.latency_hops;
  });
}

// run_verify (cube3d/verify.hpp:305-749) at the toy configuration; report into buf.
int ref_run_verify(int p, int64_t b, int64_t s, int64_t n, int64_t h, uint64_t seed, int f32,
                   char* buf, int64_t buflen) {
  VerifyOptions o;
  o.p = p;
  o.batch = b;
  o.seq = s;
  o.heads = n;
  o.hidden = h;
  o.seed = seed;
  std::ostringstream os;
  const bool ok = f32 ? run_verify<float>(o, os) : run_verify<double>(o, os);
  std::string r = os.str();
  std::strncpy(buf, r.c_str(), static_cast<std::size_t>(buflen - 1));
  buf[buflen - 1] = 0;
  return ok ? 0 : 1;
}

}  // extern "C"
