// A compiled C++ caller of the drop-in header (include/cube3d_b200.hpp over c3d.h,
// linked against paper_2105_14450_b200/libc3d.so): the reference's call shapes --
// matmul_ab_fwd(ep, a, b), linear3d_fwd(ep, x, p, gs, &saved),
// transformer_layer_fwd/bwd(ep, x, p, cfg, gs, &saved) -- on one GPU, with the
// reference's known answers (tests/test_ops3d.cpp:165-178 integer exactness,
// tests/test_nn_layers.cpp:117-137 identity pass-through, :376-392 zero blocks) and its
// error taxonomy. Prints "PASS <name>" / "FAIL <name>"; exit code = number of failures.
#include <cmath>
#include <cstdio>
#include <random>
#include <string>
#include <vector>

#include "cube3d_b200.hpp"

using namespace cube3d_b200;

static int failures = 0;
static void report(const std::string& name, bool ok, const std::string& detail = "") {
  std::printf("%s %s%s%s\n", ok ? "PASS" : "FAIL", name.c_str(), detail.empty() ? "" : ": ",
              detail.c_str());
  if (!ok) ++failures;
}

static std::vector<float> ints(size_t n, std::mt19937_64& g) {
  std::vector<float> v(n);
  for (auto& x : v) x = static_cast<float>(g() % 10);
  return v;
}

// C[M][K] = A[M][N] B[N][K] (host, exact for small integers)
static std::vector<float> mm(const std::vector<float>& a, const std::vector<float>& b, int M, int N,
                             int K, bool ta = false, bool tb = false) {
  std::vector<float> c(static_cast<size_t>(M) * K, 0.f);
  for (int i = 0; i < M; ++i)
    for (int k = 0; k < K; ++k) {
      double s = 0;
      for (int j = 0; j < N; ++j)
        s += static_cast<double>(ta ? a[j * M + i] : a[i * N + j]) * (tb ? b[k * N + j] : b[j * K + k]);
      c[static_cast<size_t>(i) * K + k] = static_cast<float>(s);
    }
  return c;
}

int main() {
  Endpoint ep(0);
  std::mt19937_64 g(5);
  // ---- 3-D matmul, integer inputs: exact in fp32 SIMT and in bf16 tensor-core mode
  for (int mode : {C3D_MODE_F32, C3D_MODE_TC}) {
    const int dt = mode == C3D_MODE_F32 ? C3D_F32 : C3D_BF16;
    const int M = 256, N = 128, K = 192;
    const DirectionTriple d;
    ShardedMatrix a = empty_matrix(ep, M, N, C3D_INPUT, d, dt);
    ShardedMatrix b = empty_matrix(ep, N, K, C3D_WEIGHT, d, dt);
    const auto ha = ints(M * N, g), hb = ints(N * K, g), hd = ints(M * K, g);
    to_device(ep, ha, *a.shard, dt);
    to_device(ep, hb, *b.shard, dt);
    ShardedMatrix c = matmul_ab_fwd(ep, a, b, mode, C3D_F32);  // exact integer sums
    const auto hc = to_host(ep, *c.shard, M * K, c.dtype);
    report(std::string("matmul_ab_fwd-integer-exact-") + (dt == C3D_F32 ? "f32" : "bf16"),
           hc == mm(ha, hb, M, N, K) && c.layout == C3D_OUTPUT && c.dirs.input == C3D_AXIS_Z);
    ShardedMatrix dc = empty_matrix(ep, M, K, C3D_OUTPUT, d.swapped(), dt);
    to_device(ep, hd, *dc.shard, dt);
    MatmulGrads gr = matmul_ab_bwd(ep, dc, a, b, mode, C3D_F32);
    const auto hda = to_host(ep, *gr.da.shard, M * N, gr.da.dtype);
    const auto hdb = to_host(ep, *gr.db.shard, N * K, gr.db.dtype);
    report(std::string("matmul_ab_bwd-integer-exact-") + (dt == C3D_F32 ? "f32" : "bf16"),
           hda == mm(hd, hb, M, K, N, false, true) && hdb == mm(ha, hd, N, M, K, true, false));
  }
  // ---- error taxonomy: validation before any work (cube3d/ops3d.hpp:117-124)
  try {
    ShardedMatrix a = empty_matrix(ep, 64, 32, C3D_INPUT, DirectionTriple{}, C3D_F32);
    ShardedMatrix b = empty_matrix(ep, 48, 64, C3D_WEIGHT, DirectionTriple{}, C3D_F32);
    matmul_ab_fwd(ep, a, b);
    report("matmul-shape-mismatch-throws", false, "no error");
  } catch (const Error& e) {
    report("matmul-shape-mismatch-throws",
           e.code() == C3D_ERR_SHAPE_MISMATCH && std::string(e.what()).rfind("ShapeMismatch:", 0) == 0,
           e.what());
  }
  // ---- linear3d: identity weight, zero bias -> y == x bitwise, group toggles
  {
    const int b = 2, s = 8, h = 16;
    LinearParams p{empty_matrix(ep, h, h, C3D_WEIGHT, triple_for_group(0), C3D_F32),
                   empty_vector(ep, h), 0};
    std::vector<float> eye(h * h, 0.f), zero(h, 0.f), x(b * s * h);
    for (int i = 0; i < h; ++i) eye[i * h + i] = 1.f;
    for (auto& v : x) v = static_cast<float>(static_cast<int>(g() % 2001) - 1000) / 1000.f;
    to_device(ep, eye, *p.weight.shard, C3D_F32);
    to_device(ep, zero, *p.bias.slice, C3D_F32);
    Activation3D X = empty_activation(ep, b, s, h, 0, C3D_F32);
    to_device(ep, x, *X.local, C3D_F32);
    GroupState gs;
    LinearSaved sv;
    Activation3D y = linear3d_fwd(ep, X, p, gs, &sv, C3D_MODE_F32);
    report("linear3d-identity-bitwise",
           to_host(ep, *y.local, x.size(), C3D_F32) == x && gs.input_group == 1 && y.group == 1);
    LinearGrads lg = linear3d_bwd(ep, y, sv, p, C3D_MODE_F32);
    report("linear3d-bwd-identity", to_host(ep, *lg.dx.local, x.size(), C3D_F32) == x &&
                                        lg.dx.group == 0);
  }
  // ---- transformer layer: zero blocks -> y == x exactly; deterministic backward
  for (int dt : {C3D_F32, C3D_BF16}) {
    const int b = 2, s = 256, n = 4, h = 256;
    const int mode = dt == C3D_F32 ? C3D_MODE_F32 : C3D_MODE_AUTO;
    TransformerConfig cfg{b, s, n, h, 1e-5};
    LayerParams p = empty_layer_params(ep, h, 0, dt);
    auto fill = [&](ShardedMatrix& m, float v) {
      to_device(ep, std::vector<float>(m.rows * m.cols, v), *m.shard, m.dtype);
    };
    auto fillv = [&](DiagonalVector& v, float x) {
      to_device(ep, std::vector<float>(v.len, x), *v.slice, v.dtype);
    };
    for (auto* m : {&p.w_qkv, &p.w_out, &p.w_fc1, &p.w_fc2}) fill(*m, 0.f);
    for (auto* v : {&p.b_qkv, &p.b_out, &p.b_fc1, &p.b_fc2, &p.ln1_beta, &p.ln2_beta}) fillv(*v, 0.f);
    fillv(p.ln1_gamma, 1.f);
    fillv(p.ln2_gamma, 1.f);
    std::vector<float> x(static_cast<size_t>(b) * s * h);
    for (auto& v : x) v = static_cast<float>(static_cast<int>(g() % 2001) - 1000) / 1000.f;
    if (dt == C3D_BF16)
      for (auto& v : x) v = from_bf16(to_bf16(v));
    Activation3D X = empty_activation(ep, b, s, h, 0, dt);
    to_device(ep, x, *X.local, dt);
    GroupState gs;
    LayerSaved sv;
    Activation3D y = transformer_layer_fwd(ep, X, p, cfg, gs, &sv, mode);
    const std::string tag = dt == C3D_F32 ? "f32" : "bf16";
    report("layer-zero-blocks-pass-residual-" + tag,
           to_host(ep, *y.local, x.size(), dt) == x && gs.input_group == 0);
    // random weights: two backward runs are bitwise identical (cube3d/verify.hpp:738-744)
    for (auto* m : {&p.w_qkv, &p.w_out, &p.w_fc1, &p.w_fc2}) {
      std::vector<float> w(m->rows * m->cols);
      for (auto& v : w) v = static_cast<float>(static_cast<int>(g() % 2001) - 1000) / 10000.f;
      to_device(ep, w, *m->shard, m->dtype);
    }
    std::vector<std::vector<float>> dxs;
    for (int rep = 0; rep < 2; ++rep) {
      GroupState gs2;
      LayerSaved sv2;
      Activation3D y2 = transformer_layer_fwd(ep, X, p, cfg, gs2, &sv2, mode);
      LayerGrads lg = transformer_layer_bwd(ep, y2, sv2, p, cfg, mode);
      dxs.push_back(to_host(ep, *lg.dx.local, x.size(), dt));
    }
    bool finite = true;
    for (float v : dxs[0]) finite = finite && std::isfinite(v);
    report("layer-bwd-deterministic-" + tag, finite && dxs[0] == dxs[1]);
  }
  ep.synchronize();
  std::printf("%d failure(s)\n", failures);
  return failures;
}
