// 3-D matmul and matrix-vector operators (cube3d/ops3d.hpp), executed per rank
// as: NCCL all-gathers along the operand axes -> one local GEMM whose operand
// views address the gathered buffers in place (no gather_cols reorder, no
// transposes) -> reduce-scatter along the result axis (fused into the GEMM epilogue over
// NVLink peer memory when the shapes allow, fused.cu) -> fused epilogue.
#include <string>

#include "common.hpp"
#include "kernels.hpp"
#include "ops.hpp"

#include <cstdlib>
#include <memory>

namespace c3d {

namespace {

bool input_family(const Mat& m) { return m.layout == kInput || m.layout == kOutput; }

void require_input_family(const Mat& m, const char* what) {
  if (!input_family(m))
    fail(C3D_ERR_SHAPE_MISMATCH, std::string(what) + " must be in the Input/Output family, got " +
                                     layout_name(m.layout));
}

View kmajor(const void* p, int dtype, int64_t ld) {
  View v;
  v.base = const_cast<void*>(p);
  v.dtype = dtype;
  v.sr = ld;
  v.sc = 1;
  return v;
}
View mnmajor(const void* p, int dtype, int64_t ld) {
  View v;
  v.base = const_cast<void*>(p);
  v.dtype = dtype;
  v.sr = 1;
  v.sc = ld;
  return v;
}
View out_view(void* p, int dtype, int64_t ld) {
  View v;
  v.base = p;
  v.dtype = dtype;
  v.sr = ld;
  v.sc = 1;
  return v;
}

void local_gemm(Cube& cube, int mode, int64_t M, int64_t N, int64_t K, const View& a,
                const View& b, const Epilogue& e, cudaStream_t s) {
  GemmProblem p;
  p.M = M;
  p.N = N;
  p.K = K;
  p.a = a;
  p.b = b;
  p.epi = e;
  run_gemm(p, mode, cube.num_sms(), s);
  cube.add_madds(static_cast<uint64_t>(M) * N * K);
}

}  // namespace

void gemm_views(Cube& cube, int mode, int64_t M, int64_t N, int64_t K, int batch, const View& a,
                const View& b, const Epilogue& e, cudaStream_t s) {
  GemmProblem p;
  p.M = M;
  p.N = N;
  p.K = K;
  p.batch = batch;
  p.a = a;
  p.b = b;
  p.epi = e;
  run_gemm(p, mode, cube.num_sms(), s);
  cube.add_madds(static_cast<uint64_t>(batch) * M * N * K);
}

Mat make_mat(const Cube& cube, void* data, int dtype, int64_t grows, int64_t gcols, int layout,
             const Dirs& dirs) {
  Mat m;
  m.data = data;
  m.dtype = dtype;
  m.grows = grows;
  m.gcols = gcols;
  m.layout = layout;
  m.dirs = dirs;
  if (dtype != kF32 && dtype != kBF16) fail(C3D_ERR_CONFIG_INVALID, "unknown dtype");
  const Bounds b = shard_bounds(layout, cube.grid(), cube.coords(), grows, gcols, dirs);
  m.rows = b.rows.size();
  m.cols = b.cols.size();
  return m;
}

Mat from_c(const Cube& cube, const c3d_matrix& m) {
  Dirs d{m.dirs[0], m.dirs[1], m.dirs[2]};
  if (m.layout < 0 || m.layout > 3) fail(C3D_ERR_SHAPE_MISMATCH, "unknown layout");
  return make_mat(cube, m.data, m.dtype, m.global_rows, m.global_cols, m.layout, d);
}

void to_c(const Mat& m, c3d_matrix* out) {
  out->data = m.data;
  out->dtype = m.dtype;
  out->global_rows = m.grows;
  out->global_cols = m.gcols;
  out->layout = m.layout;
  out->dirs[0] = m.dirs.in;
  out->dirs[1] = m.dirs.w;
  out->dirs[2] = m.dirs.out;
}

Gathered gather(Cube& cube, int axis, const void* shard, size_t count, int dtype,
                cudaStream_t s) {
  Gathered g;
  const int p = cube.extent(axis);
  if (p == 1) {
    g.ptr = shard;
    return g;
  }
  if (cube.symm() && std::getenv("C3D_DIRECT_AG")) {
    // straight into a symmetric buffer: the peers push their shards over NVLink (opt-in:
    // on this pool it measured no faster than the mailbox path, whose copy-out is cheap)
    auto sb = std::make_unique<SymBuf>(cube.symm(), count * p * dtype_size(dtype));
    if (sb->ok()) {
      cube.all_gather_sym(axis, shard, *sb, count, dtype, s);
      g.ptr = sb->local();
      g.sym = std::move(sb);
      return g;
    }
  }
  g.buf = DevBuf(count * p * dtype_size(dtype), s);
  cube.all_gather(axis, shard, g.buf.get(), count, dtype, s);
  g.ptr = g.buf.get();
  return g;
}

// ---------------------------------------------------------------- vectors

// Extents of the two alternating axes for the diagonal collectives: the cube rule
// (Pi == Po) broadcasts from the diagonal rank; with Pi == 1 every rank already holds
// its output block's slices; with Po == 1 the blocks of the whole input-axis line are
// gathered (grid.hpp, generalised diagonal placement).
namespace {
struct DiagPlan {
  int Pi, Po, px;
  bool cube_rule() const { return Pi == Po; }
  bool gather_in() const { return Pi > Po; }  // Po == 1
};
DiagPlan diag_plan(const Cube& cube, const Dirs& d) {
  const Grid& g = cube.grid();
  require_diagonal_grid(g);
  DiagPlan p{g.dims[d.in], g.dims[d.out], g.dims[kX]};
  if (p.Pi != p.Po && p.Pi != 1 && p.Po != 1)
    fail(C3D_ERR_CONFIG_INVALID, "diagonal vectors need equal input/output axis extents or one of "
                                 "them 1");
  return p;
}
}  // namespace

DevBuf expand_diagonal(Cube& cube, const Dirs& d, const Vec& v, cudaStream_t s) {
  const Grid& g = cube.grid();
  const DiagPlan pl = diag_plan(cube, d);
  const Range sl = diagonal_slice(g, cube.coords(), v.len);
  const int64_t n2 = sl.size();
  const int px = pl.px;
  const int64_t out_len = n2 * px * (pl.gather_in() ? pl.Pi : 1);
  DevBuf out(static_cast<size_t>(out_len) * sizeof(float), s);
  if (g.size() == 1) {
    k_convert(v.data, v.dtype, out.get(), kF32, n2, s);
    return out;
  }
  // cube rule: broadcast the holder's slice along the operand's input axis from position
  // owner[d.out] (the diagonal rank of that line); then all-gather along x, and along
  // the input axis when the output axis is not partitioned.
  DevBuf piece(static_cast<size_t>(n2) * dtype_size(v.dtype), s);
  if (diagonal_holder(g, cube.coords()))
    C3D_CUDA(cudaMemcpyAsync(piece.get(), v.data, n2 * dtype_size(v.dtype),
                             cudaMemcpyDeviceToDevice, s));
  if (pl.cube_rule() && pl.Pi > 1) cube.broadcast(d.in, cube.coord(d.out), piece.get(), n2, v.dtype, s);
  DevBuf xfull;
  const void* cur = piece.get();
  if (px > 1) {
    xfull = DevBuf(static_cast<size_t>(n2 * px) * dtype_size(v.dtype), s);
    cube.all_gather(kX, piece.get(), xfull.get(), n2, v.dtype, s);
    cur = xfull.get();
  }
  DevBuf infull;
  if (pl.gather_in()) {
    infull = DevBuf(static_cast<size_t>(out_len) * dtype_size(v.dtype), s);
    cube.all_gather(d.in, cur, infull.get(), n2 * px, v.dtype, s);
    cur = infull.get();
  }
  k_convert(cur, v.dtype, out.get(), kF32, out_len, s);
  return out;
}

void reduce_to_diagonal(Cube& cube, const Dirs& d, const float* colsums, int nvec,
                        const Vec* outs, cudaStream_t s) {
  std::vector<Vec> vs(outs, outs + nvec);
  // one vector at a time is the packed form with one entry per vector
  reduce_to_diagonal_multi(cube, d, colsums, vs, s);
}

DevBuf expand_diagonal_multi(Cube& cube, const Dirs& d, const std::vector<Vec>& vs,
                             std::vector<const float*>* blocks, cudaStream_t s) {
  const Grid& g = cube.grid();
  const DiagPlan pl = diag_plan(cube, d);
  const int px = pl.px;
  const int G = pl.gather_in() ? pl.Pi : 1;  // input-axis blocks per expanded vector
  const bool holder = diagonal_holder(g, cube.coords());
  std::vector<int64_t> n2(vs.size()), off(vs.size());
  int64_t S = 0;
  for (size_t k = 0; k < vs.size(); ++k) {
    n2[k] = diagonal_slice(g, cube.coords(), vs[k].len).size();
    off[k] = S;
    S += n2[k];
    if (vs[k].dtype != kF32) fail(C3D_ERR_CONFIG_INVALID, "packed expansion needs fp32 vectors");
    if (holder && vs[k].data == nullptr)
      fail(C3D_ERR_LENGTH_MISMATCH, "diagonal rank holds no buffer for its vector slice");
  }
  DevBuf out(static_cast<size_t>(S * px * G) * sizeof(float), s);
  blocks->assign(vs.size(), nullptr);
  for (size_t k = 0; k < vs.size(); ++k) (*blocks)[k] = out.as<float>() + off[k] * px * G;
  if (g.size() == 1) {
    for (size_t k = 0; k < vs.size(); ++k)
      C3D_CUDA(cudaMemcpyAsync(out.as<float>() + off[k], vs[k].data, n2[k] * sizeof(float),
                               cudaMemcpyDeviceToDevice, s));
    return out;
  }
  // holders pack their slices back to back: [k slice]; broadcast along d.in (cube rule),
  // gather along x -> [q][k slice], along d.in (Po == 1) -> [u][q][k slice]
  DevBuf piece(static_cast<size_t>(S) * sizeof(float), s);
  if (holder)
    for (size_t k = 0; k < vs.size(); ++k)
      C3D_CUDA(cudaMemcpyAsync(piece.as<float>() + off[k], vs[k].data, n2[k] * sizeof(float),
                               cudaMemcpyDeviceToDevice, s));
  if (pl.cube_rule() && pl.Pi > 1) cube.broadcast(d.in, cube.coord(d.out), piece.get(), S, kF32, s);
  DevBuf full(static_cast<size_t>(S * px * G) * sizeof(float), s);
  if (G > 1) {
    DevBuf xf(static_cast<size_t>(S * px) * sizeof(float), s);
    cube.all_gather(kX, piece.get(), xf.get(), S, kF32, s);
    cube.all_gather(d.in, xf.get(), full.get(), S * px, kF32, s);
  } else {
    cube.all_gather(kX, piece.get(), full.get(), S, kF32, s);
  }
  // [u][q][k slice] -> per-vector blocks [k][u][q slice]
  for (size_t k = 0; k < vs.size(); ++k)
    C3D_CUDA(cudaMemcpy2DAsync(out.as<float>() + off[k] * px * G, n2[k] * sizeof(float),
                               full.as<float>() + off[k], S * sizeof(float),
                               n2[k] * sizeof(float), px * G, cudaMemcpyDeviceToDevice, s));
  return out;
}

void reduce_to_diagonal_multi(Cube& cube, const Dirs& d, const float* colsums,
                              const std::vector<Vec>& outs, cudaStream_t s) {
  const Grid& g = cube.grid();
  const DiagPlan pl = diag_plan(cube, d);
  const int px = pl.px;
  const int G = pl.gather_in() ? pl.Pi : 1;
  const bool holder = diagonal_holder(g, cube.coords());
  std::vector<int64_t> n2(outs.size()), off(outs.size());
  int64_t S = 0;
  for (size_t k = 0; k < outs.size(); ++k) {
    n2[k] = diagonal_slice(g, cube.coords(), outs[k].len).size();
    off[k] = S;
    S += n2[k];
    if (holder && outs[k].data == nullptr)
      fail(C3D_ERR_LENGTH_MISMATCH, "diagonal rank holds no buffer for its vector slice");
  }
  if (g.size() == 1) {
    std::vector<ConvSeg> cv;
    for (size_t k = 0; k < outs.size(); ++k)
      cv.push_back(ConvSeg{colsums + off[k], outs[k].data, kF32, outs[k].dtype, n2[k]});
    k_convert_batch(cv.data(), static_cast<int>(cv.size()), s);
    return;
  }
  // column-sum blocks [k][u][q slice] -> position-major [u][q][k slice]; reduce-scatter
  // along d.in (Po == 1), then along x; all-reduce along d.in (cube rule, the adjoint
  // of the forward broadcast)
  DevBuf packed(static_cast<size_t>(S * px * G) * sizeof(float), s);
  for (size_t k = 0; k < outs.size(); ++k)
    C3D_CUDA(cudaMemcpy2DAsync(packed.as<float>() + off[k], S * sizeof(float),
                               colsums + off[k] * px * G, n2[k] * sizeof(float),
                               n2[k] * sizeof(float), px * G, cudaMemcpyDeviceToDevice, s));
  DevBuf xpart;
  const float* cur = packed.as<float>();
  if (G > 1) {
    xpart = DevBuf(static_cast<size_t>(S * px) * sizeof(float), s);
    cube.reduce_scatter(d.in, cur, xpart.get(), S * px, kF32, s);
    cur = xpart.as<float>();
  }
  DevBuf slice(static_cast<size_t>(S) * sizeof(float), s);
  if (px > 1) {
    cube.reduce_scatter(kX, cur, slice.get(), S, kF32, s);
  } else {
    C3D_CUDA(cudaMemcpyAsync(slice.get(), cur, S * sizeof(float), cudaMemcpyDeviceToDevice, s));
  }
  if (pl.cube_rule() && pl.Pi > 1) cube.all_reduce(d.in, slice.get(), S, kF32, false, s);
  if (holder) {
    std::vector<ConvSeg> cv;
    for (size_t k = 0; k < outs.size(); ++k)
      cv.push_back(ConvSeg{slice.as<float>() + off[k], outs[k].data, kF32, outs[k].dtype, n2[k]});
    k_convert_batch(cv.data(), static_cast<int>(cv.size()), s);
  }
}

void add_vec_fwd(Cube& cube, const Mat& a, const Vec& b, Mat& c, cudaStream_t s) {
  require_input_family(a, "A");
  if (b.len != a.gcols)
    fail(C3D_ERR_SHAPE_MISMATCH, "vector length " + std::to_string(b.len) +
                                     " does not match matrix cols " + std::to_string(a.gcols));
  DevBuf bias = expand_diagonal(cube, a.dirs, b, s);
  c = make_mat(cube, c.data, c.dtype, a.grows, a.gcols, a.layout, a.dirs);
  Epilogue e;
  e.out = out_view(c.data, c.dtype, c.cols);
  e.bias = bias.as<float>();
  k_apply_epilogue(a.data, a.dtype, a.rows, a.cols, e, s);
}

void add_vec_bwd(Cube& cube, const Mat& dc, Mat& da, const Vec& db, cudaStream_t s) {
  require_input_family(dc, "dC");
  DevBuf cs(static_cast<size_t>(dc.cols) * sizeof(float), s);
  k_colsum(dc.data, dc.dtype, nullptr, kF32, dc.rows, dc.cols, cs.as<float>(), s);
  da = make_mat(cube, da.data, da.dtype, dc.grows, dc.gcols, dc.layout, dc.dirs);
  if (da.data != dc.data) k_convert(dc.data, dc.dtype, da.data, da.dtype, dc.elems(), s);
  Vec out = db;
  out.len = dc.gcols;
  reduce_to_diagonal(cube, dc.dirs, cs.as<float>(), 1, &out, s);
}

void mul_vec_fwd(Cube& cube, const Mat& a, const Vec& b, Mat& c, cudaStream_t s) {
  require_input_family(a, "A");
  if (b.len != a.gcols) fail(C3D_ERR_SHAPE_MISMATCH, "vector length does not match matrix cols");
  DevBuf scale = expand_diagonal(cube, a.dirs, b, s);
  c = make_mat(cube, c.data, c.dtype, a.grows, a.gcols, a.layout, a.dirs);
  k_mul_cols(a.data, a.dtype, scale.as<float>(), c.data, c.dtype, a.rows, a.cols, s);
}

void mul_vec_bwd(Cube& cube, const Mat& dc, const Mat& a, const Vec& b, Mat& da, const Vec& db,
                 cudaStream_t s) {
  require_input_family(dc, "dC");
  if (dc.rows != a.rows || dc.cols != a.cols)
    fail(C3D_ERR_SHAPE_MISMATCH, "dC shape does not match the forward input");
  DevBuf cs(static_cast<size_t>(dc.cols) * sizeof(float), s);
  k_colsum(dc.data, dc.dtype, a.data, a.dtype, dc.rows, dc.cols, cs.as<float>(), s);
  DevBuf scale = expand_diagonal(cube, a.dirs, b, s);
  da = make_mat(cube, da.data, da.dtype, dc.grows, dc.gcols, dc.layout, dc.dirs);
  k_mul_cols(dc.data, dc.dtype, scale.as<float>(), da.data, da.dtype, dc.rows, dc.cols, s);
  Vec out = db;
  out.len = dc.gcols;
  reduce_to_diagonal(cube, dc.dirs, cs.as<float>(), 1, &out, s);
}

// ---------------------------------------------------------------- C = A B

namespace {

// dst[y][x][seg rows] = src[x][y][seg rows] (x < outer, y < inner): the row-block swap
// between the [input-axis block][batch][seq] order of an all-gathered activation and the
// [batch][seq] order of Activation3D (cube3d/activation.hpp:103-138) on grids with
// py != pz. One strided copy per x.
void swap_row_blocks(const void* src, void* dst, int64_t outer, int64_t inner, int64_t seg_rows,
                     int64_t cols, int dtype, cudaStream_t s) {
  const size_t blk = static_cast<size_t>(seg_rows * cols) * dtype_size(dtype);
  for (int64_t x = 0; x < outer; ++x)
    C3D_CUDA(cudaMemcpy2DAsync(static_cast<char*>(dst) + x * blk, outer * blk,
                               static_cast<const char*>(src) + x * inner * blk, blk, blk, inner,
                               cudaMemcpyDeviceToDevice, s));
}

}  // namespace

void ab_forward(Cube& cube, int mode, const Mat& a, const Mat& b, Mat& c, const LinearEpi& le,
                cudaStream_t s, const Operand* bg, Gathered* keep_a, const ActRows* ar) {
  const Dirs d = a.dirs;
  const int Pin = cube.extent(d.in), Pw = cube.extent(d.w), Pout = cube.extent(d.out);
  // a: (M/(Pw Pin)) x (N/Pout); b: (N/Pout) x (K/(Pin Pw))
  Gathered bf;
  long long b_hi = b.rows * b.cols;
  if (bg && bg->ptr) {
    bf.ptr = bg->ptr;
    b_hi = bg->s_hi;
  } else {
    bf = gather(cube, d.w, b.data, b.elems(), b.dtype, s);  // [Pw][N/Pout][K/(Pin Pw)]
  }
  const int64_t Mg = a.rows * Pin, Kg = a.cols, Ng = b.cols * Pw;
  View bv = mnmajor(bf.ptr, b.dtype, b.cols);
  if (Pw > 1) {
    bv.rsplit = b.cols;
    bv.s_hi = b_hi;
  }
  c = make_mat(cube, c.data, c.dtype, a.grows, b.gcols, kOutput, d.swapped());
  Gathered af = gather(cube, d.in, a.data, a.elems(), a.dtype, s);  // (M/Pw) x (N/Pout)
  if (ar && ar->bl > 1 && Pin != Pout) {
    // activation rows (py != pz): the output's row blocks must follow the [batch][seq]
    // order of the other group -- gathered [a][b][s] -> [b][a][s] (Pout == 1), or local
    // [b][o][s] -> [o][b][s] before the reduce-scatter into Pout blocks (Pin == 1)
    Gathered pa;
    pa.buf = DevBuf(static_cast<size_t>(Mg * a.cols) * dtype_size(a.dtype), s);
    if (Pin > Pout)
      swap_row_blocks(af.ptr, pa.buf.get(), Pin, ar->bl, ar->seq / Pin, a.cols, a.dtype, s);
    else
      swap_row_blocks(af.ptr, pa.buf.get(), ar->bl, Pout, ar->seq / Pout, a.cols, a.dtype, s);
    pa.ptr = pa.buf.get();
    af = std::move(pa);
  }
  View av = kmajor(af.ptr, a.dtype, a.cols);
  if (keep_a) *keep_a = std::move(af);  // buffer (if any) outlives this call
  Epilogue e;
  if (Pout == 1) {
    e.out = out_view(c.data, c.dtype, c.cols);
    e.bias = le.bias;
    e.act = le.act;
    e.pre_act = le.pre_act;
    e.pre_dtype = c.dtype;
    e.resid = le.resid;
    e.resid_dtype = c.dtype;
    local_gemm(cube, mode, Mg, Ng, Kg, av, bv, e, s);
    return;
  }
  Epilogue f;
  f.out = out_view(c.data, c.dtype, c.cols);
  f.bias = le.bias;
  f.act = le.act;
  f.pre_act = le.pre_act;
  f.pre_dtype = c.dtype;
  f.resid = le.resid;
  f.resid_dtype = c.dtype;
  if (gemm_reduce_scatter(cube, mode, d.out, Mg, Ng, Kg, av, bv, f, s)) return;
  DevBuf partial(static_cast<size_t>(Mg * Ng) * dtype_size(c.dtype), s);
  e.out = out_view(partial.get(), c.dtype, Ng);
  local_gemm(cube, mode, Mg, Ng, Kg, av, bv, e, s);
  cube.reduce_scatter(d.out, partial.get(), c.data, c.elems(), c.dtype, s);
  if (le.bias || le.act != kActNone || le.resid) k_apply_epilogue(c.data, c.dtype, c.rows, c.cols, f, s);
}

void ab_backward(Cube& cube, int mode, const Mat& dc, const Mat& a, const Mat& b, Mat* da,
                 Mat* db, const void* da_gelu_aux, cudaStream_t s, const Operand* bg,
                 const void* ag, const DwSink* dw, const ActRows* ar) {
  const Dirs d = a.dirs;
  const int Pin = cube.extent(d.in), Pw = cube.extent(d.w), Pout = cube.extent(d.out);
  // dC: (M/(Pw Pout)) x (K/Pin) with triple d.swapped(): gather along d.out
  Gathered dcf;
  bool have_dcf = false;
  const bool want_db = db && db->data;
  auto need_dcf = [&] {
    if (!have_dcf) dcf = gather(cube, d.out, dc.data, dc.elems(), dc.dtype, s);  // (M/Pw) x (K/Pin)
    have_dcf = true;
  };
  const int64_t Mrows = dc.rows * Pout, Kc = dc.cols;
  if (da && da->data) {
    Gathered bf;
    long long b_hi = b.rows * b.cols;
    if (bg && bg->ptr) {
      bf.ptr = bg->ptr;
      b_hi = bg->s_hi;
    } else {
      bf = gather(cube, d.w, b.data, b.elems(), b.dtype, s);
    }
    *da = make_mat(cube, da->data, da->dtype, a.grows, a.gcols, a.layout, a.dirs);
    // partial dA (M/Pw) x (N/Pout) = dc_full * b_full^T
    View bv = kmajor(bf.ptr, b.dtype, b.cols);
    if (Pw > 1) {
      bv.csplit = b.cols;
      bv.s_hi = b_hi;
    }
    need_dcf();
    // activation rows (py != pz), the adjoint of ab_forward's swaps: dC [b][a][s] ->
    // [a][b][s] before the reduce-scatter along d.in (Pout == 1); dA [o][b][s] -> [b][o][s]
    // after the product (Pin == 1)
    const bool swap = ar && ar->bl > 1 && Pin != Pout;
    DevBuf dcp;
    const void* dca = dcf.ptr;
    if (swap && Pin > Pout) {
      dcp = DevBuf(static_cast<size_t>(Mrows * Kc) * dtype_size(dc.dtype), s);
      swap_row_blocks(dcf.ptr, dcp.get(), ar->bl, Pin, ar->seq / Pin, Kc, dc.dtype, s);
      dca = dcp.get();
    }
    View av = kmajor(dca, dc.dtype, Kc);
    Epilogue e;
    if (swap && Pin < Pout) {
      DevBuf tmp(static_cast<size_t>(Mrows * b.rows) * dtype_size(da->dtype), s);
      e.out = out_view(tmp.get(), da->dtype, b.rows);
      local_gemm(cube, mode, Mrows, b.rows, Kc, av, bv, e, s);
      swap_row_blocks(tmp.get(), da->data, Pout, ar->bl, ar->seq / Pout, b.rows, da->dtype, s);
      if (da_gelu_aux) {
        Epilogue f;
        f.out = out_view(da->data, da->dtype, da->cols);
        f.act = kActMulAux;
        f.aux = da_gelu_aux;
        f.aux_dtype = da->dtype;
        k_apply_epilogue(da->data, da->dtype, da->rows, da->cols, f, s);
      }
    } else if (Pin == 1) {
      e.out = out_view(da->data, da->dtype, da->cols);
      if (da_gelu_aux) {
        e.act = kActMulAux;
        e.aux = da_gelu_aux;
        e.aux_dtype = da->dtype;
      }
      local_gemm(cube, mode, Mrows, b.rows, Kc, av, bv, e, s);
    } else {
      Epilogue f;
      f.out = out_view(da->data, da->dtype, da->cols);
      if (da_gelu_aux) {
        f.act = kActMulAux;
        f.aux = da_gelu_aux;
        f.aux_dtype = da->dtype;
      }
      if (!gemm_reduce_scatter(cube, mode, d.in, Mrows, b.rows, Kc, av, bv, f, s)) {
        DevBuf partial(static_cast<size_t>(Mrows * b.rows) * dtype_size(da->dtype), s);
        e.out = out_view(partial.get(), da->dtype, b.rows);
        local_gemm(cube, mode, Mrows, b.rows, Kc, av, bv, e, s);
        cube.reduce_scatter(d.in, partial.get(), da->data, da->elems(), da->dtype, s);
        if (da_gelu_aux) k_apply_epilogue(da->data, da->dtype, da->rows, da->cols, f, s);
      }
    }
  }
  if (want_db) {
    need_dcf();
    Gathered af;
    if (ag) af.ptr = ag;
    else af = gather(cube, d.in, a.data, a.elems(), a.dtype, s);  // (M/Pw) x (N/Pout)
    *db = make_mat(cube, db->data, db->dtype, b.grows, b.gcols, kWeight, d);
    // partial dB[k_in][n] = sum_m a_full[m][k_in] dc_full[m][n], written column-block-major
    // [Pw][N/Pout][K/(Pin Pw)] so the reduce-scatter along x lands each rank's shard.
    View av = mnmajor(af.ptr, a.dtype, a.cols);
    View bv = mnmajor(dcf.ptr, dc.dtype, Kc);
    Epilogue e;
    if (Pw == 1) {
      e.out = out_view(db->data, db->dtype, db->cols);
      local_gemm(cube, mode, a.cols, Kc, Mrows, av, bv, e, s);
    } else if (dw && dw->base) {
      e.out = out_view(dw->base, dw->dtype, db->cols);
      e.out.csplit = db->cols;
      e.out.s_hi = dw->s_hi;
      local_gemm(cube, mode, a.cols, Kc, Mrows, av, bv, e, s);
    } else {
      DevBuf partial(static_cast<size_t>(a.cols * Kc) * dtype_size(db->dtype), s);
      e.out = out_view(partial.get(), db->dtype, db->cols);
      e.out.csplit = db->cols;
      e.out.s_hi = db->rows * db->cols;
      local_gemm(cube, mode, a.cols, Kc, Mrows, av, bv, e, s);
      cube.reduce_scatter(d.w, partial.get(), db->data, db->elems(), db->dtype, s);
    }
  }
}

void matmul_ab_fwd(Cube& cube, int mode, const Mat& a, const Mat& b, Mat& c, cudaStream_t s) {
  require_input_family(a, "A");
  if (b.layout != kWeight) fail(C3D_ERR_SHAPE_MISMATCH, "B of C=AB must be Weight layout");
  if (a.dirs != b.dirs)
    fail(C3D_ERR_DIRECTION_CLASH, "A and B of C=AB must share one direction triple");
  if (a.gcols != b.grows)
    fail(C3D_ERR_SHAPE_MISMATCH, "C=AB needs A cols == B rows, got " + std::to_string(a.gcols) +
                                     " vs " + std::to_string(b.grows));
  ab_forward(cube, mode, a, b, c, LinearEpi{}, s);
}

void matmul_ab_bwd(Cube& cube, int mode, const Mat& dc, const Mat& a, const Mat& b, Mat& da,
                   Mat& db, cudaStream_t s) {
  require_input_family(dc, "dC");
  if (dc.dirs != a.dirs.swapped())
    fail(C3D_ERR_DIRECTION_CLASH, "dC of C=AB backward must carry the swapped triple");
  if (dc.grows != a.grows || dc.gcols != b.gcols)
    fail(C3D_ERR_SHAPE_MISMATCH, "dC shape does not match the forward output");
  ab_backward(cube, mode, dc, a, b, &da, &db, nullptr, s);
}

// ---------------------------------------------------------------- C = A B^T

void matmul_abt_fwd(Cube& cube, int mode, const Mat& a, const Mat& b, Mat& c, cudaStream_t s) {
  require_input_family(a, "A");
  if (b.layout != kWeightOfTranspose)
    fail(C3D_ERR_SHAPE_MISMATCH, "B of C=AB^T must be WeightOfTranspose layout");
  if (a.dirs != b.dirs)
    fail(C3D_ERR_DIRECTION_CLASH, "A and B of C=AB^T must share one direction triple");
  if (a.gcols != b.gcols)
    fail(C3D_ERR_SHAPE_MISMATCH, "C=AB^T needs A cols == B cols, got " +
                                     std::to_string(a.gcols) + " vs " + std::to_string(b.gcols));
  const Dirs d = a.dirs;
  const int Pin = cube.extent(d.in), Pw = cube.extent(d.w), Pout = cube.extent(d.out);
  Gathered af = gather(cube, d.in, a.data, a.elems(), a.dtype, s);  // (M/Pw) x (N/Pout)
  Gathered bf = gather(cube, d.w, b.data, b.elems(), b.dtype, s);   // (K/Pin) x (N/Pout)
  const int64_t Mg = a.rows * Pin, Ng = b.rows * Pw, Kg = a.cols;
  c = make_mat(cube, c.data, c.dtype, a.grows, b.grows, kOutput, d.swapped());
  Epilogue e;
  DevBuf partial;
  if (Pout == 1) {
    e.out = out_view(c.data, c.dtype, c.cols);
  } else {
    partial = DevBuf(static_cast<size_t>(Mg * Ng) * dtype_size(c.dtype), s);
    e.out = out_view(partial.get(), c.dtype, Ng);
  }
  local_gemm(cube, mode, Mg, Ng, Kg, kmajor(af.ptr, a.dtype, a.cols), kmajor(bf.ptr, b.dtype, b.cols),
             e, s);
  if (Pout > 1) cube.reduce_scatter(d.out, partial.get(), c.data, c.elems(), c.dtype, s);
}

void matmul_abt_bwd(Cube& cube, int mode, const Mat& dc, const Mat& a, const Mat& b, Mat& da,
                    Mat& db, cudaStream_t s) {
  require_input_family(dc, "dC");
  if (dc.dirs != a.dirs.swapped())
    fail(C3D_ERR_DIRECTION_CLASH, "dC of C=AB^T backward must carry the swapped triple");
  if (dc.grows != a.grows || dc.gcols != b.grows)
    fail(C3D_ERR_SHAPE_MISMATCH, "dC shape does not match the forward output");
  const Dirs d = a.dirs;
  const int Pin = cube.extent(d.in), Pw = cube.extent(d.w), Pout = cube.extent(d.out);
  Gathered dcf = gather(cube, d.out, dc.data, dc.elems(), dc.dtype, s);  // (M/Pw) x (K/Pin)
  Gathered bf = gather(cube, d.w, b.data, b.elems(), b.dtype, s);       // (K/Pin) x (N/Pout)
  const int64_t Mrows = dc.rows * Pout, Kc = dc.cols;
  {
    da = make_mat(cube, da.data, da.dtype, a.grows, a.gcols, a.layout, a.dirs);
    Epilogue e;
    DevBuf partial;
    if (Pin == 1) {
      e.out = out_view(da.data, da.dtype, da.cols);
    } else {
      partial = DevBuf(static_cast<size_t>(Mrows * b.cols) * dtype_size(da.dtype), s);
      e.out = out_view(partial.get(), da.dtype, b.cols);
    }
    local_gemm(cube, mode, Mrows, b.cols, Kc, kmajor(dcf.ptr, dc.dtype, Kc),
               mnmajor(bf.ptr, b.dtype, b.cols), e, s);
    if (Pin > 1) cube.reduce_scatter(d.in, partial.get(), da.data, da.elems(), da.dtype, s);
  }
  {
    Gathered af = gather(cube, d.in, a.data, a.elems(), a.dtype, s);  // (M/Pw) x (N/Pout)
    db = make_mat(cube, db.data, db.dtype, b.grows, b.gcols, kWeightOfTranspose, d);
    Epilogue e;
    DevBuf partial;
    if (Pw == 1) {
      e.out = out_view(db.data, db.dtype, db.cols);
    } else {
      partial = DevBuf(static_cast<size_t>(Kc * a.cols) * dtype_size(db.dtype), s);
      e.out = out_view(partial.get(), db.dtype, a.cols);
    }
    // partial (K/Pin) x (N/Pout) = dc_full^T a_full
    local_gemm(cube, mode, Kc, a.cols, Mrows, mnmajor(dcf.ptr, dc.dtype, Kc),
               mnmajor(af.ptr, a.dtype, a.cols), e, s);
    if (Pw > 1) cube.reduce_scatter(d.w, partial.get(), db.data, db.elems(), db.dtype, s);
  }
}

// ---------------------------------------------------------------- C = A^T B

void matmul_atb_fwd(Cube& cube, int mode, const Mat& a, const Mat& b, Mat& c, cudaStream_t s) {
  require_input_family(a, "A");
  require_input_family(b, "B");
  if (b.dirs != a.dirs.swapped())
    fail(C3D_ERR_DIRECTION_CLASH, "B of C=A^TB must carry A's swapped triple");
  if (a.grows != b.grows)
    fail(C3D_ERR_SHAPE_MISMATCH, "C=A^TB needs A rows == B rows, got " +
                                     std::to_string(a.grows) + " vs " + std::to_string(b.grows));
  const Dirs d = a.dirs;
  const int Pw = cube.extent(d.w);
  Gathered af = gather(cube, d.in, a.data, a.elems(), a.dtype, s);   // (M/Pw) x (N/Pout)
  Gathered bf = gather(cube, d.out, b.data, b.elems(), b.dtype, s);  // (M/Pw) x (K/Pin)
  const int64_t Mrows = a.rows * cube.extent(d.in);
  c = make_mat(cube, c.data, c.dtype, a.gcols, b.gcols, kWeight, d);
  const int64_t Kc = b.cols;
  Epilogue e;
  DevBuf partial;
  if (Pw == 1) {
    e.out = out_view(c.data, c.dtype, c.cols);
  } else {
    partial = DevBuf(static_cast<size_t>(a.cols * Kc) * dtype_size(c.dtype), s);
    e.out = out_view(partial.get(), c.dtype, c.cols);
    e.out.csplit = c.cols;
    e.out.s_hi = c.rows * c.cols;
  }
  local_gemm(cube, mode, a.cols, Kc, Mrows, mnmajor(af.ptr, a.dtype, a.cols),
             mnmajor(bf.ptr, b.dtype, Kc), e, s);
  if (Pw > 1) cube.reduce_scatter(d.w, partial.get(), c.data, c.elems(), c.dtype, s);
}

void matmul_atb_bwd(Cube& cube, int mode, const Mat& dc, const Mat& a, const Mat& b, Mat& da,
                    Mat& db, cudaStream_t s) {
  if (dc.layout != kWeight)
    fail(C3D_ERR_SHAPE_MISMATCH, "dC of C=A^TB backward must be Weight layout");
  if (dc.dirs != a.dirs) fail(C3D_ERR_DIRECTION_CLASH, "dC of C=A^TB backward must carry A's triple");
  if (dc.grows != a.gcols || dc.gcols != b.gcols)
    fail(C3D_ERR_SHAPE_MISMATCH, "dC shape does not match the forward output");
  const Dirs d = a.dirs;
  const int Pin = cube.extent(d.in), Pw = cube.extent(d.w), Pout = cube.extent(d.out);
  Gathered dcf = gather(cube, d.w, dc.data, dc.elems(), dc.dtype, s);  // [Pw][N/Pout][K/(Pin Pw)]
  const int64_t Kc = dc.cols * Pw;
  {
    Gathered bf = gather(cube, d.out, b.data, b.elems(), b.dtype, s);  // (M/Pw) x (K/Pin)
    const int64_t Mrows = b.rows * Pout;
    da = make_mat(cube, da.data, da.dtype, a.grows, a.gcols, a.layout, a.dirs);
    View bv = kmajor(dcf.ptr, dc.dtype, dc.cols);
    if (Pw > 1) {
      bv.csplit = dc.cols;
      bv.s_hi = dc.rows * dc.cols;
    }
    Epilogue e;
    DevBuf partial;
    if (Pin == 1) {
      e.out = out_view(da.data, da.dtype, da.cols);
    } else {
      partial = DevBuf(static_cast<size_t>(Mrows * dc.rows) * dtype_size(da.dtype), s);
      e.out = out_view(partial.get(), da.dtype, dc.rows);
    }
    local_gemm(cube, mode, Mrows, dc.rows, Kc, kmajor(bf.ptr, b.dtype, b.cols), bv, e, s);
    if (Pin > 1) cube.reduce_scatter(d.in, partial.get(), da.data, da.elems(), da.dtype, s);
  }
  {
    Gathered af = gather(cube, d.in, a.data, a.elems(), a.dtype, s);  // (M/Pw) x (N/Pout)
    const int64_t Mrows = a.rows * Pin;
    db = make_mat(cube, db.data, db.dtype, b.grows, b.gcols, b.layout, b.dirs);
    View bv = mnmajor(dcf.ptr, dc.dtype, dc.cols);
    if (Pw > 1) {
      bv.rsplit = dc.cols;
      bv.s_hi = dc.rows * dc.cols;
    }
    Epilogue e;
    DevBuf partial;
    if (Pout == 1) {
      e.out = out_view(db.data, db.dtype, db.cols);
    } else {
      partial = DevBuf(static_cast<size_t>(Mrows * Kc) * dtype_size(db.dtype), s);
      e.out = out_view(partial.get(), db.dtype, Kc);
    }
    local_gemm(cube, mode, Mrows, Kc, a.cols, kmajor(af.ptr, a.dtype, a.cols), bv, e, s);
    if (Pout > 1) cube.reduce_scatter(d.out, partial.get(), db.data, db.elems(), db.dtype, s);
  }
}

}  // namespace c3d
