// 3-D Linear, LayerNorm, attention, MLP and Transformer layer, forward and
// backward, per rank. Orchestration mirrors the reference call stacks
// (SURVEY.md §3 (2)/(3)); the per-slice attention loop of the reference
// (cube3d/attention.hpp:96-133, 128 iterations and 4 collectives each at
// config 3) becomes batched GEMMs over all local (batch, head) slices with one
// collective per step, and residual adds / bias / GELU / GELU' are fused into
// GEMM epilogues whenever no reduce-scatter intervenes.
#include <algorithm>
#include <cmath>
#include <string>

#include "common.hpp"
#include "kernels.hpp"
#include "nn.hpp"

#include <cstdlib>

namespace c3d {

namespace {

View mk_view(const void* base, int dtype, int64_t sr, int64_t sc) {
  View v;
  v.base = const_cast<void*>(base);
  v.dtype = dtype;
  v.sr = sr;
  v.sc = sc;
  return v;
}

const void* offset(const void* p, int64_t elems, int dtype) {
  return static_cast<const char*>(p) + elems * static_cast<int64_t>(dtype_size(dtype));
}

}  // namespace

Act make_act(const Cube& cube, void* data, int dtype, int64_t batch, int64_t seq, int64_t hidden,
             int group) {
  const ActGeom g = act_geom(cube.grid(), batch, seq, hidden, group);
  Act a;
  a.data = data;
  a.dtype = dtype;
  a.batch = batch;
  a.seq = seq;
  a.hidden = hidden;
  a.group = group;
  a.rows = g.bl * g.sl;
  a.cols = g.hl;
  return a;
}

// flatten (cube3d/activation.hpp:67-79): the activation's Input-layout matrix view.
Mat flatten(const Cube& cube, const Act& a) {
  return make_mat(cube, a.data, a.dtype, a.batch * a.seq, a.hidden, kInput,
                  triple_for_group(a.group));
}

void validate_config(const Cube& cube, const Config& cfg) {
  // TransformerConfig::validate (cube3d/nn.hpp:29-40), per-axis extents.
  const Grid& g = cube.grid();
  if (cfg.batch <= 0 || cfg.seq <= 0 || cfg.heads <= 0 || cfg.hidden <= 0)
    fail(C3D_ERR_CONFIG_INVALID, "batch, seq, heads and hidden must be positive");
  require_diagonal_grid(g);  // py == pz (the reference's cube) or one of them 1
  const int64_t py = g.dims[1], pz = g.dims[2], r = g.dims[0];
  const int64_t Q = std::max(py, pz);
  if (cfg.batch % r) fail(C3D_ERR_CONFIG_INVALID, "batch must be divisible by px");
  if (cfg.seq % py || cfg.seq % pz) fail(C3D_ERR_CONFIG_INVALID, "seq must be divisible by p");
  const int64_t p2 = g.cubic() ? Q * Q : Q * r;
  if (cfg.hidden % p2) fail(C3D_ERR_CONFIG_INVALID, "hidden must be divisible by p^2");
  if ((4 * cfg.hidden) % p2) fail(C3D_ERR_CONFIG_INVALID, "4*hidden must be divisible by p^2");
  if (cfg.heads % py || cfg.heads % pz)
    fail(C3D_ERR_HEADS_INDIVISIBLE,
         "heads=" + std::to_string(cfg.heads) + " not divisible by p=" + std::to_string(Q));
  if (cfg.hidden % cfg.heads) fail(C3D_ERR_CONFIG_INVALID, "hidden must be divisible by heads");
}

// ------------------------------------------------------------------ Linear

void linear_fwd(Cube& cube, int mode, const Act& x, const LinearP& p, int& group, Act& y,
                LinearSaved* saved, bool own_input, const LinearEpi& extra, cudaStream_t s,
                const LinearPre* pre) {
  // linear3d_fwd (cube3d/nn.hpp:81-97)
  if (x.group != group)
    fail(C3D_ERR_GROUP_MISMATCH, "activation group " + std::to_string(x.group) +
                                     " does not match state " + std::to_string(group));
  if (p.input_group != x.group)
    fail(C3D_ERR_GROUP_MISMATCH, "layer parameters were partitioned for input group " +
                                     std::to_string(p.input_group));
  Mat xf = flatten(cube, x);
  if (p.w.layout != kWeight) fail(C3D_ERR_SHAPE_MISMATCH, "B of C=AB must be Weight layout");
  if (xf.dirs != p.w.dirs)
    fail(C3D_ERR_DIRECTION_CLASH, "A and B of C=AB must share one direction triple");
  if (xf.gcols != p.w.grows)
    fail(C3D_ERR_SHAPE_MISMATCH, "C=AB needs A cols == B rows, got " +
                                     std::to_string(xf.gcols) + " vs " + std::to_string(p.w.grows));
  if (p.b.len != p.w.gcols)
    fail(C3D_ERR_SHAPE_MISMATCH, "vector length " + std::to_string(p.b.len) +
                                     " does not match matrix cols " + std::to_string(p.w.gcols));
  DevBuf bias;
  LinearEpi e = extra;
  if (pre && pre->bias) {
    e.bias = pre->bias;
  } else {
    bias = expand_diagonal(cube, xf.dirs.swapped(), p.b, s);
    e.bias = bias.as<float>();
  }
  Mat c;
  c.data = y.data;
  c.dtype = y.dtype;
  const ActRows ar{x.batch / cube.extent(kX), x.seq};
  ab_forward(cube, mode, xf, p.w, c, e, s, pre ? &pre->wg : nullptr,
             saved ? &saved->a_full : nullptr, &ar);
  group = 1 - group;
  y = make_act(cube, y.data, y.dtype, x.batch, x.seq, p.w.gcols, group);
  if (saved) {
    saved->x = xf;
    if (own_input) {
      DevBuf& cp = saved->keep(DevBuf(xf.elems() * dtype_size(xf.dtype), s));
      C3D_CUDA(cudaMemcpyAsync(cp.get(), xf.data, xf.elems() * dtype_size(xf.dtype),
                               cudaMemcpyDeviceToDevice, s));
      saved->x.data = cp.get();
    }
    // keep the gathered input only when it is a buffer of our own (p_in > 1)
    if (saved->a_full.buf.get() == nullptr) saved->a_full.ptr = nullptr;
  }
}

void linear_bwd(Cube& cube, int mode, const Act& dy, const LinearSaved& saved, const LinearP& p,
                Act* dx, Mat* dw, const Vec* db, const void* dx_gelu_aux, cudaStream_t s,
                const Operand* wg, const LinearSinks* sinks) {
  // linear3d_bwd (cube3d/nn.hpp:99-112): add_vec_bwd then matmul_ab_bwd.
  if (dy.group != 1 - p.input_group)
    fail(C3D_ERR_GROUP_MISMATCH, "upstream gradient group does not match the layer output group");
  Mat dyf = flatten(cube, dy);
  if (dyf.dirs != saved.x.dirs.swapped())
    fail(C3D_ERR_DIRECTION_CLASH, "dC of C=AB backward must carry the swapped triple");
  // The reduction is collective: every rank joins it whether or not it holds a
  // diagonal slice (non-holders pass a vector with no local data).
  if (sinks && sinks->bias_elsewhere) {
    // summed by the LayerNorm backward that reads dy as its residual (layer_bwd)
  } else if (sinks && sinks->bias_colsum) {
    k_colsum(dyf.data, dyf.dtype, nullptr, kF32, dyf.rows, dyf.cols, sinks->bias_colsum, s);
  } else if (db) {
    DevBuf cs(static_cast<size_t>(dyf.cols) * sizeof(float), s);
    k_colsum(dyf.data, dyf.dtype, nullptr, kF32, dyf.rows, dyf.cols, cs.as<float>(), s);
    Vec out = *db;
    out.len = dyf.gcols;
    reduce_to_diagonal(cube, dyf.dirs, cs.as<float>(), 1, &out, s);
  }
  Mat da, *dap = nullptr;
  if (dx && dx->data) {
    da.data = dx->data;
    da.dtype = dx->dtype;
    dap = &da;
  }
  const ActRows ar{dy.batch / cube.extent(kX), dy.seq};
  ab_backward(cube, mode, dyf, saved.x, p.w, dap, dw, dx_gelu_aux, s, wg, saved.a_full.ptr,
              sinks ? &sinks->dw : nullptr, &ar);
  if (dap) *dx = make_act(cube, dx->data, dx->dtype, dy.batch, dy.seq, saved.x.gcols, p.input_group);
}

// --------------------------------------------------------------- LayerNorm

void layernorm_fwd(Cube& cube, const Act& x, const Vec& gamma, const Vec& beta, double eps,
                   Act& y, LNSaved* saved, cudaStream_t s, const float* gpre,
                   const float* bpre) {
  // layernorm3d_fwd (cube3d/nn.hpp:140-185)
  if (gamma.len != x.hidden || beta.len != x.hidden)
    fail(C3D_ERR_SHAPE_MISMATCH, "layer norm parameter length does not match hidden size");
  const Dirs d = triple_for_group(x.group);
  const int Pout = cube.extent(d.out);
  const float inv_h = 1.f / static_cast<float>(x.hidden);
  DevBuf gown, bown;
  if (!gpre || !bpre) {
    gown = expand_diagonal(cube, d, gamma, s);
    bown = expand_diagonal(cube, d, beta, s);
  }
  const float* gb = gpre ? gpre : gown.as<float>();
  const float* bb = bpre ? bpre : bown.as<float>();
  y = make_act(cube, y.data, y.dtype, x.batch, x.seq, x.hidden, x.group);
  DevBuf xhat(x.elems() * dtype_size(x.dtype), s);
  DevBuf inv_std(static_cast<size_t>(x.rows) * sizeof(float), s);
  if (Pout == 1) {
    k_ln_fwd_fused(x.data, x.dtype, x.rows, x.cols, static_cast<float>(eps), gb, bb, y.data,
                   y.dtype, xhat.get(), x.dtype, inv_std.as<float>(), s);
  } else {
    DevBuf sums(static_cast<size_t>(x.rows) * sizeof(float), s);
    DevBuf sq(static_cast<size_t>(x.rows) * sizeof(float), s);
    DevBuf st(static_cast<size_t>(2 * x.rows) * sizeof(float), s);
    if (k_row_moments(x.data, x.dtype, x.rows, x.cols, st.as<float>(), s)) {
      // one all-gather of per-block (mean, M2) instead of two all-reduces (same elements)
      DevBuf all(static_cast<size_t>(2 * x.rows * Pout) * sizeof(float), s);
      cube.all_gather(d.out, st.get(), all.get(), static_cast<size_t>(2 * x.rows), kF32, s);
      k_combine_moments(all.as<float>(), Pout, x.rows, x.cols, sums.as<float>(), sq.as<float>(), s);
    } else {
      k_row_sum(x.data, x.dtype, x.rows, x.cols, nullptr, inv_h, sums.as<float>(), s);
      cube.all_reduce(d.out, sums.get(), x.rows, kF32, false, s);
      k_row_sum(x.data, x.dtype, x.rows, x.cols, sums.as<float>(), inv_h, sq.as<float>(), s);
      cube.all_reduce(d.out, sq.get(), x.rows, kF32, false, s);
    }
    k_ln_apply(x.data, x.dtype, x.rows, x.cols, sums.as<float>(), sq.as<float>(), inv_h,
               static_cast<float>(eps), gb, bb, y.data, y.dtype, xhat.get(), x.dtype,
               inv_std.as<float>(), s);
  }
  if (saved) {
    saved->dtype = x.dtype;
    saved->group = x.group;
    saved->hidden = x.hidden;
    saved->xhat = saved->keep(std::move(xhat)).get();
    saved->inv_std = saved->keep(std::move(inv_std)).as<float>();
    saved->gamma_block = gpre ? const_cast<float*>(gpre) : saved->keep(std::move(gown)).as<float>();
  }
}

void layernorm_bwd(Cube& cube, const Act& dy, const LNSaved& sv, Act& dx, const Vec* dgamma,
                   const Vec* dbeta, const void* resid, cudaStream_t s, float* sink,
                   float* resid_sink) {
  // layernorm3d_bwd (cube3d/nn.hpp:187-222)
  if (dy.group != sv.group || dy.hidden != sv.hidden)
    fail(C3D_ERR_SHAPE_MISMATCH, "layer norm gradient does not match the saved forward");
  const Dirs d = triple_for_group(dy.group);
  const float inv_h = 1.f / static_cast<float>(dy.hidden);
  if (sink && cube.extent(d.out) == 1 && (resid_sink || !resid)) {
    // one pass: dx, dgamma | dbeta into the sink and, with resid_sink, the residual's
    // column sum (the bias gradient of the linear whose output gradient it is)
    Act out = make_act(cube, dx.data, dx.dtype, dy.batch, dy.seq, dy.hidden, dy.group);
    if (k_ln_bwd_sums(dy.data, dy.dtype, sv.xhat, sv.dtype, sv.gamma_block, sv.inv_std, dy.rows,
                      dy.cols, resid_sink ? resid : nullptr, dx.dtype, out.data, out.dtype, sink,
                      sink + dy.cols, resid_sink, s)) {
      dx = out;
      return;
    }
  }
  if (resid_sink) k_colsum(resid, dy.dtype, nullptr, kF32, dy.rows, dy.cols, resid_sink, s);
  if (sink) {
    k_colsum(dy.data, dy.dtype, sv.xhat, sv.dtype, dy.rows, dy.cols, sink, s, sink + dy.cols);
  } else if (dgamma && dbeta) {  // collective on every rank (see linear_bwd)
    DevBuf cs(static_cast<size_t>(2 * dy.cols) * sizeof(float), s);
    k_colsum(dy.data, dy.dtype, sv.xhat, sv.dtype, dy.rows, dy.cols, cs.as<float>(), s,
             cs.as<float>() + dy.cols);
    Vec outs[2] = {*dgamma, *dbeta};
    outs[0].len = outs[1].len = dy.hidden;
    reduce_to_diagonal(cube, d, cs.as<float>(), 2, outs, s);
  }
  dx = make_act(cube, dx.data, dx.dtype, dy.batch, dy.seq, dy.hidden, dy.group);
  if (cube.extent(d.out) == 1 &&
      k_ln_bwd_fused(dy.data, dy.dtype, sv.xhat, sv.dtype, sv.gamma_block, sv.inv_std, dy.rows,
                     dy.cols, resid, dx.dtype, dx.data, dx.dtype, s))
    return;
  DevBuf rs(static_cast<size_t>(2 * dy.rows) * sizeof(float), s);
  k_ln_bwd_rows(dy.data, dy.dtype, sv.xhat, sv.dtype, sv.gamma_block, dy.rows, dy.cols,
                rs.as<float>(), s);
  cube.all_reduce(d.out, rs.get(), 2 * dy.rows, kF32, false, s);
  k_ln_bwd_dx(dy.data, dy.dtype, sv.xhat, sv.dtype, sv.gamma_block, sv.inv_std, rs.as<float>(),
              inv_h, dy.rows, dy.cols, resid, dx.dtype, dx.data, dx.dtype, s);
}

// --------------------------------------------------------------- attention

namespace {

struct AttnDims {
  int64_t bl, sl, S, H, dh, ld_qkv, hd;  // hd = H*dh
  int seq_axis, Ps;
  float scale;
};

AttnDims attn_dims(const Cube& cube, const Config& cfg, int group_after_qkv) {
  // attn_core_dims (cube3d/attention.hpp:66-76)
  AttnDims a;
  a.seq_axis = axis_of_group(group_after_qkv);
  a.Ps = cube.extent(a.seq_axis);
  const int Ph = cube.extent(axis_of_group(1 - group_after_qkv));
  if (cfg.heads % Ph)
    fail(C3D_ERR_HEADS_INDIVISIBLE, "heads=" + std::to_string(cfg.heads) +
                                        " not divisible by p=" + std::to_string(Ph));
  a.bl = cfg.batch / cube.extent(kX);
  a.sl = cfg.seq / a.Ps;
  a.S = cfg.seq;
  a.H = cfg.heads / Ph;
  a.dh = cfg.hidden / cfg.heads;
  a.hd = a.H * a.dh;
  a.ld_qkv = 3 * a.hd;
  a.scale = static_cast<float>(1.0 / std::sqrt(static_cast<double>(a.dh)));
  return a;
}

// [batch = (bi, hi)][seq position][dh] views of a packed or gathered [p][rows][H*dh] buffer
// (queries / context gradient), K-major (rows of dh) or MN-major (dh contiguous, seq as K).
View packed_view(const void* base, int dtype, const AttnDims& a, bool mn_major) {
  View v = mn_major ? mk_view(base, dtype, 1, a.hd) : mk_view(base, dtype, a.hd, 1);
  if (a.Ps > 1) {
    if (mn_major) v.csplit = a.sl;
    else v.rsplit = a.sl;
    v.s_hi = a.bl * a.sl * a.hd;
  }
  v.b_lo_n = static_cast<int>(a.H);
  v.sb_lo = a.dh;
  v.sb_hi = a.sl * a.hd;
  return v;
}

// q (part 0), k (1) or v (2) columns of the local qkv activation, per (bi, hi) slice.
View qkv_view(const void* qkv, int dtype, const AttnDims& a, int part, bool mn_major) {
  const void* base = offset(qkv, part * a.dh, dtype);
  View v = mn_major ? mk_view(base, dtype, 1, a.ld_qkv) : mk_view(base, dtype, a.ld_qkv, 1);
  v.b_lo_n = static_cast<int>(a.H);
  v.sb_lo = 3 * a.dh;
  v.sb_hi = a.sl * a.ld_qkv;
  return v;
}

// [slice][S][sl] score / probability buffers.
View scores_view(const void* base, int dtype, const AttnDims& a, bool transposed) {
  View v = transposed ? mk_view(base, dtype, 1, a.sl) : mk_view(base, dtype, a.sl, 1);
  v.b_lo_n = static_cast<int>(a.H);
  v.sb_lo = a.S * a.sl;
  v.sb_hi = a.H * a.S * a.sl;
  return v;
}

// [p][rows][H*dh] partial (reduce-scatter layout) or the [rows][H*dh] activation itself.
View packed_out(void* base, int dtype, const AttnDims& a, bool split) {
  View v = mk_view(base, dtype, a.hd, 1);
  if (split) {
    v.rsplit = a.sl;
    v.s_hi = a.bl * a.sl * a.hd;
  }
  v.b_lo_n = static_cast<int>(a.H);
  v.sb_lo = a.dh;
  v.sb_hi = a.sl * a.hd;
  return v;
}

}  // namespace

void attention_fwd(Cube& cube, int mode, const Config& cfg, const Act& x, const LinearP& qkv_p,
                   const LinearP& out_p, int& group, Act& y, AttnSaved* sv, bool own_input,
                   const void* resid, cudaStream_t s, const LinearPre* qkv_pre,
                   const LinearPre* out_pre) {
  // attention_fwd (cube3d/attention.hpp:78-136)
  validate_config(cube, cfg);
  if (x.hidden != cfg.hidden) fail(C3D_ERR_SHAPE_MISMATCH, "attention input hidden size mismatch");
  AttnSaved local;
  AttnSaved& S = sv ? *sv : local;
  const int dt = x.dtype;
  const int g_after = 1 - x.group;
  const ActGeom qg = act_geom(cube.grid(), x.batch, x.seq, 3 * cfg.hidden, g_after);
  DevBuf& qkv_buf = S.keep(DevBuf(static_cast<size_t>(qg.bl * qg.sl * qg.hl) * dtype_size(dt), s));
  Act qkv;
  qkv.data = qkv_buf.get();
  qkv.dtype = dt;
  linear_fwd(cube, mode, x, qkv_p, group, qkv, &S.qkv_lin, own_input, LinearEpi{}, s, qkv_pre);
  const AttnDims a = attn_dims(cube, cfg, qkv.group);
  if (qkv.cols != a.ld_qkv) fail(C3D_ERR_SHAPE_MISMATCH, "qkv projection width mismatch");
  S.qkv = qkv;

  const int64_t rows = a.bl * a.sl;
  const int nslices = static_cast<int>(a.bl * a.H);
  // queries of all local slices: this rank's block, or gathered along the seq axis
  View qv;
  if (a.Ps > 1) {
    DevBuf qloc(static_cast<size_t>(rows * a.hd) * dtype_size(dt), s);
    k_copy_heads(qkv.data, a.ld_qkv, 3 * a.dh, qloc.get(), a.hd, a.dh, rows, a.H, a.dh, dt, s);
    DevBuf& qf = S.keep(DevBuf(static_cast<size_t>(a.Ps * rows * a.hd) * dtype_size(dt), s));
    cube.all_gather(a.seq_axis, qloc.get(), qf.get(), rows * a.hd, dt, s);
    S.q_full = qf.get();
    qv = packed_view(qf.get(), dt, a, false);
  } else {
    qv = qkv_view(qkv.data, dt, a, 0, false);
  }
  const int64_t srows = static_cast<int64_t>(nslices) * a.S;
  const ActGeom cg = act_geom(cube.grid(), x.batch, x.seq, cfg.hidden, qkv.group);
  DevBuf& ctx_buf = S.keep(DevBuf(static_cast<size_t>(cg.bl * cg.sl * cg.hl) * dtype_size(dt), s));
  Act ctx = make_act(cube, ctx_buf.get(), dt, x.batch, x.seq, cfg.hidden, qkv.group);
  // Flash path (flash.cu): scores and probabilities stay on chip; the backward recomputes
  // them from the saved row log-sum-exp. With the key range split along the seq axis,
  // each rank's partial context is normalised over its own keys and the ranks' partials
  // are combined with the reference's two statistic all-reduces (max, then sum;
  // cube3d/attention.hpp:106-126) before the context reduce-scatter.
  bool flashed = false;
  if (mode != C3D_MODE_F32 && dt == kBF16 && flash_supported(a.S, a.sl, a.dh)) {
    const View kv = qkv_view(qkv.data, dt, a, 1, false), vv = qkv_view(qkv.data, dt, a, 2, true);
    DevBuf& lb = S.keep(DevBuf(static_cast<size_t>(srows) * sizeof(float), s));
    if (a.Ps == 1) {
      flashed = flash_fwd(qv, kv, vv, packed_out(ctx.data, dt, a, false), lb.as<float>(), a.S,
                          a.sl, a.dh, a.H, nslices, a.scale, s);
    } else {
      DevBuf partial(static_cast<size_t>(a.Ps * rows * a.hd) * dtype_size(dt), s);
      DevBuf lr(static_cast<size_t>(srows) * sizeof(float), s);
      const View pv = packed_out(partial.get(), dt, a, true);
      flashed = flash_fwd(qv, kv, vv, pv, lr.as<float>(), a.S, a.sl, a.dh, a.H, nslices, a.scale, s);
      if (flashed) {
        C3D_CUDA(cudaMemcpyAsync(lb.get(), lr.get(), static_cast<size_t>(srows) * sizeof(float),
                                 cudaMemcpyDeviceToDevice, s));
        cube.all_reduce(a.seq_axis, lb.get(), srows, kF32, true, s);
        DevBuf w(static_cast<size_t>(srows) * sizeof(float), s);
        k_flash_lse_weights(lr.as<float>(), lb.as<float>(), w.as<float>(), srows, s);
        cube.all_reduce(a.seq_axis, w.get(), srows, kF32, false, s);
        k_flash_combine(pv, lr.as<float>(), lb.as<float>(), w.as<float>(), a.S, a.dh, a.H,
                        nslices, s);
        cube.reduce_scatter(a.seq_axis, partial.get(), ctx.data, rows * a.hd, dt, s);
      }
    }
    if (flashed) {
      S.lse = lb.as<float>();
      cube.add_madds(2ull * static_cast<uint64_t>(nslices) * a.S * a.sl * a.dh);
    }
  }
  if (flashed) {
    LinearEpi oe;
    oe.resid = resid;
    linear_fwd(cube, mode, ctx, out_p, group, y, &S.out_lin, false, oe, s, out_pre);
    return;
  }
  // scores = scale * Q K^T  ([slice][S][sl], fp32)
  DevBuf& pb = S.keep(DevBuf(static_cast<size_t>(srows * a.sl) * dtype_size(dt), s));
  S.probs = pb.get();
  // unfused path (fp32-exact mode, shapes outside the flash kernels): scores GEMM,
  // distributed softmax, P V GEMM
  {
    DevBuf sc(static_cast<size_t>(srows * a.sl) * sizeof(float), s);
    Epilogue e;
    e.out = scores_view(sc.get(), kF32, a, false);
    e.alpha = a.scale;
    gemm_views(cube, mode, a.S, a.sl, a.dh, nslices, qv, qkv_view(qkv.data, dt, a, 1, false), e, s);
    // distributed softmax over the key blocks of the seq axis
    const float* scf = sc.as<float>();
    if (a.Ps == 1) {
      k_softmax_fused(scf, srows, a.sl, pb.get(), dt, s);
    } else {
      DevBuf mx(static_cast<size_t>(srows) * sizeof(float), s);
      DevBuf sm(static_cast<size_t>(srows) * sizeof(float), s);
      k_softmax_rowmax(scf, srows, a.sl, mx.as<float>(), s);
      cube.all_reduce(a.seq_axis, mx.get(), srows, kF32, true, s);
      k_softmax_rowexpsum(scf, srows, a.sl, mx.as<float>(), sm.as<float>(), s);
      cube.all_reduce(a.seq_axis, sm.get(), srows, kF32, false, s);
      k_softmax_norm(scf, srows, a.sl, mx.as<float>(), sm.as<float>(), pb.get(), dt, s);
    }
  }
  // context = P V, reduce-scattered back to this rank's seq block
  {
    Epilogue e;
    DevBuf partial;
    if (a.Ps == 1) {
      e.out = packed_out(ctx.data, dt, a, false);
    } else {
      partial = DevBuf(static_cast<size_t>(a.Ps * rows * a.hd) * dtype_size(dt), s);
      e.out = packed_out(partial.get(), dt, a, true);
    }
    gemm_views(cube, mode, a.S, a.dh, a.sl, nslices, scores_view(pb.get(), dt, a, false),
               qkv_view(qkv.data, dt, a, 2, true), e, s);
    if (a.Ps > 1) cube.reduce_scatter(a.seq_axis, partial.get(), ctx.data, rows * a.hd, dt, s);
  }
  LinearEpi oe;
  oe.resid = resid;
  linear_fwd(cube, mode, ctx, out_p, group, y, &S.out_lin, false, oe, s, out_pre);
}

void attention_bwd(Cube& cube, int mode, const Config& cfg, const Act& dy, const AttnSaved& S,
                   const LinearP& qkv_p, const LinearP& out_p, Act& dx, LayerG& g,
                   cudaStream_t s, const Operand* qkv_wg, const Operand* out_wg,
                   const LinearSinks* qkv_sinks, const LinearSinks* out_sinks) {
  // attention_bwd (cube3d/attention.hpp:138-189)
  const int dt = dy.dtype;
  const ActGeom cg = act_geom(cube.grid(), dy.batch, dy.seq, cfg.hidden, 1 - dy.group);
  DevBuf dctx_buf(static_cast<size_t>(cg.bl * cg.sl * cg.hl) * dtype_size(dt), s);
  Act dctx;
  dctx.data = dctx_buf.get();
  dctx.dtype = dt;
  linear_bwd(cube, mode, dy, S.out_lin, out_p, &dctx, &g.w_out, &g.b_out, nullptr, s, out_wg,
             out_sinks);
  const AttnDims a = attn_dims(cube, cfg, dctx.group);
  const int64_t rows = a.bl * a.sl;
  const int nslices = static_cast<int>(a.bl * a.H);
  const void* qkv = S.qkv.data;

  Gathered dcf = gather(cube, a.seq_axis, dctx.data, rows * a.hd, dt, s);
  DevBuf dqkv_buf(static_cast<size_t>(rows * a.ld_qkv) * dtype_size(dt), s);
  const int64_t srows = static_cast<int64_t>(nslices) * a.S;
  if (S.lse) {
    // flash backward: D = rowsum(dctx * ctx) (all-gathered along the seq axis when the
    // query rows are split), then dQ, dK, dV from recomputed probabilities
    DevBuf rd(static_cast<size_t>(srows) * sizeof(float), s);
    int64_t rd_split = 0;
    if (a.Ps == 1) {
      k_attn_rowdot(dcf.ptr, S.out_lin.x.data, dt, nslices, a.S, a.H, a.dh, a.sl * a.hd,
                    rd.as<float>(), s);
    } else {
      DevBuf rdl(static_cast<size_t>(nslices * a.sl) * sizeof(float), s);
      k_attn_rowdot(dctx.data, S.out_lin.x.data, dt, nslices, a.sl, a.H, a.dh, a.sl * a.hd,
                    rdl.as<float>(), s);
      cube.all_gather(a.seq_axis, rdl.get(), rd.get(), static_cast<size_t>(nslices * a.sl), kF32, s);
      rd_split = a.sl;
    }
    DevBuf ws_buf(flash_bwd_workspace_bytes(a.S, a.dh, nslices), s);
    void* ws = ws_buf.get();
    DevBuf dq_partial;
    View dqv = qkv_view(dqkv_buf.get(), dt, a, 0, false);
    if (a.Ps > 1) {
      dq_partial = DevBuf(static_cast<size_t>(a.Ps * rows * a.hd) * dtype_size(dt), s);
      dqv = packed_out(dq_partial.get(), dt, a, true);
    }
    const View qv = a.Ps > 1 ? packed_view(S.q_full, dt, a, false) : qkv_view(qkv, dt, a, 0, false);
    // b_qkv = colsum(dQKV): summed by the kernel's drain warps from the tiles they store
    // (head dim 64, unsplit query rows), per (batch, warp) partials finished here
    const bool fuse_bq = a.Ps == 1 && a.dh == 64 && qkv_sinks && qkv_sinks->bias_colsum &&
                         !qkv_sinks->bias_elsewhere;
    DevBuf bq;
    if (fuse_bq) bq = DevBuf(static_cast<size_t>(a.bl * 4 * a.H * 3 * a.dh) * sizeof(float), s);
    if (!flash_bwd(qv, qkv_view(qkv, dt, a, 1, false), qkv_view(qkv, dt, a, 2, false),
                   packed_view(dcf.ptr, dt, a, false), S.lse, rd.as<float>(), rd_split, dqv,
                   qkv_view(dqkv_buf.get(), dt, a, 1, false), qkv_view(dqkv_buf.get(), dt, a, 2, false),
                   ws, a.S, a.sl, a.dh, a.H, nslices, a.scale, s, fuse_bq ? bq.as<float>() : nullptr))
      fail(C3D_ERR_INTERNAL, "flash attention backward rejected the forward's layout");
    LinearSinks qs;
    if (qkv_sinks) qs = *qkv_sinks;
    if (fuse_bq) {
      k_colsum_parts(bq.as<float>(), static_cast<int>(a.bl * 4), a.H * 3 * a.dh,
                     qkv_sinks->bias_colsum, s);
      qs.bias_elsewhere = true;
    }
    cube.add_madds(4ull * static_cast<uint64_t>(nslices) * a.S * a.sl * a.dh);
    if (a.Ps > 1) {
      DevBuf dq(static_cast<size_t>(rows * a.hd) * dtype_size(dt), s);
      cube.reduce_scatter(a.seq_axis, dq_partial.get(), dq.get(), rows * a.hd, dt, s);
      k_copy_heads(dq.get(), a.hd, a.dh, dqkv_buf.get(), a.ld_qkv, 3 * a.dh, rows, a.H, a.dh, dt, s);
    }
    Act dqkv = make_act(cube, dqkv_buf.get(), dt, dy.batch, dy.seq, 3 * cfg.hidden, dctx.group);
    linear_bwd(cube, mode, dqkv, S.qkv_lin, qkv_p, &dx, &g.w_qkv, &g.b_qkv, nullptr, s, qkv_wg,
               qkv_sinks ? &qs : nullptr);
    return;
  }
  // unfused path: dP = dctx_full V^T (fp32)
  DevBuf dpf(static_cast<size_t>(srows * a.sl) * sizeof(float), s);
  {
    Epilogue e;
    e.out = scores_view(dpf.get(), kF32, a, false);
    gemm_views(cube, mode, a.S, a.sl, a.dh, nslices, packed_view(dcf.ptr, dt, a, false),
               qkv_view(qkv, dt, a, 2, false), e, s);
  }
  DevBuf dp(static_cast<size_t>(srows * a.sl) * dtype_size(dt), s);  // dS, activation dtype
  // dV = P^T dctx_full
  {
    Epilogue e;
    e.out = qkv_view(dqkv_buf.get(), dt, a, 2, false);
    gemm_views(cube, mode, a.sl, a.dh, a.S, nslices, scores_view(S.probs, dt, a, true),
               packed_view(dcf.ptr, dt, a, true), e, s);
  }
  // dS = P * (dP - rowdot) * scale, rowdot summed along the seq axis
  if (a.Ps == 1) {
    k_softmax_bwd_fused(dpf.as<float>(), S.probs, dt, srows, a.sl, a.scale, dp.get(), dt, s);
  } else {
    DevBuf rd(static_cast<size_t>(srows) * sizeof(float), s);
    k_softmax_bwd_rowdot(dpf.as<float>(), S.probs, dt, srows, a.sl, rd.as<float>(), s);
    cube.all_reduce(a.seq_axis, rd.get(), srows, kF32, false, s);
    k_softmax_bwd_ds(dpf.as<float>(), S.probs, dt, srows, a.sl, rd.as<float>(), a.scale,
                     dp.get(), dt, s);
  }
  // dQ = dS K (reduce-scattered), dK = dS^T Q_full
  {
    Epilogue e;
    DevBuf partial;
    if (a.Ps == 1) {
      e.out = qkv_view(dqkv_buf.get(), dt, a, 0, false);
    } else {
      partial = DevBuf(static_cast<size_t>(a.Ps * rows * a.hd) * dtype_size(dt), s);
      e.out = packed_out(partial.get(), dt, a, true);
    }
    gemm_views(cube, mode, a.S, a.dh, a.sl, nslices, scores_view(dp.get(), dt, a, false),
               qkv_view(qkv, dt, a, 1, true), e, s);
    if (a.Ps > 1) {
      DevBuf dq(static_cast<size_t>(rows * a.hd) * dtype_size(dt), s);
      cube.reduce_scatter(a.seq_axis, partial.get(), dq.get(), rows * a.hd, dt, s);
      k_copy_heads(dq.get(), a.hd, a.dh, dqkv_buf.get(), a.ld_qkv, 3 * a.dh, rows, a.H, a.dh, dt, s);
    }
  }
  {
    Epilogue e;
    e.out = qkv_view(dqkv_buf.get(), dt, a, 1, false);
    const View qv = a.Ps > 1 ? packed_view(S.q_full, dt, a, true) : qkv_view(qkv, dt, a, 0, true);
    gemm_views(cube, mode, a.sl, a.dh, a.S, nslices, scores_view(dp.get(), dt, a, true), qv, e, s);
  }
  Act dqkv = make_act(cube, dqkv_buf.get(), dt, dy.batch, dy.seq, 3 * cfg.hidden, dctx.group);
  linear_bwd(cube, mode, dqkv, S.qkv_lin, qkv_p, &dx, &g.w_qkv, &g.b_qkv, nullptr, s, qkv_wg,
             qkv_sinks);
}

// --------------------------------------------------------------------- MLP

void mlp_fwd(Cube& cube, int mode, const Config& cfg, const Act& x, const LinearP& fc1,
             const LinearP& fc2, int& group, Act& y, MlpSaved* sv, bool own_input,
             const void* resid, cudaStream_t s, const LinearPre* fc1_pre,
             const LinearPre* fc2_pre) {
  // mlp_fwd (cube3d/transformer.hpp:44-53).
  MlpSaved local;
  MlpSaved& S = sv ? *sv : local;
  const int dt = x.dtype;
  const ActGeom hg = act_geom(cube.grid(), x.batch, x.seq, 4 * cfg.hidden, 1 - x.group);
  const size_t hbytes = static_cast<size_t>(hg.bl * hg.sl * hg.hl) * dtype_size(dt);
  Act h1;
  void* h1_data = S.keep(DevBuf(hbytes, s)).get();
  h1.dtype = dt;
  S.pre_act = S.keep(DevBuf(hbytes, s)).get();
  // h1 = gelu(x), and gelu'(x) kept in S.pre_act for the backward (which only multiplies,
  // kActMulAux). Without a reduce-scatter after FC1 the GEMM epilogue produces both from
  // the fp32 accumulator; otherwise FC1 writes x into S.pre_act after the reduction and
  // one elementwise pass produces both.
  if (cube.extent(fc1.w.dirs.out) == 1) {
    h1.data = h1_data;
    LinearEpi e1;
    e1.act = kActGeluSave;
    e1.pre_act = S.pre_act;
    linear_fwd(cube, mode, x, fc1, group, h1, &S.fc1_lin, own_input, e1, s, fc1_pre);
  } else {
    Act pre;
    pre.data = S.pre_act;
    pre.dtype = dt;
    linear_fwd(cube, mode, x, fc1, group, pre, &S.fc1_lin, own_input, LinearEpi{}, s, fc1_pre);
    h1 = pre;
    h1.data = h1_data;
    k_gelu_save(S.pre_act, dt, h1.data, dt, static_cast<int64_t>(pre.elems()), s);
  }
  LinearEpi e2;
  e2.resid = resid;
  linear_fwd(cube, mode, h1, fc2, group, y, &S.fc2_lin, false, e2, s, fc2_pre);
}

void mlp_bwd(Cube& cube, int mode, const Config& cfg, const Act& dy, const MlpSaved& S,
             const LinearP& fc1, const LinearP& fc2, Act& dx, LayerG& g, cudaStream_t s,
             const Operand* fc1_wg, const Operand* fc2_wg, const LinearSinks* fc1_sinks,
             const LinearSinks* fc2_sinks) {
  // mlp_bwd (cube3d/transformer.hpp:55-70); GELU' fused into the FC2 dX epilogue.
  const int dt = dy.dtype;
  const ActGeom hg = act_geom(cube.grid(), dy.batch, dy.seq, 4 * cfg.hidden, 1 - dy.group);
  DevBuf dh(static_cast<size_t>(hg.bl * hg.sl * hg.hl) * dtype_size(dt), s);
  Act dh1;
  dh1.data = dh.get();
  dh1.dtype = dt;
  linear_bwd(cube, mode, dy, S.fc2_lin, fc2, &dh1, &g.w_fc2, &g.b_fc2, S.pre_act, s, fc2_wg,
             fc2_sinks);
  linear_bwd(cube, mode, dh1, S.fc1_lin, fc1, &dx, &g.w_fc1, &g.b_fc1, nullptr, s, fc1_wg,
             fc1_sinks);
}

// ------------------------------------------------------------------- layer

namespace {

// The layer's four weights in one order: qkv, out, fc1, fc2.
const Mat* layer_weights(const LayerP& p, int k) {
  const Mat* w[4] = {&p.qkv.w, &p.out.w, &p.fc1.w, &p.fc2.w};
  return w[k];
}

}  // namespace

void layer_fwd(Cube& cube, int mode, const Config& cfg, const Act& x, const LayerP& p, int& group,
               Act& y, LayerSaved* sv, cudaStream_t s) {
  // transformer_layer_fwd (cube3d/transformer.hpp:115-128):
  //   y1 = x + Attn(LN1(x)); y = y1 + MLP(LN2(y1)); residuals fused into the
  //   OUT and FC2 epilogues.
  // Parameter collectives are hoisted and packed: every vector of the layer is
  // expanded by one broadcast + one all-gather per direction triple, and the four
  // weights by one all-gather along x; the backward reuses both (the reference
  // re-gathers B in every matmul_ab_bwd, cube3d/ops3d.hpp:152).
  validate_config(cube, cfg);
  if (x.group != group) fail(C3D_ERR_GROUP_MISMATCH, "activation group does not match state");
  LayerSaved local;
  LayerSaved& S = sv ? *sv : local;
  const int dt = x.dtype;
  const size_t bytes = x.elems() * dtype_size(dt);
  const int g = x.group;
  bool packed_vecs = true;
  for (const Vec* v : {&p.ln1_g, &p.ln1_b, &p.out.b, &p.ln2_g, &p.ln2_b, &p.fc2.b, &p.qkv.b,
                       &p.fc1.b})
    packed_vecs = packed_vecs && v->dtype == kF32;
  LinearPre pre[4];
  if (packed_vecs) {
    S.keep(expand_diagonal_multi(cube, triple_for_group(g),
                                 {p.ln1_g, p.ln1_b, p.out.b, p.ln2_g, p.ln2_b, p.fc2.b}, &S.vec0,
                                 s));
    S.keep(expand_diagonal_multi(cube, triple_for_group(1 - g), {p.qkv.b, p.fc1.b}, &S.vec1, s));
    pre[0].bias = S.vec1[0];
    pre[1].bias = S.vec0[2];
    pre[2].bias = S.vec1[1];
    pre[3].bias = S.vec0[5];
  }
  if (cube.extent(kX) > 1) {
    bool same = true;
    int64_t T = 0, off[4];
    for (int k = 0; k < 4; ++k) {
      off[k] = T;
      T += static_cast<int64_t>(layer_weights(p, k)->elems());
      same = same && layer_weights(p, k)->dtype == p.qkv.w.dtype;
    }
    if (same) {
      const size_t es = dtype_size(p.qkv.w.dtype);
      DevBuf send(static_cast<size_t>(T) * es, s);
      for (int k = 0; k < 4; ++k)
        C3D_CUDA(cudaMemcpyAsync(static_cast<char*>(send.get()) + off[k] * es,
                                 layer_weights(p, k)->data, layer_weights(p, k)->elems() * es,
                                 cudaMemcpyDeviceToDevice, s));
      DevBuf& recv = S.keep(DevBuf(static_cast<size_t>(T) * cube.extent(kX) * es, s));
      cube.all_gather(kX, send.get(), recv.get(), T, p.qkv.w.dtype, s);
      for (int k = 0; k < 4; ++k) {
        S.wg[k].ptr = static_cast<char*>(recv.get()) + off[k] * es;
        S.wg[k].s_hi = T;
        pre[k].wg = S.wg[k];
      }
    }
  }
  Act n1;
  n1.data = S.keep(DevBuf(bytes, s)).get();
  n1.dtype = dt;
  layernorm_fwd(cube, x, p.ln1_g, p.ln1_b, cfg.eps, n1, &S.ln1, s,
                packed_vecs ? S.vec0[0] : nullptr, packed_vecs ? S.vec0[1] : nullptr);
  DevBuf y1buf(bytes, s);
  Act y1;
  y1.data = y1buf.get();
  y1.dtype = dt;
  attention_fwd(cube, mode, cfg, n1, p.qkv, p.out, group, y1, &S.attn, false, x.data, s, &pre[0],
                &pre[1]);
  Act n2;
  n2.data = S.keep(DevBuf(bytes, s)).get();
  n2.dtype = dt;
  layernorm_fwd(cube, y1, p.ln2_g, p.ln2_b, cfg.eps, n2, &S.ln2, s,
                packed_vecs ? S.vec0[3] : nullptr, packed_vecs ? S.vec0[4] : nullptr);
  mlp_fwd(cube, mode, cfg, n2, p.fc1, p.fc2, group, y, &S.mlp, false, y1.data, s, &pre[2],
          &pre[3]);
}

void layer_bwd(Cube& cube, int mode, const Config& cfg, const Act& dy, const LayerSaved& S,
               const LayerP& p, Act& dx, LayerG& g, cudaStream_t s) {
  // transformer_layer_bwd (cube3d/transformer.hpp:130-148). Vector-gradient column sums
  // and weight-gradient partials are collected into packed buffers and reduced once
  // per direction triple / once along x at the end.
  const int dt = dy.dtype;
  const size_t bytes = dy.elems() * dtype_size(dt);
  const int grp = dy.group;
  const Grid& grid = cube.grid();
  const int64_t c0 = dy.cols;                                            // h / p_out(g)
  const int64_t c1 = 3 * cfg.hidden / grid.dims[axis_of_group(grp)];     // 3h / p_out(1-g)
  const int64_t c1b = 4 * cfg.hidden / grid.dims[axis_of_group(grp)];    // 4h / p_out(1-g)
  // column-sum blocks: group-g triple [ln1 g|b, b_out, ln2 g|b, b_fc2], other [b_qkv, b_fc1]
  DevBuf cs0(static_cast<size_t>(6 * c0) * sizeof(float), s);
  DevBuf cs1(static_cast<size_t>(c1 + c1b) * sizeof(float), s);
  float* f0 = cs0.as<float>();
  float* f1 = cs1.as<float>();
  LinearSinks sk[4];
  sk[0].bias_colsum = f1;
  sk[1].bias_colsum = f0 + 2 * c0;
  sk[2].bias_colsum = f1 + c1;
  sk[3].bias_colsum = f0 + 5 * c0;
  // packed weight-gradient partials, reduce-scattered along x once
  DevBuf dwpack;
  const Mat* gw[4] = {&g.w_qkv, &g.w_out, &g.w_fc1, &g.w_fc2};
  int64_t T = 0, off[4] = {0, 0, 0, 0};
  const bool pack_dw = grid.dims[kX] > 1 && gw[0]->dtype == gw[1]->dtype &&
                       gw[0]->dtype == gw[2]->dtype && gw[0]->dtype == gw[3]->dtype &&
                       gw[0]->data && gw[1]->data && gw[2]->data && gw[3]->data;
  if (pack_dw) {
    for (int k = 0; k < 4; ++k) {
      off[k] = T;
      T += static_cast<int64_t>(layer_weights(p, k)->elems());
    }
    const size_t es = dtype_size(gw[0]->dtype);
    dwpack = DevBuf(static_cast<size_t>(T) * grid.dims[kX] * es, s);
    for (int k = 0; k < 4; ++k) {
      sk[k].dw.base = static_cast<char*>(dwpack.get()) + off[k] * es;
      sk[k].dw.s_hi = T;
      sk[k].dw.dtype = gw[0]->dtype;
    }
  }
  const Operand* wg[4];
  for (int k = 0; k < 4; ++k) wg[k] = S.wg[k].ptr ? &S.wg[k] : nullptr;
  const bool packed_vecs = !S.vec0.empty();
  if (!packed_vecs)
    for (auto& k : sk) k.bias_colsum = nullptr;  // each linear reduces its own bias grad
  // b_fc2 = colsum(dy) and b_out = colsum(dy1): the two LayerNorm backwards read dy / dy1
  // as their residuals and sum them in the same pass (with dgamma, dbeta)
  const bool ln_sums = packed_vecs && dt == kBF16 && cube.extent(triple_for_group(grp).out) == 1;
  if (ln_sums) sk[1].bias_elsewhere = sk[3].bias_elsewhere = true;

  DevBuf dn2b(bytes, s), dy1b(bytes, s), dn1b(bytes, s);
  Act dn2;
  dn2.data = dn2b.get();
  dn2.dtype = dt;
  mlp_bwd(cube, mode, cfg, dy, S.mlp, p.fc1, p.fc2, dn2, g, s, wg[2], wg[3],
          packed_vecs ? &sk[2] : (pack_dw ? &sk[2] : nullptr),
          packed_vecs ? &sk[3] : (pack_dw ? &sk[3] : nullptr));
  Act dy1;
  dy1.data = dy1b.get();
  dy1.dtype = dt;
  layernorm_bwd(cube, dn2, S.ln2, dy1, &g.ln2_g, &g.ln2_b, dy.data, s,
                packed_vecs ? f0 + 3 * c0 : nullptr,
                ln_sums ? f0 + 5 * c0 : nullptr);  // dy1 = dy + LN2'
  Act dn1;
  dn1.data = dn1b.get();
  dn1.dtype = dt;
  attention_bwd(cube, mode, cfg, dy1, S.attn, p.qkv, p.out, dn1, g, s, wg[0], wg[1],
                packed_vecs ? &sk[0] : (pack_dw ? &sk[0] : nullptr),
                packed_vecs ? &sk[1] : (pack_dw ? &sk[1] : nullptr));
  layernorm_bwd(cube, dn1, S.ln1, dx, &g.ln1_g, &g.ln1_b, dy1.data, s, packed_vecs ? f0 : nullptr,
                ln_sums ? f0 + 2 * c0 : nullptr);  // dx = dy1 + LN1'
  if (packed_vecs) {
    Vec v0[6] = {g.ln1_g, g.ln1_b, g.b_out, g.ln2_g, g.ln2_b, g.b_fc2};
    for (auto& v : v0) v.len = cfg.hidden;
    Vec v1[2] = {g.b_qkv, g.b_fc1};
    v1[0].len = 3 * cfg.hidden;
    v1[1].len = 4 * cfg.hidden;
    reduce_to_diagonal_multi(cube, triple_for_group(grp), f0, {v0, v0 + 6}, s);
    reduce_to_diagonal_multi(cube, triple_for_group(1 - grp), f1, {v1, v1 + 2}, s);
  }
  if (pack_dw) {
    const size_t es = dtype_size(gw[0]->dtype);
    DevBuf mine(static_cast<size_t>(T) * es, s);
    cube.reduce_scatter(kX, dwpack.get(), mine.get(), T, gw[0]->dtype, s);
    for (int k = 0; k < 4; ++k)
      C3D_CUDA(cudaMemcpyAsync(gw[k]->data, static_cast<char*>(mine.get()) + off[k] * es,
                               layer_weights(p, k)->elems() * es, cudaMemcpyDeviceToDevice, s));
  }
}

}  // namespace c3d

namespace c3d {

// ------------------------------------------------------------------- loss

void loss_fwd(Cube& cube, int mode, const Act& x, const LinearP& head, const int32_t* targets,
              int& group, float* loss, LossSaved* sv, cudaStream_t s) {
  if (!targets || !loss || !sv) fail(C3D_ERR_CONFIG_INVALID, "loss needs targets, output, saved");
  const int g_out = 1 - x.group;
  const ActGeom lg = act_geom(cube.grid(), x.batch, x.seq, head.w.gcols, g_out);
  DevBuf& lb = sv->keep(DevBuf(static_cast<size_t>(lg.bl * lg.sl * lg.hl) * sizeof(float), s));
  Act logits;
  logits.data = lb.get();
  logits.dtype = kF32;
  linear_fwd(cube, mode, x, head, group, logits, &sv->lin, true, LinearEpi{}, s);
  sv->logits = logits;
  const int64_t rows = logits.rows, cols = logits.cols;
  const int col_axis = lg.out_axis;
  sv->mx = sv->keep(DevBuf(static_cast<size_t>(rows) * sizeof(float), s)).as<float>();
  sv->st = sv->keep(DevBuf(static_cast<size_t>(2 * rows) * sizeof(float), s)).as<float>();
  k_softmax_rowmax(static_cast<const float*>(logits.data), rows, cols, sv->mx, s);
  cube.all_reduce(col_axis, sv->mx, rows, kF32, true, s);
  LossMap map;
  map.w = cube.coord(kX);
  map.a = cube.coord(lg.in_axis);
  map.bl = lg.bl;
  map.sl = lg.sl;
  map.seq = x.seq;
  map.col0 = static_cast<int64_t>(cube.coord(col_axis)) * cols;
  k_loss_stats(static_cast<const float*>(logits.data), rows, cols, sv->mx, targets, map, sv->st, s);
  cube.all_reduce(col_axis, sv->st, 2 * rows, kF32, false, s);
  sv->targets = targets;
  sv->col0 = map.col0;
  sv->tokens = x.batch * x.seq;
  sv->map_w = map.w;
  sv->map_a = map.a;
  k_loss_reduce(sv->mx, sv->st, rows, 1.f / static_cast<float>(sv->tokens), loss, s);
  // every token row sits on one rank of each (x, input-axis) line
  cube.all_reduce(kX, loss, 1, kF32, false, s);
  cube.all_reduce(lg.in_axis, loss, 1, kF32, false, s);
}

void loss_bwd(Cube& cube, int mode, const LossSaved& sv, const LinearP& head, Act* dx, Mat* dw,
              const Vec* db, int grad_dtype, cudaStream_t s) {
  const Act& lg = sv.logits;
  DevBuf gb(lg.elems() * dtype_size(grad_dtype), s);
  Act dl = lg;
  dl.data = gb.get();
  dl.dtype = grad_dtype;
  const ActGeom geo = act_geom(cube.grid(), lg.batch, lg.seq, lg.hidden, lg.group);
  LossMap map;
  map.w = sv.map_w;
  map.a = sv.map_a;
  map.bl = geo.bl;
  map.sl = geo.sl;
  map.seq = lg.seq;
  map.col0 = sv.col0;
  k_loss_grad(static_cast<const float*>(lg.data), lg.rows, lg.cols, sv.mx, sv.st, sv.targets, map,
              1.f / static_cast<float>(sv.tokens), dl.data, grad_dtype, s);
  linear_bwd(cube, mode, dl, sv.lin, head, dx, dw, db, nullptr, s);
}

}  // namespace c3d

namespace c3d {

// ------------------------------------------------------------------ stack

void stack_fwd(Cube& cube, int mode, const Config& cfg, const Act& x,
               const std::vector<LayerP>& ps, int& group, Act& y, StackSaved* sv,
               cudaStream_t s) {
  if (ps.empty()) fail(C3D_ERR_CONFIG_INVALID, "a stack needs at least one layer");
  if (!sv) fail(C3D_ERR_CONFIG_INVALID, "stack forward needs saved state");
  const size_t bytes = x.elems() * dtype_size(x.dtype);
  Act cur = x;
  for (size_t i = 0; i < ps.size(); ++i) {
    Act out;
    if (i + 1 == ps.size()) {
      out = y;
    } else {
      out.data = sv->keep(DevBuf(bytes, s)).get();
      out.dtype = x.dtype;
    }
    sv->layers.push_back(std::make_unique<LayerSaved>());
    layer_fwd(cube, mode, cfg, cur, ps[i], group, out, sv->layers.back().get(), s);
    cur = out;
  }
  y = cur;
}

void stack_bwd(Cube& cube, int mode, const Config& cfg, const Act& dy, const StackSaved& sv,
               const std::vector<LayerP>& ps, Act& dx, std::vector<LayerG>& gs, cudaStream_t s) {
  if (ps.size() != sv.layers.size() || gs.size() != ps.size())
    fail(C3D_ERR_CONFIG_INVALID, "stack backward: layer count differs from the forward");
  const size_t bytes = dy.elems() * dtype_size(dy.dtype);
  DevBuf tmp[2];
  Act cur = dy;
  for (size_t k = ps.size(); k-- > 0;) {
    Act out;
    if (k == 0) {
      out = dx;
    } else {
      DevBuf& b = tmp[k % 2];
      b = DevBuf(bytes, s);
      out.data = b.get();
      out.dtype = dy.dtype;
    }
    layer_bwd(cube, mode, cfg, cur, *sv.layers[k], ps[k], out, gs[k], s);
    cur = out;
  }
  dx = cur;
}

}  // namespace c3d
