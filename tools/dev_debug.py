"""Dev probe: per-block bf16 errors vs the oracle at a tensor-core shape."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from oracle import cube3d_oracle as O
from paper_2105_14450_b200 import cube3d as c3
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from helpers import bf16_round, oracle_params, to_np

b, s, n, h = (int(v) for v in sys.argv[1:5]) if len(sys.argv) > 4 else (4, 128, 4, 256)
mode = int(sys.argv[5]) if len(sys.argv) > 5 else c3.MODE_AUTO
dt = c3.BF16 if mode != c3.MODE_F32 else c3.F32
cube = c3.Cube((1, 1, 1), 0, 0)
cfg = c3.TransformerConfig(b, s, n, h)
P = O.init_layer_params(h, 99)
gp = c3.GlobalLayerParams(**{f: bf16_round(getattr(P, f)) for f in O.FIELDS})
Pq = oracle_params(gp)
r = O.Rng(99)
x = bf16_round(O.random_matrix(b * s, h, r)); dy = bf16_round(O.random_matrix(b * s, h, r))
params = c3.partition_layer_params(cube, gp, 0, dt)
X = c3.activation_to_device(cube, x, b, s, 0, dt)
def rep(name, got, want):
    err = np.abs(got - want) / np.maximum(1, np.abs(want))
    i = np.unravel_index(err.argmax(), err.shape)
    print(f"{name:10s} norm {O.normwise_err(got, want):.3e} maxrel {err.max():.3e} at {i} got {got[i]:.4f} want {want[i]:.4f}")
    bad = np.argwhere(err > 0.05)
    if len(bad):
        print("   bad rows:", np.unique(bad[:, 0])[:20], "bad cols:", np.unique(bad[:, 1])[:40], len(bad))
# attention alone
gs = c3.GroupState(0)
ya, sa = c3.attention_fwd(cube, X, params, cfg, gs, mode)
torch.cuda.synchronize()
yo, cache = O.attention_fwd(x, Pq, b, s, n)
rep("attn_fwd", to_np(ya.local), yo)
# qkv linear alone
lp = c3.LinearParams(params.w_qkv, params.b_qkv, 0)
gs = c3.GroupState(0)
yq, _ = c3.linear3d_fwd(cube, X, lp, gs, mode); torch.cuda.synchronize()
rep("qkv_lin", to_np(yq.local), x @ Pq.w_qkv + Pq.b_qkv)
gs = c3.GroupState(0)
ym, sm = c3.mlp_fwd(cube, X, params, cfg, gs, mode); torch.cuda.synchronize()
pre = x @ Pq.w_fc1 + Pq.b_fc1
rep("mlp_fwd", to_np(ym.local), O.gelu(pre) @ Pq.w_fc2 + Pq.b_fc2)
ln = c3.LayerNormParams(params.ln1_gamma, params.ln1_beta)
yl, _ = c3.layernorm3d_fwd(cube, X, ln); torch.cuda.synchronize()
rep("ln_fwd", to_np(yl.local), O.layernorm_fwd(x, Pq.ln1_gamma, Pq.ln1_beta, 1e-5)[0])
# composition
n1, _ = c3.layernorm3d_fwd(cube, X, ln); gs = c3.GroupState(0)
a1, _ = c3.attention_fwd(cube, n1, params, cfg, gs, mode); torch.cuda.synchronize()
n1o = O.layernorm_fwd(x, Pq.ln1_gamma, Pq.ln1_beta, 1e-5)[0]
rep("attn(ln1)", to_np(a1.local), O.attention_fwd(n1o, Pq, b, s, n)[0])
gs = c3.GroupState(0)
yl, sl = c3.transformer_layer_fwd(cube, X, params, cfg, gs, mode); torch.cuda.synchronize()
ylo, cache = O.layer_fwd(x, Pq, b, s, n)
rep("layer_y", to_np(yl.local), ylo)
y1o = O.attention_fwd(n1o, Pq, b, s, n)[0] + x
rep("y1-ish", to_np(a1.local) + x, y1o)
y_before = to_np(yl.local).copy()
DY = c3.activation_to_device(cube, dy, b, s, 0, dt)
dxl, gl = c3.transformer_layer_bwd(cube, DY, sl, params, cfg, mode, grad_dtype=c3.F32)
torch.cuda.synchronize()
print("y changed by bwd:", not np.array_equal(y_before, to_np(yl.local)))
rep("layer_y2", to_np(yl.local), ylo)
dxo, Go = O.layer_bwd(dy, cache, Pq, b, s, n)
rep("layer_dx", to_np(dxl.local), dxo)
for f in O.FIELDS:
    g_ = to_np(getattr(gl, f).shape if False else getattr(gl, f).shard)
    w_ = getattr(Go, f).reshape(g_.shape)
    if g_.ndim == 1: g_, w_ = g_[None], w_[None]
    rep(f, g_, w_)
