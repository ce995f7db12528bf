import os, sys
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import numpy as np, torch
from oracle import cube3d_oracle as O
from paper_2105_14450_b200 import cube3d as c3
from helpers import bf16_round, global_params_from, golden, map_params, to_np
from test_layer_gpu import run_layer
cube = c3.Cube((1, 1, 1), 0, 0)
d = golden("layer_small")
_, b, s, n, h, _ = (int(v) for v in d["cfg"])
gp = map_params(global_params_from(d), bf16_round)
y, dx, gr = run_layer(cube, gp, bf16_round(d["x"]), bf16_round(d["dy"]), b, s, n, h, c3.BF16, c3.MODE_AUTO)
print("env", os.environ.get("C3D_NO_FUSED_ATTN"), "y nan", np.isnan(y).sum(), "dx nan", np.isnan(dx).sum(),
      {f: int(np.isnan(gr[f]).sum()) for f in O.FIELDS})
P = O.LayerParams(**{f: np.asarray(getattr(gp, f), dtype=np.float64) for f in O.FIELDS})
xb, dyb = bf16_round(d["x"]), bf16_round(d["dy"])
yo, cache = O.layer_fwd(xb, P, b, s, n)
dxo, Go = O.layer_bwd(dyb, cache, P, b, s, n)
print("errs", O.normwise_err(y, yo), O.normwise_err(dx, dxo),
      {f: round(float(O.normwise_err(gr[f], getattr(Go, f).reshape(gr[f].shape))), 5) for f in O.FIELDS})
# repeat in the same process (stale memory)
for i in range(3):
    y2, dx2, gr2 = run_layer(cube, gp, xb, dyb, b, s, n, h, c3.BF16, c3.MODE_AUTO)
    print("rep", i, np.isnan(dx2).sum(), O.normwise_err(dx2, dxo), O.normwise_err(y2, yo))
