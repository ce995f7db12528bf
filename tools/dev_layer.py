"""Dev probe: one p=1 layer fwd+bwd at a given shape, finiteness + timing."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2105_14450_b200 import cube3d as c3

b, s, n, h = (int(v) for v in (sys.argv[1:5] if len(sys.argv) > 4 else (32, 512, 16, 1024)))
mode = c3.MODE_AUTO
cube = c3.Cube((1, 1, 1), 0, 0)
cfg = c3.TransformerConfig(b, s, n, h)
gp = c3.init_layer_params(cfg, 7)
params = c3.partition_layer_params(cube, gp, 0, c3.BF16)
x = c3.Activation3D(torch.randn(b * s, h, device="cuda").to(torch.bfloat16), b, s, h, 0)
dy = c3.Activation3D(torch.randn(b * s, h, device="cuda").to(torch.bfloat16), b, s, h, 0)
def step():
    gs = c3.GroupState(0)
    y, sv = c3.transformer_layer_fwd(cube, x, params, cfg, gs, mode)
    dx, g = c3.transformer_layer_bwd(cube, dy, sv, params, cfg, mode)
    return y, dx, g
y, dx, g = step(); torch.cuda.synchronize()
print("finite", torch.isfinite(y.local.float()).all().item(), torch.isfinite(dx.local.float()).all().item(),
      torch.isfinite(g.w_qkv.shard.float()).all().item(), "launches", c3.launch_count())
for _ in range(3): step()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10): step()
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
print(f"layer fwd+bwd b={b} s={s} h={h}: {ms:.3f} ms/step, {b/ms*1e3:.1f} seq/s, "
      f"{1.34e12*(b/32)*(h/1024)**2/ (ms*1e-3)/1e12:.1f} TFLOP/s (approx)")
