"""One cfg3 layer fwd+bwd step (p=1, bf16) for ncu launch lists: `warm` eager steps, then
one marked step. Run plain first, then under ncu with -s <warm*launches>."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_2105_14450_b200 import cube3d as c3
warm = int(sys.argv[1]) if len(sys.argv) > 1 else 2
cube = c3.Cube((1, 1, 1), 0, 0)
wl = bench.WORKLOADS["cfg3"]
cfg = c3.TransformerConfig(wl["b"], wl["s"], wl["n"], wl["h"])
params, x, dy = bench.make_layer_inputs(cube, wl, c3.BF16)
grads = c3.empty_like_params(cube, params, c3.F32)
def step():
    y, sv = c3.transformer_layer_fwd(cube, x, params, cfg, c3.GroupState(0))
    c3.transformer_layer_bwd(cube, dy, sv, params, cfg, grads=grads)
n0 = c3.launch_count()
step(); torch.cuda.synchronize()
per = c3.launch_count() - n0
for _ in range(warm - 1): step()
torch.cuda.synchronize()
step(); torch.cuda.synchronize()
print("launches_per_step", per)
