"""Determinism check of the mixed path: forward_backward twice on identical
parameters; gradients must agree up to fp32 atomic reordering (~1e-6)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import scenes  # noqa: E402
from gpu_common import make_pair, norm_rel  # noqa: E402
from paper_2304_05735_b200 import romap as R  # noqa: E402

BASE = dict(levels=8, log2_T=12, base_res=16, finest_res=2048.0, res_cap=128, samples_per_ray=32, rays_per_iter=256,
            seed=0, precision=1)
ctx = R.Context(0)
sc = scenes.sphere_scene(0, depth_per_view=2)
for N, rays in [(32, 256), (8, 1000), (64, 4096)]:
    h, st = make_pair(R, ctx, sc, dict(BASE, samples_per_ray=N, rays_per_iter=rays))
    gs = []
    for rep in range(4):
        ctx.set_params(h, R.BLOCK_GRAD_TABLE, np.zeros(ctx.block_bytes(h, R.BLOCK_GRAD_TABLE) // 4, np.float32))
        ctx.set_params(h, R.BLOCK_GRAD_MLP, np.zeros(ctx.block_bytes(h, R.BLOCK_GRAD_MLP) // 4, np.float32))
        ctx.forward_backward([h])
        gs.append((ctx.get_params(h, R.BLOCK_GRAD_TABLE).copy(), ctx.get_params(h, R.BLOCK_GRAD_MLP).copy()))
    for rep in range(1, 4):
        et = norm_rel(gs[rep][0], gs[0][0])
        em = norm_rel(gs[rep][1], gs[0][1])
        nz = int((gs[rep][0] != 0).sum()), int((gs[0][0] != 0).sum())
        print(f"N {N} rays {rays} rep {rep}: table {et:.2e} mlp {em:.2e} nonzero {nz}")
    ctx.destroy_object(h)
