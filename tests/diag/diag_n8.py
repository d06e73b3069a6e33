"""N = 8 gradient error: fp32 path vs mixed path vs oracle, several ray counts."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import oracle as O  # noqa: E402
import scenes  # noqa: E402
from gpu_common import make_pair, norm_rel  # noqa: E402
from paper_2304_05735_b200 import romap as R  # noqa: E402

BASE = dict(levels=8, log2_T=12, base_res=16, finest_res=2048.0, res_cap=128, samples_per_ray=32, rays_per_iter=256,
            seed=0)
ctx = R.Context(0)
sc = scenes.sphere_scene(0, depth_per_view=2)
for prec, ls in [(1, 128.0)]:
    for N, rays in [(8, 1000), (32, 256)]:
        h, st = make_pair(R, ctx, sc, dict(BASE, precision=prec, samples_per_ray=N, rays_per_iter=rays, loss_scale=ls))
        stats = ctx.forward_backward([h])[0]
        L, g, dbg = O.loss_and_grads(st, 1)
        hit = dbg["rays"]["hit"]
        rg = ctx.debug_dump(h, R.DUMP_RAY_GRADS).reshape(dbg["rays"]["R"], N, 4)[hit]
        e_ds = norm_rel(rg[..., 0], dbg["dsigma"])
        e_dc = norm_rel(rg[..., 1:], dbg["drgb"])
        e_tab = norm_rel(ctx.get_params(h, R.BLOCK_GRAD_TABLE), g["table"].reshape(-1))
        gm = ctx.get_params(h, R.BLOCK_GRAD_MLP)
        errs, off = [], 0
        for w in g["W"]:
            errs.append(norm_rel(gm[off:off + w.size], w))
            off += w.size
        print(f"ls {ls:6.0f} N {N:3d} rays {rays}: loss {abs(stats['l_total'] / L['l_total'] - 1):.1e} dsig {e_ds:.4f} "
              f"dc {e_dc:.4f} table {e_tab:.4f} W " + " ".join(f"{e:.4f}" for e in errs))
        ctx.destroy_object(h)
