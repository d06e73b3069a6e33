"""Diagnose mixed-path gradient error of network 1 vs the oracle: per hidden-layer
count, with the parameters as drawn and rounded to fp16 (so p16 == p32)."""
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

SMALL = dict(levels=8, log2_T=12, base_res=16, finest_res=2048.0, res_cap=128, samples_per_ray=32, rays_per_iter=256,
             precision=1, seed=3, network=1)
ctx = R.Context(0)
sc = scenes.sphere_scene(0, depth_per_view=2)
for net, hl in [(0, 1), (1, 1), (1, 2), (1, 3)]:
    for r16 in (False, True):
        kw = dict(SMALL, hidden_layers=hl, network=net)
        h, st = make_pair(R, ctx, sc, kw, avoid_kinks=False)
        if r16:
            tab = st.params["table"].astype(np.float16).astype(np.float64)
            W = [w.astype(np.float16).astype(np.float64) for w in st.params["W"]]
            st.params = {"table": tab, "W": W}
            ctx.set_params(h, R.BLOCK_TABLE, tab.astype(np.float32))
            ctx.set_params(h, R.BLOCK_MLP, np.concatenate([w.reshape(-1) for w in W]).astype(np.float32))
        stats = ctx.forward_backward([h])[0]
        L, g, dbg = O.loss_and_grads(st, 1)
        e_tab = norm_rel(ctx.get_params(h, R.BLOCK_GRAD_TABLE), g["table"].reshape(-1))
        gm = ctx.get_params(h, R.BLOCK_GRAD_MLP)
        errs, off = [], 0
        for w in g["W"]:
            errs.append(norm_rel(gm[off:off + w.size], w))
            off += w.size
        print(f"net {net} hl {hl} fp16-params {r16}: loss rel {abs(stats['l_total']/L['l_total']-1):.2e} "
              f"table {e_tab:.4f} W " + " ".join(f"{e:.4f}" for e in errs))
        ctx.destroy_object(h)
