"""Mesh quality of a trained cfg0 sphere object vs iso level (f2 diagnostics)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle as O  # noqa: E402
import scenes  # noqa: E402
from paper_2304_05735_b200 import romap as R  # noqa: E402

c = R.Context(0)
sc = scenes.sphere_scene(0, n_views=8)
ob = sc.objects[0]
cfg = dict(levels=8, log2_T=12, base_res=16, finest_res=2048.0, res_cap=128, samples_per_ray=32, rays_per_iter=1024,
           precision=1, seed=0)
h = c.create_object(ob.t, ob.yaw, ob.a, R.model_config(**cfg), ob.instance_id)
for fr in sc.frames:
    c.add_observation(h, fr.rgb, fr.mask, fr.T_wc, fr.K)
g = np.random.default_rng(0).normal(size=(4000, 3))
gt = 0.4 * g / np.linalg.norm(g, axis=1, keepdims=True) + np.asarray(ob.t, np.float64)
for iters in (300, 600, 1200):
    c.train_step([h], 300 if iters > 300 else 300)
    for iso in (5.0, 10.0, 20.0, 50.0):
        T = c.extract_mesh(h, 64, iso)
        if T.shape[0] == 0:
            print(iters, iso, "empty")
            continue
        m = O.mesh_metrics(O.sample_mesh_points(T, 8000), gt, tau=0.08)
        print(f"iters {iters} iso {iso}: tris {T.shape[0]} acc {m['acc']:.4f} comp {m['comp']:.4f} cr {m['cr']:.3f}")
