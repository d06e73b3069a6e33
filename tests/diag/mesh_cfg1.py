"""Mesh quality of a trained cfg1 object (20 keyframes of 640x480) against its
synthetic ground-truth surface (f2 diagnostics): Acc / Comp /
CR per iteration count and iso level, with and without the carve."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle as O  # noqa: E402
import scenes  # noqa: E402
from paper_2304_05735_b200 import romap as R  # noqa: E402


def gt_surface(ob, n=6000, seed=0, eps=2e-3):
    """points within eps of the object's SDF zero level (object frame -> world)"""
    g = np.random.default_rng(seed)
    a = np.asarray(ob.a, np.float64)
    pts = []
    while sum(len(p) for p in pts) < n:
        p = g.uniform(-a, a, size=(400000, 3))
        d = scenes.shape_sdf(torch.as_tensor(p), ob.shape).numpy()
        pts.append(p[np.abs(d) < eps])
    P = np.concatenate(pts)[:n]
    return O.to_world(P, np.asarray(ob.t, np.float64), float(ob.yaw))


def main():
    c = R.Context(0)
    c.set_deterministic(len(sys.argv) > 1 and sys.argv[1] == "det")
    sc = scenes.object_scene(1, n_views=20)
    ob = sc.objects[0]
    kw = dict(levels=16, log2_T=16, base_res=16, finest_res=512.0, res_cap=0, samples_per_ray=64, rays_per_iter=4096,
              precision=1, seed=1)
    h = c.create_object(ob.t, ob.yaw, ob.a, R.model_config(**kw), ob.instance_id)
    for fr in sc.frames:
        c.add_observation(h, fr.rgb, fr.mask, fr.T_wc, fr.K)
    gt = gt_surface(ob)
    diam = 2 * float(np.linalg.norm(ob.a))
    done = 0
    for iters in (300, 600, 1200, 2400):
        c.train_step([h], iters - done)
        done = iters
        for iso in (10.0, 20.0, 50.0, 100.0):
            for carve in (False, True):
                T = c.extract_mesh(h, 128, iso, carve=carve)
                if T.shape[0] == 0:
                    print(iters, iso, carve, "empty")
                    continue
                m = O.mesh_metrics(O.sample_mesh_points(T, 8000), gt, tau=0.01 * diam)
                print(f"iters {iters} iso {iso:5.1f} carve {int(carve)}: tris {T.shape[0]:7d} acc {m['acc']:.4f} "
                      f"comp {m['comp']:.4f} cr@1%diam {m['cr']:.3f}  (diam {diam:.3f} m)", flush=True)


if __name__ == "__main__":
    main()
