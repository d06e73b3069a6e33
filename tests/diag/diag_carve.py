"""Locate carve-mask disagreements between the GPU mesh and the oracle."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import oracle as O  # noqa: E402
import scenes  # noqa: E402
from gpu_common import make_pair  # noqa: E402
from paper_2304_05735_b200 import romap as R  # noqa: E402

CFG0M = dict(levels=8, log2_T=12, base_res=16, finest_res=2048.0, res_cap=128, samples_per_ray=32, rays_per_iter=256,
             precision=1, seed=0)
c = R.Context(0)
sc = scenes.sphere_scene(0, n_views=8)
h, st = make_pair(R, c, sc, CFG0M, avoid_kinks=False)
res = 12
P = O.lattice_points(st.box_a, res)
sig = c.query_density(h, P.reshape(-1, 3)).reshape(res + 1, res + 1, res + 1)
seen = O.observed_mask(P.reshape(-1, 3), st.box_t, st.box_yaw, st.kfs).reshape(sig.shape)
# GPU mask: iso below every sigma -> each vertex's state shows in the mesh; instead probe
# vertex by vertex with a tiny lattice is impossible, so compare meshes cell by cell
iso = float(np.median(sig))
T = c.extract_mesh(h, res, iso, carve=True)
for flip in np.argwhere(np.ones_like(seen)):
    pass
# brute force: find a mask that reproduces the GPU mesh by flipping single vertices
base = O.marching_tetrahedra(np.where(seen, sig, 0.0), P, iso)
print("gpu", T.shape, "oracle", base.shape, "seen", seen.sum(), "/", seen.size)
Tn = c.extract_mesh(h, res, iso, carve=False)
print("gpu uncarved", Tn.shape, "oracle uncarved", O.marching_tetrahedra(sig, P, iso).shape)
for idx in np.argwhere(~seen):
    print("unseen vertex", idx, P[tuple(idx)], "sigma", sig[tuple(idx)], "> iso" if sig[tuple(idx)] > iso else "")
import sys as _s
_s.exit(0)
cands = []
for idx in np.argwhere(seen | True):
    i, j, k = idx
    m = seen.copy()
    m[i, j, k] = ~m[i, j, k]
    To = O.marching_tetrahedra(np.where(m, sig, 0.0), P, iso)
    if To.shape == T.shape and np.abs(O.to_world(To, st.box_t, st.box_yaw) - T).max() < 1e-5:
        cands.append((i, j, k))
        break
print("single-vertex flips reproducing the GPU mesh:", cands)
for (i, j, k) in cands:
    p = P[i, j, k]
    print("vertex", (i, j, k), p, "oracle seen", seen[i, j, k])
    for n, kf in enumerate(st.kfs):
        Tw = np.asarray(kf.T_wc, np.float64).reshape(3, 4)
        d = p.astype(np.float64) + np.asarray(st.box_t, np.float64) - Tw[:, 3]
        xc = Tw[:, :3].T @ d
        u = kf.K[0] * xc[0] / xc[2] + kf.K[2]
        v = kf.K[1] * xc[1] / xc[2] + kf.K[3]
        print(f"  kf {n}: z {xc[2]:.6f} u {u:.9f} [{kf.x0}, {kf.x0 + kf.w}) v {v:.9f} [{kf.y0}, {kf.y0 + kf.h})")
