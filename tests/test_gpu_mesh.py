"""f2 mesh extraction (R26) on the GPU: the marching-tetrahedra mesh of
a density lattice equals the oracle's on the same lattice values (same triangle
order, fp32 rounding), and a trained object's mesh reconstructs the synthetic
ground-truth surface (Acc / Comp / CR; SPEC acceptance 5 surrogate:
completion < 5 % of the diameter, completion ratio at 10 % of it > 90 %)."""
import numpy as np
import pytest

import oracle as O
import scenes
from gpu_common import make_pair

pytestmark = pytest.mark.gpu

R = pytest.importorskip("paper_2304_05735_b200.romap")

CFG0M = dict(levels=8, log2_T=12, base_res=16, finest_res=2048.0, res_cap=128, samples_per_ray=32, rays_per_iter=256,
             precision=1, seed=0)


@pytest.mark.parametrize("precision", [0, 1])
def test_mesh_matches_oracle_on_same_lattice(precision):
    c = R.Context(0)
    sc = scenes.sphere_scene(0)
    h, st = make_pair(R, c, sc, dict(CFG0M, precision=precision), avoid_kinks=False)
    res = 10
    P = O.lattice_points(st.box_a, res)
    sig = c.query_density(h, P.reshape(-1, 3)).reshape(res + 1, res + 1, res + 1)
    iso = float(np.median(sig))
    T = c.extract_mesh(h, res, iso)
    To = O.to_world(O.marching_tetrahedra(sig, P, iso), st.box_t, st.box_yaw)
    assert T.shape == To.shape and T.shape[0] > 100
    assert np.abs(T - To).max() < 1e-5
    assert c.extract_mesh(h, res, float(sig.max()) + 1.0).shape[0] == 0          # nothing above the maximum
    for bad in (0, 513):                                                         # the lattice limits
        with pytest.raises(R.RomapError):
            c.extract_mesh(h, bad, iso)
    c.close()


def test_trained_sphere_reconstruction():
    c = R.Context(0)
    sc = scenes.sphere_scene(0, n_views=8)
    ob = sc.objects[0]
    h = c.create_object(ob.t, ob.yaw, ob.a, R.model_config(**dict(CFG0M, rays_per_iter=1024)), ob.instance_id)
    for fr in sc.frames:
        c.add_observation(h, fr.rgb, fr.mask, fr.T_wc, fr.K)
    c.train_step([h], 600)
    T = c.extract_mesh(h, 64, 20.0)
    assert T.shape[0] > 1000
    g = np.random.default_rng(0).normal(size=(4000, 3))
    gt = 0.4 * g / np.linalg.norm(g, axis=1, keepdims=True) + np.asarray(ob.t, np.float64)
    m = O.mesh_metrics(O.sample_mesh_points(T, 8000), gt, tau=0.08)
    assert m["comp"] < 0.04 and m["cr"] > 0.9, m
    c.close()


def test_carved_mesh_matches_oracle_and_keeps_the_observed_surface():
    """ROMAP_MESH_CARVE equals the oracle's carve on the same lattice; on a trained
    sphere it removes no observed surface (completion, completion ratio) and adds no
    triangles.  No accuracy gain is claimed: on these 8 views nearly every lattice
    vertex is seen by some keyframe, so the floaters that remain are in observed
    space."""
    c = R.Context(0)
    sc = scenes.sphere_scene(0, n_views=8)
    h, st = make_pair(R, c, sc, CFG0M, avoid_kinks=False)
    res = 12
    P = O.lattice_points(st.box_a, res)
    sig = c.query_density(h, P.reshape(-1, 3)).reshape(res + 1, res + 1, res + 1)
    seen = O.observed_mask(P.reshape(-1, 3), st.box_t, st.box_yaw, st.kfs).reshape(sig.shape)
    assert 0 < seen.sum() < seen.size                # the views leave box corners unseen
    iso = float(np.median(sig))
    T = c.extract_mesh(h, res, iso, carve=True)
    To = O.to_world(O.marching_tetrahedra(np.where(seen, sig, 0.0), P, iso), st.box_t, st.box_yaw)
    assert T.shape == To.shape and np.abs(T - To).max() < 1e-5
    c.close()
    # trained sphere (deterministic reductions: the same mesh every run)
    c = R.Context(0)
    c.set_deterministic(True)
    ob = sc.objects[0]
    h = c.create_object(ob.t, ob.yaw, ob.a, R.model_config(**dict(CFG0M, rays_per_iter=1024)), ob.instance_id)
    for fr in sc.frames:
        c.add_observation(h, fr.rgb, fr.mask, fr.T_wc, fr.K)
    c.train_step([h], 600)
    g = np.random.default_rng(0).normal(size=(4000, 3))
    gt = 0.4 * g / np.linalg.norm(g, axis=1, keepdims=True) + np.asarray(ob.t, np.float64)
    T0, T1 = c.extract_mesh(h, 64, 20.0), c.extract_mesh(h, 64, 20.0, carve=True)
    m0 = O.mesh_metrics(O.sample_mesh_points(T0, 8000), gt, tau=0.08)
    m1 = O.mesh_metrics(O.sample_mesh_points(T1, 8000), gt, tau=0.08)
    # carving only zeroes sigma in space no keyframe sees (R26): it adds no surface
    # (cells straddling the seen / unseen boundary may re-triangulate, at most a few)
    # and keeps the observed surface; accuracy may move by boundary cells and the
    # 8000-point sampling of the two meshes, nothing more
    assert len(T1) <= len(T0) + len(T0) // 50
    assert m1["comp"] < 0.04 and m1["cr"] > 0.9, (m0, m1)
    assert m1["acc"] <= m0["acc"] + 1e-2, (m0, m1)
    print("uncarved", m0, "carved", m1)
    c.close()
