"""Render closed forms on both device paths (a11; R11, R12, R20): an opaque
constant field puts all weight on the first sample, so the rendered depth is the
centre of the first stratum, t_near + Delta / 2 with Delta = (t_far - t_near) / N
(the inference midpoints), and the opacity is 1; a camera INSIDE the box starts
its segment at t_near = 0 (the slab's clamp).  Against the oracle's render and the
closed form, fp32 path 1e-4, mixed path 1e-3 on depth (the field is exact in
fp16: table ones, first-layer row 14 / LF)."""
import math

import numpy as np
import pytest

import oracle as O
import scenes

pytestmark = pytest.mark.gpu

R = pytest.importorskip("paper_2304_05735_b200.romap")

CFG = dict(levels=8, log2_T=12, base_res=16, finest_res=2048.0, res_cap=128, samples_per_ray=32, rays_per_iter=64,
           seed=1)
RAW0 = 14.0


def _opaque_object(c, precision):
    cfg = R.model_config(**dict(CFG, precision=precision))
    a = np.array([0.4, 0.3, 0.25], np.float32)
    t = np.array([0.1, -0.05, 0.0], np.float32)
    h = c.create_object(t, 0.3, a, cfg, 1)
    ocfg = O.ModelConfig(**{k: v for k, v in CFG.items() if k in O.ModelConfig.__dataclass_fields__})
    P = {"table": np.ones((O.table_entries(ocfg), 2)), "W": [np.zeros(s) for s in O.mlp_shapes(ocfg)]}
    P["W"][0][0, :] = RAW0 / (ocfg.levels * ocfg.feats)
    P["W"][1][0, 0] = 1.0
    c.set_params(h, R.BLOCK_TABLE, P["table"].astype(np.float32))
    c.set_params(h, R.BLOCK_MLP, np.concatenate([w.reshape(-1) for w in P["W"]]).astype(np.float32))
    return h, ocfg, P, t, a


@pytest.mark.parametrize("precision", [0, 1])
@pytest.mark.parametrize("inside", [False, True])
def test_opaque_field_depth_is_the_first_stratum_centre(precision, inside):
    c = R.Context(0)
    h, ocfg, P, t, a = _opaque_object(c, precision)
    yaw, N, W, H = 0.3, 32, 24, 18
    cam = t + (np.array([0.02, 0.01, -0.03], np.float32) if inside else np.array([0.05, 0.02, -2.0], np.float32))
    T = np.concatenate([np.eye(3), cam[:, None]], 1).astype(np.float32)        # looking down world +z
    K = (20.0, 20.0, W / 2, H / 2)
    rgb, dep, opa = c.render(h, T, K, W, H, N)
    orgb, odep, oopa = O.render(ocfg, t, yaw, a, P, T, np.asarray(K, np.float32), W, H, N)
    o, d, _ = O.make_rays(np.tile(np.arange(W), H), np.repeat(np.arange(H), W), np.asarray(K, np.float32), T, t, yaw)
    tn, tf, hit = O.ray_box(o, d, a)
    assert hit.sum() > (W * H if inside else 40) - 1
    if inside:
        assert np.all(tn[hit] == 0)                                            # the slab clamp
    first = tn[hit].astype(np.float64) + 0.5 * (tf[hit] - tn[hit]).astype(np.float64) / N
    tol = 1e-4 if precision == 0 else 1e-3
    assert np.allclose(dep.reshape(-1)[hit], first, rtol=0, atol=tol)
    assert np.allclose(dep, odep, rtol=0, atol=tol)
    assert np.allclose(opa.reshape(-1)[hit], 1.0, atol=1e-6) and np.all(opa.reshape(-1)[~hit] == 0)
    assert math.isclose(float(np.abs(rgb - orgb).max()), 0.0, abs_tol=1e-4 if precision == 0 else 2e-2)
    c.close()
