"""The model options of the ABI other tests leave at their defaults, on both device
paths against the oracle: softplus density (R3), literal Eq. 6 for
object rays (obj_bg = 1, R14), non-default loss weights (Eq. 11 lambda_1,
lambda_2), and for the mixed path a different loss scale (a power of two,
divided out exactly).  Tolerances as the default configuration:
fp32 losses 1e-5, gradients 1e-4 norm-relative per block; mixed losses 1e-2,
gradients 2e-2 per weight block and for the whole table (the per-level bound is
held by the default-configuration tests)."""
import numpy as np
import pytest

import oracle as O
import scenes
from gpu_common import make_pair, norm_rel

pytestmark = pytest.mark.gpu

R = pytest.importorskip("paper_2304_05735_b200.romap")

CFG0 = dict(levels=8, log2_T=12, base_res=16, finest_res=2048.0, res_cap=128, samples_per_ray=32, rays_per_iter=256,
            seed=3)
OPTIONS = {
    "softplus": dict(density_act=1),
    "obj_bg=1": dict(obj_bg=1),
    "lambdas": dict(lambda_depth=0.1, lambda_density=0.05),
}


@pytest.fixture(scope="module")
def scene0():
    return scenes.sphere_scene(0, depth_per_view=2)


def _run(scene, kw):
    c = R.Context(0)
    h, st = make_pair(R, c, scene, kw)
    stats = c.forward_backward([h])[0]
    L, g, _ = O.loss_and_grads(st, 1)
    gt = c.get_params(h, R.BLOCK_GRAD_TABLE).reshape(-1, 2)
    gm = c.get_params(h, R.BLOCK_GRAD_MLP)
    c.close()
    return stats, L, g, gt, gm


def _blocks(gm, W):
    off = 0
    for w in W:
        yield gm[off:off + w.size], w
        off += w.size


@pytest.mark.parametrize("name", list(OPTIONS))
def test_fp32_options(scene0, name):
    stats, L, g, gt, gm = _run(scene0, dict(CFG0, precision=0, **OPTIONS[name]))
    for k in ("l_rgb", "l_rr", "l_depth", "l_density", "l_total"):
        assert abs(stats[k] - L[k]) <= 1e-5 * max(abs(L[k]), 1e-6), (name, k, stats[k], L[k])
    assert norm_rel(gt, g["table"]) < 1e-4, name
    for a, b in _blocks(gm, g["W"]):
        assert norm_rel(a, b) < 1e-4, name


@pytest.mark.parametrize("name", list(OPTIONS) + ["loss_scale=1024"])
def test_mixed_options(scene0, name):
    opt = dict(loss_scale=1024.0) if name == "loss_scale=1024" else OPTIONS[name]
    stats, L, g, gt, gm = _run(scene0, dict(CFG0, precision=1, **opt))
    for k in ("l_rgb", "l_rr", "l_density", "l_total"):
        assert abs(stats[k] - L[k]) <= 1e-2 * max(abs(L[k]), 1e-4), (name, k, stats[k], L[k])
    assert norm_rel(gt, g["table"]) < 2e-2, name
    for a, b in _blocks(gm, g["W"]):
        assert norm_rel(a, b) < 2e-2, name


DEGENERATE = {
    "N=1": dict(samples_per_ray=1),
    "N=2": dict(samples_per_ray=2),
    "one level": dict(levels=1, finest_res=16.0),
    "T=2^4 (every level hashed into 16 entries)": dict(log2_T=4),
    "b=1 (all levels at res 16)": dict(levels=4, finest_res=16.0),
}


@pytest.mark.parametrize("name", list(DEGENERATE))
def test_fp32_degenerate_configurations(scene0, name):
    """the method's degenerate cases (one sample per ray: delta = the whole segment;
    one level; a table smaller than every level; a growth factor of 1) keep the fp32
    parity bar, including bit-exact hash indices"""
    kw = dict(CFG0, precision=0, **DEGENERATE[name])
    c = R.Context(0)
    h, st = make_pair(R, c, scene0, kw)
    stats = c.forward_backward([h])[0]
    L, g, dbg = O.loss_and_grads(st, 1)
    for k in ("l_rgb", "l_rr", "l_depth", "l_density", "l_total"):
        assert abs(stats[k] - L[k]) <= 1e-5 * max(abs(L[k]), 1e-6), (name, k, stats[k], L[k])
    rs = dbg["rays"]
    N = kw["samples_per_ray"]
    hi = c.debug_dump(h, R.DUMP_HASH_IDX).reshape(rs["R"], N, kw["levels"], 8)
    assert np.array_equal(hi[rs["hit"]].reshape(-1, kw["levels"], 8), dbg["idx"])
    gt = c.get_params(h, R.BLOCK_GRAD_TABLE).reshape(-1, 2)
    assert norm_rel(gt, g["table"]) < 1e-4, name
    for a, b in _blocks(c.get_params(h, R.BLOCK_GRAD_MLP), g["W"]):
        assert norm_rel(a, b) < 1e-4, name
    c.close()
