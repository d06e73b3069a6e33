"""Failure detection: a non-finite loss or gradient
in a step is reported as ROMAP_E_NONFINITE by the call that ran it -- from the
device-side flag the loss kernels (fp32 `k_render_loss`, the mixed fused kernel)
and `k_adam` set -- and the context stays usable: after the parameters are reset
the next step trains normally."""
import numpy as np
import pytest

import scenes
from gpu_common import flat_W, make_pair

pytestmark = pytest.mark.gpu

R = pytest.importorskip("paper_2304_05735_b200.romap")

CFG0 = dict(levels=8, log2_T=12, base_res=16, finest_res=2048.0, res_cap=128, samples_per_ray=32, rays_per_iter=256,
            seed=0)


@pytest.mark.parametrize("precision", [0, 1])
def test_nonfinite_loss_and_gradient_are_reported(precision):
    sc = scenes.sphere_scene(0)
    c = R.Context(0)
    h, st = make_pair(R, c, sc, dict(CFG0, precision=precision))
    good = c.get_params(h, R.BLOCK_MLP).copy()
    bad = good.copy()
    bad[-3 * 64:] = np.nan                           # the colour output layer W5: rgb and the loss go NaN
    # (NaN in a hidden layer would be absorbed by the ReLU, max(NaN, 0) = 0, and show
    # only in the gradients)
    c.set_params(h, R.BLOCK_MLP, bad)
    with pytest.raises(R.RomapError) as e:
        c.train_step([h], 1)
    assert e.value.status == R.E_NONFINITE and "loss" in str(e.value)
    # the context is not poisoned: reset the parameters (and the moments Adam just
    # filled with NaN), then training runs
    c.set_params(h, R.BLOCK_MLP, good)
    c.set_params(h, R.BLOCK_M_MLP, np.zeros_like(good))
    c.set_params(h, R.BLOCK_V_MLP, np.zeros_like(good))
    ne = c.get_params(h, R.BLOCK_TABLE).size
    c.set_params(h, R.BLOCK_TABLE, np.asarray(st.params["table"], np.float32).reshape(-1)[:ne])
    c.set_params(h, R.BLOCK_M_TABLE, np.zeros(ne, np.float32))
    c.set_params(h, R.BLOCK_V_TABLE, np.zeros(ne, np.float32))
    out = c.train_step([h], 2)[0]
    assert np.isfinite(out["l_total"])
    # a non-finite gradient handed to the optimiser alone (k_adam's flag)
    g = np.zeros_like(good)
    g[5] = np.inf
    c.set_params(h, R.BLOCK_GRAD_MLP, g)
    with pytest.raises(R.RomapError) as e:
        c.optimizer_step([h])
    assert e.value.status == R.E_NONFINITE and "gradient" in str(e.value)
    c.close()
