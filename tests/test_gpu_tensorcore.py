"""tcgen05 operand layouts of the mixed path vs numpy (fp16 inputs, fp32 accumulate)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from paper_2304_05735_b200 import romap as R  # noqa: E402


def test_mma_layout_selftest():
    g = np.random.default_rng(0)
    X = g.normal(size=(128, 32)).astype(np.float16).astype(np.float32)
    W = g.normal(size=(64, 32)).astype(np.float16).astype(np.float32)
    Dl = g.normal(size=(128, 64)).astype(np.float16).astype(np.float32)
    o1, o2, o3 = R.selftest_mma(X, W, Dl)
    assert np.allclose(o1, X @ W.T, rtol=1e-4, atol=1e-3)          # forward layer
    assert np.allclose(o2, Dl @ W, rtol=1e-4, atol=1e-3)           # input gradient
    assert np.allclose(o3, Dl.T @ X, rtol=1e-4, atol=1e-3)         # weight gradient (M=64)
