"""Device Adam (optim.py:115-135) and regulariser kernels against numpy restatements."""

from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _adam_ref(p, g, m, v, lr_cols, clamp_cols, step):
    b1, b2, eps = 0.9, 0.999, 1e-8
    m = b1 * m + (1 - b1) * g
    v = b2 * v + (1 - b2) * g * g
    p = p - lr_cols * (m / (1 - b1 ** step)) / (np.sqrt(v / (1 - b2 ** step)) + eps)
    p[:, clamp_cols] = np.clip(p[:, clamp_cols], -5, 5)
    return p, m, v


@pytest.mark.parametrize("n", [1, 7, 1001])
def test_device_adam_matches_reference(n):
    import torch
    from paper_2510_03312_b200 import sharding
    from paper_2510_03312_b200.engine import field_slices
    rng = np.random.default_rng(n)
    P = 38
    p0 = rng.normal(size=(n, P)).astype(np.float32) * 3
    sl = field_slices(7)
    lr = {"mu_x": 1.6e-4, "opacity_raw": 5e-2, "s_x_raw": 5e-3, "s_q_raw": 5e-3}
    lr_cols = np.full(P, 1e-3)
    for k, (s, _) in sl.items():
        lr_cols[s] = lr.get(k, 1e-3)
    clamp_cols = np.r_[sl["b_x"][0], sl["b_q"][0]]
    params = torch.tensor(p0, device="cuda")
    adam = sharding.DeviceAdam(params, 7)
    p, m, v = p0.astype(np.float64), np.zeros((n, P)), np.zeros((n, P))
    for step in range(1, 4):
        g = rng.normal(size=(n, P)).astype(np.float32)
        adam.step(torch.tensor(g, device="cuda"))
        p, m, v = _adam_ref(p, g.astype(np.float64), m, v, lr_cols, clamp_cols, step)
        got = params.cpu().numpy()
        assert np.abs(got - p).max() <= 1e-5 * max(1.0, np.abs(p).max())
    assert np.all(np.abs(params.cpu().numpy()[:, clamp_cols]) <= 5)
