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


@pytest.mark.parametrize("pdt,gdt", [("float32", "float32"), ("float64", "float32"), ("float64", "float64")])
@pytest.mark.parametrize("regularise", [True, False])
def test_adam_step_regularised_matches_separate_passes(pdt, gdt, regularise):
    """ubs_adam_step_regularised == ubs_adam_step, then zero + ubs_add_regularisers
    + ubs_regulariser_value on the updated parameters (bit for bit, sums to 1e-12)."""
    import torch
    from paper_2510_03312_b200 import sharding, synthetic as S
    from paper_2510_03312_b200.types import LossConfig, pack_records
    sc = S.synth(7, 3001, seed=4)
    p0 = torch.tensor(pack_records(sc, np.float64), device="cuda").to(getattr(torch, pdt))
    rng = np.random.default_rng(5)
    g0 = torch.tensor(rng.normal(size=p0.shape), device="cuda").to(getattr(torch, gdt))
    cfg = LossConfig(lambda_o=0.01, lambda_sigma=0.002, loss_scale=3.0)
    pa, ga = p0.clone(), g0.clone()
    a = sharding.DeviceAdam(pa, 7)
    a.step(ga)
    ga.zero_()
    be = type("B", (), {})()
    be.ds = type("D", (), {"params": pa, "n": pa.shape[0], "n_dims": 7})()
    if regularise:
        sharding.GpuViewBackend.add_regularisers(be, ga, cfg)
    ref_value = sharding.GpuViewBackend.regulariser_value(be, cfg)
    pb, gb = p0.clone(), g0.clone()
    b = sharding.DeviceAdam(pb, 7)
    nxt = b.step(gb, next_cfg=cfg, regularise=regularise)
    torch.cuda.synchronize()
    assert torch.equal(pa, pb) and torch.equal(a.m, b.m) and torch.equal(a.v, b.v)
    assert torch.equal(ga, gb)
    got_value = cfg.lambda_o * nxt.sums[0] + cfg.lambda_sigma * nxt.sums[1]
    assert abs(float(got_value) - float(ref_value)) <= 1e-12 * abs(float(ref_value))
    assert nxt.valid_for(pb, cfg) and not nxt.valid_for(pb, LossConfig())
    pb.add_(0.0)  # any in-place change of the parameters invalidates the prepared buffer
    assert not nxt.valid_for(pb, cfg)
