"""ubs_loss_image_grad (L1 + SSIM loss image gradient, gradients.py:110-116 +
metrics.py:74-114) against the oracle's ssim_and_grad, through the C ABI:
tiny images where the reflect padding folds several times, odd sizes and a
moderate frame, fp64 and fp32."""

from __future__ import annotations

import numpy as np
import pytest
import torch

from oracle import ubs_oracle as O
from paper_2510_03312_b200 import _lib

pytestmark = pytest.mark.gpu


def _gpu_loss(a, b, lam, scale, f64):
    lib = _lib.load()
    H, W = a.shape[:2]
    dt = torch.float64 if f64 else torch.float32
    ta = torch.as_tensor(a, dtype=dt, device="cuda").contiguous()
    tb = torch.as_tensor(b, dtype=dt, device="cuda").contiguous()
    g = torch.empty_like(ta)
    parts = torch.zeros(2, dtype=torch.float64, device="cuda")
    scr = torch.empty(int(lib.ubs_loss_scratch_bytes(H, W, int(f64))), dtype=torch.uint8, device="cuda")
    _lib.check(lib.ubs_loss_image_grad(ta.data_ptr(), tb.data_ptr(), H, W, int(f64), lam, scale, g.data_ptr(),
                                       parts.data_ptr(), scr.data_ptr(), torch.cuda.current_stream().cuda_stream),
               "ubs_loss_image_grad")
    return g.double().cpu().numpy(), parts.cpu().numpy()


@pytest.mark.parametrize("f64,tol", [(True, 1e-12), (False, 2e-5)])
@pytest.mark.parametrize("H,W", [(1, 1), (5, 7), (11, 13), (12, 12), (17, 6), (37, 50), (64, 96), (203, 333)])
def test_loss_gradient_matches_oracle(H, W, f64, tol):
    rng = np.random.default_rng(H * 1000 + W)
    a = rng.uniform(0, 1, (H, W, 3))
    b = np.clip(a + rng.normal(0, 0.2, (H, W, 3)), 0, 1)
    if not f64:
        a, b = a.astype(np.float32).astype(np.float64), b.astype(np.float32).astype(np.float64)
    lam, scale = 0.2, 1.7
    s, g_ssim = O.ssim_and_grad(a, b)
    diff = a - b
    n = diff.size
    want = scale * ((1 - lam) * np.sign(diff) / n - lam * g_ssim)
    got, parts = _gpu_loss(a, b, lam, scale, f64)
    ref_max = np.abs(want).max()
    assert np.abs(got - want).max() <= tol * max(ref_max, 1.0 / n)
    assert abs(parts[0] - np.abs(diff).sum()) <= 1e-9 * n
    # fp32: the variances E[a^2] - mu^2 cancel to rounding noise against C2 = 9e-4
    assert abs(parts[1] / n - s) <= (1e-12 if f64 else 5e-5)
