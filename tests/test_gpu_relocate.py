"""Device relocation / exploration noise (paper_2510_03312_b200.optim) against a
numpy restatement of the reference's mcmc_relocate and noise_inject
(optim.py:138-203) driven by the same donors and the same noise."""

from __future__ import annotations

import numpy as np
import pytest
import torch

from paper_2510_03312_b200 import optim, synthetic as S
from paper_2510_03312_b200.types import field_offsets, logit, pack_records, sigmoid

pytestmark = pytest.mark.gpu


def np_relocate(rec, n_dims, target, donors):
    """mcmc_relocate (optim.py:146-191) with the donor draw given."""
    off = field_offsets(n_dims)
    oc = off["opacity_raw"][0]
    rec = rec.copy()
    opacity = sigmoid(rec[:, oc])
    dead = np.nonzero(opacity < optim.DEAD_OPACITY)[0]
    n = rec.shape[0]
    grow = min(target - n, max(1, int(optim.GROWTH_FRACTION * n))) if n < target else 0
    if grow:
        rec = np.concatenate([rec, np.zeros((grow, rec.shape[1]))])
    recipients = np.concatenate([dead, np.arange(n, n + grow)])
    by = {}
    for d, r in zip(donors, recipients):
        by.setdefault(int(d), []).append(int(r))
    touched = []
    for d, rs in by.items():
        new_o = -np.expm1(np.log1p(-opacity[d]) / (len(rs) + 1))
        rec[rs] = rec[d]
        rec[[d] + rs, oc] = logit(new_o)
        touched += [d] + rs
    return rec, np.array(sorted(set(touched)))


@pytest.mark.parametrize("nd,target", [(7, 0), (6, 2000)])
def test_relocate_matches_reference_given_donors(nd, target):
    sc = S.random_scene(nd, 1500, seed=nd)
    off = field_offsets(nd)
    oc = off["opacity_raw"][0]
    rec = pack_records(sc, np.float64)
    rng = np.random.default_rng(3)
    rec[rng.choice(1500, 200, replace=False), oc] = logit(0.001)  # 200 dead rows
    op = sigmoid(rec[:, oc])
    alive = np.nonzero(op >= optim.DEAD_OPACITY)[0]
    n_dead = int((op < optim.DEAD_OPACITY).sum())
    grow = min(target - 1500, max(1, int(0.05 * 1500))) if 1500 < target else 0
    donors = rng.choice(alive, size=n_dead + grow, replace=True, p=op[alive] / op[alive].sum())
    want, touched = np_relocate(rec, nd, target, donors)
    got, t = optim.relocate(torch.from_numpy(rec).cuda(), nd, target, donors=torch.from_numpy(donors))
    assert got.shape[0] == 1500 + grow
    np.testing.assert_allclose(got.cpu().numpy(), want, rtol=1e-13, atol=1e-13)
    assert np.array_equal(t.cpu().numpy(), touched)
    # composited density preserved: 1 - (1 - o')^(k+1) == o for every donor
    o_new = sigmoid(got.cpu().numpy()[:, oc])
    for d in np.unique(donors)[:20]:
        k = int((donors == d).sum())
        assert abs(1 - (1 - o_new[d]) ** (k + 1) - op[d]) < 1e-12


def test_relocate_sampled_draw_and_adam_state():
    from paper_2510_03312_b200 import engine, sharding
    sc = S.random_scene(7, 800, seed=9)
    ds = engine.DeviceScene.from_scene(sc, device="cuda")
    oc = field_offsets(7)["opacity_raw"][0]
    ds.params[:100, oc] = float(logit(0.001))
    adam = sharding.DeviceAdam(ds.params, 7)
    adam.m.fill_(1.0)
    adam.v.fill_(1.0)
    g = torch.Generator(device="cuda").manual_seed(0)
    touched = optim.relocation_step(ds, adam, 900, 1.0, 1.6e-4, g)
    assert ds.n == 840 and adam.m.shape[0] == 840 and adam.params is ds.params
    assert bool((adam.m[touched] == 0).all()) and bool((adam.v[touched] == 0).all())
    assert bool((torch.sigmoid(ds.params[:100, oc].double()) >= optim.DEAD_OPACITY).all())
    assert ds._statics_key is None  # grown params: statics recomputed on the next frame


def test_noise_inject_matches_reference_given_xi():
    sc = S.random_scene(6, 500, seed=4)
    off = field_offsets(6)
    rec = pack_records(sc, np.float64)
    rec[:50, off["opacity_raw"][0]] = logit(0.004)  # near-dead: gate ~ 0.88
    xi = np.random.default_rng(1).standard_normal((500, 3))
    op = sigmoid(rec[:, off["opacity_raw"][0]])
    gate = sigmoid(-optim.NOISE_GATE_SHARPNESS * (op - optim.DEAD_OPACITY))
    a = rec[:, off["rot"][0]:off["rot"][0] + 3]
    R = np.stack([np.stack([np.ones(500), -a[:, 2], a[:, 1]], -1), np.stack([a[:, 2], np.ones(500), -a[:, 0]], -1),
                  np.stack([-a[:, 1], a[:, 0], np.ones(500)], -1)], -2)
    lx = R * np.exp(rec[:, off["s_x_raw"][0]:off["s_x_raw"][0] + 3])[:, None, :]
    want = rec.copy()
    want[:, 0:3] += 1.0 * 1.6e-4 * gate[:, None] * np.einsum("nij,nj->ni", lx, xi)
    got = optim.noise_inject(torch.from_numpy(rec).cuda(), 6, 1.0, 1.6e-4, xi=torch.from_numpy(xi))
    np.testing.assert_allclose(got.cpu().numpy(), want, rtol=1e-14, atol=1e-16)
    assert np.abs(want[:50, :3] - rec[:50, :3]).max() > 0 and np.abs(want[50:, :3] - rec[50:, :3]).max() < 1e-12


def test_clone_opacity():
    o = torch.tensor([0.0, 0.3, 0.9, 0.999], dtype=torch.float64, device="cuda")
    for k in (1, 2, 5):
        c = optim.clone_opacity(o, k)
        assert torch.allclose(1 - (1 - c) ** k, o, atol=1e-15)
    with pytest.raises(ValueError):
        optim.clone_opacity(o, 0)
