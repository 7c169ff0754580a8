"""Device-side relocation and exploration noise (reference optim.py:138-203).

The training step itself (loss + gradient, all-reduce, device Adam) lives in
``sharding``; this module adds the periodic MCMC moves that run every
``relocation_period`` iterations, on the device-resident record buffer so a
multi-million-primitive scene never round-trips through the host:

  * :func:`relocate` -- ``mcmc_relocate`` (optim.py:146-191): dead primitives
    (opacity < 0.005) and growth rows are rewritten as copies of donors drawn
    proportionally to opacity; donor and recipients share the split opacity
    ``clone_opacity(o, k + 1)``; touched rows get fresh Adam moments.
  * :func:`noise_inject` -- optim.py:194-203: covariance-shaped noise on the
    spatial means, gated to near-dead primitives.

Random draws use a ``torch.Generator`` on the device, so they do not replay
numpy's streams; given the same donors (``relocate(..., donors=...)``) and
the same noise ``xi`` the updates equal the reference's, which is what the
tests check.  These are element-wise / gather updates over the record
buffer, run once per relocation period: plain torch device ops.
"""

from __future__ import annotations

import torch

from .types import field_offsets

DEAD_OPACITY = 0.005          # optim.py:33
NOISE_GATE_SHARPNESS = 2000.0  # optim.py:34
GROWTH_FRACTION = 0.05         # optim.py:35


def clone_opacity(o: torch.Tensor, n_clones) -> torch.Tensor:
    """Opacity of each of ``n_clones`` coincident copies that composite to
    ``o``: 1 - (1 - o)^(1/n) (optim.py:138-143)."""
    n = torch.as_tensor(n_clones, dtype=torch.float64, device=o.device)
    if bool((n < 1).any()):
        raise ValueError("n_clones must be >= 1")
    return -torch.expm1(torch.log1p(-o.double()) / n)


def _logit(p: torch.Tensor) -> torch.Tensor:
    return torch.log(p) - torch.log1p(-p)


def relocate(params: torch.Tensor, n_dims: int, target_count: int, generator: torch.Generator | None = None,
             donors: torch.Tensor | None = None):
    """One relocation (optim.py:146-191) on the (n, 14+6C) record buffer.

    Returns ``(params, touched)``: ``params`` is the input tensor updated in
    place, or a new, longer tensor when the scene grew toward
    ``target_count``; ``touched`` (sorted, unique) lists every rewritten row.
    ``donors`` overrides the opacity-proportional draw (one per recipient:
    the dead rows in index order, then the growth rows)."""
    off = field_offsets(n_dims)
    oc = off["opacity_raw"][0]
    dev = params.device
    n = params.shape[0]
    opacity = torch.sigmoid(params[:, oc].double())
    dead = torch.nonzero(opacity < DEAD_OPACITY).flatten()
    alive = torch.nonzero(opacity >= DEAD_OPACITY).flatten()
    empty = torch.zeros(0, dtype=torch.int64, device=dev)
    if alive.numel() == 0:
        return params, empty
    grow = 0
    if n < target_count:
        grow = min(target_count - n, max(1, int(GROWTH_FRACTION * n)))
    total = dead.numel() + grow
    if total == 0:
        return params, empty
    if donors is None:
        probs = opacity[alive] / opacity[alive].sum()
        donors = alive[torch.multinomial(probs, total, replacement=True, generator=generator)]
    donors = donors.to(device=dev, dtype=torch.int64)
    if donors.numel() != total:
        raise ValueError(f"need {total} donors, got {donors.numel()}")
    if grow:
        params = torch.cat([params, torch.zeros((grow, params.shape[1]), dtype=params.dtype, device=dev)])
    recipients = torch.cat([dead, torch.arange(n, n + grow, device=dev)])
    # every recipient copies its donor's original record; donor and recipients
    # then take the donor's split opacity
    params[recipients] = params[donors]
    k = torch.bincount(donors, minlength=n)
    used = torch.nonzero(k).flatten()
    new_o = clone_opacity(opacity[used], k[used] + 1)
    raw = _logit(new_o).to(params.dtype)
    params[used, oc] = raw
    slot = torch.full((n,), -1, dtype=torch.int64, device=dev)
    slot[used] = torch.arange(used.numel(), device=dev)
    params[recipients, oc] = raw[slot[donors]]
    torch.autograd.graph.increment_version(params)
    touched = torch.unique(torch.cat([used, recipients]))
    return params, touched


def noise_inject(params: torch.Tensor, n_dims: int, lambda_eps: float, lr_position: float,
                 generator: torch.Generator | None = None, xi: torch.Tensor | None = None) -> torch.Tensor:
    """mu_x += lambda_eps lr g(o) (L_x xi), g = sigmoid(-2000 (o - 0.005)),
    L_x = (I + [a]_x) diag(exp(s_x_raw)) (optim.py:194-203); in place."""
    n = params.shape[0]
    if lambda_eps == 0.0 or n == 0:
        return params
    off = field_offsets(n_dims)
    p = params.double()
    if xi is None:
        xi = torch.randn((n, 3), dtype=torch.float64, device=params.device, generator=generator)
    xi = xi.to(device=params.device, dtype=torch.float64)
    opacity = torch.sigmoid(p[:, off["opacity_raw"][0]])
    gate = torch.sigmoid(-NOISE_GATE_SHARPNESS * (opacity - DEAD_OPACITY))
    a = p[:, off["rot"][0]:off["rot"][0] + 3]
    s = torch.exp(p[:, off["s_x_raw"][0]:off["s_x_raw"][0] + 3])
    one = torch.ones_like(a[:, 0])
    R = torch.stack([torch.stack([one, -a[:, 2], a[:, 1]], -1),
                     torch.stack([a[:, 2], one, -a[:, 0]], -1),
                     torch.stack([-a[:, 1], a[:, 0], one], -1)], -2)
    step = torch.einsum("nij,nj->ni", R * s[:, None, :], xi)
    mo = off["mu_x"][0]
    params[:, mo:mo + 3] = (p[:, mo:mo + 3] + lambda_eps * lr_position * gate[:, None] * step).to(params.dtype)
    torch.autograd.graph.increment_version(params)
    return params


def relocation_step(ds, adam, target_count: int, lambda_eps: float, lr_position: float,
                    generator: torch.Generator | None = None):
    """The training loop's periodic move (optim.py:240-245): relocate, grow the
    Adam state, reset touched rows, then inject noise.  ``ds`` is the
    engine.DeviceScene, ``adam`` the sharding.DeviceAdam bound to its params."""
    params, touched = relocate(ds.params, ds.n_dims, target_count, generator)
    if params is not ds.params:
        ds.params = params
        adam.rebind(params)
    if touched.numel():
        adam.reset_rows(touched)
    noise_inject(ds.params, ds.n_dims, lambda_eps, lr_position, generator)
    return touched


__all__ = ["DEAD_OPACITY", "GROWTH_FRACTION", "NOISE_GATE_SHARPNESS", "clone_opacity", "noise_inject", "relocate",
           "relocation_step"]
