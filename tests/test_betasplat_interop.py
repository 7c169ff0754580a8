"""The drop-in against the reference package's OWN objects (CPU; needs the
build container's /root/reference, skipped elsewhere).

* packing a ``betasplat.Scene`` and converting ``betasplat`` Camera / Query /
  RenderSettings to the C-ABI structs gives the same bytes as this
  package's mirror types (so the device sees identical inputs);
* ``betasplat_shim.enable`` rebinds every copy of render / render_with_cache
  / backward the reference holds, and routes ``gradients.fd_check`` to the
  fp64 path (its eps = 1e-4 central differences need the reference
  arithmetic).  The device calls are replaced by the reference's own CPU
  functions here (no GPU), recording the precision each call asked for.
"""

from __future__ import annotations

import ctypes
import os
import sys

import numpy as np
import pytest

REF = "/root/reference/pkg/src"
pytestmark = pytest.mark.skipif(not os.path.isdir(REF), reason="reference package not present")


@pytest.fixture(scope="module")
def bs():
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/ubs_numba")
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import betasplat
    return betasplat


@pytest.mark.parametrize("nd", [3, 6, 7])
def test_reference_objects_pack_and_convert_identically(bs, nd):
    from betasplat import testing as T
    from paper_2510_03312_b200 import synthetic as S
    from paper_2510_03312_b200.engine import view_struct
    from paper_2510_03312_b200.types import RenderSettings, pack_records
    ref_scene, my_scene = T.random_scene(nd, 40, seed=nd), S.random_scene(nd, 40, seed=nd)
    for dt in (np.float32, np.float64):
        assert np.array_equal(pack_records(ref_scene, dt), pack_records(my_scene, dt))
    ref_cam, my_cam = T.random_camera(48, nd + 1), S.random_camera(48, nd + 1)
    ref_q, my_q = T.random_query(nd, nd + 2), S.random_query(nd, nd + 2)
    for ref_st, my_st in ((bs.RenderSettings(), RenderSettings()),
                          (bs.RenderSettings(gate_symmetric=True, tau_sq=6.5, near_plane=0.5),
                           RenderSettings(gate_symmetric=True, tau_sq=6.5, near_plane=0.5))):
        a = view_struct(40, nd, False, ref_scene.background, ref_cam, ref_q, ref_st)
        b = view_struct(40, nd, False, my_scene.background, my_cam, my_q, my_st)
        assert ctypes.string_at(ctypes.addressof(a), ctypes.sizeof(a)) == \
            ctypes.string_at(ctypes.addressof(b), ctypes.sizeof(b))


def test_enable_routes_every_binding_and_fd_check_to_fp64(bs, monkeypatch):
    from betasplat import gradients as BG, optim as BO, raster as BR, testing as T
    from paper_2510_03312_b200 import betasplat_shim, gradients as G, raster as R
    calls = []
    orig_rwc, orig_render, orig_bwd = BR.render_with_cache, BR.render, BG.backward

    def fake_rwc(scene, cam, query, settings, *, precision=None, device=None):
        calls.append(("render_with_cache", precision))
        return orig_rwc(scene, cam, query, settings)

    def fake_render(scene, cam, query, settings, *, precision=None, device=None):
        calls.append(("render", precision))
        return orig_render(scene, cam, query, settings)

    def fake_bwd(scene, frames, cfg, settings, *, precision=None, device=None):
        calls.append(("backward", precision))
        return orig_bwd(scene, frames, cfg, settings)

    monkeypatch.setattr(R, "render_with_cache", fake_rwc)
    monkeypatch.setattr(R, "render", fake_render)
    monkeypatch.setattr(G, "backward", fake_bwd)
    betasplat_shim.enable(bs, precision="fp32")
    try:
        assert bs.render is BR.render and BO.render is BR.render and BO.backward is BG.backward
        assert BG.render_with_cache is BR.render_with_cache and bs.fd_check is BG.fd_check
        sc = T.random_scene(6, 2, seed=3)
        frames = T.random_frames(sc, 8, seed=4, count=1)
        assert calls and all(p == "fp32" for _, p in calls)  # random_frames rendered its targets
        calls.clear()
        BG.loss_value(sc, frames, BG.LossConfig(), bs.RenderSettings())
        assert calls == [("render_with_cache", "fp32")]
        calls.clear()
        rep = bs.fd_check(sc, frames, BG.LossConfig(), bs.RenderSettings())
        assert rep.total == sc.n_primitives * 32
        kinds = {k for k, _ in calls}
        assert kinds == {"backward", "render_with_cache"}
        assert all(p == "fp64" for _, p in calls)
        calls.clear()
        BO.backward(sc, frames, BG.LossConfig(), bs.RenderSettings())
        # (the stand-in device backward is the reference's, which renders through the rebound
        # render_with_cache: both at the training precision)
        assert calls[0] == ("backward", "fp32") and all(p == "fp32" for _, p in calls)
    finally:
        betasplat_shim.disable()
    assert BR.render is orig_render and BG.backward is orig_bwd and BG.render_with_cache is orig_rwc
