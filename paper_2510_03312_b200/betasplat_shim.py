"""Opt-in GPU backend for the reference package ``betasplat``.

``enable(betasplat)`` rebinds the reference's render / render_with_cache /
render_decomposition / backward at every place the reference bound them
(module attributes and the ``from .x import y`` copies in gradients.py:21,
optim.py:23-26, synthetic.py:32, cli.py:20, __init__.py:6-11), so
``optim.train``, ``optim.evaluate``, ``gradients.loss_value`` /
``fd_check``, ``synthetic.make_synthetic`` and the CLI all run on the
device path.  ``disable()`` restores the originals.

Precision: ``precision`` (default ``"fp32"``: fp64 geometry, fp32 raster with
the certified fp64 fix-up) for renders and training, while
``gradients.fd_check`` (gradients.py:338-380) runs entirely in
``fd_precision`` (default ``"fp64"``, the reference's own arithmetic): its
eps = 1e-4 central differences divide loss differences of ~1e-4 relative by
2 eps, which the fp32 raster's ~1e-6 image error would swamp.
"""

from __future__ import annotations

import contextlib
import importlib

from . import gradients as _g
from . import raster as _r
from .types import GradientError as _GradientError

_state = {"precision": "fp32", "saved": None}


def _current() -> str:
    return _state["precision"]


@contextlib.contextmanager
def use_precision(p: str):
    """Run the enclosed drop-in calls at precision ``p`` ("fp32" | "fp64")."""
    if p not in ("fp32", "fp64"):
        raise ValueError("precision must be 'fp32' or 'fp64'")
    old = _state["precision"]
    _state["precision"] = p
    try:
        yield
    finally:
        _state["precision"] = old


def _modules(pkg):
    names = ("raster", "gradients", "optim", "synthetic", "cli")
    out = {"__init__": pkg}
    for n in names:
        try:
            out[n] = importlib.import_module(f"{pkg.__name__}.{n}")
        except ImportError:  # an optional module (cli) that fails to import stays untouched
            pass
    return out


def enable(pkg=None, precision: str = "fp32", fd_precision: str = "fp64"):
    """Route ``pkg`` (the imported ``betasplat`` package, or its name) to the
    B200 path.  Returns the dict of rebound callables."""
    if isinstance(pkg, str) or pkg is None:
        pkg = importlib.import_module(pkg or "betasplat")
    if _state["saved"] is not None:
        disable()
    mods = _modules(pkg)
    _state["precision"] = precision
    R, G = mods["raster"], mods["gradients"]
    default_settings = R.DEFAULT_SETTINGS
    default_cfg = G.LossConfig()
    orig_fd = G.fd_check

    def render(scene, cam, query, settings=default_settings):
        return _r.render(scene, cam, query, settings, precision=_current())

    def render_with_cache(scene, cam, query, settings=default_settings):
        return _r.render_with_cache(scene, cam, query, settings, precision=_current())

    def render_decomposition(scene, cam, query, channel, settings=default_settings):
        return _r.render_decomposition(scene, cam, query, channel, settings)

    def backward(scene, frames, cfg=default_cfg, settings=default_settings):
        try:
            return _g.backward(scene, frames, cfg, settings, precision=_current())
        except _GradientError as e:  # re-raise as the reference's own class
            raise G.GradientError(str(e)) from e

    def fd_check(*args, **kwargs):
        with use_precision(fd_precision):
            return orig_fd(*args, **kwargs)

    new = {"render": render, "render_with_cache": render_with_cache,
           "render_decomposition": render_decomposition, "backward": backward, "fd_check": fd_check}
    saved = []
    for m in mods.values():
        for name, fn in new.items():
            if hasattr(m, name):
                saved.append((m, name, getattr(m, name)))
                setattr(m, name, fn)
    _state["saved"] = saved
    return new


def disable():
    """Restore every binding ``enable`` replaced."""
    for m, name, fn in reversed(_state["saved"] or []):
        setattr(m, name, fn)
    _state["saved"] = None
    _state["precision"] = "fp32"
