"""B200-native (sm_100a) Universal Beta Splatting render path.

Drop-in for the reference ``betasplat`` render/rasterize/backward entry points
(/root/reference/pkg/src/betasplat: raster.py:269-322, gradients.py:101-127),
with the same N-D Beta primitive layout.  Host code is Python; all per-frame
work runs in hand-written CUDA kernels behind the C ABI in
``include/ubs_b200.h`` (``libubs_b200.so``).
"""

from .types import (DEFAULT_SETTINGS, PARAM_FIELDS, Camera, DegeneratePrimitiveError, GradientError,
                    LossConfig, Query, RenderSettings, Scene, SceneGrads, logit, pack_records, quantize_f32,
                    record_width, sigmoid)

__version__ = "0.1.0"

__all__ = ["DEFAULT_SETTINGS", "PARAM_FIELDS", "Camera", "DegeneratePrimitiveError", "GradientError",
           "LossConfig", "Query", "RenderSettings", "Scene", "SceneGrads", "logit", "pack_records",
           "quantize_f32", "record_width", "sigmoid", "render", "render_with_cache", "backward",
           "FrameCache", "render_decomposition", "load_scene", "save_scene", "load_scene_device",
           "SceneFormatError", "clone_opacity", "relocate", "noise_inject"]


def __getattr__(name):
    # the GPU entry points import torch lazily so the types stay importable anywhere
    if name in ("render", "render_with_cache", "FrameCache", "render_decomposition"):
        from . import raster
        return getattr(raster, name)
    if name in ("load_scene", "save_scene", "load_scene_device", "SceneFormatError"):
        from . import sceneio
        return getattr(sceneio, name)
    if name in ("clone_opacity", "relocate", "noise_inject"):
        from . import optim
        return getattr(optim, name)
    if name == "backward":
        from .gradients import backward
        return backward
    raise AttributeError(name)
