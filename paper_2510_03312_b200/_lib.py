"""ctypes binding of ``libubs_b200.so`` (C ABI declared in ``include/ubs_b200.h``).

No fallback: if the library is missing or a CUDA device is absent the
product path raises.  ``load()`` builds the library in-tree first when the
sources are newer (nvcc cross-compiles without a GPU).
"""

from __future__ import annotations

import ctypes
from ctypes import POINTER, Structure, c_double, c_int32, c_int64, c_size_t, c_uint8, c_uint16, c_uint32, \
    c_uint64, c_ulonglong, c_void_p

from . import build as _build

UBS_OK, UBS_E_ARGS, UBS_E_CUDA, UBS_E_CAPACITY = 0, -1, -2, -3
S_PAIR_OVERFLOW, S_LIST_TRUNC = 1, 2
FULL_LISTS = 0xFFFFFFFF
F_VISIBLE, F_DEGENERATE, F_FLOOR3, F_FLOOR2, F_THIN, F_GATE_SAT = 1, 2, 4, 8, 16, 32
DEBUG_STRIDE = 144
# UBS_DEBUG_* row offsets (include/ubs_b200.h)
DEBUG = dict(vmat=32, cov2_eig=38, cov3_eig=44, beta_q=56, delta=60, m_inv=64, u=80, v=84, sigma_xq=88,
             d_raw=100, d_gate=104, l_x=108, rot=117, s_x=126, s_q=129, color=133, flags=136)
GRAD2D_STRIDE = 12
REC32_BYTES, REC64_BYTES = 64, 80


class UbsError(RuntimeError):
    pass


class UbsCamera(Structure):
    _fields_ = [("fx", c_double), ("fy", c_double), ("cx", c_double), ("cy", c_double),
                ("rot", c_double * 9), ("trans", c_double * 3), ("width", c_int32), ("height", c_int32)]


class UbsSettings(Structure):
    _fields_ = [("tau_sq", c_double), ("alpha_clamp", c_double), ("transmittance_min", c_double),
                ("near_plane", c_double), ("cull_margin", c_double), ("screen_cov_floor", c_double),
                ("psd_floor_scale", c_double), ("gate_symmetric", c_int32), ("tile_size", c_int32)]


class UbsView(Structure):
    _fields_ = [("params", c_void_p), ("n", c_int64), ("n_dims", c_int32), ("param_f64", c_int32),
                ("background", c_double * 3), ("query", c_double * 4), ("cam", UbsCamera),
                ("set", UbsSettings), ("statics", c_void_p)]


class UbsPrimBuffers(Structure):
    _fields_ = [("depth_key", c_void_p), ("rect", c_void_p), ("tile_count", c_void_p), ("flags", c_void_p),
                ("rec32", c_void_p), ("rec64", c_void_p), ("debug", c_void_p), ("n_visible", c_void_p),
                ("n_pairs", c_void_p), ("tile_grid", c_void_p),
                ("depth_range", c_void_p)]


class UbsBinBuffers(Structure):
    _fields_ = [("keys_sorted", c_void_p), ("ids_iota", c_void_p), ("order", c_void_p),
                ("tile_ids", c_void_p), ("tile_ranges", c_void_p), ("pair_capacity", c_int64),
                ("temp", c_void_p), ("temp_bytes", c_size_t), ("chunk_hist", c_void_p),
                ("chunk_hist_capacity", c_int64), ("chunk_count", c_int32), ("entries", c_void_p),
                ("seg_scratch", c_void_p), ("bucket_start", c_void_p), ("bucket_capacity", c_int64),
                ("status", c_void_p), ("list_cap", c_uint32), ("rect_sorted", c_void_p)]


class UbsImageBuffers(Structure):
    _fields_ = [("image", c_void_p), ("alpha_sum", c_void_p), ("t_stop", c_void_p), ("n_contrib", c_void_p),
                ("hit_clamp", c_void_p), ("visits", c_void_p), ("fix_list", c_void_p), ("fix_count", c_void_p),
                ("raster_f64", c_int32), ("raster_scalar", c_int32)]


class UbsGradBuffers(Structure):
    _fields_ = [("g_image", c_void_p), ("grad2d", c_void_p), ("grad_params", c_void_p), ("grad_f64", c_int32),
                ("grad2d_f64", c_int32), ("reg_opacity", c_double), ("reg_scale", c_double),
                ("nonfinite", c_void_p), ("flags", c_void_p), ("active", c_void_p), ("active_count", c_void_p),
                ("bwd_pixels_per_lane", c_int32), ("deterministic", c_int32), ("det_slot_off", c_void_p),
                ("det_partials", c_void_p), ("det_capacity", c_int64), ("det_temp", c_void_p),
                ("det_temp_bytes", c_size_t)]


ABI_VERSION = 7  # UBS_ABI_VERSION in include/ubs_b200.h
MAX_VIEWS = 8  # UBS_MAX_VIEWS

# (name, restype, argtypes) for every symbol include/ubs_b200.h declares
SIGNATURES = [
    ("ubs_abi_version", c_int32, []),
    ("ubs_build_info", ctypes.c_char_p, []),
    ("ubs_statics_bytes", c_size_t, [c_int64, c_int32, c_int32]),
    ("ubs_scene_statics", c_int32, [POINTER(UbsView), c_void_p, c_void_p]),
    ("ubs_preprocess", c_int32, [POINTER(UbsView), POINTER(UbsPrimBuffers), c_int32, c_void_p]),
    ("ubs_preprocess_views", c_int32, [POINTER(UbsView), POINTER(UbsPrimBuffers), c_int32, c_int32, c_void_p]),
    ("ubs_bin_temp_bytes", c_size_t, [c_int64, c_int64, c_int32]),
    ("ubs_bin_depth", c_int32, [POINTER(UbsView), POINTER(UbsPrimBuffers), POINTER(UbsBinBuffers), c_void_p]),
    ("ubs_bin_tiles", c_int32, [POINTER(UbsView), POINTER(UbsPrimBuffers), POINTER(UbsBinBuffers), c_int64,
                                c_void_p]),
    ("ubs_raster_forward", c_int32, [POINTER(UbsView), POINTER(UbsPrimBuffers), POINTER(UbsBinBuffers),
                                     POINTER(UbsImageBuffers), c_void_p]),
    ("ubs_raster_fixup", c_int32, [POINTER(UbsView), POINTER(UbsPrimBuffers), POINTER(UbsBinBuffers),
                                   POINTER(UbsImageBuffers), c_void_p]),
    ("ubs_loss_image_grad", c_int32, [c_void_p, c_void_p, c_int32, c_int32, c_int32, c_double, c_double,
                                      c_void_p, c_void_p, c_void_p, c_void_p]),
    ("ubs_loss_scratch_bytes", c_size_t, [c_int32, c_int32, c_int32]),
    ("ubs_det_temp_bytes", c_size_t, [c_int64]),
    ("ubs_raster_backward", c_int32, [POINTER(UbsView), POINTER(UbsPrimBuffers), POINTER(UbsBinBuffers),
                                      POINTER(UbsImageBuffers), POINTER(UbsGradBuffers), c_void_p]),
    ("ubs_prim_backward", c_int32, [POINTER(UbsView), POINTER(UbsGradBuffers), c_int32, c_void_p]),
    ("ubs_adam_step", c_int32, [c_void_p, c_int32, c_void_p, c_int32, c_void_p, c_void_p, c_int64, c_int32,
                                POINTER(c_double), c_int32, c_int32, c_void_p]),
    ("ubs_adam_step_regularised", c_int32, [c_void_p, c_int32, c_void_p, c_int32, c_void_p, c_void_p, c_int64,
                                            c_int32, POINTER(c_double), c_int32, c_int32, c_double, c_double,
                                            c_void_p, c_void_p]),
    ("ubs_add_regularisers", c_int32, [c_void_p, c_int32, c_void_p, c_int32, c_int64, c_int32, c_double,
                                       c_double, c_void_p]),
    ("ubs_regulariser_value", c_int32, [c_void_p, c_int32, c_int64, c_int32, c_void_p, c_void_p]),
]

_LIB = None


def load(build_if_needed: bool = True):
    """Load (building first if stale) the C-ABI library; raise if unavailable.

    ``UBS_B200_LIB`` names another build of the same sources (e.g. a profiling
    build with walk counters) to load instead of the in-tree library."""
    global _LIB
    if _LIB is not None:
        return _LIB
    import os
    from pathlib import Path
    path = Path(os.environ["UBS_B200_LIB"]) if os.environ.get("UBS_B200_LIB") else _build.OUT
    if path == _build.OUT and build_if_needed and _build.needs_build():
        _build.build()
    if not path.exists():
        raise UbsError(f"CUDA library {path} is missing; run python -m paper_2510_03312_b200.build")
    lib = ctypes.CDLL(str(path))
    for name, res, args in SIGNATURES:
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.ubs_abi_version() != ABI_VERSION:
        raise UbsError("libubs_b200 ABI version mismatch")
    _LIB = lib
    return lib


def check(code: int, what: str):
    if code != UBS_OK:
        names = {UBS_E_ARGS: "bad arguments", UBS_E_CUDA: "CUDA error", UBS_E_CAPACITY: "capacity"}
        raise UbsError(f"{what} failed: {names.get(code, code)}")
