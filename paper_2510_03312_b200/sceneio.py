"""UBS1 scene files (reference sceneio.py:1-85), loaded straight into HBM.

File layout (little-endian): magic ``UBS1``, uint32 n_dims (3, 6 or 7),
uint32 primitive count, 3 x f32 background, then per primitive 14 + 6C f32 in
PARAM_FIELDS order.  That record is the device layout of
:class:`engine.DeviceScene`, so :func:`load_scene_device` reads the payload
once into pinned host memory and copies it to the GPU as is -- no per-field
unpacking on the host.  :func:`load_scene` / :func:`save_scene` mirror the
reference's host API and errors (``SceneFormatError``: bad magic, truncated
header, unsupported n_dims, payload size) for the oracle and the tests.
"""

from __future__ import annotations

import struct
from pathlib import Path

import numpy as np

from .types import Scene, pack_records, record_width

SCENE_MAGIC = b"UBS1"
HEADER_BYTES = 24


class SceneFormatError(ValueError):
    pass


def _parse_header(head: bytes, payload_bytes: int):
    """(n_dims, count, background) of a UBS1 file; checks as sceneio.py:62-76."""
    if head[:4] != SCENE_MAGIC:
        raise SceneFormatError("bad magic")
    if len(head) < HEADER_BYTES:
        raise SceneFormatError("truncated header")
    n_dims, count = struct.unpack("<II", head[4:12])
    if n_dims not in (3, 6, 7):
        raise SceneFormatError(f"unsupported n_dims {n_dims}")
    background = np.frombuffer(head[12:24], dtype="<f4").astype(np.float64)
    expected = count * record_width(n_dims) * 4
    if payload_bytes != expected:
        raise SceneFormatError(f"expected {expected} payload bytes, found {payload_bytes}")
    return n_dims, count, background


def save_scene(scene: Scene, path) -> None:
    """Write ``scene`` as UBS1 (sceneio.py:49-58): f32 records."""
    n = scene.n_primitives
    record = pack_records(scene, np.float32).astype("<f4", copy=False)
    with open(path, "wb") as fh:
        fh.write(SCENE_MAGIC)
        fh.write(struct.pack("<II", scene.n_dims, n))
        fh.write(np.asarray(scene.background, dtype="<f4").tobytes())
        fh.write(record.tobytes())


def load_scene(path) -> Scene:
    """Host Scene with float64 fields (sceneio.py:61-85)."""
    blob = Path(path).read_bytes()
    n_dims, count, background = _parse_header(blob[:HEADER_BYTES], len(blob) - HEADER_BYTES)
    record = np.frombuffer(blob[HEADER_BYTES:], dtype="<f4").astype(np.float64).reshape(count,
                                                                                       record_width(n_dims))
    return Scene.from_records(n_dims, record, background)


def load_scene_device(path, device="cuda", dtype=None):
    """UBS1 file -> :class:`engine.DeviceScene` resident on ``device``.

    The payload is read into a pinned buffer and copied to HBM in one
    transfer; ``dtype=torch.float64`` widens on the device afterwards."""
    import torch

    from . import engine
    dev = engine._require_cuda(device)
    path = Path(path)
    size = path.stat().st_size
    with open(path, "rb") as fh:
        head = fh.read(HEADER_BYTES)
        n_dims, count, background = _parse_header(head, size - len(head))
        width = record_width(n_dims)
        host = torch.empty((count, width), dtype=torch.float32, pin_memory=True)
        if count:
            view = memoryview(host.numpy()).cast("B")
            got = fh.readinto(view)
            if got != count * width * 4:
                raise SceneFormatError(f"expected {count * width * 4} payload bytes, found {got}")
    params = host.to(dev, non_blocking=True)
    torch.cuda.current_stream(dev).synchronize()  # the pinned buffer is released on return
    if dtype is not None and dtype != torch.float32:
        params = params.to(dtype)
    return engine.DeviceScene(params, n_dims, background)


__all__ = ["SCENE_MAGIC", "SceneFormatError", "load_scene", "load_scene_device", "save_scene"]
