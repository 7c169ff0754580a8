"""UBS1 scene files (reference sceneio.py:1-85): host round trip and format
errors on CPU; the device loader lands the file's records in HBM unchanged."""

from __future__ import annotations

import struct

import numpy as np
import pytest

from paper_2510_03312_b200 import sceneio, synthetic as S
from paper_2510_03312_b200.types import pack_records, quantize_f32


@pytest.mark.parametrize("nd", [3, 6, 7])
def test_round_trip_is_the_packed_record(tmp_path, nd):
    sc = quantize_f32(S.random_scene(nd, 50, seed=nd))
    p = tmp_path / "s.ubs"
    sceneio.save_scene(sc, p)
    blob = p.read_bytes()
    assert blob[:4] == b"UBS1" and struct.unpack("<II", blob[4:12]) == (nd, 50)
    assert np.array_equal(np.frombuffer(blob[24:], "<f4").reshape(50, -1), pack_records(sc))
    back = sceneio.load_scene(p)
    assert np.array_equal(pack_records(back, np.float64), pack_records(sc, np.float64))
    assert np.array_equal(back.background, sc.background.astype(np.float32).astype(np.float64))


def test_empty_scene(tmp_path):
    sc = S.random_scene(7, 0, seed=1)
    p = tmp_path / "e.ubs"
    sceneio.save_scene(sc, p)
    assert sceneio.load_scene(p).n_primitives == 0


@pytest.mark.parametrize("mutate,msg", [
    (lambda b: b"UBS2" + b[4:], "bad magic"),
    (lambda b: b[:20], "truncated header"),
    (lambda b: b[:4] + struct.pack("<I", 5) + b[8:], "unsupported n_dims 5"),
    (lambda b: b[:-4], "payload bytes"),
])
def test_format_errors(tmp_path, mutate, msg):
    sc = S.random_scene(6, 4, seed=2)
    p = tmp_path / "s.ubs"
    sceneio.save_scene(sc, p)
    p.write_bytes(mutate(p.read_bytes()))
    with pytest.raises(sceneio.SceneFormatError, match=msg):
        sceneio.load_scene(p)


def test_device_loader_needs_cuda(tmp_path):
    import torch
    if torch.cuda.is_available():
        pytest.skip("CUDA present")
    sc = S.random_scene(3, 3, seed=1)
    p = tmp_path / "s.ubs"
    sceneio.save_scene(sc, p)
    with pytest.raises(Exception, match="CUDA"):
        sceneio.load_scene_device(p)


@pytest.mark.gpu
@pytest.mark.parametrize("nd", [3, 7])
def test_device_loader_lands_records_and_renders(tmp_path, nd):
    import torch
    from paper_2510_03312_b200 import engine
    sc = quantize_f32(S.random_scene(nd, 400, seed=nd + 1))
    p = tmp_path / "s.ubs"
    sceneio.save_scene(sc, p)
    ds = sceneio.load_scene_device(p, "cuda")
    assert ds.params.is_cuda and ds.params.dtype == torch.float32
    assert torch.equal(ds.params.cpu(), torch.from_numpy(pack_records(sc)))
    ref = engine.DeviceScene.from_scene(sc, device="cuda")
    cam, q = S.random_camera(64, 5), S.random_query(nd, 6)
    ws = engine.Workspace("cuda", "fp32")
    a = engine.render_frame(ws, ds, cam, q).image.clone()
    b = engine.render_frame(ws, ref, cam, q).image.clone()
    assert torch.equal(a, b)
    with pytest.raises(sceneio.SceneFormatError):
        p.write_bytes(p.read_bytes()[:-4])
        sceneio.load_scene_device(p, "cuda")


@pytest.mark.parametrize("nd", [3, 7])
def test_loaded_scenes_take_the_single_copy_upload(tmp_path, nd):
    # load_scene (here and in betasplat) leaves a 1-D float64 owner under the
    # (n, width) record view: the drop-in's packed path must still find it
    from paper_2510_03312_b200.raster import _packed_records
    sc = quantize_f32(S.random_scene(nd, 40, seed=nd + 3))
    p = tmp_path / "s.ubs"
    sceneio.save_scene(sc, p)
    back = sceneio.load_scene(p)
    rec = _packed_records(back, 40)
    assert rec is not None and rec.shape == (40, 14 + 6 * (nd - 3))
    assert np.array_equal(rec, pack_records(back, np.float64))
    assert _packed_records(back.copy(), 40) is None  # separate arrays: per-field path
