"""Seeded synthetic scenes and cameras for parity tests and benchmarks.

The generators reproduce the reference's fixture streams draw for draw so the
same seed gives the same scene on a box that has no copy of the reference:

* ``random_scene`` / ``random_camera`` / ``random_query``  follow
  testing.py:12-52 (the reference's own parity fixtures);
* ``init_scene`` follows scene.py:181-227;
* ``synth`` is the SURVEY §8(d) benchmark generator built on ``init_scene``
  (configs 2-5 of BASELINE.json), every field rounded through float32.

``tests/test_golden.py`` pins these against checksums of the reference's own
outputs.
"""

from __future__ import annotations

import numpy as np

from .types import Camera, Query, Scene, logit, quantize_f32

BENCH_EYE_ANGLE = 0.3
BENCH_FOV_X = 0.9


def random_scene(n_dims: int, count: int, seed: int, cross_scale: float = 0.3) -> Scene:
    g = np.random.default_rng(seed)
    c = n_dims - 3
    draws = {}
    draws["mu_x"] = g.uniform(-0.8, 0.8, (count, 3))
    draws["mu_q"] = g.uniform(0.0, 1.0, (count, c))
    draws["rot"] = g.uniform(-0.3, 0.3, (count, 3))
    draws["s_x_raw"] = g.uniform(np.log(0.15), np.log(0.45), (count, 3))
    draws["l_qx"] = g.uniform(-cross_scale, cross_scale, (count, c, 3))
    draws["s_q_raw"] = g.uniform(np.log(0.7), np.log(1.5), (count, c))
    draws["b_x"] = g.uniform(-1.0, 1.0, count)
    draws["b_q"] = g.uniform(-1.0, 1.0, (count, c))
    draws["opacity_raw"] = logit(g.uniform(0.2, 0.9, count))
    draws["color"] = g.uniform(0.05, 0.95, (count, 3))
    background = g.uniform(0.0, 0.3, 3)
    return Scene(n_dims=n_dims, background=background, **draws)


def random_camera(size: int, seed: int, radius: float = 3.0) -> Camera:
    g = np.random.default_rng(seed)
    az = g.uniform(0.0, 2.0 * np.pi)
    el = g.uniform(-0.5, 0.7)
    eye = radius * np.array([np.cos(az) * np.cos(el), np.sin(az) * np.cos(el), np.sin(el)])
    return Camera.look_at(eye, (0.0, 0.0, 0.0), (0.0, 0.0, 1.0), 0.9, size, size)


def random_query(n_dims: int, seed: int) -> Query:
    g = np.random.default_rng(seed)
    if n_dims == 3:
        return Query.static()
    d = g.standard_normal(3)
    if n_dims == 6:
        return Query.view(d)
    return Query.view_time(g.uniform(0.0, 1.0), d)


def _f32(x):
    return np.asarray(x, dtype=np.float32).astype(np.float64)


def init_scene(n_dims: int, count: int, seed: int,
               bounds=((-1.0, -1.0, -1.0), (1.0, 1.0, 1.0))) -> Scene:
    """Bell-like starting scene (scene.py:181-227, normalize_dirs=False)."""
    if count < 1:
        raise ValueError("count must be >= 1")
    g = np.random.default_rng(seed)
    c = n_dims - 3
    lo = np.asarray(bounds[0], dtype=np.float64)
    hi = np.asarray(bounds[1], dtype=np.float64)
    mu_x = g.uniform(lo, hi, size=(count, 3))
    mu_q = g.uniform(0.0, 1.0, size=(count, c))
    s0 = float(np.mean(hi - lo)) / count ** (1.0 / 3.0)
    color = g.uniform(0.0, 1.0, size=(count, 3))
    return Scene(n_dims=n_dims, mu_x=_f32(mu_x), mu_q=_f32(mu_q), rot=np.zeros((count, 3)),
                 s_x_raw=np.full((count, 3), _f32(np.log(s0))), l_qx=np.zeros((count, c, 3)),
                 s_q_raw=np.zeros((count, c)), b_x=np.zeros(count), b_q=np.zeros((count, c)),
                 opacity_raw=np.zeros(count), color=_f32(color))


def synth(n_dims: int, count: int, seed: int = 1) -> Scene:
    """SURVEY §8(d) benchmark scene: init_scene plus seeded shape/orientation spread.

    Config 2 (3D Gaussian-limit) keeps b_x = 0.  All fields end float32-exact.
    """
    s = init_scene(n_dims, count, seed)
    g = np.random.default_rng(seed)
    c = n_dims - 3
    s.rot = g.uniform(-0.3, 0.3, (count, 3))
    s.s_x_raw = s.s_x_raw + g.uniform(-0.3, 0.3, (count, 3))
    s.l_qx = g.uniform(-0.3, 0.3, (count, c, 3))
    b_x = g.uniform(-1.0, 1.0, count)
    s.b_x = np.zeros(count) if n_dims == 3 else b_x
    s.b_q = g.uniform(-1.0, 1.0, (count, c))
    s.opacity_raw = g.uniform(-1.0, 2.0, count)
    return quantize_f32(s)


def bench_camera(width: int = 1920, height: int = 1080, k: int = 0, n_orbit: int = 1) -> Camera:
    """Benchmark camera: eye on the r=3 orbit at angle 0.3 + 2*pi*k/n, z=1, looking at 0."""
    ang = BENCH_EYE_ANGLE + 2.0 * np.pi * k / n_orbit
    return Camera.look_at((3.0 * np.cos(ang), 3.0 * np.sin(ang), 1.0), (0.0, 0.0, 0.0),
                          (0.0, 0.0, 1.0), BENCH_FOV_X, width, height)


def bench_query(n_dims: int, cam: Camera, t: float = 0.5) -> Query:
    if n_dims == 3:
        return Query.static()
    if n_dims == 6:
        return Query.view(cam.forward)
    return Query.view_time(t, cam.forward)
