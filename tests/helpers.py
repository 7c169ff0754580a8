"""Shared comparison helpers and fixture builders for the parity tests."""

from __future__ import annotations

import numpy as np

from oracle import ubs_oracle as O
from paper_2510_03312_b200 import synthetic as S
from paper_2510_03312_b200.types import Camera, Query, RenderSettings, Scene, logit, quantize_f32

FIELDS = O.FIELDS


def grad_close(g, ref, rel=1e-3, floor=1e-3):
    """SURVEY §8(d) gradient metric, per field:
    ||g - ref|| / ||ref|| <= rel  and  |g - ref| <= rel*|ref| + floor*max|ref| elementwise."""
    bad = {}
    for k in FIELDS:
        a = np.asarray(g[k], dtype=np.float64)
        b = np.asarray(ref[k], dtype=np.float64)
        if b.size == 0:
            continue
        nb = np.linalg.norm(b)
        mx = np.abs(b).max()
        if nb == 0.0:
            if np.abs(a).max() > 1e-12:
                bad[k] = ("nonzero", float(np.abs(a).max()))
            continue
        nr = np.linalg.norm(a - b) / nb
        el = np.abs(a - b) <= rel * np.abs(b) + floor * mx
        if nr > rel or not el.all():
            bad[k] = (float(nr), int((~el).sum()))
    return bad


def branch_scene(seed=5, n=400, query=None):
    """SURVEY §8(d) branch-coverage fixture: clamp, PSD floor, screen floor, degenerate rows.

    A 7D scene where blocks of rows exercise each rarely-taken branch.  With
    ``query`` given, the PSD-floor rows are centred on it (delta = 0) so their
    sharp query block does not saturate the gate (which would make the
    reference raise GradientError)."""
    sc = S.random_scene(7, n, seed=seed)
    g = np.random.default_rng(seed + 100)
    k = n // 8
    # alpha clamp: opaque rows with a gate close to 1
    sc.opacity_raw[:k] = 9.0
    sc.s_q_raw[:k] = np.log(50.0)
    sc.l_qx[:k] = 0.0
    # PSD floor: strong cross block + sharp query shape (tests/test_slicing.py:100-111 style)
    sc.l_qx[k:2 * k] = 0.0
    sc.l_qx[k:2 * k, 1:4, :] = 2.0 * np.eye(3)[None]
    sc.s_q_raw[k:2 * k] = np.log(0.1)
    sc.b_q[k:2 * k] = np.log(5.0)
    if query is not None:
        sc.mu_q[k:2 * k] = np.asarray(query.dims)[None, :]
    # thin disks
    sc.s_x_raw[2 * k:3 * k] = np.log(np.array([0.2, 0.2, 1e-7]))
    # degenerate query block
    sc.s_q_raw[3 * k] = 800.0
    return quantize_f32(sc)


def screen_floor_case():
    """A 3D needle that engages the 1e-6 px^2 screen floor."""
    sc = Scene(n_dims=3, mu_x=np.array([[0.0, 0.0, 0.0], [0.1, 0.05, 0.0]]),
               mu_q=np.zeros((2, 0)), rot=np.zeros((2, 3)),
               s_x_raw=np.log(np.array([[1e-3, 1e-7, 1e-3], [0.05, 0.05, 0.05]])),
               l_qx=np.zeros((2, 0, 3)), s_q_raw=np.zeros((2, 0)), b_x=np.zeros(2),
               b_q=np.zeros((2, 0)), opacity_raw=np.array([2.0, 1.0]),
               color=np.array([[0.9, 0.2, 0.1], [0.1, 0.8, 0.3]]), background=(0.1, 0.1, 0.1))
    cam = Camera.look_at((3.0, 0.0, 0.0), (0.0, 0.0, 0.0), (0.0, 0.0, 1.0), 0.9, 1920, 1080)
    return quantize_f32(sc), cam, Query.static()
