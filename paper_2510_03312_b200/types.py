"""Host-side data contract: the N-D Beta primitive layout, camera, query and knobs.

These mirror the reference package's public types field for field so that a
caller holding reference objects can pass them straight to this package
(duck-typed: only attribute names are read), and so that the GPU box, which
has no copy of the reference, can build the same objects itself.

Reference anchors (paths under ``/root/reference/pkg/src/betasplat``):

* ``PARAM_FIELDS`` / ``Scene``            scene.py:17-28, 101-178
* ``Camera``                              camera.py:15-74
* ``Query``                               slicing.py:36-77
* ``RenderSettings``                      config.py:9-38
* ``LossConfig`` / ``SceneGrads`` / ``GradientError``   gradients.py:25-70

The on-device layout is the ``UBS1`` record (sceneio.py:3-11): one row of
``14 + 6C`` floats per primitive, fields in ``PARAM_FIELDS`` order.
"""

from __future__ import annotations

from dataclasses import asdict, dataclass, field

import numpy as np

# name -> per-primitive shape as a function of C (number of query dims)
PARAM_FIELDS = (
    ("mu_x", lambda c: (3,)),
    ("mu_q", lambda c: (c,)),
    ("rot", lambda c: (3,)),
    ("s_x_raw", lambda c: (3,)),
    ("l_qx", lambda c: (c, 3)),
    ("s_q_raw", lambda c: (c,)),
    ("b_x", lambda c: ()),
    ("b_q", lambda c: (c,)),
    ("opacity_raw", lambda c: ()),
    ("color", lambda c: (3,)),
)


def record_width(n_dims: int) -> int:
    """Floats per primitive in the packed record: 14 + 6C."""
    return 14 + 6 * (n_dims - 3)


def field_offsets(n_dims: int) -> dict:
    """name -> (offset, size, shape) inside one packed record."""
    c = n_dims - 3
    out, off = {}, 0
    for name, shape_fn in PARAM_FIELDS:
        shape = shape_fn(c)
        size = int(np.prod(shape)) if shape else 1
        out[name] = (off, size, shape)
        off += size
    return out


class GradientError(RuntimeError):
    """A backward pass produced a non-finite gradient (gradients.py:25)."""


class DegeneratePrimitiveError(ValueError):
    """Query-block covariance is singular even after jitter (slicing.py:32)."""


def sigmoid(x):
    """Overflow-safe logistic, same branch split as scene.py:31-38."""
    x = np.asarray(x, dtype=np.float64)
    out = np.empty_like(x)
    pos = x >= 0
    out[pos] = 1.0 / (1.0 + np.exp(-x[pos]))
    e = np.exp(x[~pos])
    out[~pos] = e / (1.0 + e)
    return out


def logit(p):
    p = np.asarray(p, dtype=np.float64)
    return np.log(p) - np.log1p(-p)


@dataclass
class Scene:
    """Structure-of-arrays scene, float64 on the host (scene.py:101-178)."""

    n_dims: int
    mu_x: np.ndarray
    mu_q: np.ndarray
    rot: np.ndarray
    s_x_raw: np.ndarray
    l_qx: np.ndarray
    s_q_raw: np.ndarray
    b_x: np.ndarray
    b_q: np.ndarray
    opacity_raw: np.ndarray
    color: np.ndarray
    background: np.ndarray = field(default_factory=lambda: np.zeros(3))

    def __post_init__(self):
        if self.n_dims not in (3, 6, 7):
            raise ValueError(f"n_dims must be 3, 6, or 7, got {self.n_dims}")
        c = self.n_dims - 3
        n = np.asarray(self.mu_x).reshape(-1, 3).shape[0]
        for name, shape_fn in PARAM_FIELDS:
            arr = np.asarray(getattr(self, name), dtype=np.float64)
            setattr(self, name, arr.reshape((n,) + shape_fn(c)))
        self.background = np.asarray(self.background, dtype=np.float64).reshape(3)

    @property
    def n_query_dims(self) -> int:
        return self.n_dims - 3

    @property
    def n_primitives(self) -> int:
        return self.mu_x.shape[0]

    @property
    def opacity(self) -> np.ndarray:
        return sigmoid(self.opacity_raw)

    def copy(self) -> "Scene":
        return Scene(self.n_dims, *(getattr(self, k).copy() for k, _ in PARAM_FIELDS),
                     background=self.background.copy())

    def take(self, idx) -> "Scene":
        return Scene(self.n_dims, *(getattr(self, k)[idx].copy() for k, _ in PARAM_FIELDS),
                     background=self.background.copy())

    @classmethod
    def empty(cls, n_dims: int, background=(0.0, 0.0, 0.0)) -> "Scene":
        c = n_dims - 3
        kw = {k: np.zeros((0,) + fn(c)) for k, fn in PARAM_FIELDS}
        return cls(n_dims=n_dims, background=np.asarray(background, dtype=np.float64), **kw)

    @classmethod
    def from_records(cls, n_dims: int, records: np.ndarray, background=(0.0, 0.0, 0.0)):
        """Inverse of :func:`pack_records` (the UBS1 body layout)."""
        records = np.asarray(records, dtype=np.float64)
        n = records.shape[0]
        kw = {}
        for name, (off, size, shape) in field_offsets(n_dims).items():
            kw[name] = records[:, off:off + size].reshape((n,) + shape)
        return cls(n_dims=n_dims, background=np.asarray(background, dtype=np.float64), **kw)


def pack_records(scene, dtype=np.float32) -> np.ndarray:
    """(n, 14+6C) packed records in PARAM_FIELDS order (sceneio.py:49-58 layout)."""
    n = scene.mu_x.shape[0]
    width = record_width(scene.n_dims)
    if n == 0:
        return np.zeros((0, width), dtype=dtype)
    out = np.empty((n, width), dtype=dtype)
    off = 0
    for k, _ in PARAM_FIELDS:  # one cast-and-copy pass per field (values as float64 -> dtype)
        part = np.asarray(getattr(scene, k), dtype=np.float64).reshape(n, -1)
        out[:, off:off + part.shape[1]] = part
        off += part.shape[1]
    return out


def quantize_f32(scene) -> Scene:
    """Copy of ``scene`` with every parameter rounded through float32."""
    rec = pack_records(scene, np.float32).astype(np.float64)
    return Scene.from_records(scene.n_dims, rec, scene.background)


@dataclass
class Camera:
    """Pinhole camera, +z forward, x right, y down (camera.py:3-51)."""

    fx: float
    fy: float
    cx: float
    cy: float
    width: int
    height: int
    world_to_cam: np.ndarray

    def __post_init__(self):
        self.world_to_cam = np.asarray(self.world_to_cam, dtype=np.float64).reshape(4, 4)
        if self.fx <= 0 or self.fy <= 0:
            raise ValueError("focal lengths must be positive")
        if self.width < 1 or self.height < 1:
            raise ValueError("image size must be at least 1x1")
        r = self.world_to_cam[:3, :3]
        if np.abs(r @ r.T - np.eye(3)).max() > 1e-6:
            raise ValueError("world_to_cam rotation block is not orthonormal")

    @property
    def rotation(self) -> np.ndarray:
        return self.world_to_cam[:3, :3]

    @property
    def translation(self) -> np.ndarray:
        return self.world_to_cam[:3, 3]

    @property
    def position(self) -> np.ndarray:
        return -self.rotation.T @ self.translation

    @property
    def forward(self) -> np.ndarray:
        # third row of R is the camera +z axis expressed in world coordinates
        return self.rotation[2].copy()

    @classmethod
    def look_at(cls, eye, target, up, fov_x: float, width: int, height: int) -> "Camera":
        """Camera at ``eye`` looking at ``target`` (camera.py:53-74 semantics)."""
        eye = np.asarray(eye, dtype=np.float64)
        fwd = np.asarray(target, dtype=np.float64) - eye
        norm = np.linalg.norm(fwd)
        if norm == 0.0:
            raise ValueError("eye and target coincide")
        fwd = fwd / norm
        up = np.asarray(up, dtype=np.float64)
        helper = up if abs(np.dot(fwd, up / np.linalg.norm(up))) < 0.999 else np.array([1.0, 0.0, 0.0])
        right = np.cross(fwd, helper)
        right = right / np.linalg.norm(right)
        down = np.cross(fwd, right)
        w2c = np.eye(4)
        w2c[:3, :3] = np.stack([right, down, fwd])
        w2c[:3, 3] = -w2c[:3, :3] @ eye
        f = focal_from_fov(fov_x, width)
        return cls(fx=f, fy=f, cx=width / 2.0, cy=height / 2.0, width=width, height=height,
                   world_to_cam=w2c)


def focal_from_fov(fov: float, pixels: int) -> float:
    return pixels / (2.0 * np.tan(fov / 2.0))


@dataclass
class Query:
    """Per-frame non-spatial coordinates: [], [dir], or [t, dir] (slicing.py:36-77)."""

    dims: np.ndarray

    def __post_init__(self):
        self.dims = np.asarray(self.dims, dtype=np.float64).reshape(-1)
        c = self.dims.shape[0]
        if c not in (0, 3, 4):
            raise ValueError(f"query must have 0, 3, or 4 dims, got {c}")
        if c >= 3 and abs(np.linalg.norm(self.dims[c - 3:]) - 1.0) > 1e-6:
            raise ValueError("view direction must be unit length")
        if c == 4 and not 0.0 <= self.dims[0] <= 1.0:
            raise ValueError("time must lie in [0, 1]")

    @classmethod
    def static(cls) -> "Query":
        return cls(np.zeros(0))

    @classmethod
    def view(cls, direction) -> "Query":
        d = np.asarray(direction, dtype=np.float64).reshape(3)
        n = np.linalg.norm(d)
        if n == 0.0:
            raise ValueError("zero view direction")
        return cls(d / n)

    @classmethod
    def view_time(cls, t: float, direction) -> "Query":
        d = np.asarray(direction, dtype=np.float64).reshape(3)
        n = np.linalg.norm(d)
        if n == 0.0:
            raise ValueError("zero view direction")
        return cls(np.concatenate([[float(t)], d / n]))


@dataclass(frozen=True)
class RenderSettings:
    """Render knobs; defaults are the reference production values (config.py:9-38).

    ``tile_size`` is fixed at 16 on the device (one 256-thread CTA per tile);
    other values are rejected.  ``threads`` is accepted for signature
    compatibility and ignored (the device parallelises over tiles itself).
    """

    tile_size: int = 16
    tau_sq: float = 8.0
    alpha_clamp: float = 0.999
    transmittance_min: float = 1e-4
    near_plane: float = 0.01
    cull_margin: float = 3.0
    screen_cov_floor: float = 1e-6
    psd_floor_scale: float = 1e-8
    gate_symmetric: bool = False
    threads: int = 1

    def to_dict(self) -> dict:
        return asdict(self)


DEFAULT_SETTINGS = RenderSettings()


@dataclass
class SliceCache:
    """Per-primitive conditioning state (reference slicing.py:153-182), filled
    from the device preprocess's debug dump (FrameCache.slices)."""

    valid: np.ndarray          # (n,) False where the query block was singular
    mean3: np.ndarray          # (n, 3)
    cov3: np.ndarray           # (n, 3, 3) floored
    beta_x: np.ndarray         # (n,)
    gated_opacity: np.ndarray  # (n,)
    color: np.ndarray          # (n, 3)
    opacity: np.ndarray        # (n,)
    gate: np.ndarray           # (n,)
    beta_q: np.ndarray         # (n, C)
    delta: np.ndarray          # (n, C)
    m_inv: np.ndarray          # (n, C, C)
    u: np.ndarray              # (n, C)
    v: np.ndarray              # (n, C)
    sigma_xq: np.ndarray       # (n, 3, C)
    d_raw: np.ndarray          # (n, C)
    s_tanh: np.ndarray         # (n, C)
    d_gate: np.ndarray         # (n, C)
    cov3_eigval: np.ndarray    # (n, 3) ascending
    cov3_eigvec: np.ndarray    # (n, 3, 3) columns, up to sign
    floor_eps: np.ndarray      # (n,)
    floored: np.ndarray        # (n,) bool
    l_x: np.ndarray            # (n, 3, 3)
    rotation: np.ndarray       # (n, 3, 3)
    s_x: np.ndarray            # (n, 3)
    s_q: np.ndarray            # (n, C)


@dataclass
class ProjectionCache:
    """Per-primitive projection state (reference raster.py:46-60)."""

    t_cam: np.ndarray        # (n, 3)
    depth: np.ndarray        # (n,)
    mean2: np.ndarray        # (n, 2)
    vmat: np.ndarray         # (n, 2, 3) jacobian @ rotation
    cov2_eigval: np.ndarray  # (n, 2) ascending, of the pre-floor cov2
    cov2_eigvec: np.ndarray  # (n, 2, 2) columns, up to sign
    floored: np.ndarray      # (n,) screen floor engaged
    cov2: np.ndarray         # (n, 2, 2)
    p2: np.ndarray           # (n, 2, 2)
    radii: np.ndarray        # (n, 2)
    visible: np.ndarray      # (n,)


@dataclass
class LossConfig:
    """Composite objective weights (gradients.py:29-40)."""

    lambda_ssim: float = 0.2
    lambda_o: float = 0.01
    lambda_sigma: float = 0.01
    loss_scale: float = 1.0


@dataclass
class SceneGrads:
    """One gradient array per PARAM_FIELDS entry (gradients.py:43-70)."""

    mu_x: np.ndarray
    mu_q: np.ndarray
    rot: np.ndarray
    s_x_raw: np.ndarray
    l_qx: np.ndarray
    s_q_raw: np.ndarray
    b_x: np.ndarray
    b_q: np.ndarray
    opacity_raw: np.ndarray
    color: np.ndarray

    @classmethod
    def zeros_like(cls, scene) -> "SceneGrads":
        return cls(**{k: np.zeros_like(np.asarray(getattr(scene, k), dtype=np.float64))
                      for k, _ in PARAM_FIELDS})

    @classmethod
    def from_records(cls, n_dims: int, records: np.ndarray) -> "SceneGrads":
        records = np.asarray(records, dtype=np.float64)
        n = records.shape[0]
        return cls(**{name: records[:, off:off + size].reshape((n,) + shape).copy()
                      for name, (off, size, shape) in field_offsets(n_dims).items()})

    def arrays(self) -> dict:
        return {k: getattr(self, k) for k, _ in PARAM_FIELDS}

    def check_finite(self):
        for name, arr in self.arrays().items():
            bad = ~np.isfinite(arr)
            if bad.any():
                prim = int(np.nonzero(bad.reshape(arr.shape[0], -1).any(axis=1))[0][0])
                raise GradientError(f"non-finite gradient in {name!r} of primitive {prim}")
