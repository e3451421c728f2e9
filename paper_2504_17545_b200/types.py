"""Host-side scene and camera containers with the reference's field names.

The render API is duck-typed: it accepts the reference's own ``ges.Scene`` /
``ges.Camera`` objects unchanged.  These light containers exist so the
package (and its tests and bench on the GPU box, where the reference is not
installed) can build scenes without it.  Field names, dtypes and validation
follow the reference:

* ``Camera``        -- ``ges/cameras.py:17-80`` (pinhole, w2c 4x4, +z forward,
                       pixel centres at +0.5, ``NEAR_PLANE = 0.01``)
* ``SurfelSet``     -- ``ges/primitives.py:42-80`` (pos, quat wxyz, log_scale, sh, w)
* ``GaussianSet``   -- ``ges/primitives.py:82-161`` (pos, raw_opacity logit,
                       quat, log_scale (N,3|2), sh, kind, filter3d)
* ``Scene``         -- ``ges/primitives.py:166-191``
* ``GradientSet``   -- ``ges/primitives.py:194-214``
"""

from __future__ import annotations

import enum
import math
from dataclasses import dataclass, field

import numpy as np

NEAR_PLANE = 0.01
W_OPAQUE = 255.0


class GaussianKind(enum.Enum):
    THREE_D = "3d"
    TWO_D = "2d"


class Stage(enum.Enum):
    SURFEL_ONLY = "surfel_only"
    JOINT = "joint"
    FROZEN = "frozen"


def num_coeffs(degree: int) -> int:
    """(degree+1)^2; degree outside [0, 3] raises like ``sh.py:24-31``."""
    if not 0 <= degree <= 3:
        raise ValueError(f"SH degree must be in [0, 3], got {degree}")
    return (degree + 1) ** 2


@dataclass(frozen=True)
class Camera:
    fx: float
    fy: float
    cx: float
    cy: float
    width: int
    height: int
    world_to_camera: np.ndarray
    position: np.ndarray = field(init=False)

    def __post_init__(self):
        if self.fx <= 0 or self.fy <= 0:
            raise ValueError("focal lengths must be positive")
        m = np.asarray(self.world_to_camera, dtype=np.float64)
        if m.shape != (4, 4):
            raise ValueError("world_to_camera must be 4x4")
        rot = m[:3, :3]
        if not np.allclose(rot @ rot.T, np.eye(3), atol=1e-5):
            raise ValueError("world_to_camera rotation is not orthonormal")
        object.__setattr__(self, "world_to_camera", m)
        object.__setattr__(self, "position", -rot.T @ m[:3, 3])

    @property
    def rotation(self):
        return self.world_to_camera[:3, :3]

    @property
    def translation(self):
        return self.world_to_camera[:3, 3]

    def to_camera(self, points):
        return np.asarray(points) @ self.rotation.T + self.translation

    def project(self, cam_points):
        p = np.asarray(cam_points)
        return np.stack([self.fx * p[..., 0] / p[..., 2] + self.cx,
                         self.fy * p[..., 1] / p[..., 2] + self.cy], axis=-1)

    def scaled(self, factor: int) -> "Camera":
        k = factor
        return Camera(self.fx * k, self.fy * k, self.cx * k, self.cy * k,
                      self.width * k, self.height * k, self.world_to_camera)


def look_at(eye, target, up=(0.0, 0.0, 1.0)) -> np.ndarray:
    """World-to-camera 4x4: rows right, down, forward (``cameras.py:83-99``)."""
    eye = np.asarray(eye, dtype=np.float64)
    fwd = np.asarray(target, dtype=np.float64) - eye
    fwd /= np.linalg.norm(fwd)
    right = np.cross(fwd, np.asarray(up, dtype=np.float64))
    if np.linalg.norm(right) < 1e-9:
        right = np.cross(fwd, np.array([1.0, 0.0, 0.0]))
    right /= np.linalg.norm(right)
    down = np.cross(fwd, right)
    m = np.eye(4)
    m[:3, :3] = np.stack([right, down, fwd])
    m[:3, 3] = -m[:3, :3] @ eye
    return m


def orbit_cameras(center, radius, n, *, height=0.0, fov_deg=50.0, width=128,
                  height_px=128, phase=0.0, sweep=2.0 * math.pi):
    """Inward-looking cameras on a circle (``cameras.py:102-114``)."""
    center = np.asarray(center, dtype=np.float64)
    f = 0.5 * width / math.tan(0.5 * math.radians(fov_deg))
    out = []
    for k in range(n):
        a = phase + sweep * k / max(n, 1)
        eye = center + np.array([radius * math.cos(a), radius * math.sin(a), height])
        out.append(Camera(f, f, width / 2.0, height_px / 2.0, width, height_px,
                          look_at(eye, center)))
    return out


@dataclass
class SurfelSet:
    pos: np.ndarray
    quat: np.ndarray
    log_scale: np.ndarray
    sh: np.ndarray
    w: np.ndarray

    @property
    def count(self) -> int:
        return int(self.pos.shape[0])

    @property
    def scale(self):
        return np.exp(self.log_scale)

    def select(self, m) -> "SurfelSet":
        return SurfelSet(self.pos[m], self.quat[m], self.log_scale[m], self.sh[m], self.w[m])

    @staticmethod
    def empty(degree: int) -> "SurfelSet":
        K = num_coeffs(degree)
        return SurfelSet(np.zeros((0, 3)), np.zeros((0, 4)), np.zeros((0, 2)),
                         np.zeros((0, K, 3)), np.zeros((0,)))


@dataclass
class GaussianSet:
    pos: np.ndarray
    raw_opacity: np.ndarray
    quat: np.ndarray
    log_scale: np.ndarray
    sh: np.ndarray
    kind: GaussianKind = GaussianKind.THREE_D
    filter3d: np.ndarray = None

    def __post_init__(self):
        if self.filter3d is None:
            self.filter3d = np.zeros(self.pos.shape[0])

    @property
    def count(self) -> int:
        return int(self.pos.shape[0])

    @property
    def dim(self) -> int:
        return int(self.log_scale.shape[1])

    def select(self, m) -> "GaussianSet":
        return GaussianSet(self.pos[m], self.raw_opacity[m], self.quat[m],
                           self.log_scale[m], self.sh[m], self.kind, self.filter3d[m])

    @staticmethod
    def empty(degree: int, kind: GaussianKind = GaussianKind.THREE_D) -> "GaussianSet":
        K = num_coeffs(degree)
        D = 3 if kind is GaussianKind.THREE_D else 2
        return GaussianSet(np.zeros((0, 3)), np.zeros((0,)), np.zeros((0, 4)),
                           np.zeros((0, D)), np.zeros((0, K, 3)), kind)


@dataclass
class Scene:
    surfels: SurfelSet
    gaussians: GaussianSet
    sh_degree: int
    stage: Stage = Stage.FROZEN


@dataclass
class GradientSet:
    """Gradients w.r.t. exposed parameter values (primitives.py:194-214)."""
    surfel_pos: np.ndarray
    surfel_quat: np.ndarray
    surfel_scale: np.ndarray
    surfel_sh: np.ndarray
    surfel_w: np.ndarray
    gaussian_pos: np.ndarray
    gaussian_opacity: np.ndarray
    gaussian_quat: np.ndarray
    gaussian_scale: np.ndarray
    gaussian_sh: np.ndarray
    surfel_screen_grad: np.ndarray = None
    gaussian_screen_grad: np.ndarray = None

    def check_finite(self):
        for name, arr in self.__dict__.items():
            if arr is not None and arr.size and not np.all(np.isfinite(arr)):
                raise FloatingPointError(f"non-finite gradient in {name}")
