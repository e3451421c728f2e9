"""Seeded synthetic scenes and cameras.

The generators draw from ``np.random.default_rng`` in the same call order as
the reference's test fixtures (``pkg/tests/conftest.py:9-57``) so a given
seed reproduces the reference's test scenes exactly.  The benchmark configs
extend them with the sizes and scale ranges pinned in SURVEY.md 8(d).
"""

from __future__ import annotations

import math

import numpy as np

from .types import (Camera, GaussianKind, GaussianSet, Scene, Stage, SurfelSet,
                    look_at, num_coeffs, orbit_cameras)


def make_camera(width=32, height=32, dist=4.0, azim=0.3, elev=0.25, fov=50.0) -> Camera:
    """conftest.py:9-13 / SURVEY 8(d) camera."""
    eye = dist * np.array([math.cos(azim) * math.cos(elev),
                           math.sin(azim) * math.cos(elev), math.sin(elev)])
    f = 0.5 * width / math.tan(0.5 * math.radians(fov))
    return Camera(f, f, width / 2, height / 2, width, height, look_at(eye, (0, 0, 0)))


def random_quats(rng, n):
    q = rng.standard_normal((n, 4))
    return q / np.linalg.norm(q, axis=1, keepdims=True)


def random_surfels(rng, n, degree=1, w=255.0, scale_range=(0.15, 0.6),
                   sh_amplitude=0.25, extent=1.2) -> SurfelSet:
    K = num_coeffs(degree)
    sh = rng.uniform(-sh_amplitude, sh_amplitude, (n, K, 3))
    pos = rng.uniform(-extent, extent, (n, 3))
    quat = random_quats(rng, n)
    log_scale = np.log(rng.uniform(*scale_range, (n, 2)))
    return SurfelSet(pos=pos, quat=quat, log_scale=log_scale, sh=sh, w=np.full(n, float(w)))


def _logit(p):
    return np.log(p / (1.0 - p))


def random_gaussians(rng, n, degree=1, kind=GaussianKind.THREE_D,
                     scale_range=(0.05, 0.35), opacity_range=(0.15, 0.9),
                     sh_amplitude=0.25, extent=1.4) -> GaussianSet:
    K = num_coeffs(degree)
    D = 3 if kind is GaussianKind.THREE_D else 2
    pos = rng.uniform(-extent, extent, (n, 3))
    raw = _logit(rng.uniform(*opacity_range, n))
    quat = random_quats(rng, n)
    log_scale = np.log(rng.uniform(*scale_range, (n, D)))
    sh = rng.uniform(-sh_amplitude, sh_amplitude, (n, K, 3))
    return GaussianSet(pos=pos, raw_opacity=raw, quat=quat, log_scale=log_scale, sh=sh, kind=kind)


def random_scene(rng, n_surfels=8, n_gaussians=12, degree=1,
                 kind=GaussianKind.THREE_D, w=255.0, stage=Stage.FROZEN) -> Scene:
    return Scene(random_surfels(rng, n_surfels, degree, w=w),
                 random_gaussians(rng, n_gaussians, degree, kind=kind), degree, stage)


def min_sampling_interval(positions, cams, margin=0.15):
    """World size of one pixel, minimised over observing cameras
    (``filters.py:39-53``)."""
    best = np.full(positions.shape[0], np.inf)
    for cam in cams:
        t = cam.to_camera(positions)
        z = t[:, 2]
        ok = z > 0.01
        px = cam.project(np.where(ok[:, None], t, np.array([0.0, 0.0, 1.0])))
        mx, my = margin * cam.width, margin * cam.height
        seen = ok & (px[:, 0] > -mx) & (px[:, 0] < cam.width + mx) \
            & (px[:, 1] > -my) & (px[:, 1] < cam.height + my)
        best = np.where(seen, np.minimum(best, z / max(cam.fx, cam.fy)), best)
    return best


def mip_world_filter(g: GaussianSet, cams, coef=0.2) -> GaussianSet:
    """Attach filter3d = coef * interval^2 (``filters.py:56-69``)."""
    var = coef * min_sampling_interval(g.pos, cams) ** 2
    return GaussianSet(g.pos, g.raw_opacity, g.quat, g.log_scale, g.sh, g.kind,
                       np.where(np.isfinite(var), var, 0.0))


# --- benchmark configurations (BASELINE.json configs) ----------
CONFIGS = {
    1: dict(ns=10_000, ng=2_000, deg=0, res=(128, 128),
            s_rng=(0.01, 0.04), g_rng=(0.005, 0.03)),
    2: dict(ns=1_000_000, ng=300_000, deg=3, res=(1920, 1080),
            s_rng=(0.002, 0.008), g_rng=(0.002, 0.01)),
    3: dict(ns=1_000_000, ng=60_000, deg=3, res=(1920, 1080),
            s_rng=(0.002, 0.008), g_rng=(0.002, 0.01)),
    4: dict(ns=1_000_000, ng=300_000, deg=3, res=(3840, 2160),
            s_rng=(0.002, 0.008), g_rng=(0.002, 0.01)),
    5: dict(ns=3_000_000, ng=1_000_000, deg=3, res=(3840, 2160),
            s_rng=(0.0012, 0.0046), g_rng=(0.0011, 0.0055)),
}


def config_scene(cfg: int, seed: int = 0, *, scale_down: int = 1) -> Scene:
    """Scene of a BASELINE config.  Config 3 is the first 60k Gaussians of the
    config-2 draw; config 4 adds the mip world filter for the 4K camera.
    ``scale_down`` divides primitive counts (for quick tests only)."""
    c = CONFIGS[cfg]
    rng = np.random.default_rng(seed)
    ns = c["ns"] // scale_down
    ng = (CONFIGS[2]["ng"] if cfg == 3 else c["ng"]) // scale_down
    s = random_surfels(rng, ns, c["deg"], scale_range=c["s_rng"], extent=1.2)
    g = random_gaussians(rng, ng, c["deg"], scale_range=c["g_rng"], extent=1.2)
    if cfg == 3:
        g = g.select(slice(0, c["ng"] // scale_down))
    if cfg == 4:
        g = mip_world_filter(g, [make_camera(3840, 2160)])
    return Scene(s, g, c["deg"], Stage.FROZEN)


def config_cameras(cfg: int):
    """Cameras of a config: one pose (configs 1-3), the 4 Mip scales (config 4)
    or the 256-view 4K orbit (config 5)."""
    if cfg in (1, 2, 3):
        w, h = CONFIGS[cfg]["res"]
        return [make_camera(w, h)]
    if cfg == 4:
        return [make_camera(3840 // k, 2160 // k) for k in (8, 4, 2, 1)]
    return orbit_cameras((0, 0, 0), 4.0, 256, height=1.0, fov_deg=50.0,
                         width=3840, height_px=2160)


def orbit_views(n, width, height, radius=4.0, elev=1.0):
    """n inward-looking views around the scene (multi-view batches)."""
    return orbit_cameras((0, 0, 0), radius, n, height=elev, fov_deg=50.0,
                         width=width, height_px=height)
