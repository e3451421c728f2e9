"""Evaluation on the GPU (the multi-view caller of the
render path): the reference's ``ges.metrics`` surface
(``/root/reference/pkg/src/ges/metrics.py:20-71``) with the views rendered by
the sm_100a path and scored on the device.

* ``psnr(a, b)``: 10 log10(1 / MSE), +inf when identical (``metrics.py:20-29``).
* ``ssim(a, b)``: mean SSIM over pixels and channels with the universal
  constants -- 11-tap Gaussian window (sigma 1.5), zero-padded separable
  correlation, C1 = 0.01^2, C2 = 0.03^2 (``losses.py:14-58``).  Computed in
  float64 with torch on the arrays' device (the render output's: cuda).
* ``evaluate(scene, dataset, views=None, settings=None) -> EvalReport``
  (``metrics.py:53-71``): default views = ``dataset.test_idx``, default
  settings ``RenderSettings(supersample=4)``; ``ms_per_frame`` is the mean
  wall time of one ``render`` call.

Accepts NumPy arrays or torch tensors; returns Python floats like the
reference.
"""

from __future__ import annotations

import json
import math
import time
from dataclasses import dataclass, field

import numpy as np
import torch

PSNR_INF = float("inf")
SSIM_WINDOW = 11
SSIM_SIGMA = 1.5
SSIM_C1 = 0.01 ** 2
SSIM_C2 = 0.03 ** 2


def _t64(a, device=None) -> torch.Tensor:
    if torch.is_tensor(a):
        return a.to(device or a.device, torch.float64)
    return torch.as_tensor(np.asarray(a, dtype=np.float64), device=device)


def _pair(a, b):
    dev = a.device if torch.is_tensor(a) else (b.device if torch.is_tensor(b) else None)
    ta, tb = _t64(a, dev), _t64(b, dev)
    if ta.shape != tb.shape:
        raise ValueError(f"shape mismatch {tuple(ta.shape)} vs {tuple(tb.shape)}")
    return ta, tb


def psnr(a, b) -> float:
    """metrics.py:20-29."""
    ta, tb = _pair(a, b)
    mse = float(torch.mean((ta - tb) ** 2))
    if mse == 0.0:
        return PSNR_INF
    return 10.0 * math.log10(1.0 / mse)


def _window(device) -> torch.Tensor:
    r = SSIM_WINDOW // 2
    x = torch.arange(-r, r + 1, dtype=torch.float64, device=device)
    w = torch.exp(-0.5 * (x / SSIM_SIGMA) ** 2)
    return w / w.sum()


def _blur(img: torch.Tensor, w: torch.Tensor) -> torch.Tensor:
    """Zero-padded separable correlation along H then W (losses.py:31-33) of
    an (H, W, C) image."""
    H, W, C = img.shape
    r = SSIM_WINDOW // 2
    k = w.view(1, 1, -1)
    x = img.permute(2, 1, 0).reshape(C * W, 1, H)                  # rows of columns: correlate along H
    x = torch.nn.functional.conv1d(x, k, padding=r).reshape(C, W, H).permute(0, 2, 1)   # (C, H, W)
    x = torch.nn.functional.conv1d(x.reshape(C * H, 1, W), k, padding=r)              # along W
    return x.reshape(C, H, W).permute(1, 2, 0)


def ssim(a, b) -> float:
    """Mean SSIM over pixels and channels (losses.py:36-58); (H, W, 3) or (H, W)."""
    ta, tb = _pair(a, b)
    if ta.shape[0] < SSIM_WINDOW or ta.shape[1] < SSIM_WINDOW:
        raise ValueError("image smaller than the SSIM window")
    if ta.dim() == 2:
        ta, tb = ta[..., None], tb[..., None]
    w = _window(ta.device)
    mu_a, mu_b = _blur(ta, w), _blur(tb, w)
    var_a = _blur(ta * ta, w) - mu_a * mu_a
    var_b = _blur(tb * tb, w) - mu_b * mu_b
    cov = _blur(ta * tb, w) - mu_a * mu_b
    s = ((2 * mu_a * mu_b + SSIM_C1) * (2 * cov + SSIM_C2)) / \
        ((mu_a * mu_a + mu_b * mu_b + SSIM_C1) * (var_a + var_b + SSIM_C2))
    return float(s.mean())


@dataclass
class EvalReport:
    """metrics.py:36-50 (same fields and JSON form)."""
    per_view_psnr: list = field(default_factory=list)
    per_view_ssim: list = field(default_factory=list)
    mean_psnr: float = 0.0
    mean_ssim: float = 0.0
    n_surfels: int = 0
    n_gaussians: int = 0
    ms_per_frame: float = 0.0
    consistency: dict = field(default_factory=dict)

    def to_json(self) -> str:
        d = dict(self.__dict__)
        d["per_view_psnr"] = [("inf" if np.isinf(v) else v) for v in self.per_view_psnr]
        return json.dumps(d, indent=1)


def evaluate(scene, dataset, views=None, settings=None) -> EvalReport:
    """metrics.py:53-71 with the views rendered and scored on the GPU."""
    from .forward import RenderSettings, render
    settings = settings or RenderSettings(supersample=4)
    views = dataset.test_idx if views is None else views
    rep = EvalReport(n_surfels=int(np.asarray(scene.surfels.pos).shape[0]),
                     n_gaussians=int(np.asarray(scene.gaussians.pos).shape[0]))
    times = []
    for vi in views:
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        out = render(scene, dataset.cameras[vi], settings, to_numpy=False)
        torch.cuda.synchronize()
        times.append(time.perf_counter() - t0)
        gt = _t64(dataset.images[vi], out.image.device)
        rep.per_view_psnr.append(psnr(out.image, gt))
        rep.per_view_ssim.append(ssim(out.image, gt))
    finite = [v for v in rep.per_view_psnr if np.isfinite(v)]
    rep.mean_psnr = float(np.mean(finite)) if finite else PSNR_INF
    rep.mean_ssim = float(np.mean(rep.per_view_ssim)) if rep.per_view_ssim else 0.0
    rep.ms_per_frame = float(np.mean(times) * 1000.0) if times else 0.0
    return rep


# --------------------------------------------------------------------------- view consistency
def camera_path(base, target, *, frames: int, angle: float = 0.02, radius_scale: float = 1.0) -> list:
    """Small orbit around ``target`` through the base camera's eye, ``angle``
    radians per frame (metrics.py:79-95)."""
    from .types import Camera, look_at
    target = np.asarray(target, dtype=np.float64)
    rel = np.asarray(base.position, dtype=np.float64) - target
    r = float(np.linalg.norm(rel[:2]))
    a0 = math.atan2(rel[1], rel[0])
    cams = []
    for k in range(frames):
        a = a0 + angle * k
        eye = target + np.array([r * radius_scale * math.cos(a), r * radius_scale * math.sin(a), rel[2]])
        cams.append(Camera(base.fx, base.fy, base.cx, base.cy, base.width, base.height, look_at(eye, target)))
    return cams


def motion_bound(prev_img, flow_px: float, quantum: float = 1.0 / 255.0) -> float:
    """Max finite-difference image gradient x max pixel displacement + the
    clamp quantum (metrics.py:98-107)."""
    gy, gx = np.gradient(np.asarray(prev_img, dtype=np.float64), axis=(0, 1))
    return float(np.maximum(np.abs(gx), np.abs(gy)).max()) * flow_px + quantum


def max_flow_px(cam_a, cam_b, points) -> float:
    """Largest screen displacement of the anchor points between two views (metrics.py:110-114)."""
    pa = cam_a.project(cam_a.to_camera(points))
    pb = cam_b.project(cam_b.to_camera(points))
    return float(np.linalg.norm(pa - pb, axis=1).max())


def consistency_probe(render_fn, cams: list, anchor_points=None, images=None) -> dict:
    """Per-pair max / mean absolute pixel change along a path, plus the
    camera-motion bounds when anchor points are given (metrics.py:116-140).
    ``images`` may be a (V, H, W, 3) device tensor: the changes are then
    computed on the device in float64."""
    if not cams:
        raise ValueError("empty camera path")
    if images is None:
        images = [render_fn(c) for c in cams]
    if torch.is_tensor(images):
        d = (images[1:].double() - images[:-1].double()).abs().flatten(1)
        max_change = [float(v) for v in d.max(dim=1).values.cpu()] if len(images) > 1 else []
        mean_change = [float(v) for v in d.mean(dim=1).cpu()] if len(images) > 1 else []
        imgs = None
    else:
        imgs = [np.asarray(im, dtype=np.float64) for im in images]
        max_change = [float(np.abs(a - b).max()) for a, b in zip(imgs, imgs[1:])]
        mean_change = [float(np.abs(a - b).mean()) for a, b in zip(imgs, imgs[1:])]
    bounds = []
    if anchor_points is not None and len(cams) > 1:
        if imgs is None:
            imgs = [im.double().cpu().numpy() for im in images]
        for (ca, cb), img in zip(zip(cams, cams[1:]), imgs):
            bounds.append(motion_bound(img, max_flow_px(ca, cb, anchor_points)))
    return {"max_change": max_change, "mean_change": mean_change, "bounds": bounds}
