"""Golden PSNR/SSIM values from the REAL reference (``ges.metrics.psnr``,
``ges.losses.ssim``; /root/reference/pkg/src/ges/metrics.py:20-33,
losses.py:14-58) on seeded images.  Run in the build container:

    python tests/golden/make_metrics_golden.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

import ges  # noqa: E402  (reference, read-only)
from ges.losses import ssim  # noqa: E402
from ges.metrics import camera_path, consistency_probe, psnr  # noqa: E402


def main():
    rng = np.random.default_rng(11)
    out = {}
    cases = [("rgb", (37, 53, 3)), ("small", (11, 11, 3)), ("gray", (24, 19)), ("wide", (12, 90, 3))]
    for name, shp in cases:
        a = rng.random(shp)
        b = np.clip(a + rng.normal(0, 0.05, shp), 0, 1)
        out[f"{name}_a"], out[f"{name}_b"] = a, b
        out[f"{name}_psnr"] = np.float64(psnr(a, b))
        out[f"{name}_ssim"] = np.float64(ssim(a, b))
    out["same_psnr"] = np.float64(psnr(out["rgb_a"], out["rgb_a"]))   # +inf
    out["same_ssim"] = np.float64(ssim(out["rgb_a"], out["rgb_a"]))
    # camera_path / consistency_probe (metrics.py:79-140)
    w2c = ges.look_at(np.array([3.0, 1.0, 1.5]), np.zeros(3))
    base = ges.Camera(60.0, 58.0, 31.5, 24.0, 64, 48, w2c)
    cams = camera_path(base, [0.1, -0.2, 0.0], frames=5, angle=0.05)
    out["path_base_w2c"] = w2c
    out["path_w2c"] = np.stack([c.world_to_camera for c in cams])
    imgs = rng.random((5, 48, 64, 3))
    pts = rng.normal(size=(20, 3))
    probe = consistency_probe(None, cams, anchor_points=pts, images=list(imgs))
    out["probe_images"], out["probe_points"] = imgs, pts
    for k in ("max_change", "mean_change", "bounds"):
        out[f"probe_{k}"] = np.array(probe[k])
    np.savez_compressed(os.path.join(HERE, "metrics.npz"), **out)
    print({k: float(v) for k, v in out.items() if v.ndim == 0})


if __name__ == "__main__":
    main()
