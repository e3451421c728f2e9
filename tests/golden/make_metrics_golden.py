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

from ges.losses import ssim  # noqa: E402  (reference, read-only)
from ges.metrics import psnr  # noqa: E402


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
    np.savez_compressed(os.path.join(HERE, "metrics.npz"), **out)
    print({k: float(v) for k, v in out.items() if v.ndim == 0})


if __name__ == "__main__":
    main()
