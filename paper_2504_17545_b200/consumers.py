"""Callers of the surfel pass beyond `render`.

``covering_counts`` is the reference's densification statistic
(``optim.py:219-230``): per surfel, the maximum over views of the number of
pixels it wins in the opaque z-buffer.  Here the winner maps stay on the
device and the per-view counts are a device bincount over the int32 winner
map the tile kernel writes.
"""

from __future__ import annotations

import numpy as np
import torch

from .forward import RenderSettings, _check_settings, _device
from .renderer import SCENE_CACHE, default_renderer


def covering_counts(scene, cams, dtype=np.float32, *, to_numpy: bool = True):
    """optim.py:219-230; ``dtype`` selects the float32 or float64 surfel pass
    like the reference's ``RenderSettings(dtype=dtype)``."""
    settings = _check_settings(RenderSettings(supersample=1, dtype=dtype))
    f64 = np.dtype(dtype) == np.float64
    dev = _device()
    ds = SCENE_CACHE.get(scene, dev, need_source=f64)
    r = default_renderer(dev)
    n = ds.n_surfels
    best = torch.zeros(n, dtype=torch.int64, device=dev)
    for cam in cams:
        if f64:
            from .renderer import render_f64
            fr = render_f64(r, ds, cam, settings, mode=1)
        else:
            fr = r.render(ds, cam, settings, mode=1, want=("s_winner",))
        w = fr.s_winner.reshape(-1)
        counts = torch.bincount(w[w >= 0].long(), minlength=n)
        best = torch.maximum(best, counts)
    return best.cpu().numpy() if to_numpy else best
