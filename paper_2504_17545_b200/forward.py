"""Drop-in replacement for the reference render API ``ges.forward``
(``/root/reference/pkg/src/ges/forward.py:36-417``).

Same names, arguments, dataclasses and exceptions; the work runs in the
sm_100a kernels of ``libges_b200.so``.  By default results are NumPy arrays
like the reference's (``to_numpy=True``); pass ``to_numpy=False`` to keep
torch CUDA tensors.  Differences, all deliberate and documented in DESIGN.md:

* ``settings.dtype`` selects the kernels: ``np.float32`` (the reference's
  default; the fused float32 tile kernel) or ``np.float64`` (the float64
  per-pixel kernels of ``ges_render_f64``, outputs float64 like the
  reference's); any other dtype raises ``NotImplementedError``.
* ``settings.threads`` is accepted and ignored.
* In supersample-4 mode depth/normal/winner are materialised arrays, not
  strided views of hi-res buffers (forward.py:205-207).
"""

from __future__ import annotations

import os
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .renderer import SCENE_CACHE, default_renderer

ALPHA_CUTOFF = 1.0 / 255.0
TILE = 16


def default_threads() -> int:
    """GES_THREADS / GES_DETERMINISTIC as in forward.py:30-33 (ignored on GPU)."""
    if os.environ.get("GES_DETERMINISTIC") == "1":
        return 1
    return max(1, int(os.environ.get("GES_THREADS", "1")))


@dataclass
class RenderSettings:
    supersample: int = 1
    background: tuple = (0.0, 0.0, 0.0)
    layers: str = "full"
    mip: bool = False
    epsilon_mode: str = "adaptive"
    epsilon_value: float = 0.0
    dtype: type = np.float32
    threads: int = field(default_factory=default_threads)
    with_geometry: bool = False

    def __post_init__(self):   # forward.py:48-54
        if self.supersample not in (1, 4):
            raise ValueError("supersample must be 1 or 4")
        if self.layers not in ("full", "surfels_only", "gaussians_only"):
            raise ValueError(f"unknown layer mode {self.layers!r}")
        if self.epsilon_mode not in ("adaptive", "constant"):
            raise ValueError(f"unknown epsilon mode {self.epsilon_mode!r}")

    @property
    def grid(self) -> int:
        return 2 if self.supersample == 4 else 1


@dataclass
class SurfelBuffers:
    color: object
    depth: object
    normal: object
    coverage: object
    winner: object


@dataclass
class GaussianBuffers:
    color: object
    weight: object
    depth: object = None
    normal: object = None


@dataclass
class RenderResult:
    image: object
    surfels: SurfelBuffers
    gaussians: GaussianBuffers


def _check_settings(settings):
    settings = settings or RenderSettings()
    if np.dtype(getattr(settings, "dtype", np.float32)) not in (np.float32, np.float64):
        raise NotImplementedError("the B200 kernels compute in float32 or float64")
    return settings


def _is_f64(settings) -> bool:
    return np.dtype(getattr(settings, "dtype", np.float32)) == np.float64


def _render_f64(scene, cam, settings, mode, surfel_depth=None):
    from .renderer import render_f64
    dev = _device()
    ds = SCENE_CACHE.get(scene, dev, need_source=True)
    return render_f64(default_renderer(dev), ds, cam, settings, mode=mode, surfel_depth=surfel_depth)


def _host(t):
    """Start the device -> host copy of ``t`` into pinned memory (torch's
    caching host allocator: blocks come back to the pool when the caller drops
    the array, so steady-state calls allocate nothing and copy at PCIe speed
    instead of through pageable staging).  Call ``_numpy`` after a sync."""
    if t is None:
        return None
    h = torch.empty(tuple(t.shape), dtype=t.dtype, pin_memory=True)
    h.copy_(t, non_blocking=True)
    return h


def _numpy(*hs):
    """Wait for the copies started by ``_host`` and view them as NumPy arrays
    (each array keeps its pinned block alive)."""
    if hs and any(h is not None for h in hs):
        torch.cuda.current_stream().synchronize()
    return tuple(None if h is None else h.numpy() for h in hs)


def _np(t):
    return _numpy(_host(t))[0]


def _device():
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2504_17545_b200 needs a CUDA device (there is no CPU fallback)")
    return torch.device("cuda", torch.cuda.current_device())


_SURF = ("color", "depth", "normal", "coverage", "winner")
_GAUSS = ("color", "weight", "depth", "normal")


def _surfel_buffers(fr, to_numpy):
    cov = torch.isfinite(fr.s_depth)
    sb = SurfelBuffers(fr.s_color, fr.s_depth, fr.s_normal, cov, fr.s_winner)
    if to_numpy:
        sb = SurfelBuffers(*_numpy(*(_host(getattr(sb, k)) for k in _SURF)))
    return sb


def _gauss_buffers(fr, to_numpy):
    gb = GaussianBuffers(fr.g_color, fr.g_weight, fr.g_depth, fr.g_normal)
    if to_numpy:
        gb = GaussianBuffers(*_numpy(*(_host(getattr(gb, k)) for k in _GAUSS)))
    return gb


def render(scene, cam, settings: RenderSettings | None = None, *, to_numpy: bool = True) -> RenderResult:
    """forward.py:403-417: both passes and the layer-selected image in one
    device frame (fused tile kernel)."""
    settings = _check_settings(settings)
    if _is_f64(settings):
        fr = _render_f64(scene, cam, settings, 3)
        if not to_numpy:
            return RenderResult(fr.image, _surfel_buffers(fr, False), _gauss_buffers(fr, False))
        cov = torch.isfinite(fr.s_depth)
        hs = [_host(t) for t in (fr.image, fr.s_color, fr.s_depth, fr.s_normal, cov, fr.s_winner,
                                 fr.g_color, fr.g_weight, fr.g_depth, fr.g_normal)]
        a = _numpy(*hs)
        return RenderResult(a[0], SurfelBuffers(*a[1:6]), GaussianBuffers(*a[6:10]))
    dev = _device()
    ds = SCENE_CACHE.get(scene, dev)
    fr = default_renderer(dev).render(ds, cam, settings, mode=3)
    if not to_numpy:
        return RenderResult(fr.image, _surfel_buffers(fr, False), _gauss_buffers(fr, False))
    # every buffer's copy is queued before the one synchronisation
    cov = torch.isfinite(fr.s_depth)
    hs = [_host(t) for t in (fr.image, fr.s_color, fr.s_depth, fr.s_normal, cov, fr.s_winner,
                             fr.g_color, fr.g_weight, fr.g_depth, fr.g_normal)]
    a = _numpy(*hs)
    return RenderResult(a[0], SurfelBuffers(*a[1:6]), GaussianBuffers(*a[6:10]))


def rasterize_surfels(scene, cam, settings: RenderSettings | None = None, *, to_numpy: bool = True) -> SurfelBuffers:
    """forward.py:127-209."""
    settings = _check_settings(settings)
    if _is_f64(settings):
        return _surfel_buffers(_render_f64(scene, cam, settings, 1), to_numpy)
    dev = _device()
    ds = SCENE_CACHE.get(scene, dev)
    fr = default_renderer(dev).render(ds, cam, settings, mode=1,
                                      want=("s_color", "s_depth", "s_normal", "s_winner"))
    return _surfel_buffers(fr, to_numpy)


def accumulate_gaussians(scene, cam, surfel_depth, settings: RenderSettings | None = None, *,
                         to_numpy: bool = True) -> GaussianBuffers:
    """forward.py:218-245 against a given (H, W) surfel depth map."""
    settings = _check_settings(settings)
    dev = _device()
    if _is_f64(settings):
        dep = torch.as_tensor(np.asarray(surfel_depth, dtype=np.float64) if not torch.is_tensor(surfel_depth)
                              else surfel_depth, dtype=torch.float64).to(dev).contiguous()
        if tuple(dep.shape) != (int(cam.height), int(cam.width)):
            raise ValueError("surfel_depth must have shape (height, width)")
        return _gauss_buffers(_render_f64(scene, cam, settings, 2, dep), to_numpy)
    ds = SCENE_CACHE.get(scene, dev)
    dep = torch.as_tensor(np.asarray(surfel_depth, dtype=np.float32) if not torch.is_tensor(surfel_depth)
                          else surfel_depth, dtype=torch.float32).to(dev).contiguous()
    if tuple(dep.shape) != (int(cam.height), int(cam.width)):
        raise ValueError("surfel_depth must have shape (height, width)")
    fr = default_renderer(dev).render(ds, cam, settings, mode=2, surfel_depth=dep,
                                      want=("g_color", "g_weight", "g_depth", "g_normal"))
    return _gauss_buffers(fr, to_numpy)


def _dev_f32(a, dev):
    if torch.is_tensor(a):
        return a.to(dev, torch.float32).contiguous()
    return torch.from_numpy(np.ascontiguousarray(np.asarray(a, dtype=np.float32))).to(dev)


def _dev_f64(a, dev):
    if torch.is_tensor(a):
        return a.to(dev, torch.float64).contiguous()
    return torch.from_numpy(np.ascontiguousarray(np.asarray(a, dtype=np.float64))).to(dev)


def _float64_inputs(*arrays) -> bool:
    """float64 buffers in -> the float64 kernels (as the reference keeps the dtype)."""
    return all((a.dtype == torch.float64) if torch.is_tensor(a) else (np.asarray(a).dtype == np.float64)
               for a in arrays)


def composite(surfel_color, gaussian: GaussianBuffers, surfel_weight: float = 1.0):
    """forward.py:384-388: (C_s * w_s + C_G) / (w_s + W_G) on the device
    (float64 kernels when the buffers are float64)."""
    dev = _device()
    as_np = not torch.is_tensor(surfel_color)
    if _float64_inputs(surfel_color, gaussian.color, gaussian.weight):
        sc, gc, gw = (_dev_f64(x, dev) for x in (surfel_color, gaussian.color, gaussian.weight))
        img = torch.empty_like(sc)
        _lib.check(_lib.lib().ges_composite_f64(sc.data_ptr(), gc.data_ptr(), gw.data_ptr(), float(surfel_weight),
                                                img.data_ptr(), gw.numel(),
                                                torch.cuda.current_stream(dev).cuda_stream), "ges_composite_f64")
        return _np(img) if as_np else img
    sc = _dev_f32(surfel_color, dev)
    gc = _dev_f32(gaussian.color, dev)
    gw = _dev_f32(gaussian.weight, dev)
    img = torch.empty_like(sc)
    n = gw.numel()
    _lib.check(_lib.lib().ges_composite(sc.data_ptr(), gc.data_ptr(), gw.data_ptr(), float(surfel_weight),
                                        img.data_ptr(), n, torch.cuda.current_stream(dev).cuda_stream),
               "ges_composite")
    return _np(img) if as_np else img


def smooth_geometry(surfel_buffers: SurfelBuffers, gaussian: GaussianBuffers):
    """forward.py:391-400."""
    if gaussian.depth is None:
        raise ValueError("gaussian buffers were rendered without geometry accumulation")
    dev = _device()
    as_np = not torch.is_tensor(surfel_buffers.depth)
    if _float64_inputs(surfel_buffers.depth, surfel_buffers.normal, gaussian.depth, gaussian.normal,
                       gaussian.weight):
        sd, sn, gd, gn, gw = (_dev_f64(x, dev) for x in (surfel_buffers.depth, surfel_buffers.normal,
                                                          gaussian.depth, gaussian.normal, gaussian.weight))
        d = torch.empty_like(sd)
        nrm = torch.empty_like(sn)
        _lib.check(_lib.lib().ges_smooth_geometry_f64(sd.data_ptr(), sn.data_ptr(), gd.data_ptr(), gn.data_ptr(),
                                                      gw.data_ptr(), d.data_ptr(), nrm.data_ptr(), sd.numel(),
                                                      torch.cuda.current_stream(dev).cuda_stream),
                   "ges_smooth_geometry_f64")
        return _numpy(_host(d), _host(nrm)) if as_np else (d, nrm)
    sd = _dev_f32(surfel_buffers.depth, dev)
    sn = _dev_f32(surfel_buffers.normal, dev)
    gd = _dev_f32(gaussian.depth, dev)
    gn = _dev_f32(gaussian.normal, dev)
    gw = _dev_f32(gaussian.weight, dev)
    d = torch.empty_like(sd)
    nrm = torch.empty_like(sn)
    _lib.check(_lib.lib().ges_smooth_geometry(sd.data_ptr(), sn.data_ptr(), gd.data_ptr(), gn.data_ptr(),
                                              gw.data_ptr(), d.data_ptr(), nrm.data_ptr(), sd.numel(),
                                              torch.cuda.current_stream(dev).cuda_stream),
               "ges_smooth_geometry")
    if as_np:
        return _numpy(_host(d), _host(nrm))
    return d, nrm
