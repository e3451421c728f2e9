"""Drop-in for the reference training renderer's joint stage
(``ges.training``, /root/reference/pkg/src/ges/training.py).

The joint stage of the reference trainer (optim.py:715-735) renders every
iteration with frozen, fully opaque surfels (``frozen_cache`` set, all
``w == 255``) and trainable Gaussians, then calls :func:`backward`.  This
module runs that step on the GPU:

* forward -- the deployment kernels: the cached opaque z-buffer of the
  supersampled camera (``ges_rasterize_surfels``, training.py:358-392), the
  surfel view colours (``ges_surfel_colors``) and the Gaussian pass
  (``ges_accumulate_gaussians`` on 16 px tiles, training.py:399-544);
* backward -- ``ges_backward_gaussians`` (training.py:646-788: a per-tile
  replay of the Gaussian pass with warp-reduced float64 partial sums, then a
  per-Gaussian float64 chain rule) and ``ges_backward_surfels_frozen``
  (training.py:612-629).

Same names and arguments as the reference (``TrainSettings``,
``TrainFrame``, ``render_training``, ``backward``, ``GradientSet``).
Deliberate differences, documented in DESIGN.md:

* the translucent surfel pass of the surfel stage (training.py:145-292,
  ``w < 255`` or no ``frozen_cache``) is not on the GPU path and raises
  ``NotImplementedError``; surfels may also be disabled
  (``surfels_enabled=False``);
* per-pixel arithmetic is float32 (``settings.dtype`` only sets the dtype of
  the returned NumPy arrays); gradients are float64;
* the frame carries no per-fragment tape; ``frame.tape`` holds the device
  state :func:`backward` needs.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from types import SimpleNamespace

import numpy as np
import torch

from . import _lib
from .forward import _host, _numpy
from .renderer import DeviceScene, camera_struct, default_renderer, settings_struct
from .types import GaussianKind, GradientSet

W_ADJUST_THRESHOLD = 30.0
W_OPAQUE = 255.0


@dataclass
class TrainSettings:
    """Training-path knobs (training.py:36-63); ``None`` = from the schedule state."""
    supersample: int | None = None
    adjust_order: bool | None = None
    background: tuple = (0.0, 0.0, 0.0)
    epsilon_mode: str = "adaptive"
    epsilon_value: float = 0.0
    mip: bool = False
    with_geometry: bool = False
    gaussians_enabled: bool = True
    surfels_enabled: bool = True
    dtype: type = np.float64
    frozen_cache: dict | None = None
    gaussian_only_norm: bool = False

    def resolve(self, scene):
        w = np.asarray(scene.surfels.w)
        wmin = w.min() if w.size else np.inf
        late = wmin >= W_ADJUST_THRESHOLD
        ss = self.supersample if self.supersample is not None else (4 if late else 1)
        adj = self.adjust_order if self.adjust_order is not None else late
        return ss, adj, late


@dataclass
class TrainFrame:
    """Forward buffers plus the device state :func:`backward` needs (training.py:66-78)."""
    image: object
    surfel_color: object
    surfel_depth: object
    gauss_color: object
    gauss_weight: object
    blend_depth: object = None
    blend_normal: object = None
    gauss_depth: object = None
    gauss_normal: object = None
    tape: dict = field(default_factory=dict)


def _count(a) -> int:
    return int(np.asarray(a).shape[0])


def _pass_settings(st: TrainSettings, **kw):
    ns = SimpleNamespace(supersample=1, layers="full", mip=st.mip, epsilon_mode=st.epsilon_mode,
                         epsilon_value=st.epsilon_value, with_geometry=st.with_geometry,
                         background=tuple(st.background), tile_mode=1)
    for k, v in kw.items():
        setattr(ns, k, v)
    return ns


def _out(t, to_numpy, dtype):
    if t is None or not to_numpy:
        return t
    return _numpy(_host(t.detach()))[0].astype(dtype, copy=False)


def _as_dev(a, dev, dtype=torch.float32):
    if a is None:
        return None
    if isinstance(a, torch.Tensor):
        return a.to(device=dev, dtype=dtype).contiguous()
    return torch.as_tensor(np.ascontiguousarray(a), dtype=dtype, device=dev).contiguous()


def _frozen_entry(ds, scene, rc, settings, cache_key, dev):
    """Cached opaque z-buffer of the (supersampled) camera (training.py:367-381)."""
    cache = settings.frozen_cache
    entry = cache.get(cache_key) if cache_key is not None else None
    if entry is not None and not entry.get("_gpu"):   # written by the reference: adopt it
        entry = {"winner": _as_dev(np.asarray(entry["winner"]).reshape(-1), dev, torch.int32),
                 "depth": _as_dev(np.asarray(entry["depth"]).reshape(-1), dev),
                 "normal": _as_dev(np.asarray(entry["normal"]).reshape(-1, 3), dev), "_gpu": True}
    if entry is None:
        fr = default_renderer(dev).render(ds, rc, _pass_settings(settings, with_geometry=False), mode=1,
                                          want=("s_depth", "s_normal", "s_winner"))
        entry = {"winner": fr.s_winner.reshape(-1), "depth": fr.s_depth.reshape(-1),
                 "normal": fr.s_normal.reshape(-1, 3), "_gpu": True}
    if "covered_any" not in entry:   # once per cached z-buffer, not per step
        entry["covered_any"] = bool((entry["winner"] >= 0).any())
        if cache_key is not None:
            cache[cache_key] = entry
    return entry


def render_training(scene, cam, settings: TrainSettings | None = None, cache_key=None, *,
                    to_numpy: bool = True, device=None, device_scene: DeviceScene | None = None) -> TrainFrame:
    """training.py:295-355 for the joint stage (frozen surfels or none) on the GPU.

    ``device_scene``: a ``DeviceScene(scene, keep_source=True)`` packed from
    the CURRENT parameter values, to skip the per-call upload and pack (the
    caller re-packs after every parameter update)."""
    settings = settings or TrainSettings()
    dev = torch.device(device or "cuda")
    if dev.index is None:
        dev = torch.device("cuda", torch.cuda.current_device())
    ns, ng = _count(scene.surfels.pos), _count(scene.gaussians.pos)
    ss, _adjust, late = settings.resolve(scene)
    grid = 2 if ss == 4 else 1
    H, W = int(cam.height), int(cam.width)
    bg = torch.tensor([float(v) for v in settings.background], dtype=torch.float32, device=dev)
    use_surfels = settings.surfels_enabled and ns > 0
    fast = (use_surfels and settings.frozen_cache is not None
            and bool(np.all(np.asarray(scene.surfels.w) == W_OPAQUE)))
    if use_surfels and not fast:
        raise NotImplementedError(
            "the translucent surfel pass (training.py:145-292) is not on the GPU path: the GPU training "
            "step needs frozen surfels (w == 255 and settings.frozen_cache) or surfels_enabled=False")
    if device_scene is not None:
        if device_scene.src is None:
            raise ValueError("device_scene must be built with keep_source=True")
        ds = device_scene
    else:
        ds = DeviceScene(scene, dev, keep_source=True)
    L = _lib.lib()
    stream = C.c_void_p(torch.cuda.current_stream(dev).cuda_stream)
    geom = bool(settings.with_geometry)
    blend_depth = blend_normal = None
    winner = None
    if fast:
        rc = cam.scaled(grid) if grid > 1 else cam
        entry = _frozen_entry(ds, scene, rc, settings, cache_key, dev)
        winner = entry["winner"]
        colors = torch.empty((ns, 3), dtype=torch.float32, device=dev)
        _lib.check(L.ges_surfel_colors(C.byref(ds.c), C.byref(camera_struct(cam)), C.c_void_p(colors.data_ptr()),
                                       stream), "surfel colours")
        # box-mean colour, gate depth (late phase, all w = 255 >= 30: the front
        # hit of sub-sample 0) and blended geometry in one kernel
        f32 = dict(dtype=torch.float32, device=dev)
        surfel_color = torch.empty((H, W, 3), **f32)
        surfel_depth = torch.empty((H, W), **f32)
        if geom:
            blend_depth = torch.empty((H, W), **f32)
            blend_normal = torch.empty((H, W, 3), **f32)
        ptr = lambda t: C.c_void_p(t.data_ptr()) if t is not None else None  # noqa: E731
        bgh = (C.c_float * 3)(*[float(v) for v in settings.background])
        _lib.check(L.ges_frozen_surfel_buffers(ptr(winner), ptr(entry["depth"]), ptr(entry["normal"]), ptr(colors),
                                               W, H, grid, C.cast(bgh, C.c_void_p), ptr(surfel_color), ptr(surfel_depth),
                                               ptr(blend_depth), ptr(blend_normal), stream), "frozen surfel buffers")
    else:
        surfel_color = bg.expand(H, W, 3).clone()
        surfel_depth = torch.full((H, W), float("inf"), dtype=torch.float32, device=dev)
        if geom and use_surfels:
            blend_depth = torch.zeros((H, W), dtype=torch.float32, device=dev)
            blend_normal = torch.zeros((H, W, 3), dtype=torch.float32, device=dev)
    gaussians = settings.gaussians_enabled and ng > 0
    gd = gn = None
    if gaussians:
        fr = default_renderer(dev).render(ds, cam, _pass_settings(settings), mode=2, surfel_depth=surfel_depth,
                                          want=("g_color", "g_weight", "g_depth", "g_normal"))
        gc, gw = fr.g_color, fr.g_weight
        if geom:
            gd, gn = fr.g_depth, fr.g_normal
    else:
        gc = torch.zeros((H, W, 3), dtype=torch.float32, device=dev)
        gw = torch.zeros((H, W), dtype=torch.float32, device=dev)
        if geom:
            gd = torch.zeros((H, W), dtype=torch.float32, device=dev)
            gn = torch.zeros((H, W, 3), dtype=torch.float32, device=dev)
    gaussian_only = settings.gaussian_only_norm and not use_surfels
    if gaussian_only:   # training.py:329-332
        image = torch.where(gw[..., None] > 0, gc / gw.clamp_min(1e-12)[..., None], bg)
    else:
        image = (surfel_color + gc) / (1.0 + gw)[..., None]
    dt = settings.dtype
    frame = TrainFrame(image=_out(image, to_numpy, dt), surfel_color=_out(surfel_color, to_numpy, dt),
                       surfel_depth=_out(surfel_depth, to_numpy, dt), gauss_color=_out(gc, to_numpy, dt),
                       gauss_weight=_out(gw, to_numpy, dt), blend_depth=_out(blend_depth, to_numpy, dt),
                       blend_normal=_out(blend_normal, to_numpy, dt), gauss_depth=_out(gd, to_numpy, dt),
                       gauss_normal=_out(gn, to_numpy, dt))
    frame.tape = {"scene": scene, "cam": cam, "settings": settings, "grid": grid, "late": late,
                  "device_scene": ds, "device": dev, "image": image, "gauss_weight": gw,
                  "surfel_depth": surfel_depth, "winner": winner, "use_surfels": use_surfels,
                  "covered_any": bool(entry["covered_any"]) if fast else False,
                  "frozen": fast, "gaussians": gaussians, "gaussian_only": gaussian_only}
    return frame


def backward(frame: TrainFrame, g_image, *, g_blend_depth=None, g_blend_normal=None,
             g_gauss_depth=None, g_gauss_normal=None, g_gauss_weight=None, to_numpy: bool = True) -> GradientSet:
    """training.py:547-609 on the GPU.  ``g_image`` is dL/dC (H, W, 3); the
    optional cotangents feed the geometry buffers.  Returns float64 gradients
    w.r.t. exposed parameter values (NumPy, or torch CUDA tensors with
    ``to_numpy=False``).  ``g_blend_*`` are accepted like the reference's and,
    as in its frozen-surfel path (training.py:612-629), do not reach any
    parameter."""
    tape = frame.tape
    if not tape:
        raise ValueError("frame carries no tape; re-render with render_training")
    scene, cam, settings = tape["scene"], tape["cam"], tape["settings"]
    dev, ds = tape["device"], tape["device_scene"]
    H, W = int(cam.height), int(cam.width)
    g_img = _as_dev(g_image, dev)
    image, gw = tape["image"], tape["gauss_weight"]
    if tape["gaussian_only"]:
        wsafe = gw.clamp_min(1e-12)
        cov = gw > 0
        g_cg = torch.where(cov[..., None], g_img / wsafe[..., None], torch.zeros((), device=dev))
        g_wg = torch.where(cov, -(g_img * image).sum(-1) / wsafe, torch.zeros((), device=dev))
        g_cs = torch.zeros_like(g_img)
    else:
        denom = 1.0 + gw
        g_cs = g_img / denom[..., None]
        g_cg = g_cs
        g_wg = -(g_img * image).sum(-1) / denom
    if g_gauss_weight is not None:
        g_wg = g_wg + _as_dev(g_gauss_weight, dev)
    g_cg, g_wg = g_cg.contiguous(), g_wg.contiguous()

    ns, ng = _count(scene.surfels.pos), _count(scene.gaussians.pos)
    K = (ds.sh_degree + 1) ** 2
    dim = ds.dim if ng else (3 if getattr(scene.gaussians, "kind", GaussianKind.THREE_D) is GaussianKind.THREE_D
                            else 2)
    f64 = dict(dtype=torch.float64, device=dev)
    out = {k: torch.zeros(shape, **f64) for k, shape in (
        ("surfel_pos", (ns, 3)), ("surfel_quat", (ns, 4)), ("surfel_scale", (ns, 2)),
        ("surfel_sh", (ns, K, 3)), ("surfel_w", (ns,)), ("gaussian_pos", (ng, 3)),
        ("gaussian_opacity", (ng,)), ("gaussian_quat", (ng, 4)), ("gaussian_scale", (ng, dim)),
        ("gaussian_sh", (ng, K, 3)), ("surfel_screen_grad", (ns,)), ("gaussian_screen_grad", (ng,)))}
    L = _lib.lib()
    stream = C.c_void_p(torch.cuda.current_stream(dev).cuda_stream)
    cam_c = camera_struct(cam)
    if tape["gaussians"]:
        gg = _lib.GaussGrads()
        gg.pos, gg.opacity = out["gaussian_pos"].data_ptr(), out["gaussian_opacity"].data_ptr()
        gg.quat, gg.scale = out["gaussian_quat"].data_ptr(), out["gaussian_scale"].data_ptr()
        gg.sh, gg.screen = out["gaussian_sh"].data_ptr(), out["gaussian_screen_grad"].data_ptr()
        st_c = settings_struct(_pass_settings(settings))
        g_gd = _as_dev(g_gauss_depth, dev)
        g_gn = _as_dev(g_gauss_normal, dev)
        scratch = torch.empty(L.ges_backward_scratch_bytes(ng), dtype=torch.uint8, device=dev)
        ptr = lambda t: C.c_void_p(t.data_ptr()) if t is not None else None  # noqa: E731
        cap = max(1 << 20, 8 * ng)
        status = torch.zeros(3, dtype=torch.int64, device=dev)
        for _ in range(3):
            nbytes = L.ges_backward_workspace_bytes(C.byref(ds.c), C.byref(cam_c), C.byref(st_c), cap)
            if nbytes == 0:
                _lib.check(_lib.GES_EINVAL, "ges_backward_workspace_bytes")
            ws = torch.empty(nbytes, dtype=torch.uint8, device=dev)
            rc = L.ges_backward_gaussians(C.byref(ds.c), C.byref(ds.src), int(ds.any_filter), C.byref(cam_c),
                                          C.byref(st_c), ptr(tape["surfel_depth"]), ptr(g_cg), ptr(g_wg),
                                          ptr(g_gd), ptr(g_gn), C.byref(gg), ptr(scratch), scratch.numel(),
                                          ptr(ws), nbytes, cap, ptr(status), stream)
            _lib.check(rc, "gaussian backward")
            st = status.cpu()
            if not int(st[2] & 0xFFFFFFFF):
                break
            cap = max(cap, int(int(st[1]) * 1.25) + 1024)
        else:
            raise RuntimeError("tile pair lists overflowed repeatedly")
    if tape["frozen"] and tape["covered_any"]:
        col = torch.empty((ns, 3), **f64)
        _lib.check(L.ges_backward_surfels_frozen(C.byref(ds.src), C.byref(cam_c), int(tape["grid"]),
                                                 C.c_void_p(tape["winner"].data_ptr()),
                                                 C.c_void_p(g_cs.contiguous().data_ptr()),
                                                 C.c_void_p(col.data_ptr()),
                                                 C.c_void_p(out["surfel_sh"].data_ptr()),
                                                 C.c_void_p(out["surfel_pos"].data_ptr()), stream),
                   "frozen surfel backward")
    if not to_numpy:
        return GradientSet(**out)
    keys = list(out)   # pinned copies, all queued before one synchronisation (forward._host)
    return GradientSet(**dict(zip(keys, _numpy(*(_host(out[k]) for k in keys)))))


def contribution_scores(scene, cams, settings: TrainSettings | None = None, cache_keys=None, *,
                        device=None) -> np.ndarray:
    """Per-Gaussian pruning statistic of the joint stage (optim.py:519-533):
    max over views and fragments of ``max_c(colour) * alpha / (1 + W_G)``.
    ``cache_keys[i]`` is the frozen-cache key of ``cams[i]`` (the trainer
    passes the view index).  Returns float64 NumPy scores (n_gaussians,)."""
    settings = settings or TrainSettings()
    dev = torch.device(device or "cuda")
    if dev.index is None:
        dev = torch.device("cuda", torch.cuda.current_device())
    ng = _count(scene.gaussians.pos)
    if ng == 0 or not settings.gaussians_enabled:
        return np.zeros(ng)
    ds = DeviceScene(scene, dev, keep_source=True)
    L = _lib.lib()
    scores = torch.zeros(ng, dtype=torch.float32, device=dev)
    st_c = settings_struct(_pass_settings(settings, with_geometry=False))
    status = torch.zeros(3, dtype=torch.int64, device=dev)
    cap = max(1 << 20, 8 * ng)
    for i, cam in enumerate(cams):
        key = cache_keys[i] if cache_keys is not None else None
        fr = render_training(scene, cam, settings, cache_key=key, to_numpy=False, device=dev, device_scene=ds)
        cam_c = camera_struct(cam)
        stream = C.c_void_p(torch.cuda.current_stream(dev).cuda_stream)
        for _ in range(3):
            nbytes = L.ges_backward_workspace_bytes(C.byref(ds.c), C.byref(cam_c), C.byref(st_c), cap)
            ws = torch.empty(nbytes, dtype=torch.uint8, device=dev)
            trial = scores.clone()
            _lib.check(L.ges_gaussian_contributions(C.byref(ds.c), C.byref(ds.src), C.byref(cam_c), C.byref(st_c),
                                                    C.c_void_p(fr.tape["surfel_depth"].data_ptr()),
                                                    C.c_void_p(fr.gauss_weight.contiguous().data_ptr()),
                                                    C.c_void_p(trial.data_ptr()), C.c_void_p(ws.data_ptr()), nbytes,
                                                    cap, C.c_void_p(status.data_ptr()), stream),
                       "gaussian contributions")
            st = status.cpu()
            if not int(st[2] & 0xFFFFFFFF):
                scores = trial
                break
            cap = max(cap, int(int(st[1]) * 1.25) + 1024)
        else:
            raise RuntimeError("tile pair lists overflowed repeatedly")
    return scores.double().cpu().numpy()
