"""`.ges` model files -> scenes (the input step before the path).

Format (reference ``ges/gesfile.py:1-13``), little-endian:

    header  : b"GES1" | u32 version=1 | u32 sh_degree | u32 flags | u64 n_surfels | u64 n_gaussians
    surfels : n_surfels  x f32[3 pos + 4 quat(wxyz) + 2 scale + 3*K sh]   (3 rgb instead of 3*K if flags&2)
    gaussians: n_gaussians x f32[3 pos + 1 sigma + 4 quat + D scale + 1 eps + 3*K sh]  (D = 2 if flags&1 else 3)

``load_ges`` returns the same ``(scene, info)`` pair as the reference's
``load_ges`` (``gesfile.py:79-126``): float64 arrays, log scales, logit
opacity (sigma clipped to [1e-7, 1-1e-7]), frozen stage, ``info`` with the
flags and the baked epsilons.  ``load_ges_device`` parses the same file and
packs it straight into a :class:`DeviceScene`.
"""

from __future__ import annotations

import struct
from pathlib import Path

import numpy as np

from .types import GaussianKind, GaussianSet, Scene, Stage, SurfelSet, W_OPAQUE

MAGIC = b"GES1"
VERSION = 1
FLAG_GAUSSIANS_2D = 1
FLAG_RGB_SURFELS = 2
HEADER = struct.Struct("<4sIIIQQ")
SH_C0 = 0.28209479177387814


class GesFileError(RuntimeError):
    pass


def _layout(deg, flags):
    K = (deg + 1) ** 2
    rgb = bool(flags & FLAG_RGB_SURFELS)
    D = 2 if flags & FLAG_GAUSSIANS_2D else 3
    s_floats = 9 + (3 if rgb else 3 * K)
    g_floats = 9 + D + 3 * K
    return K, rgb, D, s_floats, g_floats


def load_ges(path) -> tuple[Scene, dict]:
    raw = Path(path).read_bytes()
    if len(raw) < HEADER.size:
        raise GesFileError(f"{path}: truncated header")
    magic, version, deg, flags, ns, ng = HEADER.unpack_from(raw)
    if magic != MAGIC:
        raise GesFileError(f"{path}: bad magic {magic!r}")
    if version != VERSION:
        raise GesFileError(f"{path}: unsupported version {version}")
    if deg > 3:
        raise GesFileError(f"{path}: unsupported SH degree {deg}")
    K, rgb, D, sf, gf = _layout(deg, flags)
    need = HEADER.size + 4 * (ns * sf + ng * gf)
    if len(raw) != need:
        raise GesFileError(f"{path}: size {len(raw)} != expected {need}")
    body = np.frombuffer(raw, dtype="<f4", offset=HEADER.size)
    srec = body[: ns * sf].reshape(ns, sf).astype(np.float64)
    grec = body[ns * sf:].reshape(ng, gf).astype(np.float64)
    if not (np.all(np.isfinite(srec)) and np.all(np.isfinite(grec))):
        raise GesFileError(f"{path}: non-finite values")
    if rgb:   # plain RGB surfels become a DC-only SH block
        sh_s = np.zeros((ns, K, 3))
        sh_s[:, 0, :] = (srec[:, 9:12] - 0.5) / SH_C0
    else:
        sh_s = srec[:, 9:].reshape(ns, K, 3)
    surfels = SurfelSet(pos=srec[:, 0:3], quat=srec[:, 3:7],
                        log_scale=np.log(np.maximum(srec[:, 7:9], 1e-12)), sh=sh_s,
                        w=np.full(ns, W_OPAQUE))
    sig = np.clip(grec[:, 3], 1e-7, 1 - 1e-7) if ng else grec[:, 3]
    raw_op = np.log(sig / (1.0 - sig)) if ng else grec[:, 3]
    kind = GaussianKind.TWO_D if D == 2 else GaussianKind.THREE_D
    gauss = GaussianSet(pos=grec[:, 0:3], raw_opacity=raw_op, quat=grec[:, 4:8],
                        log_scale=np.log(np.maximum(grec[:, 8:8 + D], 1e-12)),
                        sh=grec[:, 9 + D:].reshape(ng, K, 3), kind=kind)
    info = {"flags": flags, "rgb_surfels": rgb, "epsilon": grec[:, 8 + D].copy()}
    return Scene(surfels, gauss, deg, Stage.FROZEN), info


def save_ges(scene: Scene, path, *, rgb_surfels: bool = False):
    """Write a frozen scene in the same format (for fixtures and round trips;
    epsilon baked from the effective scales like ``gesfile.py:42-76``), with
    the reference's export checks: frozen stage and w = 255 on every surfel
    (``gesfile.py:44-47``), finite records (``:66-69``)."""
    if getattr(scene.stage, "value", scene.stage) != getattr(Stage.FROZEN, "value", Stage.FROZEN):
        raise GesFileError("only frozen scenes can be exported")
    s, g = scene.surfels, scene.gaussians
    if not np.all(np.asarray(s.w) == W_OPAQUE):
        raise GesFileError("export requires w = 255 on every surfel")
    deg = int(scene.sh_degree)
    K = (deg + 1) ** 2
    two_d = getattr(g.kind, "value", g.kind) == "2d"
    flags = (FLAG_GAUSSIANS_2D if two_d else 0) | (FLAG_RGB_SURFELS if rgb_surfels else 0)
    sc = np.exp(s.log_scale)
    col = (np.clip(0.5 + SH_C0 * s.sh[:, 0, :], 0.0, 1.0) if rgb_surfels
           else s.sh.reshape(s.count, 3 * K))
    srec = np.concatenate([s.pos, s.quat, sc, col], axis=1).astype("<f4")
    gs = np.exp(g.log_scale)
    f3 = np.zeros(g.count) if g.filter3d is None else np.asarray(g.filter3d)
    sig = 1.0 / (1.0 + np.exp(-g.raw_opacity))
    if np.any(f3):
        es = np.sqrt(gs * gs + f3[:, None])
        sig = sig * np.prod(gs / es, axis=1)
        gs = es
    eps = (5.0 / gs.shape[1]) * gs.sum(axis=1)
    grec = np.concatenate([g.pos, sig[:, None], g.quat, gs, eps[:, None],
                           g.sh.reshape(g.count, 3 * K)], axis=1).astype("<f4")
    if srec.size and not np.all(np.isfinite(srec)):
        raise GesFileError("non-finite surfel values")
    if grec.size and not np.all(np.isfinite(grec)):
        raise GesFileError("non-finite gaussian values")
    with open(path, "wb") as f:
        f.write(HEADER.pack(MAGIC, VERSION, deg, flags, s.count, g.count))
        f.write(srec.tobytes())
        f.write(grec.tobytes())


def load_ges_device(path, device=None):
    """Parse a .ges file and pack it on the device in one step."""
    from .renderer import DeviceScene
    scene, info = load_ges(path)
    return DeviceScene(scene, device), info
