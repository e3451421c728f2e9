"""CPU oracle for the GES forward render path -- TEST INFRASTRUCTURE ONLY.

This module is a NumPy restatement of the reference's sorting-free two-pass
renderer (``/root/reference/pkg/src/ges/forward.py`` and the helpers it calls
in ``geometry.py``, ``sh.py``, ``cameras.py``, ``filters.py``,
``primitives.py``).  It exists so the parity tests, ``__graft_entry__.smoke()``
and the ``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` have a
checker that travels to the GPU box (``/root/reference`` does not).  Nothing
in the product package imports it; the CUDA path never falls back to it.

Parity of this oracle is PINNED: ``tests/golden/*.npz`` hold outputs of the
real reference (imported read-only in the build container by
``tests/golden/make_golden.py``) and ``tests/test_oracle_golden.py`` checks
this restatement against them at atol 1e-9 in float64.

Beyond the reference's outputs this oracle can
  * evaluate only a subset of 16x16 base-resolution tiles (``tiles=``; with
    supersample=4 the surfel pass covers the same pixels), which lets the GPU
    parity tests spot-check full-size frames (config 2) in seconds;
  * report per-pixel *tie flags*: pixels whose float64 decision margin is so
    small that a float32 evaluation may legitimately decide differently
    (SURVEY.md section 8(c) parity rule).  The thresholds are ``TIE_*`` below.

Inputs are duck-typed: any object with the reference's field names works
(``scene.surfels.pos/quat/log_scale/sh``, ``scene.gaussians.pos/raw_opacity/
quat/log_scale/sh/kind/filter3d``, ``cam.fx/fy/cx/cy/width/height/
world_to_camera``; settings with the ``RenderSettings`` fields).
"""

from __future__ import annotations

import math
import os
import time
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass

import numpy as np

# --- constants (reference file:line) --------------------------------------
R_OPAQUE = math.sqrt(2.0 * math.log(255.0))   # filters.py:28-30
ALPHA_CUTOFF = 1.0 / 255.0                    # forward.py:26
TILE = 16                                     # forward.py:27
NEAR = 0.01                                   # cameras.py:14
PARALLEL_EPS = 1e-8                           # geometry.py:15
SCREEN_VAR = 0.3                              # filters.py:21

# SH constants (sh.py:15-21), graphics sign convention.
_C0 = 0.28209479177387814
_C1 = 0.4886025119029199
_C2 = (1.0925484305920792, -1.0925484305920792, 0.31539156525252005,
       -1.0925484305920792, 0.5462742152960396)
_C3 = (-0.5900435899266435, 2.890611442640554, -0.4570457994644658,
       0.3731763325901154, -0.4570457994644658, 1.445305721320277,
       -0.5900435899266435)

# Tie-case thresholds for the parity rule.
TIE_DEPTH_REL = 1e-5        # competing hit depths within this relative gap
TIE_RADIUS_REL = 1e-4       # |u^2+v^2 - R^2| < TIE_RADIUS_REL * R^2
TIE_PARALLEL = 10.0         # |n.d| within 10x the parallel threshold
TIE_NEAR_ABS = 1e-6         # |t - 0.01| below this
TIE_ALPHA = 1e-3            # |255 alpha - 1| below this
TIE_GATE_REL = 1e-5         # |d - (D_s + eps)| < TIE_GATE_REL * |D_s + eps|
# Conditioning-aware float32 error model for ray-plane hits.  At grazing
# incidence the hit depth t = n.q / n.d and the disc coordinates (u, v) are
# ill-conditioned in the ray direction d (condition ~ |d| / |n.d|), so a float32
# evaluation (whose ray and plane coefficients carry ~EPS32 relative rounding)
# can move r^2 = u^2 + v^2 and t far more than the fixed relative thresholds
# above.  A decision is also a tie when its float64 margin lies within
# TIE_F32_K first-order float32 error bounds:
#   err(t)   = K * EPS32 * t * (|d| / |n.d| + 2)
#   err(r^2) = K * EPS32 * |d| * (2 (|u| |c_u| + |v| |c_v|) + 2 r^2) / |n.d|
# with c_u = (a1 (n.q) - n (a1.q)) / s1 (so that u = c_u.d / n.d), c_v alike.
EPS32 = 2.0 ** -24
TIE_F32_K = 4.0


def _is_2d(kind) -> bool:
    return getattr(kind, "value", kind) in ("2d", 2, "TWO_D")


# --- camera helpers (cameras.py:17-80) -------------------------------------
@dataclass
class Cam:
    fx: float
    fy: float
    cx: float
    cy: float
    width: int
    height: int
    R: np.ndarray      # 3x3 world->camera rotation
    t: np.ndarray      # translation

    @property
    def position(self):              # cameras.py:38
        return -self.R.T @ self.t

    def to_camera(self, p):          # cameras.py:48-50
        return p @ self.R.T + self.t

    def scaled(self, k):             # cameras.py:75-80
        return Cam(self.fx * k, self.fy * k, self.cx * k, self.cy * k,
                   self.width * k, self.height * k, self.R, self.t)

    def rays(self):
        """Pixel-centre ray directions with z = 1, float64 (cameras.py:59-73)."""
        xs = (np.arange(self.width, dtype=np.float64) + 0.5 - self.cx) / self.fx
        ys = (np.arange(self.height, dtype=np.float64) + 0.5 - self.cy) / self.fy
        d = np.ones((self.height, self.width, 3))
        d[..., 0] = xs[None, :]
        d[..., 1] = ys[:, None]
        return d


def as_cam(cam) -> Cam:
    m = np.asarray(cam.world_to_camera, dtype=np.float64)
    return Cam(float(cam.fx), float(cam.fy), float(cam.cx), float(cam.cy),
               int(cam.width), int(cam.height), m[:3, :3].copy(), m[:3, 3].copy())


# --- math helpers -----------------------------------------------------------
def rotmats(quat):
    """Normalised (w,x,y,z) -> (N,3,3) (geometry.py:18-36)."""
    q = np.atleast_2d(np.asarray(quat, dtype=np.float64))
    q = q / np.linalg.norm(q, axis=-1, keepdims=True)
    w, x, y, z = q.T
    return np.stack([
        np.stack([1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)], -1),
        np.stack([2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)], -1),
        np.stack([2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)], -1),
    ], axis=1)


def sh_colors(sh, dirs):
    """clip(0.5 + sum_k Y_k(dir) c_k, 0, 1) (sh.py:34-64, :117-133)."""
    sh = np.asarray(sh, dtype=np.float64)
    K = sh.shape[1]
    deg = int(round(math.sqrt(K))) - 1
    if (deg + 1) ** 2 != K:
        raise ValueError(f"coefficient count {K} is not a square")
    if deg > 3:
        raise ValueError(f"SH degree must be in [0, 3], got {deg}")
    x, y, z = dirs[:, 0], dirs[:, 1], dirs[:, 2]
    basis = [np.full_like(x, _C0)]
    if deg >= 1:
        basis += [-_C1 * y, _C1 * z, -_C1 * x]
    if deg >= 2:
        xx, yy, zz = x * x, y * y, z * z
        basis += [_C2[0] * x * y, _C2[1] * y * z, _C2[2] * (2.0 * zz - xx - yy),
                  _C2[3] * x * z, _C2[4] * (xx - yy)]
    if deg >= 3:
        basis += [_C3[0] * y * (3.0 * xx - yy), _C3[1] * x * y * z,
                  _C3[2] * y * (4.0 * zz - xx - yy),
                  _C3[3] * z * (2.0 * zz - 3.0 * xx - 3.0 * yy),
                  _C3[4] * x * (4.0 * zz - xx - yy), _C3[5] * z * (xx - yy),
                  _C3[6] * x * (xx - 3.0 * yy)]
    B = np.stack(basis, axis=1)                      # (N, K)
    return np.clip(0.5 + np.einsum("nk,nkc->nc", B, sh), 0.0, 1.0)


def view_colors(pos, sh, cam: Cam):
    """Per-primitive view colour, centre-to-camera dir (forward.py:99-109)."""
    pos = np.asarray(pos, dtype=np.float64)
    d = cam.position[None, :] - pos
    d = d / np.maximum(np.linalg.norm(d, axis=1, keepdims=True), 1e-12)
    return sh_colors(sh, d)


def frames(pos, quat, cam: Cam):
    """Camera-space centre and local frame (geometry.py:193-205)."""
    Rm = rotmats(quat)
    q = cam.to_camera(np.atleast_2d(np.asarray(pos, dtype=np.float64)))
    a1 = Rm[:, :, 0] @ cam.R.T
    a2 = Rm[:, :, 1] @ cam.R.T
    n = Rm[:, :, 2] @ cam.R.T
    return q, a1, a2, n


def disc_bounds(q, a1, a2, s1r, s2r, cam: Cam):
    """Screen AABB of the projected disc via the tangent quadratic
    (geometry.py:273-302).  s1r, s2r are the local half-axes (scale*radius).
    Returns (xmin, xmax, ymin, ymax) and the whole-screen mask."""
    m1 = a1 * s1r[:, None]
    m2 = a2 * s2r[:, None]
    bz = (m1[:, 2], m2[:, 2], q[:, 2])
    c2 = bz[2] ** 2 - (bz[0] ** 2 + bz[1] ** 2)
    whole = c2 <= 0
    c2s = np.where(whole, 1.0, c2)
    out = []
    for ax, (f, c) in enumerate(((cam.fx, cam.cx), (cam.fy, cam.cy))):
        A0 = f * m1[:, ax] + c * m1[:, 2]
        A1 = f * m2[:, ax] + c * m2[:, 2]
        A2 = f * q[:, ax] + c * q[:, 2]
        c1 = -2.0 * (A2 * bz[2] - (A0 * bz[0] + A1 * bz[1]))
        c0 = A2 ** 2 - (A0 ** 2 + A1 ** 2)
        root = np.sqrt(np.maximum(c1 * c1 - 4.0 * c2s * c0, 0.0))
        out += [(-c1 - root) / (2.0 * c2s), (-c1 + root) / (2.0 * c2s)]
    return np.stack(out, axis=1), whole


def pixel_ranges(bounds, whole, width, height):
    """Inclusive pixel ranges with 0.5 px padding (forward.py:85-96)."""
    def span(n, b_lo, b_hi):
        a = np.where(whole, 0.0, np.ceil(b_lo - 0.5 - 0.5))   # pad 0.5, centres at +0.5
        b = np.where(whole, n - 1.0, np.floor(b_hi + 0.5 - 0.5))
        return (np.clip(a, 0, n - 1).astype(np.int64),
                np.clip(b, 0, n - 1).astype(np.int64))
    x0, x1 = span(width, bounds[:, 0], bounds[:, 1])
    y0, y1 = span(height, bounds[:, 2], bounds[:, 3])
    return x0, x1, y0, y1


def tile_list(height, width):
    return [(y, min(y + TILE, height), x, min(x + TILE, width))
            for y in range(0, height, TILE) for x in range(0, width, TILE)]


def _select(idx, x0, x1, y0, y1, t):
    """The reference's per-tile selection (forward.py:168-169, :294-295):
    alive primitives whose pixel range overlaps the tile, ascending index."""
    ty0, ty1, tx0, tx1 = t
    return idx[(x0[idx] <= tx1 - 1) & (x1[idx] >= tx0)
               & (y0[idx] <= ty1 - 1) & (y1[idx] >= ty0)]


# Above this many (primitive x tile) range tests per frame the selection is
# done through per-tile index lists built once per frame (same lists, same
# ascending order, so results are identical; the O(N x tiles) scan of the
# reference is kept for the timed CPU baseline, see FAST_SELECT).
FAST_SELECT = [True]
_FAST_MIN = 1 << 24


class _Selector:
    """Per-tile candidate lists, identical to ``_select`` for every tile: the
    (tile, primitive) pairs are generated in ascending primitive order and
    grouped by a stable sort on the tile key."""

    def __init__(self, idx, x0, x1, y0, y1, height, width):
        self.args = (idx, x0, x1, y0, y1)
        self.ntx = (width + TILE - 1) // TILE
        nt = self.ntx * ((height + TILE - 1) // TILE)
        self.lists = None
        if not FAST_SELECT[0] or idx.size * nt < _FAST_MIN:
            return
        a0, a1 = x0[idx] // TILE, x1[idx] // TILE
        b0, b1 = y0[idx] // TILE, y1[idx] // TILE
        nx, ny = a1 - a0 + 1, b1 - b0 + 1
        cnt = nx * ny
        rep = np.repeat(np.arange(idx.size), cnt)
        k = np.arange(rep.size) - np.repeat(np.cumsum(cnt) - cnt, cnt)
        tile = (b0[rep] + k // nx[rep]) * self.ntx + a0[rep] + k % nx[rep]
        order = np.argsort(tile, kind="stable")
        self.ids = idx[rep[order]]
        self.start = np.searchsorted(tile[order], np.arange(nt + 1))
        self.lists = True

    def __call__(self, t):
        if self.lists is None:
            return _select(*self.args, t)
        ti = (t[0] // TILE) * self.ntx + t[2] // TILE
        return self.ids[self.start[ti]:self.start[ti + 1]]


# Seconds spent inside per-tile loops since the last reset (lets the CPU
# baseline separate per-frame preprocessing from per-tile work).
TILE_SECONDS = [0.0]


def _run(fn, tiles, threads):
    t0 = time.perf_counter()
    if threads <= 1:
        for t in tiles:
            fn(t)
    else:
        with ThreadPoolExecutor(max_workers=threads) as ex:
            list(ex.map(fn, tiles))
    TILE_SECONDS[0] += time.perf_counter() - t0


def _hires_tiles(tiles, base, grid):
    """Base-resolution tile indices -> the hi-res (grid x grid) tiles covering
    the same pixels, for the supersampled surfel pass."""
    if tiles is None or grid == 1:
        return tiles
    ntx = (base.width + TILE - 1) // TILE
    ntx_hi = (base.width * grid + TILE - 1) // TILE
    nty_hi = (base.height * grid + TILE - 1) // TILE
    out = []
    for t in tiles:
        by, bx = divmod(t, ntx)
        for dy in range(grid):
            for dx in range(grid):
                hy, hx = by * grid + dy, bx * grid + dx
                if hy < nty_hi and hx < ntx_hi:
                    out.append(hy * ntx_hi + hx)
    return out


def _tiles_for(height, width, tiles):
    allt = tile_list(height, width)
    if tiles is None:
        return allt
    return [allt[i] for i in tiles]


# --- output containers (forward.py:61-82) -----------------------------------
@dataclass
class SurfelOut:
    color: np.ndarray
    depth: np.ndarray
    normal: np.ndarray
    coverage: np.ndarray
    winner: np.ndarray
    tie: np.ndarray = None      # (H, W) bool, oracle extension
    depth_err: np.ndarray = None  # (H, W) float32 error bound of the winner's depth (TIE_F32_K model)
    tie_sub: np.ndarray = None    # (H, W) bool, supersample=4: a tie at sub-samples (0,1), (1,0) or
                                  # (1,1) only -- winner/depth come from sub-sample (0,0), so only
                                  # the box-mean colour may legitimately differ


@dataclass
class GaussOut:
    color: np.ndarray
    weight: np.ndarray
    depth: np.ndarray = None
    normal: np.ndarray = None
    tie: np.ndarray = None       # (H, W) bool: a depth-gate decision within TIE_GATE_REL
    tie_cut: np.ndarray = None   # (H, W) int: fragments within TIE_ALPHA of the 1/255 cutoff


@dataclass
class RenderOut:
    image: np.ndarray
    surfels: SurfelOut
    gaussians: GaussOut

    @property
    def tie(self):
        """Pixels whose result a float32 evaluation may legitimately change
        by more than one near-cutoff fragment: surfel winner/coverage ties and
        finite depth-gate ties.  These are excluded from the parity checks
        (and counted)."""
        t = self.surfels.tie
        if self.gaussians.tie is not None:
            t = t | self.gaussians.tie
        return t

    @property
    def tie_color(self):
        """supersample=4: pixels whose box-mean colour (only) may differ
        because a sub-sample other than (0, 0) is a surfel tie.  Their winner,
        depth and Gaussian sums are still checked; image and surfel colour
        are excluded (and counted)."""
        if self.surfels.tie_sub is None:
            return np.zeros(self.surfels.tie.shape, bool)
        return self.surfels.tie_sub & ~self.tie

    @property
    def tie_cut(self):
        """Per pixel, the number of contributing Gaussian fragments whose
        alpha lies within TIE_ALPHA of the 1/255 cutoff: a float32 evaluation
        may drop or add each of them, which moves the pixel by at most
        ~1/255 per fragment.  Checked against that bound, not excluded."""
        if self.gaussians.tie_cut is None:
            return np.zeros(self.surfels.tie.shape, np.int32)
        return self.gaussians.tie_cut


def _settings(settings):
    g = lambda k, d: getattr(settings, k, d) if settings is not None else d
    return dict(supersample=g("supersample", 1), background=g("background", (0.0, 0.0, 0.0)),
                layers=g("layers", "full"), mip=g("mip", False),
                epsilon_mode=g("epsilon_mode", "adaptive"),
                epsilon_value=g("epsilon_value", 0.0), dtype=g("dtype", np.float64),
                threads=g("threads", 1) or 1, with_geometry=g("with_geometry", False))


# --- pass 1: surfel z-buffer (forward.py:127-209) --------------------------
def rasterize_surfels(scene, cam, settings=None, *, tiles=None, ties=False) -> SurfelOut:
    run, finish, _ = _surfel_job(scene, cam, settings, ties)
    run(tiles)
    return finish()


def _surfel_job(scene, cam, settings, ties):
    """The surfel pass split at its tile loop: the per-frame preprocessing
    (forward.py:148-158) runs here; returns ``run(tiles)`` (the per-tile
    z-buffer of the given base-resolution tiles, forward.py:166-207),
    ``finish()`` (the supersample reduction, forward.py:201-207 -> SurfelOut)
    and the base-resolution depth map view the Gaussian pass gates against."""
    st = _settings(settings)
    dt = st["dtype"]
    grid = 2 if st["supersample"] == 4 else 1
    base = as_cam(cam)
    rc = base.scaled(grid) if grid > 1 else base
    H, W = rc.height, rc.width
    bg = np.asarray(st["background"], dtype=dt)
    color = np.empty((H, W, 3), dtype=dt)
    color[:] = bg
    depth = np.full((H, W), np.inf, dtype=dt)
    normal = np.zeros((H, W, 3), dtype=dt)
    winner = np.full((H, W), -1, dtype=np.int32)
    tie = np.zeros((H, W), dtype=bool)
    derr = np.zeros((H, W), dtype=np.float64)

    s = scene.surfels
    ns = int(np.asarray(s.pos).shape[0])
    if ns:
        q, a1, a2, n = frames(s.pos, s.quat, rc)
        scale = np.exp(np.asarray(s.log_scale, dtype=np.float64))
        cols = view_colors(s.pos, s.sh, rc).astype(dt)
        n_vis = np.where(np.sum(n * q, axis=1, keepdims=True) < 0, n, -n).astype(dt)
        bounds, whole = disc_bounds(q, a1, a2, scale[:, 0] * R_OPAQUE,
                                    scale[:, 1] * R_OPAQUE, rc)
        x0, x1, y0, y1 = pixel_ranges(bounds, whole, W, H)
        alive = (q[:, 2] > NEAR) & (x1 >= x0) & (y1 >= y0)
        idx = np.flatnonzero(alive)
        rays = rc.rays().astype(dt)
        rnorm = np.linalg.norm(rays, axis=-1)
        qd, a1d, a2d, nd_ = (v.astype(dt) for v in (q, a1, a2, n))
        s1 = scale[:, 0].astype(dt)
        s2 = scale[:, 1].astype(dt)
        nq_all = np.sum(nd_ * qd, axis=1)
        a1q_all = np.sum(a1d * qd, axis=1)
        a2q_all = np.sum(a2d * qd, axis=1)
        R2 = R_OPAQUE * R_OPAQUE
        cu_n = np.linalg.norm(a1 * np.sum(n * q, axis=1, keepdims=True)
                              - n * np.sum(a1 * q, axis=1, keepdims=True), axis=1) / scale[:, 0]
        cv_n = np.linalg.norm(a2 * np.sum(n * q, axis=1, keepdims=True)
                              - n * np.sum(a2 * q, axis=1, keepdims=True), axis=1) / scale[:, 1]
        select = _Selector(idx, x0, x1, y0, y1, H, W)

        def do_tile(t):
            ty0, ty1, tx0, tx1 = t
            sel = select(t)
            if sel.size == 0:
                return
            d = rays[ty0:ty1, tx0:tx1].reshape(-1, 3)
            dn = rnorm[ty0:ty1, tx0:tx1].reshape(1, -1)
            with np.errstate(divide="ignore", invalid="ignore", over="ignore"):
                ndot = nd_[sel] @ d.T
                th = nq_all[sel][:, None] / ndot
                u = (th * (a1d[sel] @ d.T) - a1q_all[sel][:, None]) / s1[sel][:, None]
                v = (th * (a2d[sel] @ d.T) - a2q_all[sel][:, None]) / s2[sel][:, None]
                r2 = u * u + v * v
                ok = (np.abs(ndot) > PARALLEL_EPS * dn) & (th > NEAR) & (r2 <= R2)
            dm = np.where(ok, th, np.inf).astype(dt)
            k = np.argmin(dm, axis=0)                       # first index on ties
            cols_px = np.arange(dm.shape[1])
            best = dm[k, cols_px]
            cov = np.isfinite(best)
            shp = (ty1 - ty0, tx1 - tx0)
            depth[ty0:ty1, tx0:tx1] = best.reshape(shp)
            winner[ty0:ty1, tx0:tx1] = np.where(cov, sel[k], -1).astype(np.int32).reshape(shp)
            color[ty0:ty1, tx0:tx1] = np.where(cov[:, None], cols[sel[k]], bg).reshape(shp + (3,))
            normal[ty0:ty1, tx0:tx1] = np.where(cov[:, None], n_vis[sel[k]], 0.0).reshape(shp + (3,))
            if ties:
                with np.errstate(invalid="ignore", over="ignore", divide="ignore"):
                    andot = np.abs(ndot)
                    f32 = TIE_F32_K * EPS32
                    terr = f32 * np.abs(th) * (dn / andot + 2.0)          # err(t)
                    rerr = f32 * dn * (2.0 * (np.abs(u) * cu_n[sel][:, None] + np.abs(v) * cv_n[sel][:, None])
                                       + 2.0 * r2) / andot             # err(r^2)
                    berr = np.where(cov, terr[k, cols_px], 0.0)
                    lim = np.where(cov, best * (1.0 + TIE_DEPTH_REL) + berr, np.inf)
                    lo = th - terr
                    lo[k, cols_px] = np.inf
                    close = cov & (np.where(ok, lo, np.inf).min(axis=0) <= lim)
                    fragile = ((np.abs(r2 - R2) < np.maximum(TIE_RADIUS_REL * R2, rerr))
                               | (andot < TIE_PARALLEL * PARALLEL_EPS * dn)
                               | (np.abs(th - NEAR) < np.maximum(TIE_NEAR_ABS, terr)))
                    front = (th + terr > NEAR - TIE_NEAR_ABS) & (lo <= lim[None, :])
                    front[k, cols_px] |= cov
                    near_par = andot < TIE_PARALLEL * PARALLEL_EPS * dn
                    flag = close | np.any(fragile & (front | near_par), axis=0)
                tie[ty0:ty1, tx0:tx1] = flag.reshape(shp)
                derr[ty0:ty1, tx0:tx1] = berr.reshape(shp)

    def run(tiles):
        if ns:
            _run(do_tile, _tiles_for(H, W, _hires_tiles(tiles, base, grid)), st["threads"])

    def finish():
        if grid == 1:
            return SurfelOut(color, depth, normal, np.isfinite(depth), winner, tie, derr,
                             np.zeros(tie.shape, bool))
        h, w = base.height, base.width
        tie_any = tie.reshape(h, grid, w, grid).any(axis=(1, 3))
        t0 = tie[0::grid, 0::grid]           # the reported sub-sample (forward.py:205-207)
        d0 = depth[0::grid, 0::grid]
        return SurfelOut(color.reshape(h, grid, w, grid, 3).mean(axis=(1, 3), dtype=dt), d0,
                         normal[0::grid, 0::grid], np.isfinite(d0), winner[0::grid, 0::grid], t0,
                         derr[0::grid, 0::grid], tie_any & ~t0)   # tie_sub: only the box-mean colour

    return run, finish, (depth[0::grid, 0::grid], derr[0::grid, 0::grid])


def surfel_tile_counts(scene, cam):
    """Per 16x16 tile (ss = 1), the number of alive surfels whose pixel range
    overlaps it -- the length of the reference's per-tile candidate list
    (forward.py:168-169).  Used to pick the densest tiles for sampled parity."""
    c = as_cam(cam)
    s = scene.surfels
    q, a1, a2, n = frames(s.pos, s.quat, c)
    scale = np.exp(np.asarray(s.log_scale, dtype=np.float64))
    bounds, whole = disc_bounds(q, a1, a2, scale[:, 0] * R_OPAQUE, scale[:, 1] * R_OPAQUE, c)
    x0, x1, y0, y1 = pixel_ranges(bounds, whole, c.width, c.height)
    idx = np.flatnonzero((q[:, 2] > NEAR) & (x1 >= x0) & (y1 >= y0))
    sel = _Selector(idx, x0, x1, y0, y1, c.height, c.width) if idx.size else None
    ntx = (c.width + TILE - 1) // TILE
    nt = ntx * ((c.height + TILE - 1) // TILE)
    if sel is None:
        return np.zeros(nt, np.int64)
    if sel.lists is None:
        return np.array([sel(t).size for t in tile_list(c.height, c.width)], np.int64)
    return np.diff(sel.start)


# --- pass 2: order-independent Gaussian accumulation (forward.py:212-381) ---
def gaussian_eff(g):
    """eff_scale, eff_opacity, adaptive epsilon (primitives.py:113-131)."""
    s = np.exp(np.asarray(g.log_scale, dtype=np.float64))
    sig = 1.0 / (1.0 + np.exp(-np.asarray(g.raw_opacity, dtype=np.float64)))
    f3 = getattr(g, "filter3d", None)
    f3 = np.zeros(s.shape[0]) if f3 is None else np.asarray(f3, dtype=np.float64)
    if np.any(f3):
        es = np.sqrt(s * s + f3[:, None])
        sig = sig * np.prod(s / es, axis=1)
    else:
        es = s
    eps = (5.0 / es.shape[1]) * np.sum(es, axis=1)
    return es, sig, eps


def project_ewa(pos, quat, scale, cam: Cam):
    """EWA projection (geometry.py:93-132): mean2d, cov2d, depth, valid."""
    t = cam.to_camera(np.atleast_2d(np.asarray(pos, dtype=np.float64)))
    z = t[:, 2]
    valid = z > NEAR
    ts = np.where(valid[:, None], t, np.array([0.0, 0.0, 1.0]))
    Rm = rotmats(quat)
    V = np.einsum("nij,nj,nkj->nik", Rm, scale ** 2, Rm)
    M = np.einsum("ij,njk,lk->nil", cam.R, V, cam.R)
    iz = 1.0 / ts[:, 2]
    J = np.zeros((t.shape[0], 2, 3))
    J[:, 0, 0] = cam.fx * iz
    J[:, 0, 2] = -cam.fx * ts[:, 0] * iz * iz
    J[:, 1, 1] = cam.fy * iz
    J[:, 1, 2] = -cam.fy * ts[:, 1] * iz * iz
    cov = np.einsum("nij,njk,nlk->nil", J, M, J)
    mean = np.stack([cam.fx * ts[:, 0] / ts[:, 2] + cam.cx,
                     cam.fy * ts[:, 1] / ts[:, 2] + cam.cy], axis=1)
    return mean, cov, z, valid


def object_filter_2d(q, a1, a2, scale, cam: Cam, r=SCREEN_VAR):
    """Screen low-pass back-projected into the disc frame (filters.py:84-109,
    geometry.py:305-319).  Returns (scale_mul (N,2), opacity_mul, valid)."""
    z = q[:, 2]
    J = np.empty((q.shape[0], 2, 2))
    for ax, f in enumerate((cam.fx, cam.fy)):
        m1 = a1 * scale[:, 0:1]
        m2 = a2 * scale[:, 1:2]
        J[:, ax, 0] = f * (m1[:, ax] * z - q[:, ax] * m1[:, 2]) / (z * z)
        J[:, ax, 1] = f * (m2[:, ax] * z - q[:, ax] * m2[:, 2]) / (z * z)
    det = J[:, 0, 0] * J[:, 1, 1] - J[:, 0, 1] * J[:, 1, 0]
    valid = (np.abs(det) > 1e-12) & (z > NEAR)
    dets = np.where(valid, det, 1.0)
    i00 = J[:, 1, 1] / dets
    i01 = -J[:, 0, 1] / dets
    i10 = -J[:, 1, 0] / dets
    i11 = J[:, 0, 0] / dets
    smul = np.sqrt(np.stack([1.0 + r * (i00 ** 2 + i01 ** 2),
                             1.0 + r * (i10 ** 2 + i11 ** 2)], axis=1))
    return smul, 1.0 / (smul[:, 0] * smul[:, 1]), valid


def accumulate_gaussians(scene, cam, surfel_depth, settings=None, *, tiles=None,
                         ties=False, depth_err=None) -> GaussOut:
    run, out = _gauss_job(scene, cam, surfel_depth, settings, ties, depth_err)
    run(tiles)
    return out


def _gauss_job(scene, cam, surfel_depth, settings, ties, depth_err=None):
    """The Gaussian pass split at its tile loop: per-frame preprocessing
    (projection, bounds, colours; forward.py:212-300) here; returns
    ``run(tiles)`` and the GaussOut it fills.  ``surfel_depth`` is read per
    tile when the tile runs (the same array may still be filling)."""
    st = _settings(settings)
    dt = st["dtype"]
    c = as_cam(cam)
    H, W = c.height, c.width
    out = GaussOut(np.zeros((H, W, 3), dtype=dt), np.zeros((H, W), dtype=dt))
    if st["with_geometry"]:
        out.depth = np.zeros((H, W), dtype=dt)
        out.normal = np.zeros((H, W, 3), dtype=dt)
    out.tie = np.zeros((H, W), dtype=bool)
    out.tie_cut = np.zeros((H, W), dtype=np.int32)
    g = scene.gaussians
    ng = int(np.asarray(g.pos).shape[0])
    if ng == 0:
        return (lambda tiles: None), out
    ds = surfel_depth if surfel_depth.dtype == dt else np.asarray(surfel_depth, dtype=dt)
    st["depth_err"] = np.zeros(ds.shape) if depth_err is None else np.asarray(depth_err)
    es, sigma, eps = gaussian_eff(g)
    if st["epsilon_mode"] == "constant":          # forward.py:212-215
        eps = np.full(ng, float(st["epsilon_value"]))
    eps = eps.astype(dt)
    cols = view_colors(g.pos, g.sh, c).astype(dt)
    acc = _acc_2d if _is_2d(g.kind) else _acc_3d
    return acc(g, c, ds, eps, cols, es, sigma, st, out, ties), out


def _near_gate(d, thr, err=0.0):
    """Gate decision d < D_s + eps within TIE_GATE_REL (plus the float32
    error bounds ``err`` of D_s and of d) of flipping.  An uncovered pixel has
    thr = +inf: its gate always passes (forward.py:310) and is
    never a tie."""
    return np.isfinite(thr) & (np.abs(d - thr) < TIE_GATE_REL * np.abs(thr) + err)


def _acc_3d(g, cam, ds, eps, cols, es, sigma, st, out, ties):
    """forward.py:248-321."""
    dt = st["dtype"]
    H, W = cam.height, cam.width
    ng = es.shape[0]
    mean, cov, z, valid = project_ewa(g.pos, g.quat, es, cam)
    raw_det = cov[:, 0, 0] * cov[:, 1, 1] - cov[:, 0, 1] ** 2
    c00 = cov[:, 0, 0] + SCREEN_VAR
    c11 = cov[:, 1, 1] + SCREEN_VAR
    c01 = cov[:, 0, 1]
    det = c00 * c11 - c01 ** 2
    sig = sigma
    with np.errstate(divide="ignore", invalid="ignore"):
        if st["mip"]:
            sig = sig * np.sqrt(np.maximum(raw_det, 0.0) / det)
        valid = valid & (det > 0)
        la, lb, lc = c11 / det, -c01 / det, c00 / det
        m2max = 2.0 * np.log(np.maximum(255.0 * sig, 1e-12))
        valid &= m2max > 0
        rx = np.sqrt(np.maximum(m2max * c00, 0.0))
        ry = np.sqrt(np.maximum(m2max * c11, 0.0))
    bounds = np.stack([mean[:, 0] - rx, mean[:, 0] + rx, mean[:, 1] - ry, mean[:, 1] + ry], 1)
    x0, x1, y0, y1 = pixel_ranges(bounds, np.zeros(ng, bool), W, H)
    valid &= (x1 >= x0) & (y1 >= y0)
    idx = np.flatnonzero(valid)

    nrm = None
    if st["with_geometry"]:                      # forward.py:277-284
        Rm = rotmats(g.quat)
        k = np.argmin(es, axis=1)
        nv = Rm[np.arange(ng), :, k] @ cam.R.T
        tc = cam.to_camera(np.asarray(g.pos, dtype=np.float64))
        nrm = np.where(np.sum(nv * tc, axis=1, keepdims=True) < 0, nv, -nv).astype(dt)

    mx, my = mean[:, 0].astype(dt), mean[:, 1].astype(dt)
    la, lb, lc = la.astype(dt), lb.astype(dt), lc.astype(dt)
    sg, dep = sig.astype(dt), z.astype(dt)
    xs = (np.arange(W) + 0.5).astype(dt)
    ys = (np.arange(H) + 0.5).astype(dt)

    select = _Selector(idx, x0, x1, y0, y1, H, W)

    def do_tile(t):
        ty0, ty1, tx0, tx1 = t
        sel = select(t)
        if sel.size == 0:
            return
        sel = sel[np.lexsort((sg[sel], my[sel], mx[sel], dep[sel]))]   # forward.py:298-300
        dx = xs[tx0:tx1][None, None, :] - mx[sel][:, None, None]
        dy = ys[ty0:ty1][None, :, None] - my[sel][:, None, None]
        pw = -0.5 * (la[sel][:, None, None] * dx * dx + lc[sel][:, None, None] * dy * dy) \
            - lb[sel][:, None, None] * dx * dy
        a = sg[sel][:, None, None] * np.exp(pw)
        keep = a >= ALPHA_CUTOFF
        thr = ds[ty0:ty1, tx0:tx1][None] + eps[sel][:, None, None]
        gate = dep[sel][:, None, None] < thr
        a = np.where(keep & gate, a, 0.0)
        M = sel.size
        th, tw = ty1 - ty0, tx1 - tx0
        am = a.reshape(M, -1)
        out.weight[ty0:ty1, tx0:tx1] += am.sum(axis=0).reshape(th, tw)
        out.color[ty0:ty1, tx0:tx1] += (am.T @ cols[sel]).reshape(th, tw, 3)
        if nrm is not None:
            out.depth[ty0:ty1, tx0:tx1] += (am * dep[sel][:, None]).sum(axis=0).reshape(th, tw)
            out.normal[ty0:ty1, tx0:tx1] += (am.T @ nrm[sel]).reshape(th, tw, 3)
        if ties:
            with np.errstate(invalid="ignore"):
                raw = sg[sel][:, None, None] * np.exp(pw)
                near_cut = np.abs(255.0 * raw - 1.0) < TIE_ALPHA
                near_gate = _near_gate(dep[sel][:, None, None], thr, st["depth_err"][ty0:ty1, tx0:tx1][None])
            hard = near_gate & keep
            out.tie[ty0:ty1, tx0:tx1] |= hard.any(axis=0)
            out.tie_cut[ty0:ty1, tx0:tx1] += (near_cut & (gate | near_gate) & ~hard).sum(axis=0)

    return lambda tiles: _run(do_tile, _tiles_for(H, W, tiles), st["threads"])


def _acc_2d(g, cam, ds, eps, cols, es, sigma, st, out, ties):
    """Planar Gaussians (forward.py:324-381)."""
    dt = st["dtype"]
    H, W = cam.height, cam.width
    q, a1, a2, n = frames(g.pos, g.quat, cam)
    scale, sig = es, sigma
    if st["mip"]:
        smul, omul, fvalid = object_filter_2d(q, a1, a2, es, cam)
        scale = scale * smul
        sig = sig * omul
    else:
        fvalid = np.ones(scale.shape[0], bool)
    n_vis = np.where(np.sum(n * q, axis=1, keepdims=True) < 0, n, -n).astype(dt)
    m2max = 2.0 * np.log(np.maximum(255.0 * sig, 1e-12))
    valid = fvalid & (q[:, 2] > NEAR) & (m2max > 0)
    rmax = np.sqrt(np.maximum(m2max, 0.0))
    bounds, whole = disc_bounds(q, a1, a2, scale[:, 0] * rmax, scale[:, 1] * rmax, cam)
    x0, x1, y0, y1 = pixel_ranges(bounds, whole, W, H)
    valid &= (x1 >= x0) & (y1 >= y0)
    idx = np.flatnonzero(valid)

    rays = cam.rays().astype(dt)
    rnorm = np.linalg.norm(rays, axis=-1)
    depc = q[:, 2].astype(dt)
    qd, a1d, a2d, nd_ = (v.astype(dt) for v in (q, a1, a2, n))
    s1, s2 = scale[:, 0].astype(dt), scale[:, 1].astype(dt)
    sg = sig.astype(dt)
    nq = np.sum(n * q, axis=1, keepdims=True)
    cu_n = np.linalg.norm(a1 * nq - n * np.sum(a1 * q, axis=1, keepdims=True), axis=1) / scale[:, 0]
    cv_n = np.linalg.norm(a2 * nq - n * np.sum(a2 * q, axis=1, keepdims=True), axis=1) / scale[:, 1]

    select = _Selector(idx, x0, x1, y0, y1, H, W)

    def do_tile(t):
        ty0, ty1, tx0, tx1 = t
        sel = select(t)
        if sel.size == 0:
            return
        sel = sel[np.lexsort((sg[sel], qd[sel, 1], qd[sel, 0], depc[sel]))]
        d = rays[ty0:ty1, tx0:tx1].reshape(-1, 3)
        dn = rnorm[ty0:ty1, tx0:tx1].reshape(1, -1)
        with np.errstate(divide="ignore", invalid="ignore", over="ignore"):
            ndot = nd_[sel] @ d.T
            th = np.sum(nd_[sel] * qd[sel], axis=1)[:, None] / ndot
            u = (th * (a1d[sel] @ d.T) - np.sum(a1d[sel] * qd[sel], axis=1)[:, None]) / s1[sel][:, None]
            v = (th * (a2d[sel] @ d.T) - np.sum(a2d[sel] * qd[sel], axis=1)[:, None]) / s2[sel][:, None]
            ok = (np.abs(ndot) > PARALLEL_EPS * dn) & (th > NEAR)
            raw = sg[sel][:, None] * np.exp(np.where(ok, -0.5 * (u * u + v * v), -np.inf))
            keep = raw >= ALPHA_CUTOFF
            thr = ds[ty0:ty1, tx0:tx1].reshape(1, -1) + eps[sel][:, None]
            gate = th < thr
            a = np.where(keep & gate, raw, 0.0)
        th_, tw_ = ty1 - ty0, tx1 - tx0
        out.weight[ty0:ty1, tx0:tx1] += a.sum(axis=0).reshape(th_, tw_)
        out.color[ty0:ty1, tx0:tx1] += (a.T @ cols[sel]).reshape(th_, tw_, 3)
        if out.depth is not None:
            out.depth[ty0:ty1, tx0:tx1] += np.where(a > 0, a * np.where(ok, th, 0.0), 0.0).sum(axis=0).reshape(th_, tw_)
            out.normal[ty0:ty1, tx0:tx1] += (a.T @ n_vis[sel]).reshape(th_, tw_, 3)
        if ties:
            with np.errstate(invalid="ignore", divide="ignore", over="ignore"):
                f32 = TIE_F32_K * EPS32
                andot = np.abs(ndot)
                terr = f32 * np.abs(th) * (dn / andot + 2.0)
                r2 = u * u + v * v
                rerr = f32 * dn * (2.0 * (np.abs(u) * cu_n[sel][:, None] + np.abs(v) * cv_n[sel][:, None])
                                   + 2.0 * r2) / andot
                near_cut = np.abs(255.0 * raw - 1.0) < TIE_ALPHA + 0.5 * rerr
                near_gate = _near_gate(th, thr, st["depth_err"][ty0:ty1, tx0:tx1].reshape(1, -1) + terr)
                fl = near_gate & keep
                fl |= ok & (np.abs(ndot) < TIE_PARALLEL * PARALLEL_EPS * dn) & keep
            out.tie[ty0:ty1, tx0:tx1] |= fl.any(axis=0).reshape(th_, tw_)
            out.tie_cut[ty0:ty1, tx0:tx1] += (near_cut & (gate | near_gate) & ~fl).sum(axis=0).reshape(th_, tw_)

    return lambda tiles: _run(do_tile, _tiles_for(H, W, tiles), st["threads"])


# --- composite / geometry / render (forward.py:384-417) ---------------------
def composite(surfel_color, gaussian, surfel_weight=1.0):
    den = surfel_weight + gaussian.weight
    return (surfel_color * surfel_weight + gaussian.color) / den[..., None]


def smooth_geometry(sb, gb):
    if gb.depth is None:
        raise ValueError("gaussian buffers were rendered without geometry accumulation")
    den = 1.0 + gb.weight
    d = (sb.depth + gb.depth) / den
    nn = (sb.normal + gb.normal) / den[..., None]
    norm = np.linalg.norm(nn, axis=-1, keepdims=True)
    return d, np.where(norm > 1e-12, nn / np.maximum(norm, 1e-12), 0.0)


def render(scene, cam, settings=None, *, tiles=None, ties=False) -> RenderOut:
    """forward.py:403-417 (optionally restricted to base tiles ``tiles``)."""
    steps = render_steps(scene, cam, settings, [tiles], ties=ties)
    while True:
        try:
            next(steps)
        except StopIteration as fin:
            return fin.value


def render_steps(scene, cam, settings, tile_groups, *, ties=False):
    """Generator form of render(): the first next() does the per-frame
    preprocessing of both passes and the tiles of ``tile_groups[0]``; every
    later next() renders one more group (surfel tiles, then the Gaussian
    tiles of the same group).  The RenderOut is the StopIteration value.
    bench.py's reference arm times each next() as one bounded step, so
    whole frames are measured in row strips without extrapolation."""
    st = _settings(settings)
    srun, sfinish, (d0, e0) = _surfel_job(scene, cam, settings, ties)
    grun = gb = None
    if st["layers"] != "surfels_only":
        grun, gb = _gauss_job(scene, cam, d0, settings, ties, e0)
    for grp in tile_groups:
        srun(grp)
        if grun is not None:
            grun(grp)
        yield
    sb = sfinish()
    if gb is None:
        gb = GaussOut(np.zeros_like(sb.color), np.zeros_like(sb.depth),
                      tie=np.zeros(sb.depth.shape, bool), tie_cut=np.zeros(sb.depth.shape, np.int32))
        return RenderOut(sb.color.copy(), sb, gb)
    if st["layers"] == "gaussians_only":
        bg = np.asarray(st["background"], dtype=st["dtype"])
        img = np.where(gb.weight[..., None] > 0,
                       gb.color / np.maximum(gb.weight, 1e-12)[..., None], bg)
        return RenderOut(img, sb, gb)
    return RenderOut(composite(sb.color, gb), sb, gb)


def strip_groups(height, width, nstrips):
    """Base-tile indices of ``nstrips`` horizontal strips of whole tile rows
    covering the frame (render_steps' tile groups)."""
    ntx = (width + TILE - 1) // TILE
    nty = (height + TILE - 1) // TILE
    cuts = np.linspace(0, nty, min(nstrips, nty) + 1).round().astype(int)
    return [list(range(a * ntx, b * ntx)) for a, b in zip(cuts[:-1], cuts[1:])]


def default_threads():
    return os.cpu_count() or 1
