"""CPU oracle for the GES joint-stage training step -- TEST INFRASTRUCTURE ONLY.

A float64 NumPy restatement of the reference training renderer for the
joint stage with frozen opaque surfels (or none) and trainable Gaussians,
and of its backward pass:

* forward  -- training.py:295-355 with _surfel_pass_frozen (:358-392) and
  the Gaussian passes (:399-544), built on the forward oracle
  (``ges_oracle.rasterize_surfels`` / ``accumulate_gaussians``);
* backward -- training.py:547-609 with _surfel_backward_frozen (:612-629),
  _gaussian_backward_3d (:646-719), _gaussian_backward_2d (:722-788), the
  projection / ray-plane / SH / world-filter chains they call
  (geometry.py:135-190, :229-270; training.py:123-138, :632-643, :890-911).

It is written per Gaussian (each Gaussian's pixel window is swept and its
partial sums accumulated directly) rather than over a global fragment list,
and the 2D fragment gradients are kept as full 3-vectors (the CUDA kernel
reduces them in plane coordinates), so it checks the GPU formulation
independently.  Parity of this oracle is PINNED against the real reference:
``tests/golden/train_*.npz`` are made by ``tests/golden/make_train_golden.py``
(importing /root/reference read-only in the build container) and
``tests/test_train_oracle.py`` checks this module against them at 1e-9.

Only tests and ``__graft_entry__.smoke()`` import it; the product package
never does.
"""

from __future__ import annotations

import math
from types import SimpleNamespace

import numpy as np

from . import ges_oracle as O

W_OPAQUE = 255.0
W_ADJUST = 30.0

_C0 = 0.28209479177387814
_C1 = 0.4886025119029199
_C2 = (1.0925484305920792, -1.0925484305920792, 0.31539156525252005, -1.0925484305920792, 0.5462742152960396)
_C3 = (-0.5900435899266435, 2.890611442640554, -0.4570457994644658, 0.3731763325901154,
       -0.4570457994644658, 1.445305721320277, -0.5900435899266435)


# --- SH basis and its direction Jacobian (sh.py:34-112) ---------------------
def sh_basis_and_jac(deg, d):
    """Basis (N, K) and d basis / d dir (N, K, 3) at unit directions d."""
    x, y, z = d[:, 0], d[:, 1], d[:, 2]
    n = d.shape[0]
    one, zero = np.ones(n), np.zeros(n)
    # each entry: (value, (dx, dy, dz))
    terms = [(_C0 * one, (zero, zero, zero))]
    if deg >= 1:
        terms += [(-_C1 * y, (zero, -_C1 * one, zero)), (_C1 * z, (zero, zero, _C1 * one)),
                  (-_C1 * x, (-_C1 * one, zero, zero))]
    if deg >= 2:
        a, b, c, e, f = _C2
        terms += [(a * x * y, (a * y, a * x, zero)),
                  (b * y * z, (zero, b * z, b * y)),
                  (c * (2 * z * z - x * x - y * y), (-2 * c * x, -2 * c * y, 4 * c * z)),
                  (e * x * z, (e * z, zero, e * x)),
                  (f * (x * x - y * y), (2 * f * x, -2 * f * y, zero))]
    if deg >= 3:
        c0, c1, c2, c3, c4, c5, c6 = _C3
        xx, yy, zz = x * x, y * y, z * z
        terms += [(c0 * y * (3 * xx - yy), (6 * c0 * x * y, c0 * (3 * xx - 3 * yy), zero)),
                  (c1 * x * y * z, (c1 * y * z, c1 * x * z, c1 * x * y)),
                  (c2 * y * (4 * zz - xx - yy), (-2 * c2 * x * y, c2 * (4 * zz - xx - 3 * yy), 8 * c2 * y * z)),
                  (c3 * z * (2 * zz - 3 * xx - 3 * yy),
                   (-6 * c3 * x * z, -6 * c3 * y * z, c3 * (6 * zz - 3 * xx - 3 * yy))),
                  (c4 * x * (4 * zz - xx - yy), (c4 * (4 * zz - 3 * xx - yy), -2 * c4 * x * y, 8 * c4 * x * z)),
                  (c5 * z * (xx - yy), (2 * c5 * x * z, -2 * c5 * y * z, c5 * (xx - yy))),
                  (c6 * x * (xx - 3 * yy), (c6 * (3 * xx - 3 * yy), -6 * c6 * x * y, zero))]
    B = np.stack([t[0] for t in terms], axis=1)
    Jb = np.stack([np.stack(t[1], axis=1) for t in terms], axis=1)
    return B, Jb


def colour_vjp(pos, sh, campos, g_col):
    """Gradients of clip(0.5 + B(dir) sh) w.r.t. sh and pos (training.py:123-138)."""
    sh = np.asarray(sh, dtype=np.float64)
    deg = int(round(math.sqrt(sh.shape[1]))) - 1
    diff = campos[None, :] - np.asarray(pos, dtype=np.float64)
    dist = np.linalg.norm(diff, axis=1)
    d = diff / dist[:, None]
    B, Jb = sh_basis_and_jac(deg, d)
    raw = 0.5 + np.einsum("nk,nkc->nc", B, sh)
    gc = g_col * ((raw > 0.0) & (raw < 1.0))
    g_sh = B[:, :, None] * gc[:, None, :]
    g_dir = np.einsum("nkj,nk->nj", Jb, np.einsum("nkc,nc->nk", sh, gc))
    tang = g_dir - np.sum(g_dir * d, axis=1, keepdims=True) * d
    return g_sh, -tang / dist[:, None]


def train_colours(pos, sh, campos):
    diff = campos[None, :] - np.asarray(pos, dtype=np.float64)
    d = diff / np.linalg.norm(diff, axis=1, keepdims=True)
    deg = int(round(math.sqrt(np.asarray(sh).shape[1]))) - 1
    B, _ = sh_basis_and_jac(deg, d)
    return np.clip(0.5 + np.einsum("nk,nkc->nc", B, np.asarray(sh, dtype=np.float64)), 0.0, 1.0)


# --- rotation helpers (geometry.py:18-65) -----------------------------------
def unit_quats(q):
    q = np.atleast_2d(np.asarray(q, dtype=np.float64))
    return q / np.linalg.norm(q, axis=1, keepdims=True)


def rot_vjp(qn, G):
    """sum_ij dR_ij/dq G_ij for unit quaternions qn (N,4), cotangents G (N,3,3)."""
    w, x, y, z = qn.T
    g = [G[:, i, j] for i in range(3) for j in range(3)]
    g00, g01, g02, g10, g11, g12, g20, g21, g22 = g
    return np.stack([
        2 * (-z * g01 + y * g02 + z * g10 - x * g12 - y * g20 + x * g21),
        2 * (y * g01 + z * g02 + y * g10 - 2 * x * g11 - w * g12 + z * g20 + w * g21 - 2 * x * g22),
        2 * (-2 * y * g00 + x * g01 + w * g02 + x * g10 + z * g12 - w * g20 + z * g21 - 2 * y * g22),
        2 * (-2 * z * g00 - w * g01 + x * g02 + w * g10 - 2 * z * g11 + y * g12 + x * g20 + y * g21),
    ], axis=1)


# --- settings ---------------------------------------------------------------
def resolve(settings, scene):
    w = np.asarray(scene.surfels.w)
    late = (w.min() if w.size else np.inf) >= W_ADJUST
    ss = settings.supersample if settings.supersample is not None else (4 if late else 1)
    return ss, late


def _fwd_settings(settings, **kw):
    d = dict(supersample=1, background=tuple(settings.background), layers="full", mip=settings.mip,
             epsilon_mode=settings.epsilon_mode, epsilon_value=settings.epsilon_value,
             dtype=np.float64, threads=1, with_geometry=settings.with_geometry)
    d.update(kw)
    return SimpleNamespace(**d)


# --- forward ----------------------------------------------------------------
def render_training(scene, cam, settings, cache=None, cache_key=None):
    """Joint-stage forward: frozen opaque surfels (or none) + Gaussians."""
    c = O.as_cam(cam)
    H, W = c.height, c.width
    ns = int(np.asarray(scene.surfels.pos).shape[0])
    ng = int(np.asarray(scene.gaussians.pos).shape[0])
    ss, late = resolve(settings, scene)
    grid = 2 if ss == 4 else 1
    bg = np.asarray(settings.background, dtype=np.float64)
    use_s = settings.surfels_enabled and ns > 0
    if use_s and not (settings.frozen_cache is not None and np.all(np.asarray(scene.surfels.w) == W_OPAQUE)):
        raise NotImplementedError("oracle covers frozen surfels only")
    geom = settings.with_geometry
    out = dict(grid=grid, use_s=use_s, blend_depth=None, blend_normal=None, winner=None)
    if use_s:
        entry = cache.get(cache_key) if (cache is not None and cache_key is not None) else None
        if entry is None:
            rc = cam.scaled(grid) if grid > 1 else cam
            sb = O.rasterize_surfels(scene, rc, _fwd_settings(settings, with_geometry=False, background=(0, 0, 0)))
            entry = dict(winner=sb.winner.reshape(-1), depth=sb.depth.reshape(-1), normal=sb.normal.reshape(-1, 3))
            if cache is not None and cache_key is not None:
                cache[cache_key] = entry
        win = entry["winner"]
        cov = win >= 0
        cols = train_colours(scene.surfels.pos, scene.surfels.sh, c.position)
        hi = np.where(cov[:, None], cols[np.maximum(win, 0)], bg[None, :])
        out["surfel_color"] = hi.reshape(H, grid, W, grid, 3).mean(axis=(1, 3))
        out["surfel_depth"] = entry["depth"].reshape(H * grid, W * grid)[0::grid, 0::grid].copy()
        if geom:
            out["blend_depth"] = np.where(cov, entry["depth"], 0.0).reshape(H, grid, W, grid).mean(axis=(1, 3))
            out["blend_normal"] = np.where(cov[:, None], entry["normal"], 0.0).reshape(
                H, grid, W, grid, 3).mean(axis=(1, 3))
        out["winner"] = win
    else:
        out["surfel_color"] = np.broadcast_to(bg, (H, W, 3)).copy()
        out["surfel_depth"] = np.full((H, W), np.inf)
    if settings.gaussians_enabled and ng:
        gb = O.accumulate_gaussians(scene, cam, out["surfel_depth"], _fwd_settings(settings))
        gc, gw, gd, gn = gb.color, gb.weight, gb.depth, gb.normal
    else:
        gc, gw = np.zeros((H, W, 3)), np.zeros((H, W))
        gd = np.zeros((H, W)) if geom else None
        gn = np.zeros((H, W, 3)) if geom else None
    gonly = settings.gaussian_only_norm and not use_s
    if gonly:
        image = np.where(gw[..., None] > 0, gc / np.maximum(gw, 1e-12)[..., None], bg)
    else:
        image = (out["surfel_color"] + gc) / (1.0 + gw)[..., None]
    out.update(image=image, gauss_color=gc, gauss_weight=gw, gauss_depth=gd, gauss_normal=gn,
               gaussian_only=gonly, gaussians=bool(settings.gaussians_enabled and ng))
    return out


# --- Gaussian backward: per-Gaussian sweeps ----------------------------------
def _windows(x0, x1, y0, y1, W):
    for i in range(len(x0)):
        if x1[i] < x0[i] or y1[i] < y0[i]:
            yield i, None
            continue
        xs = np.arange(x0[i], x1[i] + 1)
        ys = np.arange(y0[i], y1[i] + 1)
        X, Y = np.meshgrid(xs, ys)
        yield i, (X.reshape(-1), Y.reshape(-1))


def _eps(g, settings, es):
    if settings.epsilon_mode == "constant":
        return np.full(es.shape[0], float(settings.epsilon_value))
    return (5.0 / es.shape[1]) * np.sum(es, axis=1)


def _effective(g):
    s = np.exp(np.asarray(g.log_scale, dtype=np.float64))
    sig = 1.0 / (1.0 + np.exp(-np.asarray(g.raw_opacity, dtype=np.float64)))
    lam = np.asarray(g.filter3d, dtype=np.float64) if getattr(g, "filter3d", None) is not None else np.zeros(len(s))
    anyf = bool(np.any(lam))
    es = np.sqrt(s * s + lam[:, None]) if anyf else s
    sig_e = sig * np.prod(s / es, axis=1) if anyf else sig
    return s, sig, lam, anyf, es, sig_e


def _chain_eff(s, sig, lam, anyf, es, sig_e, g_es, g_sig_e):
    if not anyf:
        return g_es, g_sig_e
    g_s = g_es * (s / es) + (g_sig_e * sig_e)[:, None] * (1.0 / s - s / (es * es))
    return g_s, g_sig_e * (sig_e / sig)


def _screen(pos, g_pos, c):
    z = np.maximum(c.to_camera(np.asarray(pos, dtype=np.float64))[:, 2], O.NEAR)
    gcam = g_pos @ c.R.T
    return np.hypot(gcam[:, 0] * z / c.fx * (c.width / 2.0), gcam[:, 1] * z / c.fy * (c.height / 2.0))


def _backward_3d(scene, c, settings, ds, g_cg, g_wg, g_gd, g_gn, wg):
    g = scene.gaussians
    n = int(np.asarray(g.pos).shape[0])
    H, W = c.height, c.width
    s, sig, lam, anyf, es, sig_e = _effective(g)
    qn = unit_quats(g.quat)
    Rq = O.rotmats(qn)
    pos = np.asarray(g.pos, dtype=np.float64)
    t = c.to_camera(pos)
    x, y, z = t[:, 0], t[:, 1], t[:, 2]
    valid = z > O.NEAR
    zs = np.where(valid, z, 1.0)
    xs_, ys_ = np.where(valid, x, 0.0), np.where(valid, y, 0.0)
    J = np.zeros((n, 2, 3))
    J[:, 0, 0], J[:, 0, 2] = c.fx / zs, -c.fx * xs_ / zs ** 2
    J[:, 1, 1], J[:, 1, 2] = c.fy / zs, -c.fy * ys_ / zs ** 2
    S3 = np.einsum("nik,nk,njk->nij", Rq, es ** 2, Rq)
    M = np.einsum("ab,nbc,dc->nad", c.R, S3, c.R)
    Craw = np.einsum("nab,nbc,ndc->nad", J, M, J)
    Cf = Craw + O.SCREEN_VAR * np.eye(2)
    det = Cf[:, 0, 0] * Cf[:, 1, 1] - Cf[:, 0, 1] ** 2
    rdet = Craw[:, 0, 0] * Craw[:, 1, 1] - Craw[:, 0, 1] ** 2
    with np.errstate(divide="ignore", invalid="ignore"):
        kc = np.sqrt(np.maximum(rdet, 1e-300) / det) if settings.mip else np.ones(n)
        amp = sig_e * kc
        Lam = np.stack([np.stack([Cf[:, 1, 1], -Cf[:, 0, 1]], -1), np.stack([-Cf[:, 0, 1], Cf[:, 0, 0]], -1)],
                       1) / det[:, None, None]
        m2 = 2.0 * np.log(np.maximum(255.0 * amp, 1e-12))
    valid &= (det > 0) & (m2 > 0)
    mean = np.stack([c.fx * xs_ / zs + c.cx, c.fy * ys_ / zs + c.cy], 1)
    rx = np.sqrt(np.maximum(m2 * Cf[:, 0, 0], 0.0))
    ry = np.sqrt(np.maximum(m2 * Cf[:, 1, 1], 0.0))
    x0, x1, y0, y1 = O.pixel_ranges(np.stack([mean[:, 0] - rx, mean[:, 0] + rx, mean[:, 1] - ry, mean[:, 1] + ry], 1),
                                    np.zeros(n, bool), W, H)
    eps = _eps(g, settings, es)
    cols = train_colours(pos, g.sh, c.position)
    nrm = None
    if settings.with_geometry:
        k = np.argmin(es, axis=1)
        nv = Rq[np.arange(n), :, k] @ c.R.T
        nrm = np.where(np.sum(nv * t, axis=1, keepdims=True) < 0, nv, -nv)
    S_gp = np.zeros(n)
    S_m = np.zeros((n, 2))
    S_L = np.zeros((n, 2, 2))
    S_col = np.zeros((n, 3))
    S_d = np.zeros(n)
    S_con = np.zeros(n)
    for i, win in _windows(x0, x1, y0, y1, W):
        if win is None or not valid[i]:
            continue
        X, Y = win
        dlt = np.stack([X + 0.5 - mean[i, 0], Y + 0.5 - mean[i, 1]], 1)
        pw = -0.5 * np.einsum("fa,ab,fb->f", dlt, Lam[i], dlt)
        a = amp[i] * np.exp(pw)
        ok = (a >= O.ALPHA_CUTOFF) & (z[i] < ds[Y, X] + eps[i])
        if not np.any(ok):
            continue
        X, Y, dlt, a = X[ok], Y[ok], dlt[ok], a[ok]
        S_con[i] = np.max(cols[i].max() * a / (1.0 + wg[Y, X]))   # optim.py:526-533
        ga = g_cg[Y, X] @ cols[i] + g_wg[Y, X]
        if g_gd is not None:
            ga = ga + z[i] * g_gd[Y, X]
            S_d[i] += np.sum(a * g_gd[Y, X])
        if g_gn is not None and nrm is not None:
            ga = ga + g_gn[Y, X] @ nrm[i]
        gp = ga * a
        S_gp[i] += gp.sum()
        S_m[i] += (gp[:, None] * (dlt @ Lam[i])).sum(0)
        S_L[i] += -0.5 * np.einsum("f,fa,fb->ab", gp, dlt, dlt)
        S_col[i] += a @ g_cg[Y, X]
    # dL/dC' = -Lam S_L Lam ; amplitude and mip compensation
    gC = -np.einsum("nab,nbc,ncd->nad", Lam, S_L, Lam)
    with np.errstate(divide="ignore", invalid="ignore"):
        g_amp = np.where(S_gp != 0, S_gp / amp, 0.0)
    g_sig_e = g_amp * kc
    if settings.mip:
        gk = g_amp * sig_e
        inv_r = np.linalg.inv(Craw + 1e-12 * np.eye(2))
        inv_f = np.linalg.inv(Cf)
        gC = gC + (0.5 * kc * gk)[:, None, None] * (inv_r - inv_f)
    # EWA: C = J M J^T, mean = (fx x/z + cx, fy y/z + cy), depth = z
    gM = np.einsum("nai,nab,nbj->nij", J, gC, J)
    gJ = 2.0 * np.einsum("nab,nbc,ncd->nad", gC, J, M)
    g_t = np.zeros((n, 3))
    g_t[:, 0] = gJ[:, 0, 2] * (-c.fx / zs ** 2) + S_m[:, 0] * c.fx / zs
    g_t[:, 1] = gJ[:, 1, 2] * (-c.fy / zs ** 2) + S_m[:, 1] * c.fy / zs
    g_t[:, 2] = (gJ[:, 0, 0] * (-c.fx / zs ** 2) + gJ[:, 0, 2] * (2 * c.fx * xs_ / zs ** 3)
                 + gJ[:, 1, 1] * (-c.fy / zs ** 2) + gJ[:, 1, 2] * (2 * c.fy * ys_ / zs ** 3)
                 - S_m[:, 0] * c.fx * xs_ / zs ** 2 - S_m[:, 1] * c.fy * ys_ / zs ** 2 + S_d)
    g_pos = g_t @ c.R
    gS3 = np.einsum("ai,nab,bj->nij", c.R, gM, c.R)
    gS3 = 0.5 * (gS3 + np.swapaxes(gS3, 1, 2))
    # S3 = sum_k es_k^2 r_k r_k^T
    gcolk = 2.0 * np.einsum("nij,njk->nik", gS3, Rq)           # column k: 2 gS3 r_k
    g_es = es * np.einsum("nik,nik->nk", gcolk, Rq)
    g_quat_u = rot_vjp(qn, gcolk * (es ** 2)[:, None, :])
    g_sh, g_pos_sh = colour_vjp(pos, g.sh, c.position, S_col)
    g_pos = g_pos + g_pos_sh
    g_scale, g_sigma = _chain_eff(s, sig, lam, anyf, es, sig_e, g_es, g_sig_e)
    touched = (S_gp != 0) | np.any(S_col != 0, axis=1) | (S_d != 0) | np.any(S_m != 0, axis=1)
    out = _pack(touched, qn, pos, g_pos, g_quat_u, g_scale, g_sigma, g_sh, c)
    out["contrib"] = S_con
    return out


def _backward_2d(scene, c, settings, ds, g_cg, g_wg, g_gd, g_gn, wg):
    g = scene.gaussians
    n = int(np.asarray(g.pos).shape[0])
    H, W = c.height, c.width
    s, sig, lam, anyf, es, sig_e = _effective(g)
    qn = unit_quats(g.quat)
    pos = np.asarray(g.pos, dtype=np.float64)
    q, a1, a2, nn = O.frames(pos, qn, c)
    if settings.mip:
        smul, omul, fvalid = O.object_filter_2d(q, a1, a2, es, c)
    else:
        smul, omul, fvalid = np.ones((n, 2)), np.ones(n), np.ones(n, bool)
    scl = es * smul
    sgm = sig_e * omul
    with np.errstate(divide="ignore"):
        m2 = 2.0 * np.log(np.maximum(255.0 * sgm, 1e-12))
    valid = fvalid & (q[:, 2] > O.NEAR) & (m2 > 0)
    rmax = np.sqrt(np.maximum(m2, 0.0))
    bnd, whole = O.disc_bounds(q, a1, a2, scl[:, 0] * rmax, scl[:, 1] * rmax, c)
    x0, x1, y0, y1 = O.pixel_ranges(bnd, whole, W, H)
    eps = _eps(g, settings, es)
    cols = train_colours(pos, g.sh, c.position)
    sign = np.where(np.sum(nn * q, axis=1) < 0, 1.0, -1.0)
    rays = c.rays()
    Gq, Ga1, Ga2, Gn = (np.zeros((n, 3)) for _ in range(4))
    Gs = np.zeros((n, 2))
    Gsig = np.zeros(n)
    S_col = np.zeros((n, 3))
    S_nv = np.zeros((n, 3))
    S_con = np.zeros(n)
    for i, win in _windows(x0, x1, y0, y1, W):
        if win is None or not valid[i]:
            continue
        X, Y = win
        d = rays[Y, X]
        with np.errstate(divide="ignore", invalid="ignore"):
            nd = d @ nn[i]
            t = (nn[i] @ q[i]) / nd
            h = t[:, None] * d - q[i][None, :]
            u = (h @ a1[i]) / scl[i, 0]
            v = (h @ a2[i]) / scl[i, 1]
            ok = (np.abs(nd) > O.PARALLEL_EPS * np.linalg.norm(d, axis=1)) & (t > O.NEAR)
            G = np.where(ok, np.exp(-0.5 * (u * u + v * v)), 0.0)
        a = sgm[i] * G
        keep = ok & (a >= O.ALPHA_CUTOFF) & (t < ds[Y, X] + eps[i])
        if not np.any(keep):
            continue
        X, Y, d, nd, t, h, u, v, G, a = (w[keep] for w in (X, Y, d, nd, t, h, u, v, G, a))
        S_con[i] = np.max(cols[i].max() * a / (1.0 + wg[Y, X]))   # optim.py:526-533
        ga = g_cg[Y, X] @ cols[i] + g_wg[Y, X]
        gt_direct = np.zeros_like(t)
        if g_gd is not None:
            ga = ga + t * g_gd[Y, X]
            gt_direct = a * g_gd[Y, X]
        if g_gn is not None:
            ga = ga + g_gn[Y, X] @ (sign[i] * nn[i])
            S_nv[i] += a @ g_gn[Y, X]
        Gsig[i] += np.sum(ga * G)
        gu = -u * a * ga
        gv = -v * a * ga
        # u = a1.(t d - q)/s1, v likewise, t = (n.q)/(n.d)
        g_tt = gu * (d @ a1[i]) / scl[i, 0] + gv * (d @ a2[i]) / scl[i, 1] + gt_direct
        Gq[i] += np.sum(g_tt / nd) * nn[i] - np.sum(gu) / scl[i, 0] * a1[i] - np.sum(gv) / scl[i, 1] * a2[i]
        Gn[i] += -((g_tt / nd)[:, None] * h).sum(0)
        Ga1[i] += (gu[:, None] * h).sum(0) / scl[i, 0]
        Ga2[i] += (gv[:, None] * h).sum(0) / scl[i, 1]
        Gs[i, 0] += -np.sum(gu * u) / scl[i, 0]
        Gs[i, 1] += -np.sum(gv * v) / scl[i, 1]
        S_col[i] += a @ g_cg[Y, X]
    Gn = Gn + sign[:, None] * S_nv
    g_pos = Gq @ c.R
    cols_g = np.stack([Ga1 @ c.R, Ga2 @ c.R, Gn @ c.R], axis=-1)
    g_quat_u = rot_vjp(qn, cols_g)
    g_sh, g_pos_sh = colour_vjp(pos, g.sh, c.position, S_col)
    g_pos = g_pos + g_pos_sh
    g_scale, g_sigma = _chain_eff(s, sig, lam, anyf, es, sig_e, Gs * smul, Gsig * omul)
    touched = (Gsig != 0) | np.any(S_col != 0, axis=1) | np.any(Gq != 0, axis=1)
    out = _pack(touched, qn, pos, g_pos, g_quat_u, g_scale, g_sigma, g_sh, c)
    out["contrib"] = S_con
    return out


def _pack(touched, qn, pos, g_pos, g_quat_u, g_scale, g_sigma, g_sh, c):
    g_quat = g_quat_u - np.sum(qn * g_quat_u, axis=1, keepdims=True) * qn
    out = dict(gaussian_pos=g_pos, gaussian_quat=g_quat, gaussian_scale=g_scale, gaussian_opacity=g_sigma,
               gaussian_sh=g_sh, gaussian_screen_grad=_screen(pos, g_pos, c))
    for k, v in out.items():   # primitives without fragments get exact zeros
        v[~touched] = 0.0
    return out


def backward(scene, cam, settings, frame, g_image, *, g_gauss_depth=None, g_gauss_normal=None,
             g_gauss_weight=None):
    """training.py:547-609 for the joint stage; returns a dict of float64 arrays
    (plus ``contrib``: this view's contribution scores, optim.py:519-533)."""
    c = O.as_cam(cam)
    g_img = np.asarray(g_image, dtype=np.float64)
    gw, image = frame["gauss_weight"], frame["image"]
    if frame["gaussian_only"]:
        wsafe = np.maximum(gw, 1e-12)
        cov = gw > 0
        g_cg = np.where(cov[..., None], g_img / wsafe[..., None], 0.0)
        g_wg = np.where(cov, -np.sum(g_img * image, axis=-1) / wsafe, 0.0)
        g_cs = np.zeros_like(g_img)
    else:
        den = 1.0 + gw
        g_cs = g_img / den[..., None]
        g_cg = g_cs
        g_wg = -np.sum(g_img * image, axis=-1) / den
    if g_gauss_weight is not None:
        g_wg = g_wg + np.asarray(g_gauss_weight, dtype=np.float64)
    ns = int(np.asarray(scene.surfels.pos).shape[0])
    ng = int(np.asarray(scene.gaussians.pos).shape[0])
    K = np.asarray(scene.surfels.sh if ns else scene.gaussians.sh).shape[1]
    D = int(np.asarray(scene.gaussians.log_scale).shape[1]) if ng else 3
    out = dict(surfel_pos=np.zeros((ns, 3)), surfel_quat=np.zeros((ns, 4)), surfel_scale=np.zeros((ns, 2)),
               surfel_sh=np.zeros((ns, K, 3)), surfel_w=np.zeros(ns), gaussian_pos=np.zeros((ng, 3)),
               gaussian_opacity=np.zeros(ng), gaussian_quat=np.zeros((ng, 4)), gaussian_scale=np.zeros((ng, D)),
               gaussian_sh=np.zeros((ng, K, 3)), surfel_screen_grad=np.zeros(ns),
               gaussian_screen_grad=np.zeros(ng), contrib=np.zeros(ng))
    if frame["gaussians"]:
        gd = None if g_gauss_depth is None else np.asarray(g_gauss_depth, dtype=np.float64)
        gn = None if g_gauss_normal is None else np.asarray(g_gauss_normal, dtype=np.float64)
        fn = _backward_2d if O._is_2d(scene.gaussians.kind) else _backward_3d
        out.update(fn(scene, c, settings, frame["surfel_depth"], g_cg, g_wg, gd, gn, frame["gauss_weight"]))
    win = frame["winner"]
    if win is not None and np.any(win >= 0):
        grid = frame["grid"]
        H, W = c.height, c.width
        up = np.repeat(np.repeat(g_cs / (grid * grid), grid, axis=0), grid, axis=1).reshape(-1, 3)
        cov = win >= 0
        g_col = np.zeros((ns, 3))
        np.add.at(g_col, win[cov], up[cov])
        g_sh, g_pos = colour_vjp(scene.surfels.pos, scene.surfels.sh, c.position, g_col)
        hit = np.any(g_col != 0, axis=1)
        g_sh[~hit] = 0.0
        g_pos[~hit] = 0.0
        out["surfel_sh"], out["surfel_pos"] = g_sh, g_pos
    return out
