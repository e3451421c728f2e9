"""Parity comparator: GPU float32 outputs vs the float64 oracle.

Rule (north_star): the surfel-ID map must be bit-exact except
on pixels the oracle flags as ties (float64 decision margin below the TIE_*
thresholds in oracle/ges_oracle.py); depth relative error <= DEPTH_REL and
RGB max-abs error <= RGB_TOL on the remaining pixels; PSNR >= 60 dB over all
pixels.  The report counts the excluded pixels, and the excluded count is
bounded (EXCLUDED_FRAC).  Pixels where a Gaussian fragment sits at the 1/255
alpha cutoff are not excluded: they are checked against the bound one
flipped fragment can cause (CUT_FLIP per flagged fragment).
"""

from __future__ import annotations

import numpy as np

RGB_TOL = 1e-4
DEPTH_REL = 1e-5
PSNR_MIN = 60.0
# excluded (hard-tie) pixels may be at most this fraction of the compared
# pixels (or EXCLUDED_MIN pixels on tiny frames)
EXCLUDED_FRAC = 0.005
EXCLUDED_MIN = 2
# one Gaussian fragment at the 1/255 cutoff moves a pixel's image, weight or
# accumulated colour by at most alpha ~ 1/255 (TIE_ALPHA slack included)
CUT_FLIP = (1.0 + 1e-3) / 255.0


def psnr(a, b):
    mse = float(np.mean((np.asarray(a, np.float64) - np.asarray(b, np.float64)) ** 2))
    return float("inf") if mse == 0 else 10.0 * np.log10(1.0 / mse)


def compare_oracle(gpu, ref, ora, *, region=None):
    """compare() with every flag taken from an oracle RenderOut ``ora``
    (rendered with ties=True): hard ties, cut-flagged fragments, colour-only
    sub-sample ties (supersample=4) and the winner depths' float32 error
    bounds.  ``ref`` holds the values compared against (oracle or golden)."""
    ref = dict(ref)
    ref.setdefault("s_depth_err", ora.surfels.depth_err)
    return compare(gpu, ref, ora.tie, region=region, tie_cut=ora.tie_cut, tie_color=ora.tie_color)


def compare(gpu, ora, tie, *, region=None, tie_cut=None, tie_color=None):
    """gpu / ora: dicts with image, s_winner, s_depth (+ optional s_color,
    g_weight, g_color ...).  tie: (H, W) bool hard ties (excluded and
    counted).  tie_cut: (H, W) int, per pixel the number of Gaussian
    fragments at the alpha cutoff: those pixels are checked against
    RGB_TOL + n * CUT_FLIP instead of RGB_TOL.  region: optional (H, W) bool
    mask restricting the comparison (tile-sampled oracle).  tie_color: (H, W)
    bool, pixels whose colour only may differ (supersample=4 sub-sample
    ties): excluded from the image / s_color checks and counted."""
    H, W = tie.shape
    region = np.ones((H, W), bool) if region is None else region
    cut = np.zeros((H, W), np.int32) if tie_cut is None else np.asarray(tie_cut)
    keep = region & ~tie
    strict = keep & (cut == 0)
    tcol = np.zeros((H, W), bool) if tie_color is None else (np.asarray(tie_color) & keep)
    rep = dict(pixels=int(region.sum()), excluded=int((region & tie).sum()),
               cut_flagged=int((keep & (cut > 0)).sum()), color_flagged=int(tcol.sum()))
    gw, ow = gpu["s_winner"], ora["s_winner"]
    rep["winner_mismatch"] = int(((gw != ow) & keep).sum())
    rep["winner_mismatch_incl_ties"] = int(((gw != ow) & region).sum())
    gd, od = gpu["s_depth"].astype(np.float64), ora["s_depth"]
    both = keep & np.isfinite(od) & (gw == ow)
    rep["coverage_mismatch"] = int((np.isfinite(gd) != np.isfinite(od))[keep].sum())
    # depth: relative error beyond the winner's float32 conditioning bound
    # (oracle s_depth_err, nonzero only at grazing incidence)
    derr = ora.get("s_depth_err")
    derr = np.zeros(od.shape) if derr is None else derr
    with np.errstate(invalid="ignore"):
        exc = np.maximum(np.abs(gd - od) - derr, 0.0)
    rep["depth_rel_max"] = float(np.max(exc[both] / np.abs(od[both]))) if both.any() else 0.0
    for k in ("image", "s_color", "s_normal", "g_color", "g_weight", "g_depth", "g_normal"):
        if k in gpu and k in ora and gpu[k] is not None and ora[k] is not None:
            diff = np.abs(gpu[k].astype(np.float64) - ora[k])
            if diff.ndim == 3:
                diff = diff.max(axis=-1)
            sk = strict & ~tcol if k in ("image", "s_color") else strict
            rep[f"{k}_maxabs"] = float(diff[sk].max()) if sk.any() else 0.0
            if k in ("image", "g_weight", "g_color"):
                # flagged pixels: the excess over the per-pixel flip bound
                m = keep & (cut > 0) & (~tcol if k == "image" else True)
                rep[f"{k}_cut_excess"] = float((diff - cut * CUT_FLIP)[m].max()) if m.any() else -1.0
    r = region
    rep["psnr"] = psnr(gpu["image"][r], ora["image"][r])
    return rep


def assert_parity(rep, *, rgb_tol=RGB_TOL, depth_rel=DEPTH_REL, psnr_min=PSNR_MIN,
                  weight_tol=None, excluded_frac=EXCLUDED_FRAC):
    assert rep["excluded"] <= max(excluded_frac * rep["pixels"], EXCLUDED_MIN), rep
    assert rep.get("color_flagged", 0) <= max(excluded_frac * rep["pixels"], EXCLUDED_MIN), rep
    assert rep["winner_mismatch"] == 0, rep
    assert rep["coverage_mismatch"] == 0, rep
    assert rep["depth_rel_max"] <= depth_rel, rep
    assert rep["image_maxabs"] <= rgb_tol, rep
    assert rep.get("image_cut_excess", -1.0) <= rgb_tol, rep
    if "s_color_maxabs" in rep:
        assert rep["s_color_maxabs"] <= rgb_tol, rep
    if "g_color_maxabs" in rep and weight_tol is not None:
        assert rep["g_weight_maxabs"] <= weight_tol, rep
        assert rep["g_color_maxabs"] <= weight_tol, rep
        assert rep.get("g_weight_cut_excess", -1.0) <= weight_tol, rep
        assert rep.get("g_color_cut_excess", -1.0) <= weight_tol, rep
    assert rep["psnr"] >= psnr_min, rep
