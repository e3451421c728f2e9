"""The CPU oracle (oracle/ges_oracle.py) against golden vectors produced by
the real reference renderer (tests/golden/make_golden.py).  Tolerance is the
reference's own oracle tolerance, atol 1e-9 in float64
(/root/reference/pkg/tests/test_forward.py:151-160, :209-238)."""

import hashlib

import numpy as np
import pytest

from golden_io import load, names, settings_ns
from oracle import ges_oracle as O


def _digest(scene):
    h = hashlib.sha256()
    s, g = scene.surfels, scene.gaussians
    for a in (s.pos, s.quat, s.log_scale, s.sh, g.pos, g.raw_opacity, g.quat,
              g.log_scale, g.sh, g.filter3d):
        h.update(np.ascontiguousarray(a, dtype=np.float64).tobytes())
    return h.hexdigest()


def _close(a, b, atol=1e-9):
    both_inf = np.isinf(a) & np.isinf(b)
    assert np.array_equal(np.isinf(a), np.isinf(b))
    assert np.allclose(a[~both_inf], b[~both_inf], atol=atol, rtol=0)


@pytest.mark.parametrize("name", names())
def test_oracle_matches_reference_golden(name):
    scene, cam, st, gold, digest = load(name)
    assert _digest(scene) == digest, "scene generator drifted from the golden"
    out = O.render(scene, cam, settings_ns(st))
    assert np.array_equal(out.surfels.winner, gold["s_winner"])
    _close(out.surfels.depth, gold["s_depth"])
    _close(out.surfels.color, gold["s_color"])
    _close(out.surfels.normal, gold["s_normal"])
    _close(out.gaussians.weight, gold["g_weight"])
    _close(out.gaussians.color, gold["g_color"])
    _close(out.image, gold["image"])
    if "g_depth" in gold:
        _close(out.gaussians.depth, gold["g_depth"])
        _close(out.gaussians.normal, gold["g_normal"])


def test_oracle_tile_subset_matches_full():
    scene, cam, st, gold, _ = load("deg3_64x48")
    tiles = [1, 4, 7]
    out = O.render(scene, cam, settings_ns(st), tiles=tiles)
    for ti in tiles:
        ty0, ty1, tx0, tx1 = O.tile_list(cam.height, cam.width)[ti]
        _close(out.image[ty0:ty1, tx0:tx1], gold["image"][ty0:ty1, tx0:tx1])


def test_tie_flags_are_rare():
    scene, cam, st, gold, _ = load("config1")
    out = O.render(scene, cam, settings_ns(st), ties=True)
    frac = out.tie.mean()
    assert frac < 0.01, frac


def test_oracle_fp32_close_to_fp64():
    scene, cam, st, gold, _ = load("config1")
    out = O.render(scene, cam, settings_ns(st, np.float32))
    assert np.max(np.abs(out.image - gold["image"])) < 1e-4


def test_oracle_tile_subset_supersampled():
    scene, cam, st, gold, _ = load("deg3_64x48_ss4")
    tiles = [0, 5, 10]
    out = O.render(scene, cam, settings_ns(st), tiles=tiles)
    for ti in tiles:
        ty0, ty1, tx0, tx1 = O.tile_list(cam.height, cam.width)[ti]
        _close(out.image[ty0:ty1, tx0:tx1], gold["image"][ty0:ty1, tx0:tx1])
