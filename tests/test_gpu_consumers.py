"""GPU tests of the callers either side of the path:
.ges -> device render, the CLI, and the winner-map consumer covering_counts."""

import json
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2504_17545_b200 as G  # noqa: E402
from paper_2504_17545_b200 import cli, scenes as S  # noqa: E402
from paper_2504_17545_b200.consumers import covering_counts  # noqa: E402
from paper_2504_17545_b200.gesfile import load_ges  # noqa: E402
from paper_2504_17545_b200.types import Camera  # noqa: E402
from golden_io import settings_ns  # noqa: E402
from oracle import ges_oracle as O  # noqa: E402
from parity import assert_parity, compare  # noqa: E402

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _cam(z):
    return Camera(float(z["fx"]), float(z["fy"]), float(z["cx"]), float(z["cy"]), int(z["width"]),
                  int(z["height"]), z["w2c"])


@pytest.mark.parametrize("name", ["ges_3d_deg3", "ges_2d_rgb"])
def test_ges_file_renders_like_reference(name):
    scene, _ = load_ges(os.path.join(GOLD, name + ".ges"))
    z = np.load(os.path.join(GOLD, name + "_load.npz"))
    cam = _cam(z)
    out = G.render(scene, cam)
    ora = O.render(scene, cam, settings_ns({}), ties=True)
    rep = compare(dict(image=out.image, s_winner=out.surfels.winner, s_depth=out.surfels.depth),
                  dict(image=z["image"], s_winner=z["s_winner"], s_depth=z["s_depth"]), ora.tie, tie_cut=ora.tie_cut)
    assert_parity(rep)


def test_cli_render_writes_png(tmp_path):
    from PIL import Image
    z = np.load(os.path.join(GOLD, "ges_3d_deg3_load.npz"))
    cam = _cam(z)
    (tmp_path / "cams.json").write_text(json.dumps([cli.camera_to_entry(cam)]))
    rc = cli.main(["render", "--model", os.path.join(GOLD, "ges_3d_deg3.ges"), "--camera",
                   str(tmp_path / "cams.json"), "--out", str(tmp_path / "o.png"), "--ss", "1"])
    assert rc == 0
    img = np.asarray(Image.open(tmp_path / "o.png")).astype(int)
    ref = np.clip(z["image"] * 255.0 + 0.5, 0, 255).astype(int)
    scene, _ = load_ges(os.path.join(GOLD, "ges_3d_deg3.ges"))
    tie = O.render(scene, cam, settings_ns({}), ties=True).tie
    assert np.abs(img - ref)[~tie].max() <= 1


def test_cli_path_and_errors(tmp_path):
    z = np.load(os.path.join(GOLD, "ges_2d_rgb_load.npz"))
    (tmp_path / "cams.json").write_text(json.dumps(cli.camera_to_entry(_cam(z))))
    rc = cli.main(["path", "--model", os.path.join(GOLD, "ges_2d_rgb.ges"), "--camera",
                   str(tmp_path / "cams.json"), "--out", str(tmp_path / "p"), "--frames", "5"])
    assert rc == 0
    assert len(list((tmp_path / "p").glob("frame_*.png"))) == 5
    # cli.py:154-174: the small orbit (metrics.camera_path) and the consistency probe
    from paper_2504_17545_b200 import metrics as M
    from paper_2504_17545_b200.forward import RenderSettings, render
    from paper_2504_17545_b200.gesfile import load_ges
    cams = M.camera_path(_cam(z), [0.0, 0.0, 0.0], frames=5, angle=0.02)
    path = json.loads((tmp_path / "p" / "path.json").read_text())
    assert np.allclose([e["w2c"] for e in path], [c.world_to_camera.reshape(-1) for c in cams])
    probe = json.loads((tmp_path / "p" / "probe.json").read_text())
    scene, _ = load_ges(os.path.join(GOLD, "ges_2d_rgb.ges"))
    imgs = [render(scene, c, RenderSettings(supersample=1)).image for c in cams]
    want = M.consistency_probe(None, cams, images=imgs)
    assert len(probe["max_change"]) == 4 and probe["bounds"] == []
    assert np.allclose(probe["max_change"], want["max_change"], atol=1e-5)
    assert np.allclose(probe["mean_change"], want["mean_change"], atol=1e-6)
    assert cli.main(["render", "--model", str(tmp_path / "missing.ges"), "--camera",
                     str(tmp_path / "cams.json"), "--out", str(tmp_path / "x.png")]) == 1


def test_covering_counts_match_oracle_winners():
    scene = S.random_scene(np.random.default_rng(8), 60, 0, degree=1)
    cams = S.orbit_views(3, 48, 40)
    got = covering_counts(scene, cams)
    best = np.zeros(60, np.int64)
    ties = 0
    for c in cams:
        o = O.rasterize_surfels(scene, c, settings_ns({}), ties=True)
        w = o.winner.reshape(-1)
        best = np.maximum(best, np.bincount(w[w >= 0], minlength=60))
        ties += int(o.tie.sum())
    # each flagged pixel can move at most one count from one surfel to another
    assert ties <= 2
    assert int(np.abs(got - best).sum()) <= 2 * ties
    assert got.sum() > 0
    # in float64 (the reference's covering_counts(..., dtype=np.float64)) the counts are exact
    got64 = covering_counts(scene, cams, dtype=np.float64)
    assert np.array_equal(got64, best)


def test_covering_counts_exact_like_reference():
    """test_optim.py:141-178: 10 stacked random surfels at 32x32 (rng 1234),
    per-surfel frontmost counts equal the brute-force scan exactly (the
    oracle flags no tie pixel on this scene)."""
    from paper_2504_17545_b200.types import GaussianSet, Scene, Stage
    rng = np.random.default_rng(1234)
    cam = S.make_camera()
    scene = Scene(S.random_surfels(rng, 10), GaussianSet.empty(1), 1, Stage.FROZEN)
    o = O.rasterize_surfels(scene, cam, settings_ns({}), ties=True)
    assert not o.tie.any()
    ref = np.bincount(o.winner[o.winner >= 0], minlength=10)
    assert np.array_equal(covering_counts(scene, [cam]), ref)


def test_scene_cache_replaced_and_invalidated_arrays():
    """Replacing an array re-packs the scene; in-place edits need invalidate()."""
    rng = np.random.default_rng(8)
    scene = S.random_scene(rng, 40, 30, degree=1)
    cam = S.make_camera(48, 40)
    a = G.render(scene, cam).image
    scene.surfels.pos = scene.surfels.pos + np.array([0.05, 0.0, 0.0])   # new array: detected
    b = G.render(scene, cam).image
    assert not np.array_equal(a, b)
    np.testing.assert_allclose(b, O.render(scene, cam, None).image, atol=1e-4)
    scene.gaussians.sh[...] *= 0.0                                        # in place: needs invalidate
    G.invalidate(scene)
    c = G.render(scene, cam).image
    np.testing.assert_allclose(c, O.render(scene, cam, None).image, atol=1e-4)
