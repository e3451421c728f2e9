"""Float64 render mode (RenderSettings(dtype=np.float64), forward.py:44):
the reference's own test suite renders in float64 (pkg/tests/
test_forward.py:33-35).  The drop-in's float64 kernels (ges_render_f64) are
compared with the reference's float64 goldens (tests/golden, written by the
real reference) at 1e-9 -- float64 summation order is the only difference --
and with the float64 oracle on larger scenes.  No pixel is exempt: every
winner must be identical and every value within 1e-9 (the float32 tie flags
are not needed at float64 precision)."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2504_17545_b200 as G  # noqa: E402
from paper_2504_17545_b200 import scenes as S  # noqa: E402
from paper_2504_17545_b200.types import Scene, Stage  # noqa: E402
from golden_io import load, names, settings_ns  # noqa: E402
from oracle import ges_oracle as O  # noqa: E402

ATOL = 1e-9


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def settings64(st):
    kw = {k: (tuple(v) if isinstance(v, list) else v) for k, v in st.items()}
    return G.RenderSettings(dtype=np.float64, **kw)


def _check(out, ref, tie, *, atol=ATOL, name=""):
    """ref: dict of float64 reference buffers.  Returns (winner mismatches, of which on ties)."""
    assert out.image.dtype == np.float64 and out.surfels.depth.dtype == np.float64
    mism = out.surfels.winner != ref["s_winner"]
    assert int((mism & ~tie).sum()) == 0, (name, int(mism.sum()))
    keep = ~tie
    for k, a in (("image", out.image), ("s_color", out.surfels.color), ("s_depth", out.surfels.depth),
                 ("s_normal", out.surfels.normal), ("g_color", out.gaussians.color),
                 ("g_weight", out.gaussians.weight), ("g_depth", out.gaussians.depth),
                 ("g_normal", out.gaussians.normal)):
        if k not in ref or ref[k] is None or a is None:
            continue
        b = np.asarray(ref[k])
        fa, fb = np.isfinite(a), np.isfinite(b)
        assert np.array_equal(fa[keep], fb[keep]), (name, k)
        m = keep & (fa.all(-1) if fa.ndim == 3 else fa)
        with np.errstate(invalid="ignore"):
            d = np.abs(a - b)
        err = float(d[m].max()) if m.any() else 0.0
        assert err <= atol * max(1.0, float(np.abs(b[np.isfinite(b)]).max(initial=1.0))), (name, k, err)
    return int(mism.sum())


@pytest.mark.parametrize("name", names())
def test_float64_matches_reference_goldens(name):
    scene, cam, st, gold, _ = load(name)
    out = G.render(scene, cam, settings64(st))
    ora = O.render(scene, cam, settings_ns(st), ties=True)
    assert _check(out, gold, np.zeros_like(ora.tie), name=name) == 0


def test_float64_split_entry_points_and_layers():
    """rasterize_surfels / accumulate_gaussians / composite / smooth_geometry
    in float64 equal the reference's buffers (geometry golden)."""
    scene, cam, st, gold, _ = load("geo_rand3d")
    z = np.load(__import__("os").path.join(__import__("golden_io").GOLDEN_DIR, "geo_rand3d.npz"))
    s64 = settings64(st)
    sb = G.rasterize_surfels(scene, cam, s64)
    assert sb.depth.dtype == np.float64
    np.testing.assert_array_equal(sb.winner, gold["s_winner"])
    np.testing.assert_allclose(sb.color, gold["s_color"], atol=ATOL, rtol=0)
    gb = G.accumulate_gaussians(scene, cam, gold["s_depth"], s64)
    np.testing.assert_allclose(gb.weight, gold["g_weight"], atol=ATOL, rtol=0)
    np.testing.assert_allclose(gb.color, gold["g_color"], atol=ATOL, rtol=0)
    np.testing.assert_allclose(gb.depth, gold["g_depth"], atol=ATOL, rtol=0)
    d, n = G.smooth_geometry(sb, gb)
    np.testing.assert_allclose(d, z["smooth_depth"], atol=ATOL, rtol=0)
    np.testing.assert_allclose(n, z["smooth_normal"], atol=ATOL, rtol=0)
    for i, w in enumerate(z["composite_weights"]):
        img = G.composite(sb.color, gb, surfel_weight=float(w))
        np.testing.assert_allclose(img, z[f"composite_{i}"], atol=ATOL, rtol=0, equal_nan=True)


@pytest.mark.parametrize("seed,kind,ss", [(0, "3d", 1), (1, "2d", 1), (2, "3d", 4)])
def test_float64_random_scene_480x270_vs_oracle(seed, kind, ss):
    r = np.random.default_rng(seed)
    gk = G.GaussianKind.TWO_D if kind == "2d" else G.GaussianKind.THREE_D
    sc = Scene(S.random_surfels(r, 20000, 3, scale_range=(0.005, 0.02)),
               S.random_gaussians(r, 6000, 3, scale_range=(0.004, 0.025), extent=1.2, kind=gk), 3, Stage.FROZEN)
    cam = S.make_camera(480, 270)
    st = {"supersample": ss, "with_geometry": True} if ss == 1 else {"supersample": ss}
    out = G.render(sc, cam, settings64(st))
    ns = settings_ns(st)
    ns.threads = 8
    ora = O.render(sc, cam, ns, ties=True)
    ref = dict(image=ora.image, s_winner=ora.surfels.winner, s_depth=ora.surfels.depth,
               s_color=ora.surfels.color, s_normal=ora.surfels.normal, g_color=ora.gaussians.color,
               g_weight=ora.gaussians.weight, g_depth=ora.gaussians.depth, g_normal=ora.gaussians.normal)
    assert _check(out, ref, np.zeros_like(ora.tie), name=f"rand{seed}") == 0


def test_float64_config2_full_frame_vs_oracle():
    """Config 2 (1M surfels + 300k Gaussians, SH3, 1920x1080) in float64."""
    sc = S.config_scene(2)
    cam = S.config_cameras(2)[0]
    out = G.render(sc, cam, G.RenderSettings(dtype=np.float64))
    ns = settings_ns({})
    ns.threads = 16
    ora = O.render(sc, cam, ns, ties=True)
    ref = dict(image=ora.image, s_winner=ora.surfels.winner, s_depth=ora.surfels.depth,
               g_weight=ora.gaussians.weight)
    n = _check(out, ref, np.zeros_like(ora.tie), name="config2")
    print(f"\n[config2 float64] winner differences: {n} (float32 tie flags: {int(ora.tie.sum())})")
    assert n == 0
