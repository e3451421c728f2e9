"""Randomised parity sweep: 96 seeded combinations of every render setting
(Gaussian kind, SH degree, supersample, mip, layers, geometry, epsilon mode,
background, tile layout), scene density and primitive size, camera distance
and odd resolutions.  The float32 kernels are held to the parity rule
(tests/parity.py) against the float64 oracle; the float64 kernels must match
the oracle to 1e-9 on every pixel."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2504_17545_b200 as G  # noqa: E402
from paper_2504_17545_b200 import scenes as S  # noqa: E402
from paper_2504_17545_b200.types import GaussianKind, GaussianSet, Scene, Stage  # noqa: E402
from golden_io import settings_ns  # noqa: E402
from oracle import ges_oracle as O  # noqa: E402
from parity import assert_parity, compare_oracle  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _case(seed):
    r = np.random.default_rng(1000 + seed)
    kind = GaussianKind.TWO_D if r.random() < 0.4 else GaussianKind.THREE_D
    deg = int(r.integers(0, 4))
    ns = int(r.integers(50, 3000)) if seed % 16 else 0   # every 16th case: Gaussians only
    ng = int(r.integers(0, 1500)) if r.random() < 0.9 else 0
    s_lo = float(r.uniform(0.005, 0.05))
    g_lo = float(r.uniform(0.004, 0.05))
    surf = S.random_surfels(r, ns, deg, scale_range=(s_lo, s_lo * r.uniform(1.5, 4.0)))
    if seed % 16 == 8:   # ... and every 16th a single surfel
        surf = surf.select(np.arange(1))
    gs = (S.random_gaussians(r, ng, deg, kind=kind, scale_range=(g_lo, g_lo * r.uniform(1.5, 4.0)), extent=1.2)
          if ng else GaussianSet.empty(deg))
    w, h = int(r.integers(16, 200)), int(r.integers(16, 150))
    cam = S.make_camera(w, h, dist=float(r.uniform(0.8, 6.0)), azim=float(r.uniform(0, 6.28)),
                        elev=float(r.uniform(-0.8, 0.8)), fov=float(r.uniform(20, 80)))
    mip = bool(r.random() < 0.3)
    if mip and ng and kind is GaussianKind.THREE_D:
        gs = S.mip_world_filter(gs, [S.make_camera(w * 2, h * 2)])
    st = {"supersample": 4 if r.random() < 0.3 else 1, "mip": mip,
          "layers": ["full", "full", "surfels_only", "gaussians_only"][int(r.integers(0, 4))],
          "with_geometry": bool(r.random() < 0.3),
          "background": [float(x) for x in r.uniform(0, 1, 3)] if r.random() < 0.5 else [0.0, 0.0, 0.0]}
    if r.random() < 0.25:
        st.update(epsilon_mode="constant", epsilon_value=float(r.uniform(0.0, 0.1)))
    tile_mode = int(r.integers(0, 3))
    return Scene(surf, gs, deg, Stage.FROZEN), cam, st, tile_mode


def _settings(st, dtype):
    kw = {k: (tuple(v) if isinstance(v, list) else v) for k, v in st.items()}
    return G.RenderSettings(dtype=dtype, **kw)


def _dicts(out, ora):
    g = dict(image=out.image, s_winner=out.surfels.winner, s_depth=out.surfels.depth, s_color=out.surfels.color,
             g_color=out.gaussians.color, g_weight=out.gaussians.weight)
    o = dict(image=ora.image, s_winner=ora.surfels.winner, s_depth=ora.surfels.depth, s_color=ora.surfels.color,
             g_color=ora.gaussians.color, g_weight=ora.gaussians.weight)
    return g, o


@pytest.mark.parametrize("seed", range(96))
def test_fuzz_float32_and_float64(seed):
    scene, cam, st, tile_mode = _case(seed)
    ora = O.render(scene, cam, settings_ns(st), ties=True)
    s32 = _settings(st, np.float32)
    s32.tile_mode = tile_mode
    out = G.render(scene, cam, s32)
    g, o = _dicts(out, ora)
    assert_parity(compare_oracle(g, o, ora), weight_tol=5e-4)
    out64 = G.render(scene, cam, _settings(st, np.float64))
    np.testing.assert_array_equal(out64.surfels.winner, ora.surfels.winner)
    for a, b in ((out64.image, ora.image), (out64.surfels.depth, ora.surfels.depth),
                 (out64.gaussians.weight, ora.gaussians.weight), (out64.gaussians.color, ora.gaussians.color)):
        fa, fb = np.isfinite(a), np.isfinite(b)
        assert np.array_equal(fa, fb)
        if fb.any():
            assert float(np.max(np.abs(a[fb] - b[fb]))) <= 1e-9 * max(1.0, float(np.abs(b[fb]).max()))
