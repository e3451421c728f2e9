"""GPU parity: the sm_100a kernels (through the C ABI via the drop-in API)
against the float64 oracle and the reference golden vectors.  Mirrors the
reference's own hot-path tests (pkg/tests/test_forward.py) with the float32
parity rule of tests/parity.py."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2504_17545_b200 as G  # noqa: E402
from paper_2504_17545_b200 import scenes as S  # noqa: E402
from paper_2504_17545_b200.types import (Camera, GaussianKind, GaussianSet, Scene, Stage,  # noqa: E402
                                         SurfelSet)
from golden_io import load, names, settings_ns  # noqa: E402
from oracle import ges_oracle as O  # noqa: E402
from parity import assert_parity, compare_oracle  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def gpu_dict(out):
    d = dict(image=out.image, s_winner=out.surfels.winner, s_depth=out.surfels.depth,
             s_color=out.surfels.color, s_normal=out.surfels.normal,
             g_color=out.gaussians.color, g_weight=out.gaussians.weight)
    if out.gaussians.depth is not None:
        d.update(g_depth=out.gaussians.depth, g_normal=out.gaussians.normal)
    return d


def ora_dict(out):
    d = dict(image=out.image, s_winner=out.surfels.winner, s_depth=out.surfels.depth,
             s_depth_err=out.surfels.depth_err, s_color=out.surfels.color, s_normal=out.surfels.normal,
             g_color=out.gaussians.color, g_weight=out.gaussians.weight)
    if out.gaussians.depth is not None:
        d.update(g_depth=out.gaussians.depth, g_normal=out.gaussians.normal)
    return d


def settings32(st):
    kw = {k: (tuple(v) if isinstance(v, list) else v) for k, v in st.items()}
    return G.RenderSettings(dtype=np.float32, **kw)


@pytest.mark.parametrize("name", names())
def test_golden_parity(name):
    """GPU vs the reference's own float64 output, ties from the oracle."""
    scene, cam, st, gold, _ = load(name)
    out = G.render(scene, cam, settings32(st))
    ora = O.render(scene, cam, settings_ns(st), ties=True)
    ref = dict(image=gold["image"], s_winner=gold["s_winner"], s_depth=gold["s_depth"],
               s_depth_err=ora.surfels.depth_err,
               s_color=gold["s_color"], s_normal=gold["s_normal"], g_color=gold["g_color"],
               g_weight=gold["g_weight"])
    if "g_depth" in gold:
        ref.update(g_depth=gold["g_depth"], g_normal=gold["g_normal"])
    rep = compare_oracle(gpu_dict(out), ref, ora)
    assert_parity(rep, weight_tol=5e-4)
    if "g_depth_maxabs" in rep:
        assert rep["g_depth_maxabs"] < 5e-4 and rep["g_normal_maxabs"] < 5e-4, rep


@pytest.mark.parametrize("seed", [0, 1])
def test_random_scene_480x270(seed):
    """Denser stress scene (the survey's fp32-vs-fp64 noise-floor setup, scaled)."""
    r = np.random.default_rng(seed)
    sc = Scene(S.random_surfels(r, 20000, 3, scale_range=(0.005, 0.02)),
               S.random_gaussians(r, 6000, 3, scale_range=(0.004, 0.025), extent=1.2), 3, Stage.FROZEN)
    cam = S.make_camera(480, 270)
    out = G.render(sc, cam)
    ora = O.render(sc, cam, settings_ns({}), ties=True)
    rep = compare_oracle(gpu_dict(out), ora_dict(ora), ora)
    assert_parity(rep)


def test_config2_tile_sample():
    """Full-size config 2 (1M surfels + 300k Gaussians, 1080p): GPU frame vs
    the oracle on a sample of tiles including the densest ones."""
    sc = S.config_scene(2)
    cam = S.config_cameras(2)[0]
    out = G.render(sc, cam)
    ntx = (cam.width + 15) // 16
    nt = ntx * ((cam.height + 15) // 16)
    rng = np.random.default_rng(5)
    tiles = sorted(set(rng.choice(nt, 12, replace=False).tolist() + [nt // 2 + ntx // 2, nt // 2]))
    ora = O.render(sc, cam, settings_ns({}, np.float64), tiles=tiles, ties=True)
    region = np.zeros((cam.height, cam.width), bool)
    for ti in tiles:
        ty0, ty1, tx0, tx1 = O.tile_list(cam.height, cam.width)[ti]
        region[ty0:ty1, tx0:tx1] = True
    rep = compare_oracle(gpu_dict(out), ora_dict(ora), ora, region=region)
    assert_parity(rep)
    assert rep["pixels"] >= 12 * 256


def test_config2_full_frame_properties():
    """Every pixel of the full config-2 frame through size-independent
    properties: the fused render equals its split entry points (surfel pass
    alone: identical winner/depth maps -- min over packed keys is order-free;
    Gaussian pass against that depth: the same accumulations to fp32 order
    noise; composite of the two: the image), coverage == finite depth, the
    winner's surfel is in view, and layer modes are consistent."""
    import torch
    sc = S.config_scene(2)
    cam = S.config_cameras(2)[0]
    full = G.render(sc, cam, to_numpy=False)
    sb = G.rasterize_surfels(sc, cam, to_numpy=False)
    assert torch.equal(full.surfels.winner, sb.winner)
    assert torch.equal(full.surfels.depth, sb.depth)
    assert torch.equal(full.surfels.coverage, torch.isfinite(full.surfels.depth))
    assert torch.equal(full.surfels.coverage, full.surfels.winner >= 0)
    assert float(full.surfels.coverage.float().mean()) > 0.5
    gb = G.accumulate_gaussians(sc, cam, sb.depth, to_numpy=False)
    assert torch.allclose(gb.weight, full.gaussians.weight, rtol=1e-5, atol=1e-6)
    assert torch.allclose(gb.color, full.gaussians.color, rtol=1e-5, atol=1e-6)
    img = G.composite(full.surfels.color, full.gaussians)
    assert float((img - full.image).abs().max()) <= 1e-6
    so = G.render(sc, cam, G.RenderSettings(layers="surfels_only"), to_numpy=False)
    assert torch.equal(so.image, full.surfels.color) and float(so.gaussians.weight.abs().max()) == 0.0
    # winners are surfels whose centre projects near the pixel (within the largest disc radius)
    ys, xs = torch.nonzero(full.surfels.coverage, as_tuple=True)
    pick = torch.randperm(len(ys), generator=torch.Generator().manual_seed(0))[:2000].to(ys.device)
    w = full.surfels.winner[ys[pick], xs[pick]].cpu().numpy()
    pc = sc.surfels.pos[w] @ np.asarray(cam.world_to_camera)[:3, :3].T + np.asarray(cam.world_to_camera)[:3, 3]
    px = cam.fx * pc[:, 0] / pc[:, 2] + cam.cx
    py = cam.fy * pc[:, 1] / pc[:, 2] + cam.cy
    rmax = 3.33 * float(np.exp(sc.surfels.log_scale.max())) * cam.fx / pc[:, 2].min()
    d = np.hypot(px - xs[pick].cpu().numpy() - 0.5, py - ys[pick].cpu().numpy() - 0.5)
    assert float(d.max()) <= rmax + 1.0


# ---- known-answer tests (test_forward.py:79-145) --------------------------------
def frontal(color=0.2, depth=3.0, scale=1.0):
    sh = np.zeros((1, 1, 3))
    sh[0, 0] = (color - 0.5) / 0.28209479177387814
    s = SurfelSet(np.array([[0.0, 0.0, depth]]), np.array([[1.0, 0, 0, 0]]),
                  np.log(np.full((1, 2), scale)), sh, np.array([255.0]))
    return Scene(s, GaussianSet.empty(0), 0, Stage.FROZEN)


def ident(w=32, h=32, f=40.0):
    return Camera(f, f, w / 2, h / 2, w, h, np.eye(4))


def test_single_surfel_centre():
    b = G.rasterize_surfels(frontal(0.8, 3.0), ident())
    assert b.coverage[16, 16]
    assert np.allclose(b.color[16, 16], 0.8, atol=1e-6)
    assert np.isclose(b.depth[16, 16], 3.0, rtol=1e-6)
    assert np.allclose(b.normal[16, 16], [0, 0, -1])
    assert b.winner[16, 16] == 0


def test_zbuffer_nearest_and_background():
    near, far = frontal(0.9, 2.0), frontal(0.1, 5.0)
    sc = Scene(SurfelSet(*(np.concatenate([getattr(far.surfels, k), getattr(near.surfels, k)])
                           for k in ("pos", "quat", "log_scale", "sh", "w"))),
               GaussianSet.empty(0), 0, Stage.FROZEN)
    b = G.rasterize_surfels(sc, ident(), G.RenderSettings(background=(0.25, 0.5, 0.75)))
    assert b.winner[16, 16] == 1 and np.allclose(b.color[16, 16], 0.9, atol=1e-6)
    small = G.rasterize_surfels(frontal(scale=0.1), ident(), G.RenderSettings(background=(0.25, 0.5, 0.75)))
    assert not small.coverage[0, 0] and np.isinf(small.depth[0, 0]) and small.winner[0, 0] == -1
    assert np.allclose(small.color[0, 0], [0.25, 0.5, 0.75])


def test_empty_scene_background():
    sc = Scene(SurfelSet.empty(0), GaussianSet.empty(0), 0, Stage.FROZEN)
    out = G.render(sc, ident(), G.RenderSettings(background=(0.1, 0.2, 0.3)))
    assert np.allclose(out.image, [0.1, 0.2, 0.3])


def test_footprint_boundary_radius():
    R = O.R_OPAQUE
    b = G.rasterize_surfels(frontal(1.0, 4.0, 1.0), ident(512, 512, 256.0))
    ys, xs = np.nonzero(b.coverage)
    rad = np.hypot(xs + 0.5 - 256.0, ys + 0.5 - 256.0) * 4.0 / 256.0
    assert rad.max() <= R + 1e-5
    xx, yy = np.meshgrid(np.arange(512) + 0.5, np.arange(512) + 0.5)
    inside = np.hypot(xx - 256.0, yy - 256.0) * 4.0 / 256.0 <= R - 0.01
    assert np.all(b.coverage[inside])


def test_centered_gaussian_weight():
    sh = np.zeros((1, 1, 3))
    sh[0, 0] = (0.9 - 0.5) / 0.28209479177387814
    g = GaussianSet(np.array([[0.0, 0.0, 2.0]]), np.log(np.array([0.8]) / 0.2), np.array([[1.0, 0, 0, 0]]),
                    np.log(np.full((1, 3), 0.3)), sh)
    sc = Scene(SurfelSet.empty(0), g, 0, Stage.FROZEN)
    gb = G.accumulate_gaussians(sc, ident(), np.full((32, 32), np.inf))
    d = np.array([0.5, 0.5])
    cov = (40.0 * 0.3 / 2.0) ** 2 * np.eye(2) + 0.3 * np.eye(2)
    expect = 0.8 * np.exp(-0.5 * d @ np.linalg.inv(cov) @ d)
    assert np.isclose(gb.weight[16, 16], expect, rtol=1e-5)
    assert np.allclose(gb.color[16, 16], expect * 0.9, rtol=1e-5)


def test_depth_gate():
    r = np.random.default_rng(1234)
    g = S.random_gaussians(r, 1, degree=0)
    g.pos[0] = [0.0, 0.0, 5.0]
    sc = Scene(SurfelSet.empty(0), g, 0, Stage.FROZEN)
    eps = O.gaussian_eff(g)[2][0]
    assert np.all(G.accumulate_gaussians(sc, ident(), np.full((32, 32), 5.0 - 2 * eps)).weight == 0)
    assert G.accumulate_gaussians(sc, ident(), np.full((32, 32), 5.0 + eps)).weight.max() > 0


def test_epsilon_monotonicity_and_pass_separation():
    r = np.random.default_rng(3)
    sc = S.random_scene(r, 10, 30)
    cam = S.make_camera()
    base = G.render(sc, cam)
    big = G.accumulate_gaussians(sc, cam, base.surfels.depth,
                                 G.RenderSettings(epsilon_mode="constant", epsilon_value=1e9))
    assert np.all(big.weight >= base.gaussians.weight - 1e-6)
    only = G.render(sc, cam, G.RenderSettings(layers="surfels_only"))
    gb = G.accumulate_gaussians(sc, cam, only.surfels.depth)
    re = G.composite(only.surfels.color, gb)
    assert np.max(np.abs(re - base.image)) <= 1e-6


def test_order_independence_permutation():
    r = np.random.default_rng(9)
    sc = S.random_scene(r, 10, 60)
    cam = S.make_camera()
    a = G.render(sc, cam)
    perm = r.permutation(60)
    sc2 = Scene(sc.surfels, sc.gaussians.select(perm), sc.sh_degree, sc.stage)
    b = G.render(sc2, cam)
    assert np.max(np.abs(a.image - b.image)) <= 1e-4
    sp = r.permutation(10)
    sc3 = Scene(sc.surfels.select(sp), sc.gaussians, sc.sh_degree, sc.stage)
    c = G.render(sc3, cam)
    inv = np.argsort(sp)
    mapped = np.where(c.surfels.winner >= 0, sp[np.maximum(c.surfels.winner, 0)], -1)
    assert np.array_equal(mapped, a.surfels.winner)


def test_run_to_run_deterministic_surfels():
    sc = S.config_scene(1)
    cam = S.config_cameras(1)[0]
    a = G.render(sc, cam)
    b = G.render(sc, cam)
    assert np.array_equal(a.surfels.winner, b.surfels.winner)
    assert np.array_equal(a.surfels.depth, b.surfels.depth)
    assert np.max(np.abs(a.image - b.image)) <= 1e-6


def test_near_plane_crossing_surfel():
    """A surfel spanning the focal plane gets whole-screen bounds
    (geometry.py:295-297) and still matches the oracle."""
    r = np.random.default_rng(4)
    s = S.random_surfels(r, 40, 1, scale_range=(0.1, 0.5))
    s.pos[0] = S.make_camera().position * 0.98
    s.log_scale[0] = np.log([2.0, 2.0])
    sc = Scene(s, S.random_gaussians(r, 30, 1), 1, Stage.FROZEN)
    cam = S.make_camera(64, 64)
    out = G.render(sc, cam)
    ora = O.render(sc, cam, settings_ns({}), ties=True)
    assert_parity(compare_oracle(gpu_dict(out), ora_dict(ora), ora))


def test_settings_validation():
    with pytest.raises(ValueError):
        G.RenderSettings(supersample=2)
    with pytest.raises(ValueError):
        G.RenderSettings(layers="nope")
    with pytest.raises(ValueError):
        G.RenderSettings(epsilon_mode="x")
    sc = S.random_scene(np.random.default_rng(0), 3, 3)
    with pytest.raises(NotImplementedError):
        G.render(sc, S.make_camera(), G.RenderSettings(dtype=np.float16))
    bad = Scene(S.random_surfels(np.random.default_rng(0), 3, 1), GaussianSet.empty(1), 1, Stage.FROZEN)
    bad.surfels.sh = np.zeros((3, 5, 3))
    with pytest.raises(ValueError):
        G.render(bad, S.make_camera())


def test_smooth_geometry_identity():
    sc = S.random_scene(np.random.default_rng(2), 10, 0)
    out = G.render(sc, S.make_camera(), G.RenderSettings(with_geometry=True))
    d, n = G.smooth_geometry(out.surfels, out.gaussians)
    assert np.array_equal(d, out.surfels.depth)
    cov = out.surfels.coverage
    assert np.allclose(n[cov], out.surfels.normal[cov], atol=1e-6)
    with pytest.raises(ValueError):
        G.smooth_geometry(out.surfels, G.GaussianBuffers(out.gaussians.color, out.gaussians.weight))


def test_supersample4_480x270_stress():
    r = np.random.default_rng(21)
    sc = Scene(S.random_surfels(r, 15000, 2, scale_range=(0.006, 0.02)),
               S.random_gaussians(r, 4000, 2, scale_range=(0.004, 0.02), extent=1.2), 2, Stage.FROZEN)
    cam = S.make_camera(480, 270)
    st = {"supersample": 4, "background": [0.1, 0.2, 0.3]}
    out = G.render(sc, cam, settings32(st))
    ora = O.render(sc, cam, settings_ns(st), ties=True)
    assert_parity(compare_oracle(gpu_dict(out), ora_dict(ora), ora))


def test_mip_filtered_scene_multiscale():
    """Config-4 style: world-filtered Gaussians + mip=True at two scales."""
    r = np.random.default_rng(22)
    g = S.random_gaussians(r, 5000, 3, scale_range=(0.002, 0.02), extent=1.2)
    sc = Scene(S.random_surfels(r, 12000, 3, scale_range=(0.004, 0.016)),
               S.mip_world_filter(g, [S.make_camera(960, 540)]), 3, Stage.FROZEN)
    for w, h in ((120, 68), (480, 270)):
        cam = S.make_camera(w, h)
        out = G.render(sc, cam, settings32({"mip": True}))
        ora = O.render(sc, cam, settings_ns({"mip": True}), ties=True)
        assert_parity(compare_oracle(gpu_dict(out), ora_dict(ora), ora))


def test_pair_list_overflow_grows_and_rerenders():
    """A too-small pair capacity is detected on the device, reported in the
    frame status, and the checked render grows the lists and re-renders."""
    from paper_2504_17545_b200.renderer import DeviceScene, Renderer
    sc = S.random_scene(np.random.default_rng(6), 300, 200, degree=1)
    cam = S.make_camera(96, 64)
    ds = DeviceScene(sc)
    r = Renderer()
    st = G.RenderSettings()
    r._caps(ds, 1)
    r.cap_s, r.cap_g = 16, 16                      # force overflow
    orig_caps = r._caps
    r._caps = lambda ds_, ss: None                 # keep the tiny capacity for the first attempt
    fr = r.render(ds, cam, st, check=False)
    sp, gp, ovf = fr.pairs()
    assert ovf and sp > 16
    r._caps = orig_caps
    fr = r.render(ds, cam, st, check=True)
    assert fr.pairs()[2] == 0
    ref = G.render(sc, cam)
    assert np.array_equal(fr.s_winner.cpu().numpy(), ref.surfels.winner)
    assert np.max(np.abs(fr.image.cpu().numpy() - ref.image)) <= 1e-6


def test_view_batch_streams_and_graph_match_single_renders():
    from paper_2504_17545_b200.multiview import ViewBatchRenderer
    from paper_2504_17545_b200.renderer import DeviceScene, Renderer
    sc = S.random_scene(np.random.default_rng(10), 2000, 800, degree=3)
    cams = S.orbit_views(6, 128, 96)
    ds = DeviceScene(sc)
    st = G.RenderSettings()
    vb = ViewBatchRenderer(Renderer(), ds, cams, st, want=("image", "s_winner", "image_rgba8"), streams=2)
    for rr in vb.pool:
        for c, fr in zip(vb.cams, vb.frames):
            rr.render(ds, c, st, frame=fr, check=True)
    assert vb.capture()
    for _ in range(2):
        vb.render()
    torch.cuda.synchronize()
    assert not vb.overflowed()
    for c, fr, rgba in zip(cams, vb.frames, vb.rgba):
        ref = G.render(sc, c)
        assert np.array_equal(fr.s_winner.cpu().numpy(), ref.surfels.winner)
        assert np.max(np.abs(fr.image.cpu().numpy() - ref.image)) <= 1e-6
        q = np.clip(ref.image * 255.0 + 0.5, 0, 255).astype(np.int32)
        assert np.abs(rgba[..., :3].cpu().numpy().astype(np.int32) - q).max() <= 1


def test_view_batch_float_outputs_only():
    """Without "image_rgba8" (the N = 1 bench batch) no RGBA8 frame exists and
    the float outputs are those of single renders."""
    from paper_2504_17545_b200.multiview import ViewBatchRenderer
    from paper_2504_17545_b200.renderer import DeviceScene, Renderer
    sc = S.random_scene(np.random.default_rng(11), 2000, 800, degree=3)
    cams = S.orbit_views(4, 128, 96)
    ds = DeviceScene(sc)
    st = G.RenderSettings()
    vb = ViewBatchRenderer(Renderer(), ds, cams, st, want=("image", "s_depth", "s_winner"), streams=2)
    assert vb.rgba is None and all(fr.image_rgba8 is None for fr in vb.frames)
    for rr in vb.pool:
        for c, fr in zip(vb.cams, vb.frames):
            rr.render(ds, c, st, frame=fr, check=True)
    assert vb.capture()
    assert vb.render() is None
    torch.cuda.synchronize()
    assert not vb.overflowed()
    for c, fr in zip(cams, vb.frames):
        ref = G.render(sc, c)
        assert np.array_equal(fr.s_winner.cpu().numpy(), ref.surfels.winner)
        assert np.max(np.abs(fr.image.cpu().numpy() - ref.image)) <= 1e-6
        d, rd = fr.s_depth.cpu().numpy(), ref.surfels.depth
        assert np.array_equal(np.isinf(d), np.isinf(rd))
        assert np.max(np.abs(d - rd)[np.isfinite(rd)]) <= 1e-6 * max(1.0, np.abs(rd[np.isfinite(rd)]).max())


def _tile_region(cam, tiles):
    region = np.zeros((cam.height, cam.width), bool)
    for ti in tiles:
        ty0, ty1, tx0, tx1 = O.tile_list(cam.height, cam.width)[ti]
        region[ty0:ty1, tx0:tx1] = True
    return region


def test_camera_inside_scene_near_plane():
    """Camera inside the primitive cloud: many surfels straddle the focal
    plane (whole-screen ranges, geometry.py:295-297) or lie behind it."""
    r = np.random.default_rng(33)
    sc = Scene(S.random_surfels(r, 3000, 2, scale_range=(0.01, 0.05)),
               S.random_gaussians(r, 1500, 2, scale_range=(0.01, 0.05), extent=1.2), 2, Stage.FROZEN)
    cam = S.make_camera(160, 120, dist=0.3)
    out = G.render(sc, cam)
    ora = O.render(sc, cam, settings_ns({}), ties=True)
    assert_parity(compare_oracle(gpu_dict(out), ora_dict(ora), ora))


def test_4k_supersampled_config2_scene_tile_sample():
    """The config-2 scene at 3840x2160 with supersample=4 (7680x4320 surfel
    pass): GPU frame vs the oracle on sampled tiles."""
    sc = S.config_scene(2, scale_down=4)
    cam = S.make_camera(3840, 2160)
    st = {"supersample": 4}
    out = G.render(sc, cam, settings32(st))
    nt = ((cam.width + 15) // 16) * ((cam.height + 15) // 16)
    tiles = sorted(np.random.default_rng(9).choice(nt, 6, replace=False).tolist() + [nt // 2 + 120])
    ora = O.render(sc, cam, settings_ns(st), tiles=tiles, ties=True)
    rep = compare_oracle(gpu_dict(out), ora_dict(ora), ora, region=_tile_region(cam, tiles))
    assert_parity(rep)


def test_8k_frame_tile_sample_and_consistency():
    """7680x4320 (and its 15360x8640 supersampled surfel pass): span packing,
    tile counts and pair capacities at 8K; sampled tiles against the oracle
    and, over every pixel, coverage == finite depth == winner >= 0."""
    sc = S.config_scene(2, scale_down=4)
    cam = S.make_camera(7680, 4320)
    for ss in (1, 4):
        st = {"supersample": ss}
        out = G.render(sc, cam, settings32(st))
        cov = out.surfels.winner >= 0
        assert np.array_equal(cov, np.isfinite(out.surfels.depth)) and np.isfinite(out.image).all()
        assert cov.mean() > 0.1
        nt = ((cam.width + 15) // 16) * ((cam.height + 15) // 16)
        tiles = sorted(np.random.default_rng(10 + ss).choice(nt, 6, replace=False).tolist() + [nt // 2 + 240])
        ora = O.render(sc, cam, settings_ns(st), tiles=tiles, ties=True)
        assert_parity(compare_oracle(gpu_dict(out), ora_dict(ora), ora, region=_tile_region(cam, tiles)))


def test_planar_gaussians_dense_with_geometry():
    r = np.random.default_rng(44)
    sc = Scene(S.random_surfels(r, 8000, 1, scale_range=(0.008, 0.03)),
               S.random_gaussians(r, 4000, 1, kind=GaussianKind.TWO_D, scale_range=(0.006, 0.03),
                                  extent=1.2), 1, Stage.FROZEN)
    cam = S.make_camera(320, 200)
    st = {"with_geometry": True, "mip": True}
    out = G.render(sc, cam, settings32(st))
    ora = O.render(sc, cam, settings_ns(st), ties=True)
    rep = compare_oracle(gpu_dict(out), ora_dict(ora), ora)
    assert_parity(rep)
    assert rep["g_depth_maxabs"] < 1e-3 and rep["g_normal_maxabs"] < 1e-3, rep


@pytest.mark.parametrize("kind,tile_mode", [("3d", 2), ("3d", 1), ("2d", 2)])
def test_offscreen_and_edge_straddling_primitives(kind, tile_mode):
    """The preprocess drops primitives whose (padded) support box misses the
    image, where the reference clamps them onto the edge tiles and rejects
    them pixel by pixel (forward.py:85-96): a close, narrow view of the cloud
    leaves most primitives off-screen on every side and many straddling the
    edges; every pixel, both tile layouts, against the oracle."""
    r = np.random.default_rng(46)
    gk = GaussianKind.TWO_D if kind == "2d" else GaussianKind.THREE_D
    sc = Scene(S.random_surfels(r, 20000, 2, scale_range=(0.005, 0.03)),
               S.random_gaussians(r, 8000, 2, kind=gk, scale_range=(0.004, 0.03), extent=1.2), 2, Stage.FROZEN)
    cam = S.make_camera(640, 120, dist=2.2, fov=20.0)   # wide, short frame: top/bottom edges cut the cloud
    s32 = settings32({})
    s32.tile_mode = tile_mode
    out = G.render(sc, cam, s32)
    ora = O.render(sc, cam, settings_ns({}), ties=True)
    assert_parity(compare_oracle(gpu_dict(out), ora_dict(ora), ora))
    # most candidates really were off-screen: the pair count stays far below the reference's
    # clamped candidate lists' total
    full = int(O.surfel_tile_counts(sc, cam).sum()) if tile_mode == 1 else None
    if full is not None:
        from paper_2504_17545_b200.renderer import SCENE_CACHE, default_renderer
        ds = SCENE_CACHE.get(sc, torch.device("cuda", torch.cuda.current_device()))
        fr = default_renderer().render(ds, cam, s32, mode=1, want=("s_winner",))
        sp, _, _ = fr.pairs()
        assert sp < full, (sp, full)


def test_odd_sizes_and_aspect():
    sc = S.random_scene(np.random.default_rng(45), 400, 200, degree=1)
    for w, h in ((17, 33), (1, 1), (257, 3)):
        cam = S.make_camera(w, h)
        out = G.render(sc, cam)
        ora = O.render(sc, cam, settings_ns({}), ties=True)
        assert_parity(compare_oracle(gpu_dict(out), ora_dict(ora), ora))


@pytest.mark.parametrize("name", ["g3d_500", "g2d_901", "bg_gonly", "bg_sonly", "eps_const", "mip3d",
                                  "deg3_64x48", "config1"])
def test_golden_parity_2x2_pixel_tiles(name):
    """The 32x32-tile / 2x2-pixels-per-thread kernel variant (auto-selected
    for large plain frames) forced on the golden cases."""
    scene, cam, st, gold, _ = load(name)
    s32 = settings32(st)
    s32.tile_mode = 2
    out = G.render(scene, cam, s32)
    ora = O.render(scene, cam, settings_ns(st), ties=True)
    ref = dict(image=gold["image"], s_winner=gold["s_winner"], s_depth=gold["s_depth"],
               s_depth_err=ora.surfels.depth_err,
               s_color=gold["s_color"], s_normal=gold["s_normal"], g_color=gold["g_color"],
               g_weight=gold["g_weight"])
    assert_parity(compare_oracle(gpu_dict(out), ref, ora), weight_tol=5e-4)


def test_tile_modes_agree_480x270():
    r = np.random.default_rng(46)
    sc = Scene(S.random_surfels(r, 20000, 3, scale_range=(0.005, 0.02)),
               S.random_gaussians(r, 6000, 3, scale_range=(0.004, 0.025), extent=1.2), 3, Stage.FROZEN)
    cam = S.make_camera(481, 271)
    outs = []
    for mode in (1, 2):
        st = G.RenderSettings()
        st.tile_mode = mode
        outs.append(G.render(sc, cam, st))
    assert np.array_equal(outs[0].surfels.winner, outs[1].surfels.winner)
    assert np.max(np.abs(outs[0].image - outs[1].image)) <= 1e-5
    ora = O.render(sc, cam, settings_ns({}), ties=True)
    assert_parity(compare_oracle(gpu_dict(outs[1]), ora_dict(ora), ora))


GEO = ("geo_match", "geo_bridge", "geo_rand3d", "geo_rand2d")


def _golden_npz(name):
    import os
    from golden_io import GOLDEN_DIR
    return np.load(os.path.join(GOLDEN_DIR, name + ".npz"))


def _close_nan(a, b, tol, mask=None):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    if mask is not None:
        a, b = a[mask], b[mask]
    assert np.array_equal(np.isnan(a), np.isnan(b)) and np.array_equal(np.isinf(a), np.isinf(b))
    f = np.isfinite(b)
    err = float(np.max(np.abs(a[f] - b[f]))) if f.any() else 0.0
    assert err <= tol, err
    return err


@pytest.mark.parametrize("name", GEO)
def test_smooth_geometry_and_composite_ops_on_reference_buffers(name):
    """The device smooth_geometry / composite kernels applied to the
    reference's own float64 buffers (forward.py:384-400) reproduce the
    reference's outputs (test_forward.py:163-180, :255-300 scenes)."""
    z = _golden_npz(name)
    sb = G.SurfelBuffers(z["s_color"], z["s_depth"], z["s_normal"], np.isfinite(z["s_depth"]), z["s_winner"])
    gb = G.GaussianBuffers(z["g_color"], z["g_weight"], z["g_depth"], z["g_normal"])
    d, n = G.smooth_geometry(sb, gb)
    _close_nan(d, z["smooth_depth"], 1e-5)
    _close_nan(n, z["smooth_normal"], 1e-5)
    for i, w in enumerate(z["composite_weights"]):
        _close_nan(G.composite(z["s_color"], gb, surfel_weight=float(w)), z[f"composite_{i}"], 1e-5)


@pytest.mark.parametrize("name", GEO)
def test_smooth_geometry_and_composite_end_to_end(name):
    """Render with geometry on the device, then smooth_geometry and
    composite(surfel_weight in 0, 0.5, 1, 2) against the reference's float64
    results on the same scene.  Hard ties (oracle) are excluded and bounded;
    pixels with a Gaussian fragment at the 1/255 cutoff (tests/parity.py)
    are checked against the change one flipped fragment can cause (alpha
    <= CUT_FLIP times the value range, divided by the blend denominator),
    except composite(surfel_weight=0), whose pure-Gaussian ratio has no such
    bound (counted instead); every other pixel within 1e-4."""
    from parity import CUT_FLIP
    scene, cam, st, gold, _ = load(name)
    z = _golden_npz(name)
    out = G.render(scene, cam, settings32(st))
    ora = O.render(scene, cam, settings_ns(st), ties=True)
    hard = ora.tie
    cut = np.where(hard, 0, ora.tie_cut)
    assert hard.sum() <= max(0.005 * hard.size, 2)
    keep = ~hard
    gw = np.asarray(z["g_weight"])
    d, n = G.smooth_geometry(out.surfels, out.gaussians)
    sd = z["smooth_depth"]
    fin = np.isfinite(sd)
    assert np.array_equal(np.isfinite(d)[keep], fin[keep])
    # one flipped fragment (alpha ~ 1/255, depth t <= the frame's depth range) per flagged count
    dr = float(np.max(np.abs(sd[fin]))) if fin.any() else 1.0
    tol_d = 1e-4 * np.maximum(np.abs(sd), 1.0) + cut * CUT_FLIP * 2.0 * dr / (1.0 + gw)
    m = keep & fin
    assert np.all(np.abs(d[m] - sd[m]) <= tol_d[m])
    tol_n = 1e-4 + cut * CUT_FLIP * 4.0 / (1.0 + gw)
    assert np.all(np.abs(n - z["smooth_normal"]).max(axis=-1)[keep] <= tol_n[keep])
    cmax = float(np.max(np.abs(z["s_color"]))) + float(np.max(np.abs(z["g_color"] / np.maximum(gw, 1e-12)[..., None])))
    for i, w in enumerate(z["composite_weights"]):
        img = G.composite(out.surfels.color, out.gaussians, surfel_weight=float(w))
        ref = z[f"composite_{i}"]
        if w == 0.0:
            m = keep & (cut == 0)
            assert (keep & (cut > 0)).sum() <= 0.05 * keep.size
            _close_nan(img, ref, 1e-4, mask=m)
        else:
            tol = 1e-4 + cut * CUT_FLIP * 2.0 * cmax / (w + gw)
            err = np.abs(np.asarray(img, np.float64) - ref).max(axis=-1)
            assert np.all(err[keep] <= tol[keep])
    if name == "geo_match":   # test_forward.py:263-276: depth unchanged by an on-plane Gaussian
        assert abs(float(d[16, 16]) - 3.0) <= 1e-5
    if name == "geo_bridge":  # test_forward.py:278-300: the seam is softened
        row = 16
        f = np.isfinite(out.surfels.depth[row])
        assert np.abs(np.diff(d[row][f])).max() < np.abs(np.diff(out.surfels.depth[row][f])).max()
