"""Evaluation surface: PSNR/SSIM against golden values
produced by the real reference (tests/golden/make_metrics_golden.py), the
dataset loader, and -- on the GPU -- ``metrics.evaluate`` and ``eval``."""
import json
import os

import numpy as np
import pytest

from paper_2504_17545_b200 import datasets as D, metrics as M

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "metrics.npz")


@pytest.mark.parametrize("case", ["rgb", "small", "gray", "wide"])
def test_psnr_ssim_match_reference(case):
    g = np.load(GOLD)
    a, b = g[f"{case}_a"], g[f"{case}_b"]
    assert M.psnr(a, b) == pytest.approx(float(g[f"{case}_psnr"]), rel=1e-12)
    assert M.ssim(a, b) == pytest.approx(float(g[f"{case}_ssim"]), rel=1e-10)


def test_identical_and_errors():
    g = np.load(GOLD)
    a = g["rgb_a"]
    assert M.psnr(a, a) == float("inf") == float(g["same_psnr"])
    assert M.ssim(a, a) == pytest.approx(1.0, abs=1e-12)
    with pytest.raises(ValueError):
        M.psnr(a, a[:-1])
    with pytest.raises(ValueError):
        M.ssim(a[:10], a[:10])   # smaller than the 11-pixel window
    rep = M.EvalReport(per_view_psnr=[float("inf"), 30.0])
    assert json.loads(rep.to_json())["per_view_psnr"] == ["inf", 30.0]


def _write_dataset(root, cams, imgs, ply=True):
    from PIL import Image

    from paper_2504_17545_b200.cli import camera_to_entry
    (root / "images").mkdir(parents=True, exist_ok=True)
    entries = []
    for i, (c, im) in enumerate(zip(cams, imgs)):
        rel = f"images/{i:04d}.png"
        Image.fromarray(np.clip(im * 255.0 + 0.5, 0, 255).astype(np.uint8)).save(root / rel)
        entries.append(dict(camera_to_entry(c), image=rel))
    (root / "cameras.json").write_text(json.dumps(entries))
    if ply:
        pts = np.arange(12, dtype=np.float32).reshape(4, 3)
        hdr = (b"ply\nformat binary_little_endian 1.0\nelement vertex 4\nproperty float x\n"
               b"property float y\nproperty float z\nproperty uchar red\nproperty uchar green\n"
               b"property uchar blue\nend_header\n")
        rec = np.zeros(4, dtype=[("xyz", "<f4", 3), ("rgb", "u1", 3)])
        rec["xyz"], rec["rgb"] = pts, 255
        (root / "points.ply").write_bytes(hdr + rec.tobytes())


def test_load_dataset_split_and_errors(tmp_path):
    from paper_2504_17545_b200 import scenes as S
    cams = [S.make_camera(24, 16, azim=0.1 * k) for k in range(10)]
    rng = np.random.default_rng(0)
    imgs = [rng.random((16, 24, 3)) for _ in cams]
    _write_dataset(tmp_path, cams, imgs)
    ds = D.load_dataset(tmp_path, test_every=4)
    assert ds.test_idx == [0, 4, 8] and len(ds.train_idx) == 7
    assert np.abs(ds.images[3] - imgs[3]).max() <= 0.5 / 255 + 1e-12   # 8-bit round trip
    assert ds.cameras[2].width == 24 and np.allclose(ds.cameras[2].world_to_camera, cams[2].world_to_camera)
    assert ds.points.shape == (4, 3) and np.all(ds.point_colors == 1.0)
    with pytest.raises(D.DatasetError):
        D.load_dataset(tmp_path / "missing")
    (tmp_path / "images" / "0001.png").unlink()
    with pytest.raises(D.DatasetError):
        D.load_dataset(tmp_path)


@pytest.mark.gpu
def test_evaluate_and_eval_command_on_gpu(tmp_path):
    import paper_2504_17545_b200 as G
    from paper_2504_17545_b200 import cli, scenes as S
    from paper_2504_17545_b200.gesfile import save_ges
    rng = np.random.default_rng(5)
    scene = G.Scene(S.random_surfels(rng, 3000, 3, scale_range=(0.02, 0.08)),
                    S.random_gaussians(rng, 800, 3, scale_range=(0.01, 0.05), extent=1.2), 3, G.Stage.FROZEN)
    cams = [S.make_camera(64, 48, azim=0.3 + 0.2 * k) for k in range(6)]
    st = G.RenderSettings(supersample=4)
    imgs = [G.render(scene, c, st).image for c in cams]
    imgs[2] = np.clip(imgs[2] + 0.02, 0, 1)
    ds = D.Dataset(cams, imgs)
    ds.split(2)                                   # test views 0, 2, 4
    rep = M.evaluate(scene, ds, settings=st)
    # renders repeat to ~1e-7 (Gaussian sums in list order, which the atomic binning fixes per run)
    assert rep.per_view_psnr[0] > 120.0 and rep.per_view_ssim[0] == pytest.approx(1.0, abs=1e-9)
    assert rep.per_view_psnr[1] == pytest.approx(M.psnr(G.render(scene, cams[2], st).image, imgs[2]), rel=1e-6)
    assert rep.n_surfels == 3000 and rep.n_gaussians == 800 and rep.ms_per_frame > 0
    # the CLI on the same model written as .ges and the views written as a dataset directory
    model = tmp_path / "m.ges"
    save_ges(scene, model)
    _write_dataset(tmp_path / "ds", cams, [G.render(scene, c, st).image for c in cams], ply=False)
    out = tmp_path / "report.json"
    assert cli.main(["eval", "--model", str(model), "--scene", str(tmp_path / "ds"), "--out", str(out),
                     "--test-every", "3"]) == 0
    r = json.loads(out.read_text())
    assert len(r["per_view_psnr"]) == 2 and r["mean_psnr"] > 40.0 and r["mean_ssim"] > 0.99


def test_camera_path_and_probe_match_reference():
    import torch

    from paper_2504_17545_b200.types import Camera
    g = np.load(GOLD)
    base = Camera(60.0, 58.0, 31.5, 24.0, 64, 48, g["path_base_w2c"])
    cams = M.camera_path(base, [0.1, -0.2, 0.0], frames=5, angle=0.05)
    assert np.allclose(np.stack([c.world_to_camera for c in cams]), g["path_w2c"], rtol=0, atol=1e-12)
    imgs = g["probe_images"]
    p = M.consistency_probe(None, cams, anchor_points=g["probe_points"], images=list(imgs))
    for k in ("max_change", "mean_change", "bounds"):
        assert np.allclose(p[k], g[f"probe_{k}"], rtol=1e-12, atol=0)
    # the tensor form (device batches in the path command) gives the same changes
    pt = M.consistency_probe(None, cams, images=torch.as_tensor(imgs))
    assert np.allclose(pt["max_change"], g["probe_max_change"], rtol=1e-12)
    assert np.allclose(pt["mean_change"], g["probe_mean_change"], rtol=1e-12) and pt["bounds"] == []
    with pytest.raises(ValueError):
        M.consistency_probe(None, [])
