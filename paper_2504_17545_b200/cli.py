"""Command line front end for the GPU render path,
mirroring the reference's ``ges render`` / ``ges path`` / ``ges eval`` (``cli.py:126-174``):

  python -m paper_2504_17545_b200 render --model m.ges --camera cams.json --out o.png
         [--view K] [--ss {1,4}] [--layer {full,surfels,gaussians}] [--mip] [--background R G B]
  python -m paper_2504_17545_b200 path --model m.ges --camera cams.json --out DIR
         [--target X Y Z] [--frames N] [--angle RAD] [--ss {1,4}]
  python -m paper_2504_17545_b200 eval --model m.ges --scene DATASET_DIR --out report.json
         [--test-every N] [--ss {1,4}]
  python -m paper_2504_17545_b200 export --model m.ges --out n.ges

Camera files use the reference's dataset entries ({fx, fy, cx, cy, width,
height, w2c[16]}, ``datasets.py:125-137``).  Exit codes: 0 ok, 1 error,
2 usage (argparse).
"""

from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

import numpy as np

from .gesfile import load_ges
from .types import Camera


def camera_from_entry(e: dict) -> Camera:
    w2c = np.array(e["w2c"], dtype=np.float64).reshape(4, 4)
    return Camera(e["fx"], e["fy"], e["cx"], e["cy"], int(e["width"]), int(e["height"]), w2c)


def camera_to_entry(c) -> dict:
    return {"fx": c.fx, "fy": c.fy, "cx": c.cx, "cy": c.cy, "width": c.width, "height": c.height,
            "w2c": [float(x) for x in np.asarray(c.world_to_camera).reshape(-1)]}


def save_image(path, img):
    """clip(x*255+0.5) -> 8-bit PNG (datasets.py:54-56)."""
    from PIL import Image
    arr = np.clip(np.asarray(img) * 255.0 + 0.5, 0, 255).astype(np.uint8)
    Image.fromarray(arr).save(path)


def _settings(args):
    from .forward import RenderSettings
    layers = {"full": "full", "surfels": "surfels_only", "gaussians": "gaussians_only"}[args.layer]
    return RenderSettings(supersample=args.ss, layers=layers, mip=args.mip,
                          background=tuple(args.background))


def _load_cams(path):
    spec = json.loads(Path(path).read_text())
    return spec if isinstance(spec, list) else [spec]


def cmd_render(args) -> int:
    from .forward import render
    scene, _ = load_ges(args.model)
    cam = camera_from_entry(_load_cams(args.camera)[args.view])
    out = render(scene, cam, _settings(args))
    save_image(Path(args.out), out.image)
    print(f"wrote {args.out}")
    return 0


def cmd_path(args) -> int:
    """``ges path`` (cli.py:154-174): the small orbit of metrics.camera_path
    rendered as one batch on the GPU (views pipelined over CUDA streams),
    frames written as PNG, plus path.json and the consistency probe
    (probe.json, computed on the device)."""
    import torch

    from .forward import _device
    from .metrics import camera_path, consistency_probe
    from .multiview import ViewBatchRenderer
    from .renderer import SCENE_CACHE, default_renderer
    scene, _ = load_ges(args.model)
    base = camera_from_entry(_load_cams(args.camera)[0])
    cams = camera_path(base, args.target, frames=args.frames, angle=args.angle)
    out_dir = Path(args.out)
    out_dir.mkdir(parents=True, exist_ok=True)
    dev = _device()
    ds = SCENE_CACHE.get(scene, dev)
    vb = ViewBatchRenderer(default_renderer(dev), ds, cams, _settings(args), want=("image", "image_rgba8"),
                           streams=4)
    for r in vb.pool:                             # size every workspace's pair lists, then render the batch
        for c, fr in zip(vb.cams, vb.frames):
            r.render(ds, c, vb.settings, frame=fr, check=True)
    vb.render(check=False)
    torch.cuda.synchronize(dev)
    if vb.overflowed():
        vb.render(check=True)
    from PIL import Image
    rgba = vb.rgba if isinstance(vb.rgba, list) else list(vb.rgba.unbind(0))
    for k, f in enumerate(rgba):
        Image.fromarray(f[..., :3].cpu().numpy()).save(out_dir / f"frame_{k:04d}.png")
    probe = consistency_probe(None, cams, images=torch.stack([fr.image for fr in vb.frames]))
    (out_dir / "path.json").write_text(json.dumps([camera_to_entry(c) for c in cams], indent=1))
    (out_dir / "probe.json").write_text(json.dumps(probe, indent=1))
    print(f"wrote {len(rgba)} frames to {out_dir}")
    return 0


def cmd_eval(args) -> int:
    """``ges eval`` (cli.py:138-144): render the dataset's test views on the
    GPU and write the PSNR/SSIM report (metrics.evaluate)."""
    from .datasets import load_dataset
    from .forward import RenderSettings
    from .metrics import evaluate
    scene, _ = load_ges(args.model)
    dataset = load_dataset(Path(args.scene), test_every=args.test_every)
    rep = evaluate(scene, dataset, settings=RenderSettings(supersample=args.ss))
    Path(args.out).write_text(rep.to_json())
    print(f"mean PSNR {rep.mean_psnr:.2f} dB  SSIM {rep.mean_ssim:.4f} -> {args.out}")
    return 0


def cmd_export(args) -> int:
    """``ges export`` (cli.py:147-151): re-write a model in the normal layout."""
    from .gesfile import save_ges
    scene, info = load_ges(args.model)
    save_ges(scene, args.out, rgb_surfels=bool(info["rgb_surfels"]))
    print(f"wrote {args.out}")
    return 0


def build_parser():
    p = argparse.ArgumentParser(prog="paper_2504_17545_b200")
    sub = p.add_subparsers(dest="cmd", required=True)

    def common(sp, ss_default=4):
        sp.add_argument("--model", required=True)
        sp.add_argument("--camera", required=True)
        sp.add_argument("--out", required=True)
        sp.add_argument("--ss", type=int, default=ss_default, choices=[1, 4])
        sp.add_argument("--layer", default="full", choices=["full", "surfels", "gaussians"])
        sp.add_argument("--mip", action="store_true")
        sp.add_argument("--background", type=float, nargs=3, default=[0.0, 0.0, 0.0])

    r = sub.add_parser("render", help="render one view of a .ges model")
    common(r)
    r.add_argument("--view", type=int, default=0)
    r.set_defaults(fn=cmd_render)
    pa = sub.add_parser("path", help="render an orbit path as a batch and probe consistency")
    common(pa, ss_default=1)
    pa.add_argument("--target", type=float, nargs=3, default=[0.0, 0.0, 0.0])
    pa.add_argument("--frames", type=int, default=24)
    pa.add_argument("--angle", type=float, default=0.02, help="radians per frame")
    pa.set_defaults(fn=cmd_path)
    ev = sub.add_parser("eval", help="PSNR/SSIM of a model on a dataset's test views")
    ev.add_argument("--model", required=True)
    ev.add_argument("--scene", required=True, help="dataset directory (cameras.json + images)")
    ev.add_argument("--out", required=True)
    ev.add_argument("--test-every", type=int, default=8)
    ev.add_argument("--ss", type=int, default=4, choices=[1, 4])
    ev.set_defaults(fn=cmd_eval)
    x = sub.add_parser("export", help="re-export a model file (normalizes layout)")
    x.add_argument("--model", required=True)
    x.add_argument("--out", required=True)
    x.set_defaults(fn=cmd_export)
    return p


def main(argv=None) -> int:
    args = build_parser().parse_args(argv)
    try:
        return args.fn(args)
    except Exception as e:   # noqa: BLE001  (reference CLI maps failures to exit 1, cli.py:255-262)
        print(f"error: {e}", file=sys.stderr)
        return 1


if __name__ == "__main__":
    sys.exit(main())
