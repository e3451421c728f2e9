"""Golden vectors of the REAL reference training step (joint stage).

Run in the build container (the only place ``/root/reference`` exists):

    python tests/golden/make_train_golden.py

Each case builds a seeded scene with ``paper_2504_17545_b200.scenes``,
renders it with the reference's ``ges.training.render_training``
(training.py:295-355; frozen surfels through ``frozen_cache``, float64) and
runs ``ges.training.backward`` (training.py:547-609) on seeded cotangents.
``train_<case>.npz`` stores scene arrays, camera, settings, cotangents, the
forward buffers and every gradient array.
"""

from __future__ import annotations

import json
import os
import sys
import zlib

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/src")

from ges.training import TrainSettings, backward, render_training  # noqa: E402  (reference, read-only)

from make_golden import to_ref, to_ref_cam  # noqa: E402
from paper_2504_17545_b200 import scenes as S  # noqa: E402
from paper_2504_17545_b200.types import GaussianKind, Scene, Stage  # noqa: E402

GRAD_FIELDS = ("surfel_pos", "surfel_quat", "surfel_scale", "surfel_sh", "surfel_w", "gaussian_pos",
               "gaussian_opacity", "gaussian_quat", "gaussian_scale", "gaussian_sh", "surfel_screen_grad",
               "gaussian_screen_grad")


def scene_of(seed, ns, ng, deg=1, kind=GaussianKind.THREE_D, mip_cam=None, s_rng=(0.1, 0.4),
             g_rng=(0.05, 0.3)):
    r = np.random.default_rng(seed)
    s = S.random_surfels(r, ns, deg, scale_range=s_rng)
    g = S.random_gaussians(r, ng, deg, kind=kind, scale_range=g_rng)
    if mip_cam is not None:
        g = S.mip_world_filter(g, [mip_cam])
    return Scene(s, g, deg, Stage.FROZEN)


def cases():
    cam = S.make_camera(40, 32)
    big = S.make_camera(64, 64)
    yield "t3d_frozen", scene_of(300, 14, 24), cam, {}, {}
    yield "t3d_mip_geom", scene_of(301, 12, 24, deg=2, mip_cam=big), cam, \
        {"mip": True, "with_geometry": True}, {"depth": True, "normal": True, "weight": True}
    yield "t2d_frozen", scene_of(302, 14, 20, kind=GaussianKind.TWO_D), cam, {}, {}
    yield "t2d_mip_geom", scene_of(303, 12, 20, kind=GaussianKind.TWO_D), cam, \
        {"mip": True, "with_geometry": True, "epsilon_mode": "constant", "epsilon_value": 0.08}, \
        {"depth": True, "normal": True}
    yield "t3d_gonly", scene_of(304, 10, 24, deg=3), cam, \
        {"surfels_enabled": False, "gaussian_only_norm": True, "background": [0.2, 0.4, 0.6]}, {}
    yield "t2d_nosurf", scene_of(305, 0, 20, kind=GaussianKind.TWO_D), cam, \
        {"background": [0.5, 0.25, 0.1]}, {"weight": True}
    yield "t3d_ss1", scene_of(306, 14, 24, deg=3), S.make_camera(48, 40), {"supersample": 1}, {}


def main():
    only = set(sys.argv[1:])
    for name, scene, cam, st, cot in cases():
        if only and name not in only:
            continue
        rs = to_ref(scene)
        kw = {k: (tuple(v) if isinstance(v, list) else v) for k, v in st.items()}
        settings = TrainSettings(dtype=np.float64, frozen_cache={}, **kw)
        frame = render_training(rs, to_ref_cam(cam), settings, cache_key=0)
        rng = np.random.default_rng(zlib.crc32(name.encode()))
        H, W = cam.height, cam.width
        g_img = rng.standard_normal((H, W, 3))
        extras = {}
        if cot.get("depth"):
            extras["g_gauss_depth"] = 0.1 * rng.standard_normal((H, W))
        if cot.get("normal"):
            extras["g_gauss_normal"] = 0.1 * rng.standard_normal((H, W, 3))
        if cot.get("weight"):
            extras["g_gauss_weight"] = 0.1 * rng.standard_normal((H, W))
        grads = backward(frame, g_img, **extras)
        s, g = scene.surfels, scene.gaussians
        d = dict(settings=json.dumps(st), fx=cam.fx, fy=cam.fy, cx=cam.cx, cy=cam.cy, width=cam.width,
                 height=cam.height, w2c=cam.world_to_camera, sh_degree=scene.sh_degree,
                 kind="2d" if g.kind is GaussianKind.TWO_D else "3d",
                 sp=s.pos, sq=s.quat, sl=s.log_scale, ssh=s.sh, sw=s.w,
                 gp=g.pos, go=g.raw_opacity, gq=g.quat, gl=g.log_scale, gsh=g.sh, gf=g.filter3d,
                 g_image=g_img, image=frame.image, surfel_color=frame.surfel_color,
                 surfel_depth=frame.surfel_depth, gauss_color=frame.gauss_color,
                 gauss_weight=frame.gauss_weight)
        for k, v in extras.items():
            d[k] = v
        for k in ("blend_depth", "blend_normal", "gauss_depth", "gauss_normal"):
            if getattr(frame, k) is not None:
                d[k] = getattr(frame, k)
        for k in GRAD_FIELDS:
            d["grad_" + k] = getattr(grads, k)
        # optim.py:526-533 (Trainer.contribution_scores) for this one view,
        # from the reference's own fragment tape
        gt = frame.tape["gauss"]
        contrib = np.zeros(g.count)
        if gt.get("count"):
            denom = (1.0 + frame.gauss_weight).reshape(-1)
            cmax = gt["colors"].max(axis=1)
            np.maximum.at(contrib, gt["gid"], cmax[gt["gid"]] * gt["alpha"] / denom[gt["pix"]])
        d["contrib"] = contrib
        np.savez_compressed(os.path.join(HERE, f"train_{name}.npz"), **d)
        print(name, "gauss frags:", frame.tape["gauss"].get("count", 0),
              "|g_pos|:", float(np.abs(grads.gaussian_pos).max()) if g.count else 0.0)


if __name__ == "__main__":
    main()
