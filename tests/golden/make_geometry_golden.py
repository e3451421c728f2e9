"""Golden vectors for ``smooth_geometry`` and ``composite(surfel_weight)``
from the REAL reference (build container only, where ``/root/reference``
exists):

    python tests/golden/make_geometry_golden.py

Scenes follow ``/root/reference/pkg/tests/test_forward.py``:

* ``geo_match``  -- a 2D Gaussian on the surfel plane (:263-276,
  ``test_matching_gaussian_keeps_depth``), 32x32 identity camera, f=40;
* ``geo_bridge`` -- two fractured surfels plus a bridging 3D Gaussian
  (:278-300, ``test_bridging_gaussians_soften_seam``), f=60;
* ``geo_rand3d`` / ``geo_rand2d`` -- seeded random scenes (3D / planar
  Gaussians) rendered with geometry.

Each file stores the scene, the camera, the reference's float64 render
(``forward.py:403-417`` with ``with_geometry=True``), its
``smooth_geometry`` output (``forward.py:391-400``) and
``composite(surfel_color, gaussians, surfel_weight)`` for
surfel_weight in (0, 0.5, 1, 2) (``forward.py:384-388``;
``test_forward.py:163-180``).
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, HERE)
sys.path.insert(0, "/root/reference/pkg/src")

from ges.forward import RenderSettings, composite, render, smooth_geometry  # noqa: E402

from make_golden import scene_digest, to_ref, to_ref_cam  # noqa: E402
from paper_2504_17545_b200 import scenes as S  # noqa: E402
from paper_2504_17545_b200.types import (Camera, GaussianKind, GaussianSet, Scene, Stage,  # noqa: E402
                                         SurfelSet)

WEIGHTS = (0.0, 0.5, 1.0, 2.0)


def _logit(p):
    return np.log(p) - np.log1p(-p)


def identity_cam(width=32, height=32, f=40.0):
    return Camera(f, f, width / 2, height / 2, width, height, np.eye(4))


def frontal(color, depth, scale):
    sh = np.zeros((1, 1, 3))
    sh[0, 0] = (color - 0.5) / 0.28209479177387814
    return SurfelSet(np.array([[0.0, 0.0, depth]]), np.array([[1.0, 0.0, 0.0, 0.0]]),
                     np.log(np.full((1, 2), scale)), sh, np.array([255.0]))


def cases():
    # test_forward.py:263-276
    g = GaussianSet(np.array([[0.0, 0.0, 3.0]]), _logit(np.array([0.9])), np.array([[1.0, 0, 0, 0]]),
                    np.log(np.full((1, 2), 0.5)), np.zeros((1, 1, 3)), GaussianKind.TWO_D, np.zeros(1))
    yield "geo_match", Scene(frontal(0.5, 3.0, 2.0), g, 0, Stage.FROZEN), identity_cam()
    # test_forward.py:278-300
    surf = SurfelSet(np.array([[-0.55, 0.0, 2.6], [0.55, 0.0, 3.4]]), np.array([[1.0, 0, 0, 0], [1.0, 0, 0, 0]]),
                     np.log(np.full((2, 2), 0.2)), np.zeros((2, 1, 3)), np.full(2, 255.0))
    g = GaussianSet(np.array([[0.1, 0.0, 3.0]]), _logit(np.array([0.95])), np.array([[1.0, 0, 0, 0]]),
                    np.log(np.full((1, 3), 0.3)), np.zeros((1, 1, 3)), GaussianKind.THREE_D, np.zeros(1))
    yield "geo_bridge", Scene(surf, g, 0, Stage.FROZEN), identity_cam(f=60.0)
    yield "geo_rand3d", S.random_scene(np.random.default_rng(61), 14, 40), S.make_camera()
    yield "geo_rand2d", S.random_scene(np.random.default_rng(62), 12, 30, kind=GaussianKind.TWO_D), \
        S.make_camera(40, 28)


def main():
    for name, scene, cam in cases():
        out = render(to_ref(scene), to_ref_cam(cam), RenderSettings(dtype=np.float64, threads=1,
                                                                    with_geometry=True))
        d_sm, n_sm = smooth_geometry(out.surfels, out.gaussians)
        s, g = scene.surfels, scene.gaussians
        d = dict(settings=json.dumps({"with_geometry": True}), fx=cam.fx, fy=cam.fy, cx=cam.cx, cy=cam.cy,
                 width=cam.width, height=cam.height, w2c=cam.world_to_camera, sh_degree=scene.sh_degree,
                 kind="2d" if g.kind is GaussianKind.TWO_D else "3d", digest=scene_digest(scene),
                 image=out.image, s_color=out.surfels.color, s_depth=out.surfels.depth,
                 s_normal=out.surfels.normal, s_winner=out.surfels.winner,
                 g_color=out.gaussians.color, g_weight=out.gaussians.weight,
                 g_depth=out.gaussians.depth, g_normal=out.gaussians.normal,
                 smooth_depth=d_sm, smooth_normal=n_sm,
                 composite_weights=np.array(WEIGHTS),
                 sp=s.pos, sq=s.quat, sl=s.log_scale, ssh=s.sh, sw=s.w,
                 gp=g.pos, go=g.raw_opacity, gq=g.quat, gl=g.log_scale, gsh=g.sh,
                 gf=np.asarray(g.filter3d, dtype=np.float64))
        for i, w in enumerate(WEIGHTS):
            with np.errstate(divide="ignore", invalid="ignore"):
                d[f"composite_{i}"] = composite(out.surfels.color, out.gaussians, surfel_weight=w)
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **d)
        print(name, "covered px:", int(np.isfinite(out.surfels.depth).sum()),
              "gauss w>0 px:", int((out.gaussians.weight > 0).sum()))


if __name__ == "__main__":
    main()
