"""Generate golden vectors from the REAL reference renderer.

Run in the build container (the only place ``/root/reference`` exists):

    python tests/golden/make_golden.py

For every case it builds a seeded scene with ``paper_2504_17545_b200.scenes``
(same RNG call order as ``/root/reference/pkg/tests/conftest.py``), converts
it to the reference's own containers, renders it with
``ges.forward.render(..., RenderSettings(dtype=np.float64, threads=1))``
(``/root/reference/pkg/src/ges/forward.py:403-417``) and stores scene arrays,
camera, settings and every output buffer as float64 in ``<case>.npz``.
The config-1 scene is too large to store; its arrays are regenerated from
the seed and pinned by a sha256 recorded in the file.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/src")

import ges  # noqa: E402  (reference, read-only)
from ges import filters as rfilters  # noqa: E402
from ges.forward import RenderSettings, render  # noqa: E402
from ges.primitives import GaussianKind as RKind  # noqa: E402

from paper_2504_17545_b200 import scenes as S  # noqa: E402
from paper_2504_17545_b200.types import GaussianKind, Scene, Stage  # noqa: E402


def to_ref(scene: Scene):
    s, g = scene.surfels, scene.gaussians
    rs = ges.SurfelSet(s.pos, s.quat, s.log_scale, s.sh, s.w)
    kind = RKind.TWO_D if g.kind is GaussianKind.TWO_D else RKind.THREE_D
    rg = ges.GaussianSet(g.pos, g.raw_opacity, g.quat, g.log_scale, g.sh, kind,
                         np.asarray(g.filter3d, dtype=np.float64).copy())
    return ges.Scene(rs, rg, scene.sh_degree, ges.Stage.FROZEN)


def to_ref_cam(cam):
    return ges.Camera(cam.fx, cam.fy, cam.cx, cam.cy, cam.width, cam.height,
                      cam.world_to_camera)


def scene_digest(scene: Scene) -> str:
    h = hashlib.sha256()
    for a in (scene.surfels.pos, scene.surfels.quat, scene.surfels.log_scale,
              scene.surfels.sh, scene.gaussians.pos, scene.gaussians.raw_opacity,
              scene.gaussians.quat, scene.gaussians.log_scale, scene.gaussians.sh,
              scene.gaussians.filter3d):
        h.update(np.ascontiguousarray(a, dtype=np.float64).tobytes())
    return h.hexdigest()


def cases():
    cam32 = S.make_camera()
    for seed in range(100, 108):                       # test_forward.py:151-160
        r = np.random.default_rng(seed)
        sc = Scene(S.random_surfels(r, 25), S.GaussianSet.empty(1), 1, Stage.FROZEN)
        yield f"surf_{seed}", sc, cam32, {}
    for seed in range(500, 506):                       # test_forward.py:209-218
        yield f"g3d_{seed}", S.random_scene(np.random.default_rng(seed), 8, 20), cam32, {}
    for seed in range(900, 906):                       # test_forward.py:220-229
        sc = S.random_scene(np.random.default_rng(seed), 6, 15, kind=GaussianKind.TWO_D)
        yield f"g2d_{seed}", sc, cam32, {}
    r = np.random.default_rng(1234)                    # test_forward.py:286-300
    yield "ss4_surf", S.random_scene(r, 12, 0), cam32, {"supersample": 4}
    yield "ss4_full", S.random_scene(np.random.default_rng(21), 12, 30), cam32, {"supersample": 4}
    sc = S.random_scene(np.random.default_rng(7), 10, 25)
    yield "bg_gonly", sc, cam32, {"background": [0.2, 0.3, 0.4], "layers": "gaussians_only"}
    yield "bg_sonly", sc, cam32, {"background": [0.6, 0.1, 0.9], "layers": "surfels_only"}
    yield "bg_full", sc, cam32, {"background": [0.25, 0.5, 0.75]}
    yield "eps_const", sc, cam32, {"epsilon_mode": "constant", "epsilon_value": 0.05}
    yield "geom3d", sc, cam32, {"with_geometry": True}
    sc = S.random_scene(np.random.default_rng(11), 10, 25)
    sc = Scene(sc.surfels, S.mip_world_filter(sc.gaussians, [S.make_camera(64, 64)]),
               sc.sh_degree, Stage.FROZEN)
    yield "mip3d", sc, cam32, {"mip": True}
    sc2 = S.random_scene(np.random.default_rng(12), 8, 20, kind=GaussianKind.TWO_D)
    yield "mip2d", sc2, cam32, {"mip": True}
    yield "geom2d", sc2, cam32, {"with_geometry": True}
    r = np.random.default_rng(31)
    sc = Scene(S.random_surfels(r, 300, 3, scale_range=(0.03, 0.12)),
               S.random_gaussians(r, 100, 3, scale_range=(0.02, 0.1)), 3, Stage.FROZEN)
    yield "deg3_64x48", sc, S.make_camera(64, 48), {}
    yield "deg3_64x48_ss4", sc, S.make_camera(64, 48), {"supersample": 4, "mip": True}
    yield "config1", S.config_scene(1), S.config_cameras(1)[0], {}


def ges_goldens():
    """.ges fixtures written by the reference's export_ges (gesfile.py:42-76),
    with the reference's load_ges result and its float64 render of the
    float32-quantised scene."""
    from ges.gesfile import export_ges, load_ges
    r = np.random.default_rng(41)
    sc3 = Scene(S.random_surfels(r, 120, 3, scale_range=(0.05, 0.15)),
                S.random_gaussians(r, 60, 3, scale_range=(0.03, 0.1)), 3, Stage.FROZEN)
    sc3 = Scene(sc3.surfels, S.mip_world_filter(sc3.gaussians, [S.make_camera(64, 64)]), 3, Stage.FROZEN)
    sc2 = S.random_scene(np.random.default_rng(42), 40, 30, degree=1, kind=GaussianKind.TWO_D)
    cam = S.make_camera(48, 40)
    for name, sc, rgb in (("ges_3d_deg3", sc3, False), ("ges_2d_rgb", sc2, True)):
        path = os.path.join(HERE, name + ".ges")
        export_ges(to_ref(sc), path, rgb_surfels=rgb)
        rs, info = load_ges(path)
        out = render(rs, to_ref_cam(cam), RenderSettings(dtype=np.float64, threads=1))
        np.savez_compressed(os.path.join(HERE, name + "_load.npz"),
                            sp=rs.surfels.pos, sq=rs.surfels.quat, sl=rs.surfels.log_scale,
                            ssh=rs.surfels.sh, gp=rs.gaussians.pos, go=rs.gaussians.raw_opacity,
                            gq=rs.gaussians.quat, gl=rs.gaussians.log_scale, gsh=rs.gaussians.sh,
                            eps=info["epsilon"], flags=info["flags"],
                            fx=cam.fx, fy=cam.fy, cx=cam.cx, cy=cam.cy, width=cam.width,
                            height=cam.height, w2c=cam.world_to_camera,
                            image=out.image, s_winner=out.surfels.winner, s_depth=out.surfels.depth)
        print(name, os.path.getsize(path), "bytes")


def main():
    only = set(sys.argv[1:])
    if not only or "ges" in only:
        ges_goldens()
    for name, scene, cam, st in cases():
        if only and name not in only:
            continue
        settings = RenderSettings(dtype=np.float64, threads=1,
                                  **{k: (tuple(v) if isinstance(v, list) else v)
                                     for k, v in st.items()})
        out = render(to_ref(scene), to_ref_cam(cam), settings)
        d = dict(settings=json.dumps(st), fx=cam.fx, fy=cam.fy, cx=cam.cx, cy=cam.cy,
                 width=cam.width, height=cam.height, w2c=cam.world_to_camera,
                 sh_degree=scene.sh_degree,
                 kind="2d" if scene.gaussians.kind is GaussianKind.TWO_D else "3d",
                 digest=scene_digest(scene),
                 image=out.image, s_color=out.surfels.color, s_depth=out.surfels.depth,
                 s_normal=out.surfels.normal, s_winner=out.surfels.winner,
                 g_color=out.gaussians.color, g_weight=out.gaussians.weight)
        if out.gaussians.depth is not None:
            d.update(g_depth=out.gaussians.depth, g_normal=out.gaussians.normal)
        if name != "config1":
            s, g = scene.surfels, scene.gaussians
            d.update(sp=s.pos, sq=s.quat, sl=s.log_scale, ssh=s.sh, sw=s.w,
                     gp=g.pos, go=g.raw_opacity, gq=g.quat, gl=g.log_scale,
                     gsh=g.sh, gf=g.filter3d)
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **d)
        print(name, "covered px:", int(np.isfinite(out.surfels.depth).sum()),
              "gauss w>0 px:", int((out.gaussians.weight > 0).sum()))


if __name__ == "__main__":
    main()
