"""Load the golden cases written by ``tests/golden/make_golden.py``."""

from __future__ import annotations

import glob
import json
import os
from types import SimpleNamespace

import numpy as np

from paper_2504_17545_b200 import scenes as S
from paper_2504_17545_b200.types import (Camera, GaussianKind, GaussianSet, Scene,
                                         Stage, SurfelSet)

GOLDEN_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def names():
    """Render golden cases (the .ges, training and metrics fixtures are separate)."""
    return sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN_DIR, "*.npz"))
                  if not os.path.basename(p).startswith(("ges_", "train_", "metrics")))


def train_names():
    """Training-step cases written by ``tests/golden/make_train_golden.py``."""
    return sorted(os.path.basename(p)[6:-4] for p in glob.glob(os.path.join(GOLDEN_DIR, "train_*.npz")))


TRAIN_GRADS = ("surfel_pos", "surfel_quat", "surfel_scale", "surfel_sh", "surfel_w", "gaussian_pos",
               "gaussian_opacity", "gaussian_quat", "gaussian_scale", "gaussian_sh", "surfel_screen_grad",
               "gaussian_screen_grad")


def train_settings(d, settings_cls=None):
    """TrainSettings of a case (the package's own class unless given)."""
    if settings_cls is None:
        from paper_2504_17545_b200.training import TrainSettings as settings_cls
    kw = {k: (tuple(v) if isinstance(v, list) else v) for k, v in d.items()}
    return settings_cls(frozen_cache={}, **kw)


def load_train(name):
    z = np.load(os.path.join(GOLDEN_DIR, f"train_{name}.npz"))
    cam = Camera(float(z["fx"]), float(z["fy"]), float(z["cx"]), float(z["cy"]),
                 int(z["width"]), int(z["height"]), z["w2c"])
    kind = GaussianKind.TWO_D if str(z["kind"]) == "2d" else GaussianKind.THREE_D
    scene = Scene(SurfelSet(z["sp"], z["sq"], z["sl"], z["ssh"], z["sw"]),
                  GaussianSet(z["gp"], z["go"], z["gq"], z["gl"], z["gsh"], kind, z["gf"]),
                  int(z["sh_degree"]), Stage.FROZEN)
    st = json.loads(str(z["settings"]))
    cot = {k: z[k] for k in ("g_gauss_depth", "g_gauss_normal", "g_gauss_weight") if k in z.files}
    fwd = {k: z[k] for k in ("image", "surfel_color", "surfel_depth", "gauss_color", "gauss_weight",
                             "blend_depth", "blend_normal", "gauss_depth", "gauss_normal") if k in z.files}
    grads = {k: z["grad_" + k] for k in TRAIN_GRADS}
    grads["contrib"] = z["contrib"]
    return scene, cam, st, z["g_image"], cot, fwd, grads


def settings_ns(d, dtype=np.float64):
    base = dict(supersample=1, background=(0.0, 0.0, 0.0), layers="full", mip=False,
                epsilon_mode="adaptive", epsilon_value=0.0, dtype=dtype, threads=1,
                with_geometry=False)
    for k, v in d.items():
        base[k] = tuple(v) if isinstance(v, list) else v
    return SimpleNamespace(**base)


def load(name):
    z = np.load(os.path.join(GOLDEN_DIR, name + ".npz"))
    cam = Camera(float(z["fx"]), float(z["fy"]), float(z["cx"]), float(z["cy"]),
                 int(z["width"]), int(z["height"]), z["w2c"])
    st = json.loads(str(z["settings"]))
    if "sp" in z:
        kind = GaussianKind.TWO_D if str(z["kind"]) == "2d" else GaussianKind.THREE_D
        scene = Scene(SurfelSet(z["sp"], z["sq"], z["sl"], z["ssh"], z["sw"]),
                      GaussianSet(z["gp"], z["go"], z["gq"], z["gl"], z["gsh"], kind, z["gf"]),
                      int(z["sh_degree"]), Stage.FROZEN)
    else:
        scene = S.config_scene(1)
    out = {k: z[k] for k in z.files if k in ("image", "s_color", "s_depth", "s_normal",
                                             "s_winner", "g_color", "g_weight",
                                             "g_depth", "g_normal")}
    return scene, cam, st, out, str(z["digest"])
