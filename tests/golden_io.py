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
    """Render golden cases (the .ges fixtures have their own *_load.npz)."""
    return sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN_DIR, "*.npz"))
                  if not os.path.basename(p).startswith("ges_"))


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
