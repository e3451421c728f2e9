"""Joint-stage training step on the GPU at benchmark scale.

    python tools/train_bench.py [--config 2] [--steps 10] [--warmup 3] [--kind 3d|2d]

One step = render_training (frozen surfels, cached z-buffer, supersample 4 as
the reference's late phase; Gaussian pass at base resolution) + backward on
an L2 image cotangent, with the scene resident on the device (one
DeviceScene, as a trainer that re-packs only after parameter updates would
hold it between forward and backward).  Prints one JSON line with the step
time, the forward / backward split (CUDA events on the current stream) and
the Gaussian tile-pair count.
"""

import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2504_17545_b200 import scenes as S, training as TR  # noqa: E402
from paper_2504_17545_b200.renderer import DeviceScene  # noqa: E402
from paper_2504_17545_b200.types import GaussianKind, GaussianSet, Scene, Stage  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--kind", default="3d", choices=["3d", "2d"])
    ap.add_argument("--ss", type=int, default=4, choices=[1, 4])
    a = ap.parse_args()
    sc = S.config_scene(a.config)
    if a.kind == "2d":
        g = sc.gaussians
        g = GaussianSet(g.pos, g.raw_opacity, g.quat, g.log_scale[:, :2], g.sh, GaussianKind.TWO_D)
        sc = Scene(sc.surfels, g, sc.sh_degree, Stage.FROZEN)
    cam = S.config_cameras(a.config)[0]
    ds = DeviceScene(sc, keep_source=True)
    st = TR.TrainSettings(frozen_cache={}, supersample=a.ss, dtype=np.float32)
    target = torch.rand((cam.height, cam.width, 3), device="cuda")

    def step(ev=None):
        if ev:
            ev[0].record()
        fr = TR.render_training(sc, cam, st, cache_key=0, to_numpy=False, device_scene=ds)
        if ev:
            ev[1].record()
        g = TR.backward(fr, 2.0 * (fr.image - target), to_numpy=False)
        if ev:
            ev[2].record()
        return g

    for _ in range(a.warmup):
        step()
    torch.cuda.synchronize()
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(a.steps)]
    t0 = time.perf_counter()
    for k in range(a.steps):
        step(evs[k])
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) / a.steps
    fwd = float(np.median([e[0].elapsed_time(e[1]) for e in evs]))
    bwd = float(np.median([e[1].elapsed_time(e[2]) for e in evs]))
    # the reference-facing form: NumPy frame out, NumPy cotangent in, NumPy gradients out
    tgt = target.cpu().numpy()

    def step_np():
        fr = TR.render_training(sc, cam, st, cache_key=0, device_scene=ds)
        return TR.backward(fr, 2.0 * (fr.image - tgt))

    for _ in range(2):
        step_np()
    t0 = time.perf_counter()
    for _ in range(3):
        step_np()
    np_wall = (time.perf_counter() - t0) / 3
    print(json.dumps({"metric": "train_step_ms", "value": fwd + bwd, "unit": "ms", "forward_ms": fwd,
                      "backward_ms": bwd, "wall_ms": wall * 1e3, "numpy_wall_ms": np_wall * 1e3,
                      "steps": a.steps, "warmup": a.warmup,
                      "config": {"workload": f"config{a.config} joint-stage step, {a.kind} Gaussians, ss={a.ss}",
                                 "surfels": ds.n_surfels, "gaussians": ds.n_gaussians,
                                 "resolution": [cam.width, cam.height]}}))


if __name__ == "__main__":
    main()
