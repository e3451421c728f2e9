"""Wall time of the Python drop-in API (what a reference caller sees):
forward.render(scene, cam) returning NumPy (all RenderResult buffers copied
to host) and torch CUDA tensors (to_numpy=False), config-2 scene, 1080p.

  python tools/dropin_bench.py
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2504_17545_b200 as G  # noqa: E402
from paper_2504_17545_b200 import scenes as S  # noqa: E402

sc = S.config_scene(2)
cam = S.config_cameras(2)[0]
for to_np in (False, True):
    for _ in range(3):
        G.render(sc, cam, to_numpy=to_np)
    torch.cuda.synchronize()
    n = 20
    t0 = time.perf_counter()
    for _ in range(n):
        out = G.render(sc, cam, to_numpy=to_np)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / n
    print(f"render(to_numpy={to_np}): {dt * 1e3:.2f} ms/frame ({1 / dt:.0f} frames/s)")

# scene (re)pack: what a caller pays when it hands over new parameter arrays
from paper_2504_17545_b200.renderer import DeviceScene  # noqa: E402
for k in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ds = DeviceScene(sc)
    torch.cuda.synchronize()
    print(f"DeviceScene pack #{k}: {(time.perf_counter() - t0) * 1e3:.1f} ms")
    del ds
