"""Device time of the float64 render mode (ges_render_f64) at a BASELINE
config, next to the float32 path: python tools/f64_bench.py [config]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2504_17545_b200 as G  # noqa: E402
from paper_2504_17545_b200 import scenes as S  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
sc = S.config_scene(cfg)
cam = S.config_cameras(cfg)[0]
for dt in (np.float32, np.float64):
    st = G.RenderSettings(dtype=dt, mip=(cfg == 4))
    G.render(sc, cam, st, to_numpy=False)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 5
    e0.record()
    for _ in range(n):
        G.render(sc, cam, st, to_numpy=False)
    e1.record()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    G.render(sc, cam, st)
    wall = time.perf_counter() - t0
    print(f"config {cfg} {np.dtype(dt).name}: {e0.elapsed_time(e1) / n:.2f} ms per render call (device, "
          f"to_numpy=False, includes the overflow check sync); {wall * 1e3:.1f} ms with NumPy outputs")
