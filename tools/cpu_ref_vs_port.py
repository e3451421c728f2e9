"""Pin the CPU baseline's stand-in: time the REAL reference renderer and the
oracle port (oracle/ges_oracle.py, what bench.py's cpu_baseline and
``--impl reference`` run on the GPU box, where /root/reference does not exist)
on the same host, scenes and settings.  Build container only:

    OPENBLAS_NUM_THREADS=1 python tools/cpu_ref_vs_port.py > profiles/cpu_ref_vs_port.json
"""
from __future__ import annotations

import json
import os
import sys
import time
from types import SimpleNamespace

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))

import numpy as np  # noqa: E402

from make_golden import to_ref, to_ref_cam  # noqa: E402  (imports the reference read-only)
from ges.forward import RenderSettings, render as ref_render  # noqa: E402
from oracle import ges_oracle as O  # noqa: E402
from paper_2504_17545_b200 import scenes as S  # noqa: E402
from paper_2504_17545_b200.types import Scene, Stage  # noqa: E402


def best_of(fn, n):
    ts = []
    for _ in range(n):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return min(ts)


def main():
    threads = os.cpu_count() or 1
    cases = []
    sc1 = S.config_scene(1)
    cases.append(("config1 10k+2k SH0 128x128", sc1, S.config_cameras(1)[0], 5))
    rng = np.random.default_rng(3)
    sc2 = Scene(S.random_surfels(rng, 100_000, 3, scale_range=(0.004, 0.016)),
                S.random_gaussians(rng, 30_000, 3, scale_range=(0.004, 0.02), extent=1.2), 3, Stage.FROZEN)
    cases.append(("100k+30k SH3 480x270", sc2, S.make_camera(480, 270), 1))
    out = {"host_threads": threads, "openblas_threads": os.environ["OPENBLAS_NUM_THREADS"], "cases": []}
    for name, sc, cam, reps in cases:
        rs, rc = to_ref(sc), to_ref_cam(cam)
        rst = RenderSettings(dtype=np.float32, threads=threads)
        ost = SimpleNamespace(supersample=1, background=(0.0, 0.0, 0.0), layers="full", mip=False,
                              epsilon_mode="adaptive", epsilon_value=0.0, dtype=np.float32,
                              threads=threads, with_geometry=False)
        t_ref = best_of(lambda: ref_render(rs, rc, rst), reps)
        t_port = best_of(lambda: O.render(sc, cam, ost), reps)
        img_r = ref_render(rs, rc, rst).image
        img_p = O.render(sc, cam, ost).image
        out["cases"].append({"case": name, "reference_s": t_ref, "port_s": t_port,
                             "port_over_reference": t_port / t_ref,
                             "image_max_abs_diff": float(np.max(np.abs(img_r.astype(np.float64) - img_p)))})
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
