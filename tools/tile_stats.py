"""Work counters of the tile kernel for one config-2 frame (tuning aid).

  python -m paper_2504_17545_b200._build stats
  GES_B200_LIB=paper_2504_17545_b200/libges_b200_stats.so python tools/tile_stats.py [--ss 4]
  (or a -DGES_TIMING build with --timing: warp lifetimes and the slowest warps)
"""
import argparse
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2504_17545_b200 as G  # noqa: E402
from paper_2504_17545_b200 import _lib, scenes as S  # noqa: E402

NAMES = ["surfel batches", "surfel entries staged", "  with live mask", "surfel warp tests",
         "candidate lanes", "gauss batches", "gauss entries walked (x warps)", "  surviving the warp cull",
         "gauss warp tests", "contributing lanes", "tiles", "tiles with uncovered px",
         "surfel warp tests at wmx=inf", "sample tests: not covered", "sample tests: covered",
         "  covered, sample still empty", "surfel warp tests covering no sample", "surfel entries in the warp patch (range)",
         "gauss entries in the warp patch (range)", "gauss batches (chunk iterations)",
         "surfel tests: range in one x half", "surfel tests: range in one y half", "surfel tests: range in one quadrant", "-"]

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--ss", type=int, default=1)
ap.add_argument("--timing", action="store_true", help="library built with -DGES_TIMING (warp lifetimes)")
a = ap.parse_args()
sc = S.config_scene(a.config)
cam = S.config_cameras(a.config)[0]
ds = G.DeviceScene(sc)
r = G.Renderer()
st = G.RenderSettings(supersample=a.ss)
fr = r.render(ds, cam, st, check=True)
buf = (C.c_uint64 * 24)()
_lib.lib().ges_debug_stats(buf)            # reset after the sizing render
fr = r.render(ds, cam, st, check=True)
torch.cuda.synchronize()
_lib.lib().ges_debug_stats(buf)
sp, gp, _ = fr.pairs()
print(f"pairs: surfel {sp}  gaussian {gp}   pixels {cam.width * cam.height}")
if a.timing:
    nw = ((cam.width + 31) // 32) * ((cam.height + 31) // 32) * 8
    ntx = (cam.width + 31) // 32
    k = buf[18]
    t = (k >> 3) % (1 << 21)
    print(f"warps {nw}: mean lifetime {buf[16] / nw:.0f} cycles, max {buf[17]} "
          f"(tile ({t % ntx}, {t // ntx}), warp {k & 7})")
    n = max(buf[19], 1)
    print(f"warps over 50 us: {buf[19]}; their mean list length {buf[12] / n:.0f}, "
          f"chunks walked {buf[13] / n:.1f}, warp tests {buf[14] / n:.1f}; "
          f"cycles: pass 1 {buf[5] / n:.0f}, pass 2 {buf[6] / n:.0f} "
          f"(Gaussian chunks {buf[7] / n:.1f}, warp tests {buf[8] / n:.1f})")
else:
    for n, v in zip(NAMES, buf):
        print(f"{n:28s} {v:14d}")
