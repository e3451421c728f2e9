"""Host-side cost of one drop-in render() call (config 2, to_numpy=False):
cProfile of 50 calls after warm-up."""
import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2504_17545_b200 as G  # noqa: E402
from paper_2504_17545_b200 import scenes as S  # noqa: E402

sc = S.config_scene(2)
cam = S.config_cameras(2)[0]
for _ in range(3):
    G.render(sc, cam, to_numpy=False)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(50):
    G.render(sc, cam, to_numpy=False)
torch.cuda.synchronize()
print(f"{(time.perf_counter() - t0) / 50 * 1e3:.3f} ms per render(to_numpy=False) call")
cProfile.run("for _ in range(50): G.render(sc, cam, to_numpy=False)", "/tmp/hprof")
pstats.Stats("/tmp/hprof").sort_stats("tottime").print_stats(12)
