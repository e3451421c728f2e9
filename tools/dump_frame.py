"""Render a config frame on the GPU and save winner/depth/image maps (debug aid)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2504_17545_b200 as G
from paper_2504_17545_b200 import scenes as S

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
ss = int(sys.argv[2]) if len(sys.argv) > 2 else 1
out = sys.argv[3] if len(sys.argv) > 3 else f"gpurun_out/frame_c{cfg}_ss{ss}.npz"
sc = S.config_scene(cfg)
cam = S.config_cameras(cfg)[0]
r = G.render(sc, cam, G.RenderSettings(supersample=ss, mip=cfg == 4))
np.savez_compressed(out, winner=r.surfels.winner, depth=r.surfels.depth, image=r.image,
                    g_weight=r.gaussians.weight)
print("saved", out)
