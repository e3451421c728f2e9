import sys, time; sys.path.insert(0, '/root/repo')
import numpy as np, torch
import paper_2504_17545_b200 as G
from paper_2504_17545_b200 import scenes as S
sc = S.config_scene(5)
for (w, h, ss) in ((3840, 2160, 4), (7680, 4320, 1), (7680, 4320, 4)):
    cam = S.make_camera(w, h)
    t0 = time.perf_counter()
    out = G.render(sc, cam, G.RenderSettings(supersample=ss), to_numpy=False)
    torch.cuda.synchronize()
    wn = out.surfels.winner; d = out.surfels.depth
    ok = bool(((wn >= 0) == torch.isfinite(d)).all())
    print(w, h, ss, "render s", round(time.perf_counter() - t0, 2), "winner/depth consistent", ok,
          "covered", float((wn >= 0).float().mean()), "img finite", bool(torch.isfinite(out.image).all()))
