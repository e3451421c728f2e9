"""Benchmark of the GES forward render path on B200 (contract: one JSON line).

Default workload = BASELINE config 2: 1M surfels + 300k Gaussians, SH degree
3, 1920x1080, float32, seeded synthetic scene.  One step = one
batch of ``--views`` views per rank (azimuths around the 8(d) pose, same
distance/elevation); value = frames/s over all ranks (weak scaling: fixed
views per GPU).  For N > 1 each step ends with the frame exchange: the RGBA8
frames are gathered to rank 0 over NCCL.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config 2] [--views 8]
  python bench.py --impl reference ...   # the reference algorithm on host cores
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=50)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", default="ges", choices=["ges", "reference"])
    p.add_argument("--config", type=int, default=2, choices=[1, 2, 3, 4, 5])
    p.add_argument("--views", type=int, default=None, help="views per rank per step")
    p.add_argument("--ss", type=int, default=1, choices=[1, 4])
    p.add_argument("--streams", type=int, default=16, help="CUDA streams pipelining the views of a step")
    p.add_argument("--layers", default="full", choices=["full", "surfels_only", "gaussians_only"])
    p.add_argument("--gather", default="peer", choices=["peer", "nccl"],
                   help="N > 1: frames to rank 0 through peer memory written by the tile kernel, or NCCL gather")
    p.add_argument("--no-graph", action="store_true", help="launch kernels eagerly instead of one CUDA graph per step")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline sample")
    p.add_argument("--tile-mode", type=int, default=0, choices=[0, 1, 2],
                   help="tile kernel layout: 0 auto, 1 16x16 tiles (1 px/thread), 2 32x32 tiles (2x2 px/thread)")
    p.add_argument("--no-others", action="store_true",
                   help="skip the short measurements of configs 3, 4, 5 in the default run")
    p.add_argument("--cpu-tiles", type=int, default=1 << 30,
                   help="tiles in the CPU sample (default: the whole frame, about 12 s of CPU work at config 2)")
    p.add_argument("--profile-only", action="store_true", help="render a few frames, no JSON (for ncu)")
    p.add_argument("--strips", action="store_true",
                   help="one frame per step split into row strips over the ranks (SURVEY 8(e) single huge frame)")
    return p.parse_args()


ARGS = parse()
if ARGS.impl == "reference":
    # the reference's CPU tile threads; keep BLAS single-threaded per tile thread
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    os.environ.setdefault("OMP_NUM_THREADS", "1")

import numpy as np  # noqa: E402

from paper_2504_17545_b200 import scenes as S  # noqa: E402

METRIC = "frames/sec at 1080p (1M surfels+300k Gaussians) per B200, views/s at 1/2/4/8 GPUs"
WORKLOADS = {
    1: "config1: 10k surfels + 2k Gaussians, SH0, 128x128",
    2: "config2: 1M surfels + 300k Gaussians, SH3, 1920x1080",
    3: "config3 (Speedy): 1M surfels + 60k Gaussians, SH3, 1920x1080",
    4: "config4 (Mip): 1M surfels + 300k filtered Gaussians, SH3, 3840x2160, mip=True",
    5: "config5: 3M surfels + 1M Gaussians, SH3, 3840x2160 orbit views",
}
DEFAULT_VIEWS = {1: 32, 2: 32, 3: 32, 4: 4, 5: None}
ORBIT_VIEWS = 256   # config 5: the 256-camera orbit, split over the ranks (strong scaling)


def per_rank_views(cfg, world, views):
    """Views per rank per step: --views, else the config default; config 5
    is the fixed 256-camera batch in contiguous blocks of ceil(256 / P)."""
    if views:
        return views
    if cfg == 5:
        return math.ceil(ORBIT_VIEWS / world)
    return DEFAULT_VIEWS[cfg]


def views_for(cfg, rank, world, per_rank):
    """Cameras of this rank's views."""
    total = per_rank * world
    ks = range(rank * per_rank, (rank + 1) * per_rank)
    if cfg == 5:   # 256-camera 4K orbit, contiguous blocks per rank
        from paper_2504_17545_b200.multiview import shard
        cams = S.orbit_cameras((0, 0, 0), 4.0, ORBIT_VIEWS, height=1.0, fov_deg=50.0,
                               width=3840, height_px=2160)
        if per_rank * world >= ORBIT_VIEWS and per_rank == math.ceil(ORBIT_VIEWS / world):
            return [cams[k] for k in shard(ORBIT_VIEWS, rank, world)]
        return [cams[k % ORBIT_VIEWS] for k in ks]
    if cfg == 4:   # the 8(d) pose at 1/8, 1/4, 1/2 and full 4K resolution
        return [S.make_camera(3840 // f, 2160 // f, azim=0.3 + 2.0 * math.pi * k / total)
                for k in ks for f in (8, 4, 2, 1)][:per_rank]
    w, h = S.CONFIGS[cfg]["res"]
    return [S.make_camera(w, h, azim=0.3 + 2.0 * math.pi * k / total) for k in ks]


def out_bytes_per_px(cfg):
    """Output bytes per pixel of the bench workload: fp32 RGB image, depth and
    winner id (20 B) -- config 5's 256-view batch keeps the RGBA8 frame the
    gather delivers (4 B)."""
    return 4 if cfg == 5 else 20


def b_alg(cfg, cams):
    """Algorithmic bytes per frame: scene read once + the
    output bytes per pixel, averaged over the step's views."""
    c = S.CONFIGS[cfg]
    K = (c["deg"] + 1) ** 2
    px = sum(int(v.width) * int(v.height) for v in cams) / len(cams)
    return c["ns"] * (36 + 12 * K) + c["ng"] * (44 + 12 * K) + px * out_bytes_per_px(cfg)


def base_config(cfg, per_rank, world, ss):
    w, h = S.CONFIGS[cfg]["res"]
    l2 = ("inputs larger than L2 (packed scene > 126 MB; no flush needed)" if cfg != 1 else
          "inputs fit in L2 (config 1 is the CPU-runnable parity case, not the headline)")
    return {"workload": WORKLOADS[cfg], "views_per_rank_per_step": per_rank,
            "resolution": [w, h] if cfg != 4 else "480x270, 960x540, 1920x1080, 3840x2160",
            "supersample": ss, "parallelism": f"views x{world}", "streams_per_gpu": ARGS.streams,
            "cuda_graph": not ARGS.no_graph, "layers": ARGS.layers,
            "frame_gather": ("none (N=1)" if world == 1 else
                             "peer: tile kernel writes RGBA8 frames into rank 0 over NVLink (CUDA IPC)"
                             if ARGS.gather == "peer" else "NCCL gather of RGBA8 frames"),
            "scene": "seeded synthetic (SURVEY 8(d), seed 0)", "l2": l2}


# ----------------------------------------------------------------------------- CPU
def cpu_model() -> str:
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def _oracle_settings(cfg, threads, ss):
    from types import SimpleNamespace
    return SimpleNamespace(supersample=ss, background=(0.0, 0.0, 0.0), layers="full", mip=cfg == 4,
                           epsilon_mode="adaptive", epsilon_value=0.0, dtype=np.float32,
                           threads=threads, with_geometry=False)


def cpu_sample(cfg, scene, cam, n_tiles, threads, ss=1):
    """Time the reference algorithm (oracle/ges_oracle.py, float32 like the
    reference default) on a bounded sample: the full per-frame preprocessing
    plus ``n_tiles`` random tiles of the frame; the tile time is extrapolated
    to all tiles (no extrapolation when n_tiles covers the frame).  Returns
    (frame seconds, wall seconds, tiles, total tiles)."""
    from oracle import ges_oracle as O
    st = _oracle_settings(cfg, threads, ss)
    nt = ((cam.width + 15) // 16) * ((cam.height + 15) // 16)
    rng = np.random.default_rng(7)
    tiles = None if n_tiles >= nt else sorted(rng.choice(nt, n_tiles, replace=False).tolist())
    O.TILE_SECONDS[0] = 0.0
    t0 = time.perf_counter()
    O.render(scene, cam, st, tiles=tiles)
    wall = time.perf_counter() - t0
    tile_s = O.TILE_SECONDS[0]
    frame_s = wall if tiles is None else (wall - tile_s) + tile_s * nt / len(tiles)
    return frame_s, wall, min(n_tiles, nt), nt


# strips per frame of the reference arm: one step = one strip of tile rows, so
# a step is a bounded ~1-3 s of host work at every config
STRIPS_TARGET = {1: 1, 2: 8, 3: 4, 4: 16, 5: 32}


def strips_for(cfg, steps):
    """Strips per frame: the smallest divisor of ``steps`` >= the config's
    target (so the timed steps are exactly steps / strips whole frames), or
    ``steps`` itself when it is smaller than the target."""
    tgt = STRIPS_TARGET[cfg]
    for d in range(tgt, steps + 1):
        if steps % d == 0:
            return d
    return max(steps, 1)


def single_thread_sample(cfg, scene, cam, ss):
    """BASELINE.md section 2 variant (b): threads=1 with default (multi-
    threaded) OpenBLAS, one whole frame (config 2: ~15 s on the box)."""
    from oracle import ges_oracle as O
    try:
        from threadpoolctl import threadpool_limits
    except ImportError:   # pragma: no cover
        threadpool_limits = None
    st = _oracle_settings(cfg, 1, ss)
    ctx = threadpool_limits(limits=os.cpu_count() or 1, user_api="blas") if threadpool_limits else None
    try:
        if ctx is not None:
            ctx.__enter__()
        t0 = time.perf_counter()
        O.render(scene, cam, st)
        wall = time.perf_counter() - t0
    finally:
        if ctx is not None:
            ctx.__exit__(None, None, None)
    return {"value": 1.0 / wall, "unit": "frames/s", "cores": 1, "kind": "port",
            "sample": "threads=1, default OpenBLAS threading (BASELINE.md 2(b)): one whole frame",
            "frame_s": wall, "measured_wall_s": wall}


def faithful_frame(cfg, scene, cam, ss, threads):
    """One whole frame with the reference's own candidate selection -- the
    O(N x tiles) scan of forward.py:168-169, :294-295 -- instead of the
    port's per-tile lists (oracle FAST_SELECT off): the reference algorithm
    exactly as written, all host threads."""
    from oracle import ges_oracle as O
    st = _oracle_settings(cfg, threads, ss)
    old = O.FAST_SELECT[0]
    O.FAST_SELECT[0] = False
    try:
        t0 = time.perf_counter()
        O.render(scene, cam, st)
        wall = time.perf_counter() - t0
    finally:
        O.FAST_SELECT[0] = old
    return {"value": 1.0 / wall, "unit": "frames/s", "cores": threads, "kind": "port",
            "sample": "one whole frame with the reference's per-tile O(N x tiles) selection scan "
                      "(forward.py:168-169); the main value uses per-tile candidate lists (faster, same results)",
            "frame_s": wall}


def reference_other(cfg, threads):
    """The reference algorithm on the other BASELINE configurations (the
    default reference run carries them, next to the GPU line's
    other_configs): configs 3 and 4 in whole frames (config 4: one frame at
    each of its four scales); config 5 (3M + 1M at 4K, ~1 min per frame on
    the box) as its per-frame preprocessing plus 4 of 32 row strips spread
    over the frame, extrapolated to the frame and labelled so."""
    from oracle import ges_oracle as O
    scene = S.config_scene(cfg)
    cams = views_for(cfg, 0, 1, 4 if cfg == 4 else 1)
    st = _oracle_settings(cfg, threads, 1)
    if cfg != 5:
        t0 = time.perf_counter()
        for c in cams:
            O.render(scene, c, st)
        wall = time.perf_counter() - t0
        return {"workload": WORKLOADS[cfg], "value": len(cams) / wall, "unit": "frames/s", "cores": threads,
                "kind": "port", "sample": f"{len(cams)} whole frame(s)", "measured_wall_s": wall}
    cam = cams[0]
    groups = O.strip_groups(cam.height, cam.width, 32)
    sample = [groups[k] for k in (0, 8, 16, 24)]   # strips spread over the frame
    steps = O.render_steps(scene, cam, st, sample)
    t0 = time.perf_counter()
    next(steps)                       # preprocessing + strip 0
    t1 = time.perf_counter()
    for _ in range(3):                # strips 8, 16, 24
        next(steps)
    t2 = time.perf_counter()
    strip_s = (t2 - t1) / 3
    frame_s = (t1 - t0) + strip_s * (len(groups) - 1)
    return {"workload": WORKLOADS[cfg], "value": 1.0 / frame_s, "unit": "frames/s", "cores": threads,
            "kind": "port", "sample": f"preprocessing + 4 of {len(groups)} row strips (0, 8, 16, 24) of one "
                                      f"3840x2160 view, extrapolated to the frame", "frame_s": frame_s,
            "measured_wall_s": t2 - t0}


def run_reference(args, rank, world):
    """--impl reference: the reference algorithm (oracle/ges_oracle.py, the
    NumPy restatement pinned to the reference's goldens; float32 like the
    reference default) on this box's host cores, all threads, timed in whole
    frames.  One step = one strip of tile rows of the frame (the first strip
    of a frame also does the frame's preprocessing), so K steps are exactly
    K / strips frames and ms_per_step is the measured wall time per step."""
    if rank != 0:
        return
    from oracle import ges_oracle as O
    cfg = args.config
    scene = S.config_scene(cfg)
    cam = views_for(cfg, 0, 1, 1)[0]
    threads = os.cpu_count() or 1
    st = _oracle_settings(cfg, threads, args.ss)
    nstrips = strips_for(cfg, args.steps)
    groups = O.strip_groups(cam.height, cam.width, nstrips)
    nstrips = len(groups)

    def strips():
        while True:   # an endless sequence of frames, one strip per step
            yield from O.render_steps(scene, cam, st, groups)

    seq = strips()
    for _ in range(args.warmup):
        next(seq)
    seq = strips()   # the timed steps start at a frame boundary
    t0 = time.perf_counter()
    for _ in range(args.steps):
        next(seq)
    wall = time.perf_counter() - t0
    frames = args.steps / nstrips
    fps = frames / wall
    single = None if args.no_cpu else single_thread_sample(cfg, scene, cam, args.ss)
    faithful = None if args.no_cpu else faithful_frame(cfg, scene, cam, args.ss, threads)
    others = None
    if cfg == 2 and args.ss == 1 and not args.no_others:
        others = {f"config{oc}": reference_other(oc, threads) for oc in (3, 4, 5)}
    sample = (f"{args.steps} steps = {frames:g} whole {cam.width}x{cam.height} frames, each rendered as "
              f"{nstrips} strips of tile rows (one strip per step, the frame's preprocessing in its first "
              f"strip); oracle/ges_oracle.py float32 with per-tile candidate lists (faster than the "
              f"reference's O(N x tiles) selection scan, forward.py:168-169); {threads} tile threads, "
              f"OPENBLAS_NUM_THREADS=1 (BASELINE.md 2(a))")
    line = {"metric": METRIC, "value": fps, "unit": "frames/s", "impl": "reference",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": wall * 1e3 / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {**base_config(cfg, 1, world, args.ss), "strips_per_frame": nstrips,
                       "views_per_rank_per_step": f"1/{nstrips} of a view"},
            "cpu_baseline": {"value": fps, "unit": "frames/s", "cores": threads, "kind": "port",
                             "cpu_model": cpu_model(), "sample": sample, "measured_wall_s": wall,
                             "frame_s": wall / frames, "single_thread": single,
                             "reference_selection": faithful},
            "e2e": {"value": fps, "unit": "frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "other_configs": others}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for ln in self.proc.stdout:
            self.lines.append(ln.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for ln in self.lines:
            p = [x.strip() for x in ln.split(",")]
            if len(p) < 8:
                continue
            try:
                sm.append(float(p[0]))
                mx = float(p[1])
            except ValueError:
                continue
            for n, v in zip(names, p[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ----------------------------------------------------------------------------- GPU
def measure_config(cfg, dev, streams, steps=5, warmup=3):
    """One other BASELINE configuration, device-timed like the main line (its
    default views per step in one CUDA graph over `streams` streams, CUDA
    events around `steps` steps): frames/s, ms/step and the isolated-frame
    time are reported as extra keys of the default run's line so they are
    observed by the driver's run."""
    import torch

    import paper_2504_17545_b200 as G
    from paper_2504_17545_b200.multiview import ViewBatchRenderer

    t0 = time.perf_counter()
    per = per_rank_views(cfg, 1, None)
    cams = views_for(cfg, 0, 1, per)
    scene = S.config_scene(cfg)
    settings = G.RenderSettings(mip=(cfg == 4))
    ds = G.DeviceScene(scene, dev)
    rend = G.Renderer(dev)
    vb = ViewBatchRenderer(rend, ds, cams, settings,
                           want=("image_rgba8",) if cfg == 5 else ("image", "s_depth", "s_winner"),
                           streams=streams)
    for i, r in enumerate(vb.pool):
        for c, fr in list(zip(vb.cams, vb.frames))[i::len(vb.pool)]:
            r.render(ds, c, settings, frame=fr, check=True)
    vb.capture()
    for _ in range(warmup):
        vb.render()
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        vb.render()
    e1.record(stream)
    torch.cuda.synchronize()
    el = e0.elapsed_time(e1) / 1e3
    if vb.overflowed():
        raise RuntimeError(f"config {cfg}: tile pair lists overflowed inside the timed region")
    # isolated frame: the last view alone, eager, on the main stream, through the
    # renderer (workspace) that rendered it inside the graph
    lane = vb.pool[(len(cams) - 1) % len(vb.pool)]
    lane.render(ds, cams[-1], settings, frame=vb.frames[-1], check=False)   # (warm)
    torch.cuda.synchronize()
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    f0.record(stream)
    lane.render(ds, cams[-1], settings, frame=vb.frames[-1], check=False)
    f1.record(stream)
    torch.cuda.synchronize()
    out = {"workload": WORKLOADS[cfg], "value": per * steps / el, "unit": "frames/s",
           "scaling": "strong" if cfg == 5 else "weak", "views_per_step": per, "steps": steps,
           "warmup": warmup, "ms_per_step": el * 1e3 / steps,
           "isolated_frame_ms": f0.elapsed_time(f1), "b_alg_bytes_per_frame": b_alg(cfg, cams),
           "setup_s": time.perf_counter() - t0}
    del vb, rend, ds
    return out


def run_gpu(args, rank, world, local_rank):
    import ctypes as C

    import torch
    import torch.distributed as dist

    import paper_2504_17545_b200 as G
    from paper_2504_17545_b200 import _lib
    from paper_2504_17545_b200.multiview import PeerFrameGather, ViewBatchRenderer, gather_frames
    from paper_2504_17545_b200.renderer import camera_struct, settings_struct

    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    cfg = args.config
    per_rank = per_rank_views(cfg, world, args.views)
    # N > 1: rank 0 builds and packs the scene, the other ranks receive the packed
    # blob by one broadcast (SURVEY 8(e) scene replication)
    scene = S.config_scene(cfg) if (world == 1 or rank == 0) else None
    cams = views_for(cfg, rank, world, per_rank)
    strips = None
    if args.strips:   # one frame per step: this rank's band of rows as a camera of its own
        from paper_2504_17545_b200.multiview import strip_bounds, strip_camera
        full_cam = views_for(cfg, 0, 1, 1)[0]
        strips = strip_bounds(int(full_cam.height), world)
        cams = [strip_camera(full_cam, *strips[rank])]
        per_rank = 1
    settings = G.RenderSettings(supersample=args.ss, mip=(cfg == 4), layers=args.layers)
    settings.tile_mode = args.tile_mode   # (not a reference field: 0 auto, 1 16x16, 2 32x32 tiles)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    if world == 1:
        ds = G.DeviceScene(scene, dev)
    else:
        from paper_2504_17545_b200.multiview import broadcast_scene
        ds = broadcast_scene(scene, src=0, device=dev)
    torch.cuda.synchronize()
    upload_ms = (time.perf_counter() - t0) * 1e3
    rend = G.Renderer(dev)
    # B_alg outputs (image fp32, depth, winner) + the RGBA8 frames of the gather (N > 1): with
    # --gather peer the tile kernel writes them straight into rank 0's batch over NVLink
    same_res = len({(int(c.height), int(c.width)) for c in cams}) == 1
    sink = None
    gather_used = "none (N=1)" if world == 1 else "nccl"
    if world > 1 and args.gather == "peer" and same_res:
        # every rank agrees on the form: if any rank cannot map rank 0's buffer
        # (no peer access), all of them fall back to the NCCL gather
        err = None
        try:
            if strips is not None:
                sink = PeerFrameGather(1, int(full_cam.height), int(full_cam.width), dst=0, device=dev,
                                       strips=strips)
            else:
                sink = PeerFrameGather(per_rank, int(cams[0].height), int(cams[0].width), dst=0, device=dev)
            if os.environ.get("GES_BENCH_PEER_FAIL") == str(rank):   # test-only: exercise the fallback
                raise RuntimeError("peer mapping disabled by GES_BENCH_PEER_FAIL")
        except RuntimeError as e:
            err = str(e)
        ok = torch.tensor([0 if err else 1], device=dev, dtype=torch.int32)
        dist.all_reduce(ok, op=dist.ReduceOp.MIN)
        if int(ok.item()) == 0:
            if sink is not None:
                sink.close()
                sink = None
            if rank == 0:
                print(f"peer frame gather unavailable ({err or 'on another rank'}); using the NCCL gather",
                      file=sys.stderr)
        else:
            gather_used = "peer"
    # config 5 keeps only the RGBA8 frames (256 4K views); the others the float
    # outputs (plus the RGBA8 send buffer of the NCCL gather at N > 1)
    want = (("image_rgba8",) if cfg == 5 else ("image", "s_depth", "s_winner")) + \
        (("image_rgba8",) if world > 1 and sink is None and cfg != 5 else ())
    rgba_out = sink.slots if sink is not None else None
    strip_pad = None
    if strips is not None and sink is None and world > 1:
        # NCCL form of the strip gather: every rank's band padded to the tallest one
        from paper_2504_17545_b200.multiview import DevicePointer
        hmax = max(y1 - y0 for y0, y1 in strips)
        strip_pad = torch.zeros((1, hmax, int(full_cam.width), 4), dtype=torch.uint8, device=dev)
        rgba_out = [DevicePointer(strip_pad.data_ptr(), strip_pad.numel())]
    vb = ViewBatchRenderer(rend, ds, cams, settings, want=want, streams=args.streams, rgba_out=rgba_out)
    # size every workspace's pair lists from a checked frame of every view
    for i, r in enumerate(vb.pool):   # (each lane renders views i, i + lanes, ...)
        for c, fr in list(zip(vb.cams, vb.frames))[i::len(vb.pool)]:
            r.render(ds, c, settings, frame=fr, check=True)
    graphed = False if args.no_graph else vb.capture()
    stream = torch.cuda.current_stream(dev)

    def step():
        vb.render(check=False)
        if sink is not None:
            sink.fence()
        elif strip_pad is not None:
            gather_frames(strip_pad, dst=0)
        elif world > 1 and torch.is_tensor(vb.rgba):
            gather_frames(vb.rgba, dst=0)

    if args.profile_only:
        for _ in range(max(args.warmup, 1) + args.steps):
            step()
        torch.cuda.synchronize()
        return

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    phys = os.environ.get("CUDA_VISIBLE_DEVICES", "").split(",")
    smi_index = phys[local_rank] if len(phys) > local_rank and phys[local_rank] else local_rank
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(smi_index) as clk:
        time.sleep(0.3)
        torch.cuda.synchronize()
        ev0.record(stream)
        for _ in range(args.steps):
            step()
        ev1.record(stream)
        torch.cuda.synchronize()
        time.sleep(0.2)
    if world > 1:
        dist.barrier()
    elapsed = ev0.elapsed_time(ev1) / 1e3
    if world > 1:
        t = torch.tensor([elapsed], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        elapsed = float(t.item())
    if vb.overflowed():
        raise RuntimeError("tile pair lists overflowed inside the timed region")
    frames = args.steps if strips is not None else per_rank * world * args.steps
    fps = frames / elapsed
    ms_step = elapsed * 1e3 / args.steps
    s_pairs, g_pairs, _ = vb.frames[0].pairs()

    # ---- per-phase breakdown (separate pass, events on the launching stream)
    L = _lib.lib()
    n_prof = max(4, min(3 * per_rank, 24))
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(6)] for _ in range(n_prof)]
    for row in evs:
        for e in row:
            e.record(stream)
    torch.cuda.synchronize()
    st_c = settings_struct(settings)
    for i in range(n_prof):
        c = vb.cams[i % per_rank]
        fr = vb.frames[i % per_rank]
        cam_c = camera_struct(c)
        ws, nbytes = rend.workspace(ds, cam_c, st_c)
        arr = (C.c_void_p * 6)(*[e.cuda_event for e in evs[i]])
        _lib.check(L.ges_render_profiled(C.byref(ds.c), C.byref(cam_c), C.byref(st_c),
                                         C.byref(rend._outputs(fr)), C.c_void_p(ws.data_ptr()), nbytes,
                                         rend.cap_s, rend.cap_g, C.c_void_p(fr.status.data_ptr()),
                                         C.c_void_p(stream.cuda_stream), arr), "profiled render")
    torch.cuda.synchronize()
    names = ["memsets", "prep", "tile_scan", "tile_fill", "tile_render"]
    phase = {n: statistics.mean(row[k].elapsed_time(row[k + 1]) for row in evs) for k, n in enumerate(names)}
    frame_ms_profiled = statistics.mean(row[0].elapsed_time(row[5]) for row in evs)
    # the isolated frame itself: one ges_render per frame with events only around it (the
    # phase events above also cut the programmatic-dependent-launch overlap between kernels)
    fevs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n_prof)]
    for i in range(n_prof):
        c = vb.cams[i % per_rank]
        fr = vb.frames[i % per_rank]
        cam_c = camera_struct(c)
        ws, nbytes = rend.workspace(ds, cam_c, st_c)
        fevs[i][0].record(stream)
        _lib.check(L.ges_render(C.byref(ds.c), C.byref(cam_c), C.byref(st_c), C.byref(rend._outputs(fr)),
                                C.c_void_p(ws.data_ptr()), nbytes, rend.cap_s, rend.cap_g,
                                C.c_void_p(fr.status.data_ptr()), C.c_void_p(stream.cuda_stream)), "render")
        fevs[i][1].record(stream)
    torch.cuda.synchronize()
    frame_ms = statistics.mean(e0.elapsed_time(e1) for e0, e1 in fevs)

    # ---- end-to-end through the C ABI with host buffers (ges_render_views_host)
    e2e = e2e_u8 = None
    if not args.no_e2e and cfg != 5 and strips is None and len({(c.width, c.height) for c in cams}) == 1:
        W, H = cams[0].width, cams[0].height
        cams_c = (_lib.Camera * per_rank)(*[camera_struct(c) for c in cams])
        cam_pin = torch.empty(C.sizeof(cams_c), dtype=torch.uint8, pin_memory=True)
        C.memmove(cam_pin.data_ptr(), cams_c, C.sizeof(cams_c))
        cams_pinned = C.cast(C.c_void_p(cam_pin.data_ptr()), C.POINTER(_lib.Camera))
        statuses = torch.zeros((per_rank, 3), dtype=torch.int64, device=dev)
        copy_stream = torch.cuda.Stream(dev)
        # one lane per stream of the view batch: its renderer's workspace and stream
        lanes = len(vb.pool)
        wss = [r.workspace(ds, camera_struct(cams[0]), st_c) for r in vb.pool]
        nbytes = max(n for _, n in wss)
        ws_arr = (C.c_void_p * lanes)(*[w.data_ptr() for w, _ in wss])
        lane_streams = [stream] + [sx for sx in vb.streams[1:]]
        st_arr = (C.c_void_p * lanes)(*[sx.cuda_stream for sx in lane_streams])
        caps = (min(r.cap_s for r in vb.pool), min(r.cap_g for r in vb.pool))

        def e2e_run(fmt, lanes):
            shape, dt = ((H, W, 3), torch.float32) if fmt == _lib.GES_IMAGE_F32_RGB else ((H, W, 4), torch.uint8)
            host = torch.empty((per_rank,) + shape, dtype=dt, pin_memory=True)
            imgdev = torch.empty((2 * lanes,) + shape, dtype=dt, device=dev)

            def e2e_step():
                _lib.check(L.ges_render_views_host(C.byref(ds.c), cams_pinned, per_rank, C.byref(st_c), fmt,
                                                   C.c_void_p(host.data_ptr()), lanes, ws_arr, nbytes,
                                                   caps[0], caps[1], C.c_void_p(imgdev.data_ptr()),
                                                   C.c_void_p(statuses.data_ptr()), st_arr,
                                                   C.c_void_p(copy_stream.cuda_stream)), "views_host")

            for _ in range(args.warmup):
                e2e_step()
            torch.cuda.synchronize()
            if world > 1:
                dist.barrier()
            t0 = time.perf_counter()
            for _ in range(args.steps):
                e2e_step()
            copy_stream.synchronize()
            torch.cuda.synchronize(dev)
            e_el = time.perf_counter() - t0
            if world > 1:
                t = torch.tensor([e_el], device=dev, dtype=torch.float64)
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
                e_el = float(t.item())
            if fmt == _lib.GES_IMAGE_F32_RGB:
                ref_img = vb.frames[0].image.cpu().numpy()
                assert np.allclose(host[0].numpy(), ref_img, atol=1e-6), "e2e image differs from device render"
            else:
                # fp32 Gaussian sums may differ in the last bit between renders (atomic list
                # order), which can move an 8-bit rounding by one step
                if vb.rgba is None:   # (N = 1: the step writes float frames only)
                    dev_rgba = (vb.frames[0].image * 255.0 + 0.5).clamp(0, 255).to(torch.uint8)
                    dev_rgba = torch.cat([dev_rgba, torch.full_like(dev_rgba[..., :1], 255)], dim=-1)
                else:
                    dev_rgba = (vb.rgba[0] if torch.is_tensor(vb.rgba[0]) else
                                sink.frames[0] if sink is not None and sink.frames is not None else None)
                if dev_rgba is not None:   # (ranks > 0 of the peer gather hold no local frame copy)
                    dif = (host[0].int() - dev_rgba.cpu().int()).abs().max().item()
                    assert dif <= 1, f"e2e RGBA8 frame differs from device render by {dif}"
            return per_rank * world * args.steps / e_el, host[0].numel() * host.element_size() * per_rank

        # fp32 frames saturate PCIe with one render stream (more streams only contend)
        v32, b32 = e2e_run(_lib.GES_IMAGE_F32_RGB, 1)
        # the e2e path's roofline: this box's pinned device->host copy bandwidth
        probe_n = int(W) * int(H) * 12
        psrc = torch.empty(probe_n, dtype=torch.uint8, device=dev)
        pdst = torch.empty(probe_n, dtype=torch.uint8, pin_memory=True)
        pdst.copy_(psrc)
        torch.cuda.synchronize()
        tp = time.perf_counter()
        for _ in range(16):
            pdst.copy_(psrc, non_blocking=True)
        torch.cuda.synchronize()
        d2h_gbs = 16 * probe_n / (time.perf_counter() - tp) / 1e9
        del psrc, pdst
        e2e = {"value": v32, "unit": "frames/s", "h2d_bytes_per_step": per_rank * C.sizeof(_lib.Camera),
               "d2h_bytes_per_step": b32,
               "path": "ges_render_views_host (C ABI): host camera structs in, pinned fp32 RGB frames "
                       "(RenderResult.image) out on a copy stream overlapped with the next render; "
                       "PCIe-bound at 1080p (24.9 MB per frame)",
               "roofline": {"bound": "pcie_d2h", "achieved": v32 * b32 / per_rank / 1e9,
                            "peak": d2h_gbs, "unit": "GB/s", "frac": v32 * b32 / per_rank / 1e9 / d2h_gbs,
                            "peak_source": "measured here: 16 pinned device->host copies of one frame"}}
        v8, b8 = e2e_run(_lib.GES_IMAGE_RGBA8, lanes)
        e2e_u8 = {"value": v8, "unit": "frames/s", "h2d_bytes_per_step": per_rank * C.sizeof(_lib.Camera),
                  "d2h_bytes_per_step": b8,
                  "path": f"same, RGBA8 frames (the saved 8-bit image, datasets.py:54-56) out, "
                          f"views on {lanes} render streams"}

    # ---- the other BASELINE configurations, measured in the same run (rank 0, N=1, default workload)
    others = None
    if rank == 0 and world == 1 and cfg == 2 and args.ss == 1 and not args.strips and not args.no_others:
        others = {}
        for oc in (3, 4, 5):
            others[f"config{oc}"] = measure_config(oc, dev, args.streams, steps=5, warmup=3)
            torch.cuda.empty_cache()

    # ---- CPU baseline sample (rank 0, N=1 only)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        threads = os.cpu_count() or 1
        fs, wall, nt, tot = cpu_sample(cfg, scene, cams[0], args.cpu_tiles, threads, args.ss)
        cpu = {"value": 1.0 / fs, "unit": "frames/s", "cores": threads, "kind": "port", "cpu_model": cpu_model(),
               "sample": f"oracle/ges_oracle.py (reference algorithm, float32), full per-frame "
                         f"preprocessing + {nt} of {tot} tiles of one view"
                         f"{'' if nt == tot else ', extrapolated'}; "
                         f"{threads} tile threads; {wall:.1f} s of CPU work",
               "frame_s": fs}

    if rank != 0:
        return
    balg = b_alg(cfg, [full_cam] if strips is not None else cams)
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except (OSError, ValueError):
        pass
    peak = float(peaks.get("hbm_gbs", 6650.0))
    achieved = balg / (frame_ms / 1e3) / 1e9
    traffic = None
    issue = None
    tp = os.path.join(ROOT, "profiles", f"traffic_config{cfg}.json")
    if os.path.exists(tp) and args.ss == 1 and args.layers == "full":
        prof = json.load(open(tp))
        traffic = prof.get("dram_bytes_per_frame")
        wi = prof.get("warp_instructions_per_frame")
        if wi:
            # instruction-issue view of the same frame: warp-instructions per frame (ncu, profiles/)
            # x frames/s per GPU against 148 SMs x 4 schedulers x the SM clock
            sm_mhz = clk.summary().get("sm_mhz")
            issue_peak = 148 * 4 * sm_mhz * 1e6 if sm_mhz else None
            if issue_peak:
                ach = wi * fps / world
                issue = {"warp_instructions_per_frame": wi, "achieved_per_s": ach, "peak_per_s": issue_peak,
                         "frac": ach / issue_peak, "source": "profiles/" + os.path.basename(tp)}
    line = {
        "metric": METRIC, "value": fps, "unit": "frames/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "strong" if (cfg == 5 and not args.views) or strips is not None else "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {**base_config(cfg, per_rank, world, args.ss),
                   **({"parallelism": f"row strips x{world}", "strips": strips,
                       "views_per_rank_per_step": "one band of one frame"} if strips is not None else {}),
                   **({} if gather_used != "nccl" or args.gather == "nccl" else
                      {"frame_gather": "NCCL gather of RGBA8 frames (peer buffer unavailable)"})},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic,
                     "unit_of_work": "one frame (ges_render: 5 kernels + 2 memsets)",
                     "b_alg_bytes_per_frame": balg, "frame_ms": frame_ms, "frame_ms_profiled": frame_ms_profiled,
                     "achieved_pipelined": balg * fps / world / 1e9,
                     "note": "achieved = B_alg / isolated frame time (single stream, one ges_render, events "
                             "around it; phase_ms from ges_render_profiled); "
                             "achieved_pipelined = B_alg x frames/s per GPU of the multi-stream step. The tile "
                             "kernel is issue/latency-bound, not HBM-bound (profiles/README.md)",
                     "issue": issue,
                     "peak_source": "MEASURED_PEAKS.json hbm_gbs" if peaks else "fallback 6650 GB/s",
                     "phase_ms": phase, "dominant": max(phase, key=phase.get)},
        "cpu_baseline": cpu,
        "e2e": e2e if cfg != 5 else {"value": None, "note": "config 5 (256 x 4K RGBA8 = 8.5 GB per step) "
                                     "is measured device-side only; e2e is config 2's"},
        "e2e_rgba8": e2e_u8,
        "gpu_launches": frames * (5 if ds.n_gaussians else 4),
        "clocks": clk.summary(),
        "scene_upload_ms": upload_ms,
        "scene_replication": "one scene per rank" if world == 1 else
                             f"rank 0 packs, packed blob ({ds.nbytes / 1e6:.0f} MB) broadcast over {dist.get_backend()}",
        "pairs_per_frame": {"surfel": s_pairs, "gaussian": g_pairs},
        "cuda_graph_captured": graphed,
        "other_configs": others,
    }
    print(json.dumps(line), flush=True)


def main():
    args = ARGS
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    import torch
    import torch.distributed as dist
    if "GES_BENCH_DEVICE" in os.environ:
        # functional test of the N > 1 code path on a one-GPU box (all ranks on one
        # device, gloo): not a measurement
        local_rank = int(os.environ["GES_BENCH_DEVICE"])
    if world > 1:
        torch.cuda.set_device(local_rank)
        backend = os.environ.get("GES_BENCH_BACKEND", "nccl")
        if backend == "nccl":
            # communicator lines (nRanks, NVLS/P2P transport) on stderr for the run's log
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        else:
            dist.init_process_group(backend)
    try:
        run_gpu(args, rank, world, local_rank)
    finally:
        if world > 1:
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
