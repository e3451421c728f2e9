"""Multi-view batches and their distribution over GPUs.

Views are independent units (``render`` is a pure function of scene and
camera, forward.py:403); the reference's multi-view callers loop over them
(metrics.py:60-66, cli.py:165-168).  Here each rank holds a full scene
replica, renders a contiguous block of views, and the only inter-GPU
traffic is one frame gather to the destination rank over NCCL (NVLink),
of RGBA8 frames the tile kernel writes straight into the send buffer.
"""

from __future__ import annotations

import math

import torch
import torch.distributed as dist


def shard(n_views: int, rank: int, world: int) -> range:
    """Contiguous block of ceil(n/world) views for ``rank``."""
    per = math.ceil(n_views / world) if world else 0
    lo = min(n_views, rank * per)
    return range(lo, min(n_views, lo + per))


def gather_frames(local: torch.Tensor, dst: int = 0, group=None):
    """Gather equally-shaped per-rank frame batches (V, H, W, C) to ``dst``.
    Returns the (world*V, H, W, C) batch on ``dst`` and None elsewhere."""
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return local
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    if rank == dst:
        out = torch.empty((world,) + tuple(local.shape), dtype=local.dtype, device=local.device)
        dist.gather(local.contiguous(), gather_list=list(out.unbind(0)), dst=dst, group=group)
        return out.reshape((world * local.shape[0],) + tuple(local.shape[1:]))
    dist.gather(local.contiguous(), gather_list=None, dst=dst, group=group)
    return None


class ViewBatchRenderer:
    """Renders a batch of views of one packed scene, asynchronously on the
    current stream, into preallocated outputs: a (V, H, W, 4) RGBA8 send
    buffer when all views share one resolution (a list of (H, W, 4) buffers
    otherwise, e.g. the multi-scale Mip views), plus any other requested
    buffers (fp32 image, depth, winner ...)."""

    def __init__(self, renderer, scene, cams, settings, *, want=("image_rgba8",), streams: int = 1):
        """``streams`` > 1 pipelines consecutive views on that many CUDA
        streams, each with its own frame workspace, so one view's
        preprocessing/binning overlaps another view's tile kernel."""
        self.r = renderer
        self.pool = [renderer] + [type(renderer)(renderer.device) for _ in range(max(streams, 1) - 1)]
        self.streams = [None] + [torch.cuda.Stream(renderer.device) for _ in range(max(streams, 1) - 1)]
        self.scene = scene
        self.cams = list(cams)
        self.settings = settings
        shapes = {(int(c.height), int(c.width)) for c in self.cams}
        dev = renderer.device
        self.frames = []
        if len(shapes) == 1:
            H, W = shapes.pop()
            self.rgba = torch.empty((len(self.cams), H, W, 4), dtype=torch.uint8, device=dev)
            bufs = list(self.rgba.unbind(0))
        else:
            bufs = [torch.empty((int(c.height), int(c.width), 4), dtype=torch.uint8, device=dev)
                    for c in self.cams]
            self.rgba = bufs
        for c, b in zip(self.cams, bufs):
            fr = renderer.alloc(c, settings, want=[k for k in want if k != "image_rgba8"])
            fr.image_rgba8 = b
            self.frames.append(fr)

    def capture(self) -> bool:
        """Record the whole batch (all views, all streams) into one CUDA graph
        so a step is a single graph launch.  Call after a checked render has
        sized every workspace; returns False (and keeps eager launches) if
        capture is unavailable."""
        try:
            torch.cuda.synchronize(self.r.device)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                self._launch(check=False)
            self.graph = g
            return True
        except RuntimeError:
            self.graph = None
            return False

    def render(self, check: bool = False):
        if getattr(self, "graph", None) is not None and not check:
            self.graph.replay()
            return self.rgba
        return self._launch(check)

    def _launch(self, check: bool):
        if len(self.pool) == 1:
            for c, fr in zip(self.cams, self.frames):
                self.r.render(self.scene, c, self.settings, frame=fr, check=check)
            return self.rgba
        main = torch.cuda.current_stream(self.r.device)
        start = main.record_event()
        for s in self.streams[1:]:
            s.wait_event(start)          # outputs may still be read by earlier work on main
        k = len(self.pool)
        for v, (c, fr) in enumerate(zip(self.cams, self.frames)):
            s = self.streams[v % k]
            if s is None:
                self.pool[0].render(self.scene, c, self.settings, frame=fr, check=check)
            else:
                with torch.cuda.stream(s):
                    self.pool[v % k].render(self.scene, c, self.settings, frame=fr, check=check)
        for s in self.streams[1:]:
            main.wait_stream(s)
        return self.rgba

    def overflowed(self) -> bool:
        st = torch.stack([f.status for f in self.frames]).cpu()
        return bool(((st[:, 2] & 0xFFFFFFFF) != 0).any())
