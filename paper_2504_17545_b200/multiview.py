"""Multi-view batches and their distribution over GPUs.

Views are independent units (``render`` is a pure function of scene and
camera, forward.py:403); the reference's multi-view callers loop over them
(metrics.py:60-66, cli.py:165-168).  Here each rank holds a full scene
replica, renders a contiguous block of views, and the only inter-GPU
traffic is the frame gather to the destination rank.  Two forms:

* ``PeerFrameGather`` (default for the multi-GPU bench): the destination
  rank exports one device buffer through CUDA IPC; every rank's tile kernel
  writes its RGBA8 frames straight into its slice of that buffer over NVLink
  while it renders, so the transfer overlaps the tile work and no collective
  moves frames; a one-word all-reduce per step orders the writes before the
  destination reads them.
* ``gather_frames``: the plain NCCL ``gather`` of per-rank send buffers
  (baseline, also used on CPU/gloo).

One huge frame is split into screen strips instead (``strip_bounds`` /
``strip_camera``): rank r renders rows [y0, y1) as a camera of its own (the
principal point moved up by y0) -- preprocessing is repeated per rank, the
binning is clipped to the strip -- and ``PeerFrameGather(..., strips=...)``
lets each rank's tile kernel write its rows straight into the destination's
frame.
"""

from __future__ import annotations

import ctypes as C
import math

import numpy as np

import torch
import torch.distributed as dist


def shard(n_views: int, rank: int, world: int) -> range:
    """Contiguous block of ceil(n/world) views for ``rank``."""
    per = math.ceil(n_views / world) if world else 0
    lo = min(n_views, rank * per)
    return range(lo, min(n_views, lo + per))


def broadcast_scene(scene=None, src: int = 0, group=None, device=None):
    """Scene replication: rank ``src`` loads and packs the scene
    once (K0; ``scene`` is a reference ``Scene`` or an already packed
    ``DeviceScene``), every other rank receives the packed blob through one
    ``broadcast`` (NCCL over NVLink: ~0.3 GB at config 2, instead of each
    rank uploading the float64 source arrays and packing its own copy).
    Other ranks pass ``scene=None``.  Returns this rank's ``DeviceScene``
    (render-only on the receivers: the float64 source arrays stay on
    ``src``)."""
    from .renderer import DeviceScene

    if not dist.is_initialized():
        return scene if isinstance(scene, DeviceScene) else DeviceScene(scene, device)
    rank = dist.get_rank()   # (src is a global rank, as in dist.broadcast)
    ds = None
    hdr = [None]
    if rank == src:
        if scene is None:
            raise ValueError("the source rank needs the scene")
        ds = scene if isinstance(scene, DeviceScene) else DeviceScene(scene, device)
        hdr = [ds.header()]
    dist.broadcast_object_list(hdr, src=src, group=group)
    if rank == src:
        blob = ds.blob
    else:
        dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        blob = torch.empty(int(hdr[0]["nbytes"]), dtype=torch.uint8, device=dev)
    dist.broadcast(blob, src=src, group=group)
    return ds if rank == src else DeviceScene.from_blob(hdr[0], blob)


def strip_bounds(height: int, world: int, weights=None, align: int = 32) -> list:
    """Screen-strip partition of one frame (single huge frame):
    ``world`` bands of whole rows [y0, y1), cut at multiples of ``align``
    rows (the tile height) where possible.  ``weights``: optional per-row
    cost estimate (e.g. the pair counts of a previous frame's tile rows,
    repeated per row); the cuts then balance the summed weight instead of
    the row count."""
    if world <= 1:
        return [(0, height)]
    if weights is None:
        w = np.ones(height)
    else:
        w = np.asarray(weights, dtype=np.float64).reshape(-1)
        if w.size != height:
            raise ValueError("one weight per row")
        w = np.maximum(w, 0.0) + 1e-9
    c = np.concatenate([[0.0], np.cumsum(w)])
    cuts = [0]
    for r in range(1, world):
        y = int(np.searchsorted(c, c[-1] * r / world))
        y = int(round(y / align)) * align if align > 1 else y
        cuts.append(min(max(y, cuts[-1]), height))
    cuts.append(height)
    return [(cuts[i], cuts[i + 1]) for i in range(world)]


def strip_camera(cam, y0: int, y1: int):
    """The camera of rows [y0, y1) of ``cam``'s frame: same intrinsics and
    pose with the principal point moved up by y0, so every pixel centre ray
    (cameras.py:59-73) is the full frame's, and the strip renders exactly the
    full frame's rows (the per-pixel tests do not depend on the tiling)."""
    return type(cam)(cam.fx, cam.fy, cam.cx, cam.cy - y0, cam.width, y1 - y0, cam.world_to_camera)


def gather_frames(local: torch.Tensor, dst: int = 0, group=None):
    """Gather equally-shaped per-rank frame batches (V, H, W, C) to ``dst``.
    Returns the (world*V, H, W, C) batch on ``dst`` and None elsewhere."""
    if not dist.is_initialized():
        return local
    if dist.get_world_size(group) == 1 and dist.get_backend(group) != "nccl":
        return local   # (a one-rank NCCL communicator still runs the collective)
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    if local.is_cuda and dist.get_backend(group) != "nccl":   # gloo gathers host tensors only
        out = gather_frames(local.cpu(), dst, group)
        return out.to(local.device) if out is not None else None
    if rank == dst:
        out = torch.empty((world,) + tuple(local.shape), dtype=local.dtype, device=local.device)
        dist.gather(local.contiguous(), gather_list=list(out.unbind(0)), dst=dst, group=group)
        return out.reshape((world * local.shape[0],) + tuple(local.shape[1:]))
    dist.gather(local.contiguous(), gather_list=None, dst=dst, group=group)
    return None


class DevicePointer:
    """A raw device address with the ``data_ptr()`` the renderer's output
    binding reads (slices of a peer buffer are not torch allocations)."""

    def __init__(self, ptr: int, nbytes: int):
        self.ptr, self.nbytes = int(ptr), int(nbytes)

    def data_ptr(self) -> int:
        return self.ptr


class _CudaArray:
    """``__cuda_array_interface__`` view of a device buffer (torch.as_tensor)."""

    def __init__(self, ptr, shape):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": "|u1", "data": (int(ptr), False),
                                         "version": 3, "strides": None}


class PeerFrameGather:
    """Frame gather through peer memory (SURVEY 8(e) exchange step, fused with
    the rendering): ``dst`` allocates the (world * V, H, W, 4) RGBA8 batch and
    shares it by CUDA IPC; rank r's views go to rows [r*V, (r+1)*V).  Pass
    ``slots`` to ``ViewBatchRenderer(rgba_out=...)``; after each step call
    ``fence()`` on every rank; ``frames`` (dst only) is the gathered batch."""

    def __init__(self, frames_per_rank: int, height: int, width: int, *, dst: int = 0, group=None, device=None,
                 strips=None):
        """``strips``: screen-strip form instead of view batches -- one
        (height, width, 4) frame on ``dst``, this rank's slot the rows
        strips[rank] = (y0, y1) (``frames_per_rank`` must be 1)."""
        from . import _lib
        self.L = _lib.lib()
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.dst = dst
        self.device = torch.device(device or "cuda", torch.cuda.current_device()) if device is None \
            else torch.device(device)
        self.frame_bytes = height * width * 4
        V = frames_per_rank
        if strips is not None and V != 1:
            raise ValueError("the strip form gathers one frame")
        total = (1 if strips is not None else self.world * V) * self.frame_bytes
        handle = None
        self._owned = self._opened = None
        if self.rank == dst:
            ptr = C.c_void_p()
            hbuf = (C.c_char * 64)()
            if self.L.ges_peer_alloc(total, C.byref(ptr), hbuf) == 0:
                self._owned = ptr.value
                handle = bytes(hbuf)
        if self.world > 1:   # always reached by every rank, so a failure cannot strand the others
            obj = [handle]
            dist.broadcast_object_list(obj, src=dst, group=group)
            handle = obj[0]
        if handle is None:
            raise RuntimeError(f"peer buffer allocation failed on rank {dst}: {self.L.ges_last_error().decode(errors='replace')}"
                               if self.rank == dst else f"peer buffer allocation failed on rank {dst}")
        if self.rank == dst:
            base = self._owned
        else:
            ptr = C.c_void_p()
            _lib.check(self.L.ges_peer_open(handle, self.device.index, C.byref(ptr)), "peer buffer open")
            self._opened = base = ptr.value
        self.base = base
        if strips is not None:
            y0, y1 = strips[self.rank]
            self.slots = [DevicePointer(base + y0 * width * 4, (y1 - y0) * width * 4)]
            nf = 1
        else:
            first = self.rank * V * self.frame_bytes
            self.slots = [DevicePointer(base + first + k * self.frame_bytes, self.frame_bytes) for k in range(V)]
            nf = self.world * V
        self.frames = (torch.as_tensor(_CudaArray(base, (nf, height, width, 4)), device=self.device)
                       if self.rank == dst else None)
        self._flag = torch.zeros(1, device=self.device) if dist.is_initialized() else None

    def fence(self):
        """Order every rank's frame writes of this step before the
        destination's later work: one stream-ordered one-word all-reduce with
        NCCL (a rank's all-reduce starts only after its render kernels have
        finished); host synchronisation + barrier with other backends."""
        if not dist.is_initialized():
            return
        if dist.get_backend(self.group) == "nccl":
            dist.all_reduce(self._flag, group=self.group)
        else:
            torch.cuda.current_stream(self.device).synchronize()
            dist.barrier(group=self.group)

    def close(self):
        if self._opened:
            self.L.ges_peer_close(C.c_void_p(self._opened))
            self._opened = None
        if self._owned:
            torch.cuda.synchronize(self.device)
            self.frames = None
            self.L.ges_peer_free(C.c_void_p(self._owned))
            self._owned = None


class ViewBatchRenderer:
    """Renders a batch of views of one packed scene, asynchronously on the
    current stream, into preallocated outputs: the requested buffers (fp32
    image, depth, winner ...) and, when ``"image_rgba8"`` is requested or
    ``rgba_out`` is given, a (V, H, W, 4) RGBA8 send buffer when all views
    share one resolution (a list of (H, W, 4) buffers otherwise, e.g. the
    multi-scale Mip views); without either, ``rgba`` is None and no RGBA8
    frame is written."""

    def __init__(self, renderer, scene, cams, settings, *, want=("image_rgba8",), streams: int = 1,
                 rgba_out=None):
        """``streams`` > 1 pipelines consecutive views on that many CUDA
        streams, each with its own frame workspace, so one view's
        preprocessing/binning overlaps another view's tile kernel.
        ``rgba_out``: per-view RGBA8 destinations (e.g.
        ``PeerFrameGather.slots``) instead of a local send buffer."""
        self.r = renderer
        self.pool = [renderer] + [type(renderer)(renderer.device) for _ in range(max(streams, 1) - 1)]
        self.streams = [None] + [torch.cuda.Stream(renderer.device) for _ in range(max(streams, 1) - 1)]
        self.scene = scene
        self.cams = list(cams)
        self.settings = settings
        shapes = {(int(c.height), int(c.width)) for c in self.cams}
        dev = renderer.device
        self.frames = []
        # RGBA8 frames only when asked for (or given a destination): the
        # float outputs alone are the reference's RenderResult
        if rgba_out is None and "image_rgba8" not in want:
            bufs = [None] * len(self.cams)
            self.rgba = None
        elif rgba_out is not None:
            if len(rgba_out) != len(self.cams):
                raise ValueError("one RGBA8 destination per view")
            self.rgba = bufs = list(rgba_out)
        elif len(shapes) == 1:
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
