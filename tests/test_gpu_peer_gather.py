"""Peer-memory frame gather (multiview.PeerFrameGather): two
processes (gloo group) share the one GPU of the box -- CUDA IPC maps the
destination's buffer into the other process exactly as it maps it across
GPUs -- and each renders its block of views straight into the destination
rank's batch.  The kernels of the two ranks never wait on each other; only
the fence orders them before the destination reads the batch.  The result
must equal a local render of all views (RGBA8, within 1 LSB: Gaussian sums
are order-free up to float rounding)."""

import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n_views, out_path):
    import paper_2504_17545_b200 as G
    from paper_2504_17545_b200 import scenes as S
    from paper_2504_17545_b200.multiview import PeerFrameGather, ViewBatchRenderer, shard
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        scene = S.random_scene(np.random.default_rng(5), 120, 60, degree=2)
        cams = S.orbit_views(n_views, 64, 48)
        mine = list(shard(n_views, rank, world))
        ds = G.DeviceScene(scene)
        settings = G.RenderSettings()
        sink = PeerFrameGather(len(mine), 48, 64, dst=0)
        vb = ViewBatchRenderer(G.Renderer(), ds, [cams[v] for v in mine], settings, want=("image_rgba8",),
                               rgba_out=sink.slots, streams=2)
        vb.render(check=True)
        vb.capture()                      # the graph replays into the peer buffer too
        vb.render()
        sink.fence()
        if rank == 0:
            got = sink.frames.cpu().numpy().copy()
            ref = ViewBatchRenderer(G.Renderer(), ds, cams, settings, want=("image_rgba8",))
            ref.render(check=True)
            torch.cuda.synchronize()
            np.savez(out_path, got=got, ref=ref.rgba.cpu().numpy())
        dist.barrier()
        sink.close()
    finally:
        dist.destroy_process_group()


def test_peer_gather_matches_local_render(tmp_path):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    out = str(tmp_path / "peer.npz")
    mp.start_processes(_worker, args=(2, _free_port(), 4, out), nprocs=2, join=True, start_method="spawn")
    z = np.load(out)
    got, ref = z["got"].astype(int), z["ref"].astype(int)
    assert got.shape == ref.shape == (4, 48, 64, 4)
    assert np.abs(got - ref).max() <= 1
    assert (got[..., 3] == 255).all()
