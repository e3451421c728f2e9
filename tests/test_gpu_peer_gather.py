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


def _nccl_worker(rank, world, port, out_path, log_path):
    import paper_2504_17545_b200 as G
    from paper_2504_17545_b200 import scenes as S
    from paper_2504_17545_b200.multiview import PeerFrameGather, ViewBatchRenderer, gather_frames
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), NCCL_DEBUG="INFO",
                      NCCL_DEBUG_SUBSYS="INIT", NCCL_DEBUG_FILE=log_path)
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", 0))
    try:
        scene = S.random_scene(np.random.default_rng(6), 120, 60, degree=2)
        cams = S.orbit_views(3, 64, 48)
        ds = G.DeviceScene(scene)
        settings = G.RenderSettings()
        # peer-memory form: IPC buffer, tile kernel writes into it, NCCL fence
        sink = PeerFrameGather(3, 48, 64, dst=0)
        vb = ViewBatchRenderer(G.Renderer(), ds, cams, settings, want=("image_rgba8",), rgba_out=sink.slots)
        vb.render(check=True)
        sink.fence()
        peer = sink.frames.cpu().numpy().copy()
        # NCCL gather form (the bench's fallback)
        # scene replication by NCCL broadcast (one rank: the source keeps its own scene)
        from paper_2504_17545_b200.multiview import broadcast_scene
        assert broadcast_scene(ds, src=0) is ds
        vb2 = ViewBatchRenderer(G.Renderer(), ds, cams, settings, want=("image_rgba8",))
        vb2.render(check=True)
        got = gather_frames(vb2.rgba, dst=0)
        torch.cuda.synchronize()
        np.savez(out_path, peer=peer, gathered=got.cpu().numpy(), local=vb2.rgba.cpu().numpy(),
                 backend=dist.get_backend(), world=dist.get_world_size())
        sink.close()
    finally:
        dist.destroy_process_group()


def test_nccl_one_rank_fence_and_gather(tmp_path):
    """The NCCL code paths of the multi-GPU bench on the one GPU this box has:
    process-group init with device_id, the peer buffer's NCCL fence
    (all-reduce) and the NCCL frame gather, in a one-rank communicator (the
    collectives run; a one-GPU box cannot run two NCCL ranks)."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    out = str(tmp_path / "nccl.npz")
    log = str(tmp_path / "nccl.log")
    mp.start_processes(_nccl_worker, args=(1, _free_port(), out, log), nprocs=1, join=True, start_method="spawn")
    z = np.load(out)
    assert str(z["backend"]) == "nccl" and int(z["world"]) == 1
    assert z["gathered"].shape == z["local"].shape == z["peer"].shape == (3, 48, 64, 4)
    assert np.array_equal(z["gathered"], z["local"])
    assert np.abs(z["peer"].astype(int) - z["local"].astype(int)).max() <= 1
    text = open(log).read() if os.path.exists(log) else ""
    assert "NCCL INFO" in text and "nRanks 1" in text, text[-2000:]


def _strip_worker(rank, world, port, out_path):
    import paper_2504_17545_b200 as G
    from paper_2504_17545_b200 import scenes as S
    from paper_2504_17545_b200.multiview import PeerFrameGather, ViewBatchRenderer, strip_bounds, strip_camera
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        r = np.random.default_rng(8)
        scene = G.Scene(S.random_surfels(r, 20000, 2, scale_range=(0.005, 0.02)),
                        S.random_gaussians(r, 6000, 2, scale_range=(0.004, 0.025), extent=1.2), 2,
                        G.Stage.FROZEN)
        cam = S.make_camera(640, 360)
        bounds = strip_bounds(cam.height, world)
        ds = G.DeviceScene(scene)
        settings = G.RenderSettings()
        sink = PeerFrameGather(1, cam.height, cam.width, dst=0, strips=bounds)
        y0, y1 = bounds[rank]
        vb = ViewBatchRenderer(G.Renderer(), ds, [strip_camera(cam, y0, y1)], settings, want=("image_rgba8",),
                               rgba_out=sink.slots)
        vb.render(check=True)
        sink.fence()
        if rank == 0:
            got = sink.frames[0].cpu().numpy().copy()
            ref = ViewBatchRenderer(G.Renderer(), ds, [cam], settings, want=("image_rgba8",))
            ref.render(check=True)
            torch.cuda.synchronize()
            np.savez(out_path, got=got, ref=ref.rgba[0].cpu().numpy(), bounds=np.array(bounds))
        dist.barrier()
        sink.close()
    finally:
        dist.destroy_process_group()


def test_screen_strips_assemble_the_full_frame(tmp_path):
    """Screen-strip partition of one frame: two ranks render
    the two row bands as cameras of their own straight into rank 0's frame;
    the assembled frame equals the full render (RGBA8 within 1 LSB; the
    per-pixel tests do not depend on the tiling, fp32 sums on the order)."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    out = str(tmp_path / "strips.npz")
    mp.start_processes(_strip_worker, args=(2, _free_port(), out), nprocs=2, join=True, start_method="spawn")
    z = np.load(out)
    got, ref = z["got"].astype(int), z["ref"].astype(int)
    assert got.shape == ref.shape == (360, 640, 4)
    assert tuple(z["bounds"][1]) == (z["bounds"][0][1], 360)
    d = np.abs(got - ref).max(axis=-1)
    assert (d > 1).mean() <= 1e-3, int((d > 1).sum())   # (a winner flip on a depth tie can exceed 1 LSB)
    assert (got[..., 3] == 255).all()


def _bcast_worker(rank, world, port, out_path):
    import paper_2504_17545_b200 as G
    from paper_2504_17545_b200 import scenes as S
    from paper_2504_17545_b200.multiview import broadcast_scene
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        r = np.random.default_rng(12)
        cam = S.make_camera(160, 120)
        scene = None
        if rank == 0:
            scene = G.Scene(S.random_surfels(r, 3000, 3, scale_range=(0.01, 0.04)),
                            S.random_gaussians(r, 1500, 3, scale_range=(0.01, 0.05), extent=1.2), 3, G.Stage.FROZEN)
        ds = broadcast_scene(scene, src=0, device="cuda:0")
        fr = G.Renderer().render(ds, cam, G.RenderSettings(), want=("image", "s_winner"))
        img, win = fr.image.cpu().numpy(), fr.s_winner.cpu().numpy()
        torch.cuda.synchronize()
        objs = [None, None]
        dist.all_gather_object(objs, (img, win))
        if rank == 0:
            np.savez(out_path, img0=objs[0][0], win0=objs[0][1], img1=objs[1][0], win1=objs[1][1])
        dist.barrier()
    finally:
        dist.destroy_process_group()


def test_broadcast_scene_renders_like_the_source(tmp_path):
    """Scene replication (multiview.broadcast_scene): rank 0
    packs, rank 1 receives the packed blob by broadcast and renders the same
    frame from it (winners identical, image within float rounding of the
    order-free Gaussian sums)."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    out = str(tmp_path / "bcast.npz")
    mp.start_processes(_bcast_worker, args=(2, _free_port(), out), nprocs=2, join=True, start_method="spawn")
    z = np.load(out)
    assert np.array_equal(z["win0"], z["win1"]) and (z["win0"] >= 0).any()
    assert np.abs(z["img0"] - z["img1"]).max() <= 1e-5


def test_from_blob_copy_renders_identically():
    """DeviceScene.from_blob over a copy of a packed scene's bytes: every
    array pointer rebased, same frame."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2504_17545_b200 as G
    from paper_2504_17545_b200 import scenes as S
    r = np.random.default_rng(13)
    scene = G.Scene(S.random_surfels(r, 3000, 2, scale_range=(0.01, 0.04)),
                    S.random_gaussians(r, 1500, 2, kind=G.GaussianKind.TWO_D, scale_range=(0.01, 0.05), extent=1.2),
                    2, G.Stage.FROZEN)
    ds = G.DeviceScene(scene)
    cp = G.DeviceScene.from_blob(ds.header(), ds.blob.clone())
    assert cp.blob.data_ptr() != ds.blob.data_ptr()
    cam = S.make_camera(200, 150)
    rend = G.Renderer()
    a = rend.render(ds, cam, G.RenderSettings(), want=("image", "s_winner"))
    a_img, a_win = a.image.cpu().numpy(), a.s_winner.cpu().numpy()
    del ds   # the copy must not read the source blob
    torch.cuda.empty_cache()
    b = rend.render(cp, cam, G.RenderSettings(), want=("image", "s_winner"))
    assert np.array_equal(a_win, b.s_winner.cpu().numpy()) and (a_win >= 0).any()
    assert np.abs(a_img - b.image.cpu().numpy()).max() <= 1e-5
