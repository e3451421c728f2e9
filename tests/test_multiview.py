"""Multi-GPU view sharding and frame gather, exercised on CPU
with the gloo backend at world_size 2: each rank renders its block of views
with the CPU oracle (stand-in for the device renderer, which needs a GPU) and
the frames are gathered to rank 0 in view order."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2504_17545_b200 import scenes as S
from paper_2504_17545_b200.multiview import gather_frames, shard


def test_shard_blocks_cover_views_exactly_once():
    for n in (1, 7, 8, 256, 257):
        for world in (1, 2, 3, 4, 8):
            seen = []
            for r in range(world):
                seen += list(shard(n, r, world))
            assert seen == list(range(n))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _render_rgba(scene, cam):
    from oracle import ges_oracle as O
    img = O.render(scene, cam, None).image
    u8 = np.clip(img * 255.0 + 0.5, 0, 255).astype(np.uint8)
    out = np.full(u8.shape[:2] + (4,), 255, np.uint8)
    out[..., :3] = u8
    return out


def _worker(rank, world, port, n_views, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        scene = S.random_scene(np.random.default_rng(3), 30, 20)
        cams = S.orbit_views(n_views, 24, 16)
        mine = shard(n_views, rank, world)
        local = torch.from_numpy(np.stack([_render_rgba(scene, cams[v]) for v in mine]))
        out = gather_frames(local, dst=0)
        if rank == 0:
            q.put(out.numpy())
        else:
            assert out is None
    finally:
        dist.destroy_process_group()


def test_gather_frames_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    n_views = 6
    procs = [ctx.Process(target=_worker, args=(r, 2, port, n_views, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    scene = S.random_scene(np.random.default_rng(3), 30, 20)
    cams = S.orbit_views(n_views, 24, 16)
    expect = np.stack([_render_rgba(scene, c) for c in cams])
    assert got.shape == expect.shape
    assert np.array_equal(got, expect)


def test_strip_bounds_and_cameras_tile_the_frame():
    """Screen strips (SURVEY 8(e) single huge frame): the bands cover the
    rows exactly once, and each strip camera's pixel-centre rays are the
    full camera's rays of those rows (cameras.py:59-73)."""
    import numpy as np
    from oracle import ges_oracle as O
    from paper_2504_17545_b200 import scenes as S
    from paper_2504_17545_b200.multiview import strip_bounds, strip_camera
    cam = S.make_camera(200, 150)
    full = O.as_cam(cam).rays()
    for world in (1, 2, 3, 4, 8):
        b = strip_bounds(cam.height, world, align=16)
        assert b[0][0] == 0 and b[-1][1] == cam.height and len(b) == world
        assert all(b[i][1] == b[i + 1][0] for i in range(world - 1))
        assert all(y0 % 16 == 0 for y0, _ in b)
        for y0, y1 in b:
            if y1 > y0:
                sc = strip_camera(cam, y0, y1)
                assert (sc.height, sc.width) == (y1 - y0, cam.width)
                np.testing.assert_array_equal(O.as_cam(sc).rays(), full[y0:y1])
    # cost-weighted cuts: all the weight in the bottom half moves the cut down
    w = np.r_[np.zeros(75), np.ones(75)]
    (a0, a1), (b0, b1) = strip_bounds(150, 2, weights=w, align=1)
    assert a1 > 100


def _fake_header(nbytes):
    offs = {n: 256 * i for i, n in enumerate(("s_pos_s1", "s_quat", "s_s2", "s_sh", "s_id", "s_pack", "g_pos_op",
                                              "g_quat", "g_scale_eps", "g_sh"))}
    offs["g_sh"] = None   # (an array the pack left unset)
    return {"n_surfels": 5, "n_gaussians": 3, "sh_degree": 1, "dim": 3, "nbytes": nbytes, "offsets": offs,
            "bounds": [0.5, -1.0, 2.0, 3.0, 4.0, 5.0, 0.25], "any_filter": True}


def _bcast_worker(rank, world, port, q):
    from paper_2504_17545_b200.multiview import broadcast_scene
    from paper_2504_17545_b200.renderer import DeviceScene
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n = 4096
        src = None
        if rank == 0:   # a host blob stands in for the packed device scene (gloo moves host tensors)
            src = DeviceScene.from_blob(_fake_header(n), (torch.arange(n) * 7 % 251).to(torch.uint8))
        ds = broadcast_scene(src, src=0, device="cpu")
        base = ds.blob.data_ptr()
        ptrs = {k: getattr(ds.c, k) for k in DeviceScene._PTRS}
        q.put((rank, ds.blob.numpy().copy(), {k: (None if v is None else v - base) for k, v in ptrs.items()},
               (ds.c.n_surfels, ds.c.n_gaussians, ds.c.sh_degree, ds.c.gaussian_dim, list(ds.c.bounds),
                ds.any_filter, ds.header())))
    finally:
        dist.destroy_process_group()


def test_broadcast_scene_gloo_world2():
    """rank 0 packs, the other ranks rebuild the scene from the
    broadcast blob -- same bytes, every array pointer rebased onto the
    receiver's own blob, same counts and slab bounds."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_bcast_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = dict((r, rest) for r, *rest in (q.get(timeout=120) for _ in range(2)))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    hdr = _fake_header(4096)
    for r in (0, 1):
        blob, offs, (ns, ng, deg, dim, bounds, anyf, h) = got[r]
        assert np.array_equal(blob, (np.arange(4096) * 7 % 251).astype(np.uint8))
        assert offs == hdr["offsets"]
        assert (ns, ng, deg, dim, bounds, anyf) == (5, 3, 1, 3, hdr["bounds"], True)
        assert h == hdr


def test_from_blob_rejects_bad_blobs():
    from paper_2504_17545_b200.renderer import DeviceScene
    with pytest.raises(ValueError):
        DeviceScene.from_blob(_fake_header(4096), torch.zeros(100, dtype=torch.uint8))
    with pytest.raises(ValueError):
        DeviceScene.from_blob(_fake_header(4096), torch.zeros(4096, dtype=torch.float32))
    bad = _fake_header(4096)
    bad["offsets"]["s_quat"] = 5000
    with pytest.raises(ValueError):
        DeviceScene.from_blob(bad, torch.zeros(4096, dtype=torch.uint8))
