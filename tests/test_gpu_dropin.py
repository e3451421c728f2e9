"""The drop-in's "pure function, thread-safe" contract (
the reference's render has no hidden state): concurrent Python threads get
the same frames as sequential calls, and in-place edits of a scene's arrays
are seen by the next render (scene cache fingerprint)."""

import threading

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2504_17545_b200 as G  # noqa: E402
from paper_2504_17545_b200 import scenes as S  # noqa: E402
from paper_2504_17545_b200.renderer import SCENE_CACHE  # noqa: E402
from paper_2504_17545_b200.types import Scene, Stage  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _scene(seed, ns=20000, ng=6000):
    r = np.random.default_rng(seed)
    return Scene(S.random_surfels(r, ns, 2, scale_range=(0.005, 0.02)),
                 S.random_gaussians(r, ng, 2, scale_range=(0.004, 0.025), extent=1.2), 2, Stage.FROZEN)


def test_four_threads_match_sequential_renders():
    scenes = [_scene(40), _scene(41)]
    jobs = [(scenes[k % 2], S.make_camera(320 + 32 * k, 200 + 16 * k, azim=0.4 * k),
             G.RenderSettings(supersample=4 if k % 3 == 0 else 1)) for k in range(8)]
    seq = [G.render(sc, cam, st) for sc, cam, st in jobs]
    got = [None] * len(jobs)
    errors = []
    barrier = threading.Barrier(4)

    def worker(t):
        try:
            barrier.wait()
            for rep in range(3):
                for k in range(t, len(jobs), 4):
                    sc, cam, st = jobs[k]
                    # half the threads on their own CUDA stream, half on the default one
                    if t % 2:
                        with torch.cuda.stream(torch.cuda.Stream()):
                            got[k] = G.render(sc, cam, st)
                    else:
                        got[k] = G.render(sc, cam, st)
        except Exception as e:   # pragma: no cover - reported below
            errors.append(e)

    th = [threading.Thread(target=worker, args=(t,)) for t in range(4)]
    for x in th:
        x.start()
    for x in th:
        x.join()
    assert not errors, errors
    for a, b in zip(seq, got):
        np.testing.assert_array_equal(a.surfels.winner, b.surfels.winner)
        np.testing.assert_array_equal(a.surfels.depth, b.surfels.depth)
        # Gaussian sums are order-independent up to fp32 rounding of the atomic list order
        assert float(np.max(np.abs(a.image - b.image))) <= 1e-5


def test_in_place_edit_is_seen_without_invalidate():
    sc = _scene(42, 5000, 2000)
    cam = S.make_camera(160, 120)
    a = G.render(sc, cam)
    sc.surfels.pos[:] += np.array([0.05, 0.0, 0.0])          # optimiser-style whole-array edit
    sc.gaussians.raw_opacity[:] -= 0.5
    b = G.render(sc, cam)
    assert not np.array_equal(a.surfels.winner, b.surfels.winner)
    fresh = Scene(G.SurfelSet(sc.surfels.pos.copy(), sc.surfels.quat.copy(), sc.surfels.log_scale.copy(),
                              sc.surfels.sh.copy(), sc.surfels.w.copy()),
                  G.GaussianSet(sc.gaussians.pos.copy(), sc.gaussians.raw_opacity.copy(), sc.gaussians.quat.copy(),
                                sc.gaussians.log_scale.copy(), sc.gaussians.sh.copy(), sc.gaussians.kind,
                                sc.gaussians.filter3d.copy()), sc.sh_degree, Stage.FROZEN)
    c = G.render(fresh, cam)
    np.testing.assert_array_equal(b.surfels.winner, c.surfels.winner)
    assert float(np.max(np.abs(b.image - c.image))) <= 1e-5   # fp32 sums in atomic list order


def test_single_element_edit_full_verify_and_invalidate():
    sc = _scene(43, 3000, 0)
    cam = S.make_camera(96, 64)
    a = G.render(sc, cam)
    cov = np.flatnonzero(a.surfels.winner.ravel() >= 0)
    i = int(a.surfels.winner.ravel()[cov[len(cov) // 2]])
    old = SCENE_CACHE.verify
    try:
        SCENE_CACHE.verify = "full"
        sc.surfels.pos[i, 2] += 10.0          # push one visible surfel far away
        b = G.render(sc, cam)
        assert not np.any(b.surfels.winner == i) or not np.array_equal(a.surfels.depth, b.surfels.depth)
    finally:
        SCENE_CACHE.verify = old
    sc.surfels.pos[i, 2] -= 10.0
    G.invalidate(sc)
    c = G.render(sc, cam)
    np.testing.assert_array_equal(a.surfels.winner, c.surfels.winner)
