"""GPU joint-stage training step: the CUDA forward and
backward of paper_2504_17545_b200.training against the real reference's
training step (golden vectors, tests/golden/make_train_golden.py) and against
the float64 oracle (oracle/ges_train_oracle.py) on larger random scenes.

Tolerances: the GPU evaluates pixels in float32 (forward buffers within
TOL_FWD of the float64 reference) and sums fragments with float64 atomics;
gradients agree to REL_GRAD of each array's largest entry.  A fragment at
the 1/255 alpha cutoff or the depth gate may flip between float32 and
float64; its contribution is bounded by the cutoff, well inside REL_GRAD.
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2504_17545_b200 import scenes as S  # noqa: E402
from paper_2504_17545_b200 import training as TR  # noqa: E402
from paper_2504_17545_b200.types import GaussianKind, Scene, Stage  # noqa: E402
from golden_io import TRAIN_GRADS, load_train, train_names, train_settings  # noqa: E402
from oracle import ges_train_oracle as TO  # noqa: E402

TOL_FWD = 2e-4
REL_GRAD = 2e-3


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _flags(scene, cam, st):
    """The parity rule's per-pixel flags (tests/parity.py) for the training
    forward of this case: the frozen surfel pass is the supersampled opaque
    z-buffer and the Gaussian pass is gated by sub-sample (0,0)'s depth, as in
    render() with the same settings (training.py:358-392)."""
    from golden_io import settings_ns
    from oracle import ges_oracle as O
    w = np.asarray(scene.surfels.w)
    ss = st.get("supersample") or (4 if (w.size == 0 or w.min() >= 30.0) else 1)
    keys = ("mip", "with_geometry", "epsilon_mode", "epsilon_value", "background")
    o = O.render(scene, cam, settings_ns(dict({k: st[k] for k in keys if k in st}, supersample=ss)), ties=True)
    return o.tie, o.tie_color, o.tie_cut


def _fwd_close(name, a, b, flags, tol=TOL_FWD):
    """Every pixel within tol except the oracle's hard ties (excluded, at most
    0.5 %) and colour-only sub-sample ties; pixels holding fragments at the
    1/255 cutoff within tol + one flipped fragment's change per flagged
    fragment (alpha <= CUT_FLIP times the value range)."""
    from parity import CUT_FLIP
    a, b = np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64)
    assert a.shape == b.shape, name
    tie, tie_color, cut = flags
    assert tie.sum() <= max(0.005 * tie.size, 2), (name, int(tie.sum()))
    keep = ~tie & ~(tie_color if name in ("image", "surfel_color") else np.zeros_like(tie))
    inf = np.isinf(b)
    assert np.array_equal(np.isinf(a)[keep], inf[keep]), name
    m = keep & ~(inf.any(-1) if inf.ndim == 3 else inf)
    with np.errstate(invalid="ignore"):
        err = np.abs(a - b)
    if err.ndim == 3:
        err = err.max(axis=-1)
    fin = np.isfinite(b)
    span = float(np.abs(b[fin]).max()) if fin.any() else 1.0
    allow = tol + cut * CUT_FLIP * 2.0 * max(span, 1.0)
    bad = m & (err > allow)
    assert not bad.any(), (name, float(err[m].max()), int(bad.sum()))


def _grad_close(name, a, b, rel=REL_GRAD):
    assert a.shape == b.shape, name
    if b.size == 0:
        return
    scale = max(float(np.abs(b).max()), 1e-6)
    err = float(np.abs(a - b).max())
    assert err <= rel * scale, (name, err, scale)


@pytest.mark.parametrize("name", train_names())
def test_training_step_matches_reference(name):
    scene, cam, st, g_img, cot, fwd, grads = load_train(name)
    settings = train_settings(st, TR.TrainSettings)
    frame = TR.render_training(scene, cam, settings, cache_key=0)
    flags = _flags(scene, cam, st)
    for k, v in fwd.items():
        _fwd_close(k, getattr(frame, k), v, flags)
    out = TR.backward(frame, g_img, **cot)
    for k in TRAIN_GRADS:
        _grad_close(k, getattr(out, k), grads[k])
    out.check_finite()
    # the joint stage's pruning statistic for this view (optim.py:519-533)
    sc = TR.contribution_scores(scene, [cam], train_settings(st, TR.TrainSettings), cache_keys=[0])
    _grad_close("contrib", sc, grads["contrib"], rel=1e-4)


def _random_case(seed, kind, ns=60, ng=150, deg=2, res=(96, 80), mip=False):
    r = np.random.default_rng(seed)
    s = S.random_surfels(r, ns, deg, scale_range=(0.05, 0.2))
    g = S.random_gaussians(r, ng, deg, kind=kind, scale_range=(0.03, 0.15))
    if mip:
        g = S.mip_world_filter(g, [S.make_camera(128, 128)])
    return Scene(s, g, deg, Stage.FROZEN), S.make_camera(*res)


@pytest.mark.parametrize("kind", [GaussianKind.THREE_D, GaussianKind.TWO_D])
@pytest.mark.parametrize("mip,geom", [(False, False), (True, True)])
def test_training_step_matches_oracle_random(kind, mip, geom):
    scene, cam = _random_case(71 + mip, kind, mip=mip)
    st = dict(mip=mip, with_geometry=geom)
    rng = np.random.default_rng(3)
    H, W = cam.height, cam.width
    g_img = rng.standard_normal((H, W, 3))
    cot = {}
    if geom:
        cot = dict(g_gauss_depth=0.1 * rng.standard_normal((H, W)),
                   g_gauss_normal=0.1 * rng.standard_normal((H, W, 3)))
    so = train_settings(st, TR.TrainSettings)
    ref = TO.render_training(scene, cam, so, cache=so.frozen_cache, cache_key=1)
    rout = TO.backward(scene, cam, so, ref, g_img, **cot)
    sg = train_settings(st, TR.TrainSettings)
    frame = TR.render_training(scene, cam, sg, cache_key=1)
    flags = _flags(scene, cam, st)
    _fwd_close("image", frame.image, ref["image"], flags)
    _fwd_close("gauss_weight", frame.gauss_weight, ref["gauss_weight"], flags)
    out = TR.backward(frame, g_img, **cot)
    for k in TRAIN_GRADS:
        _grad_close(k, getattr(out, k), rout[k])
    sc = TR.contribution_scores(scene, [cam], train_settings(st, TR.TrainSettings), cache_keys=[1])
    _grad_close("contrib", sc, rout["contrib"], rel=1e-4)


def test_frozen_cache_is_reused_and_translucent_pass_raises():
    scene, cam = _random_case(5, GaussianKind.THREE_D, ns=30, ng=40)
    st = TR.TrainSettings(frozen_cache={})
    f1 = TR.render_training(scene, cam, st, cache_key="v0")
    entry = st.frozen_cache["v0"]
    f2 = TR.render_training(scene, cam, st, cache_key="v0")
    assert st.frozen_cache["v0"] is entry
    assert np.array_equal(f1.image, f2.image)
    soft = Scene(scene.surfels.select(np.arange(30)), scene.gaussians, scene.sh_degree, Stage.JOINT)
    soft.surfels.w = np.full(30, 40.0)
    with pytest.raises(NotImplementedError):
        TR.render_training(soft, cam, TR.TrainSettings(frozen_cache={}))
    with pytest.raises(NotImplementedError):
        TR.render_training(scene, cam, TR.TrainSettings())   # no frozen cache: translucent pass
    with pytest.raises(ValueError):
        TR.backward(TR.TrainFrame(None, None, None, None, None), np.zeros((cam.height, cam.width, 3)))


def test_training_gradient_descends_loss():
    """One SGD step on the Gaussians along -grad lowers an L2 image loss."""
    scene, cam = _random_case(9, GaussianKind.THREE_D, ns=40, ng=80, deg=1)
    target = np.random.default_rng(1).uniform(0, 1, (cam.height, cam.width, 3))
    st = TR.TrainSettings(frozen_cache={})

    def loss_and_grad(sc):
        fr = TR.render_training(sc, cam, st, cache_key=0)
        diff = fr.image - target
        return float(np.sum(diff ** 2)), TR.backward(fr, 2.0 * diff)

    l0, g = loss_and_grad(scene)
    lr = 1e-4
    gs = scene.gaussians
    new_g = type(gs)(gs.pos - lr * g.gaussian_pos, gs.raw_opacity, gs.quat, gs.log_scale,
                     gs.sh - lr * 10 * g.gaussian_sh, gs.kind, gs.filter3d)
    l1, _ = loss_and_grad(Scene(scene.surfels, new_g, scene.sh_degree, scene.stage))
    assert l1 < l0


def test_contribution_scores_max_over_views():
    scene, cam0 = _random_case(13, GaussianKind.THREE_D, ns=50, ng=120)
    cams = [cam0, S.make_camera(96, 80, azim=1.1), S.make_camera(96, 80, azim=2.3, elev=0.5)]
    so = TR.TrainSettings(frozen_cache={})
    ref = np.zeros(scene.gaussians.count)
    for k, c in enumerate(cams):
        fr = TO.render_training(scene, c, so, cache=so.frozen_cache, cache_key=k)
        out = TO.backward(scene, c, so, fr, np.zeros((c.height, c.width, 3)))
        ref = np.maximum(ref, out["contrib"])
    got = TR.contribution_scores(scene, cams, TR.TrainSettings(frozen_cache={}), cache_keys=[0, 1, 2])
    assert got.shape == ref.shape and np.count_nonzero(ref) > 10
    _grad_close("contrib", got, ref, rel=1e-4)
