"""The training-step oracle (oracle/ges_train_oracle.py) against golden
vectors of the real reference training step (tests/golden/make_train_golden.py:
ges.training.render_training + backward, float64).  Forward buffers at atol
1e-9; gradients at 1e-9 relative to each array's magnitude (the oracle sums
fragments per Gaussian, the reference over a sorted fragment list)."""

import numpy as np
import pytest

from golden_io import TRAIN_GRADS, load_train, train_names, train_settings
from oracle import ges_train_oracle as T


def _close_fwd(a, b):
    assert a.shape == b.shape
    inf = np.isinf(a) & np.isinf(b)
    assert np.array_equal(np.isinf(a), np.isinf(b))
    assert np.allclose(a[~inf], b[~inf], atol=1e-9, rtol=0)


def _close_grad(name, a, b, rel=1e-9):
    assert a.shape == b.shape, name
    scale = max(1.0, float(np.abs(b).max()) if b.size else 0.0)
    err = float(np.abs(a - b).max()) if b.size else 0.0
    assert err <= rel * scale, (name, err, scale)


@pytest.mark.parametrize("name", train_names())
def test_train_oracle_matches_reference(name):
    scene, cam, st, g_img, cot, fwd, grads = load_train(name)
    settings = train_settings(st)
    frame = T.render_training(scene, cam, settings, cache=settings.frozen_cache, cache_key=0)
    for k, v in fwd.items():
        _close_fwd(np.asarray(frame[k]), v)
    out = T.backward(scene, cam, settings, frame, g_img, **cot)
    for k in TRAIN_GRADS + ("contrib",):
        _close_grad(k, out[k], grads[k])


def test_sh_jacobian_matches_finite_differences():
    rng = np.random.default_rng(5)
    d = rng.standard_normal((7, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    B, J = T.sh_basis_and_jac(3, d)
    h = 1e-6
    for j in range(3):
        e = np.zeros(3)
        e[j] = h
        num = (T.sh_basis_and_jac(3, d + e)[0] - T.sh_basis_and_jac(3, d - e)[0]) / (2 * h)
        assert np.allclose(num, J[:, :, j], atol=1e-7)
