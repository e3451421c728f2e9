"""The C-ABI library loads without a GPU and exports every function that
include/ges_b200.h declares; argument validation maps to the reference's
exception types (no compute calls here)."""

import ctypes as C
import os
import re

import pytest

from paper_2504_17545_b200 import _lib, _build

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    src = open(os.path.join(ROOT, "include", "ges_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ges_\w+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    L = _lib.lib()
    declared = header_functions()
    assert declared, "no declarations parsed"
    assert set(declared) == set(_lib.EXPORTS)
    for name in declared:
        assert hasattr(L, name), name
    assert L.ges_abi_version() == 3


def test_library_is_sm100a():
    so = _lib.LIB_PATH
    data = open(so, "rb").read()
    assert b"sm_100a" in data or b"compute_100a" in data


def test_scene_bytes_and_workspace_validation():
    L = _lib.lib()
    assert L.ges_scene_bytes(0, 0, 0) == 0
    assert L.ges_scene_bytes(10, 0, 5) == 0            # bad degree
    b = L.ges_scene_bytes(1000, 500, 3)
    assert b >= 1000 * (16 + 16 + 4 + 192) + 500 * (48 + 192)
    sc = _lib.Scene(n_surfels=1000, n_gaussians=500, sh_degree=3, gaussian_dim=3)
    cam = _lib.Camera(fx=100.0, fy=100.0, cx=64.0, cy=64.0, width=128, height=128)
    st = _lib.Settings(supersample=1, layers=0, mip=0, epsilon_mode=0)
    assert L.ges_workspace_bytes(C.byref(sc), C.byref(cam), C.byref(st), 1 << 16, 1 << 16) > 0
    st.supersample = 2
    assert L.ges_workspace_bytes(C.byref(sc), C.byref(cam), C.byref(st), 1 << 16, 1 << 16) == 0


def test_scene_bytes_pad_gaussian_sh_rows():
    """ABI 3: the packed Gaussian SH rows are padded to 4 / 12 / 28 / 52 floats
    (an odd number of 16-byte units, one bulk copy per warp in the
    preprocess); surfel SH rows stay 3K floats."""
    L = _lib.lib()
    n = 1 << 16   # (multiples of the 256-byte carve alignment)
    for deg, stride in ((0, 4), (1, 12), (2, 28), (3, 52)):
        k3 = 3 * (deg + 1) ** 2
        g = L.ges_scene_bytes(0, n, deg)
        assert g == n * (3 * 16 + 4 * stride)
        assert L.ges_scene_bytes(n, 0, deg) == n * (16 + 16 + 4 + 4 * k3 + 4 + 4)


def test_error_codes_map_to_reference_exceptions():
    L = _lib.lib()
    sc = _lib.Scene(n_surfels=0, n_gaussians=0, sh_degree=7, gaussian_dim=3)
    cam = _lib.Camera(fx=100.0, fy=100.0, cx=64.0, cy=64.0, width=128, height=128)
    st = _lib.Settings(supersample=1)
    out = _lib.Outputs()
    rc = L.ges_render(C.byref(sc), C.byref(cam), C.byref(st), C.byref(out), None, 0, 0, 0, None, None)
    assert rc == _lib.GES_EDEGREE
    with pytest.raises(ValueError, match="degree"):
        _lib.check(rc, "render")
    sc.sh_degree = 1
    st.layers = 9
    rc = L.ges_render(C.byref(sc), C.byref(cam), C.byref(st), C.byref(out), None, 0, 0, 0, None, None)
    assert rc == _lib.GES_EINVAL
    st.layers = 0
    rc = L.ges_render(C.byref(sc), C.byref(cam), C.byref(st), C.byref(out), None, 0, 0, 0, None, None)
    assert rc == _lib.GES_EWORKSPACE
    with pytest.raises(RuntimeError):
        _lib.check(rc, "render")


def test_build_is_up_to_date():
    assert not _build.stale(), "libges_b200.so older than its sources: run __graft_entry__.build()"


def test_missing_library_fails_loudly(tmp_path):
    """No CPU fallback: without the CUDA library the render API raises."""
    import subprocess
    import sys
    code = ("import numpy as np, paper_2504_17545_b200 as G\n"
            "from paper_2504_17545_b200 import scenes as S\n"
            "sc = S.random_scene(np.random.default_rng(0), 3, 3)\n"
            "G.render(sc, S.make_camera())\n")
    env = dict(os.environ, GES_B200_LIB=str(tmp_path / "nope.so"))
    p = subprocess.run([sys.executable, "-c", code], cwd=ROOT, env=env, capture_output=True, text=True)
    assert p.returncode != 0
    assert "ImportError" in p.stderr or "RuntimeError" in p.stderr


def test_float64_entry_validation():
    """ges_render_f64 / ges_workspace_bytes_f64 argument checks (no compute):
    missing source scene, bad mode, missing depth for mode 2, mismatched
    source, workspace too small."""
    L = _lib.lib()
    sc = _lib.Scene(n_surfels=10, n_gaussians=5, sh_degree=1, gaussian_dim=3)
    src = _lib.SceneSrc(n_surfels=10, n_gaussians=5, sh_degree=1, gaussian_dim=3)
    cam = _lib.Camera(fx=100.0, fy=100.0, cx=64.0, cy=64.0, width=128, height=128)
    st = _lib.Settings(supersample=1)
    out = _lib.OutputsF64()
    need = L.ges_workspace_bytes_f64(C.byref(sc), C.byref(cam), C.byref(st), 1 << 10, 1 << 10)
    assert need > L.ges_workspace_bytes(C.byref(sc), C.byref(cam), C.byref(st), 1 << 10, 1 << 10)
    args = (None, 0, 1 << 10, 1 << 10, None, None)
    assert L.ges_render_f64(C.byref(sc), None, C.byref(cam), C.byref(st), 3, None, C.byref(out), *args) \
        == _lib.GES_EINVAL
    assert L.ges_render_f64(C.byref(sc), C.byref(src), C.byref(cam), C.byref(st), 4, None, C.byref(out), *args) \
        == _lib.GES_EINVAL
    assert L.ges_render_f64(C.byref(sc), C.byref(src), C.byref(cam), C.byref(st), 2, None, C.byref(out), *args) \
        == _lib.GES_EINVAL
    rc = L.ges_render_f64(C.byref(sc), C.byref(src), C.byref(cam), C.byref(st), 3, None, C.byref(out), *args)
    assert rc == _lib.GES_EINVAL and "source scene arrays missing" in L.ges_last_error().decode()
    src2 = _lib.SceneSrc(n_surfels=11, n_gaussians=5, sh_degree=1, gaussian_dim=3)
    rc = L.ges_render_f64(C.byref(sc), C.byref(src2), C.byref(cam), C.byref(st), 3, None, C.byref(out), *args)
    assert rc == _lib.GES_EINVAL and "does not match" in L.ges_last_error().decode()
    empty = _lib.Scene(n_surfels=0, n_gaussians=0, sh_degree=1, gaussian_dim=3)
    esrc = _lib.SceneSrc(n_surfels=0, n_gaussians=0, sh_degree=1, gaussian_dim=3)
    rc = L.ges_render_f64(C.byref(empty), C.byref(esrc), C.byref(cam), C.byref(st), 3, None, C.byref(out), *args)
    assert rc == _lib.GES_EWORKSPACE
    with pytest.raises(RuntimeError):
        _lib.check(rc, "render_f64")
