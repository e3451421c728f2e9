"""The drop-in API accepts the reference's own objects (duck typing): the
host-side conversions to the C-ABI structs give the same values for a
reference ges.Scene/ges.Camera/ges.RenderSettings as for this package's
mirrors.  Runs only where /root/reference exists (the build container)."""

import os
import sys

import numpy as np
import pytest

from paper_2504_17545_b200 import _lib
from paper_2504_17545_b200 import scenes as S
from paper_2504_17545_b200.forward import RenderSettings
from paper_2504_17545_b200.renderer import (_degree, _kind_dim, camera_struct, scene_bounds,
                                            settings_struct)

REF = "/root/reference/pkg/src"
pytestmark = pytest.mark.skipif(not os.path.isdir(REF), reason="reference not mounted")


@pytest.fixture(scope="module")
def ges():
    sys.path.insert(0, REF)
    import ges as g
    return g


def test_reference_objects_convert_like_mirrors(ges):
    sc = S.random_scene(np.random.default_rng(5), 20, 10, degree=2)
    rs = ges.Scene(ges.SurfelSet(sc.surfels.pos, sc.surfels.quat, sc.surfels.log_scale, sc.surfels.sh,
                                 sc.surfels.w),
                   ges.GaussianSet(sc.gaussians.pos, sc.gaussians.raw_opacity, sc.gaussians.quat,
                                   sc.gaussians.log_scale, sc.gaussians.sh),
                   2, ges.Stage.FROZEN)
    assert _kind_dim(rs.gaussians) == _kind_dim(sc.gaussians) == 3
    assert _degree(rs.surfels.sh) == 2
    assert scene_bounds(rs.surfels, rs.gaussians, 20, 10) == scene_bounds(sc.surfels, sc.gaussians, 20, 10)
    cam = S.make_camera(40, 30)
    rc = ges.Camera(cam.fx, cam.fy, cam.cx, cam.cy, cam.width, cam.height, cam.world_to_camera)
    a, b = camera_struct(cam), camera_struct(rc)
    assert bytes(a) == bytes(b)
    st_ref = ges.RenderSettings(supersample=4, background=(0.1, 0.2, 0.3), layers="gaussians_only",
                                mip=True, epsilon_mode="constant", epsilon_value=0.25,
                                with_geometry=True)
    st_own = RenderSettings(supersample=4, background=(0.1, 0.2, 0.3), layers="gaussians_only",
                            mip=True, epsilon_mode="constant", epsilon_value=0.25, with_geometry=True)
    assert bytes(settings_struct(st_ref)) == bytes(settings_struct(st_own))
    two_d = ges.GaussianSet(np.zeros((1, 3)), np.zeros(1), np.array([[1.0, 0, 0, 0]]),
                            np.zeros((1, 2)), np.zeros((1, 9, 3)), ges.GaussianKind.TWO_D)
    assert _kind_dim(two_d) == 2


def test_settings_validation_matches_reference(ges):
    for kw in (dict(supersample=2), dict(layers="x"), dict(epsilon_mode="y")):
        with pytest.raises(ValueError):
            ges.RenderSettings(**kw)
        with pytest.raises(ValueError):
            RenderSettings(**kw)
    with pytest.raises(ValueError):
        _degree(np.zeros((3, 25, 3)))          # degree 4: UnsupportedDegreeError in the reference
    with pytest.raises(ValueError):
        _degree(np.zeros((3, 5, 3)))           # not a square
    assert _lib.LAYERS["gaussians_only"] == 2
