"""`.ges` loading against fixtures written and loaded by the
reference (tests/golden/make_golden.py): bit-identical arrays, the reference's
f32 round-trip identity (test_io.py:173-182) and its error cases."""

import os
import struct

import numpy as np
import pytest

from paper_2504_17545_b200.gesfile import GesFileError, HEADER, load_ges, save_ges

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
CASES = ("ges_3d_deg3", "ges_2d_rgb")


@pytest.mark.parametrize("name", CASES)
def test_load_matches_reference_loader(name):
    scene, info = load_ges(os.path.join(GOLD, name + ".ges"))
    z = np.load(os.path.join(GOLD, name + "_load.npz"))
    s, g = scene.surfels, scene.gaussians
    for a, k in ((s.pos, "sp"), (s.quat, "sq"), (s.log_scale, "sl"), (s.sh, "ssh"), (g.pos, "gp"),
                 (g.raw_opacity, "go"), (g.quat, "gq"), (g.log_scale, "gl"), (g.sh, "gsh")):
        assert np.array_equal(a, z[k]), k
    assert np.array_equal(info["epsilon"], z["eps"])
    assert info["flags"] == int(z["flags"])


@pytest.mark.parametrize("name", CASES)
def test_save_load_roundtrip_is_bitwise(name, tmp_path):
    scene, info = load_ges(os.path.join(GOLD, name + ".ges"))
    p = tmp_path / "again.ges"
    save_ges(scene, p, rgb_surfels=info["rgb_surfels"])
    again, info2 = load_ges(p)
    for a, b in ((scene.surfels.pos, again.surfels.pos), (scene.surfels.sh, again.surfels.sh),
                 (scene.gaussians.quat, again.gaussians.quat),
                 (scene.gaussians.log_scale, again.gaussians.log_scale)):
        assert np.array_equal(a, b)
    # geometry/SH floats are copied through unchanged; the baked epsilon is
    # recomputed from the loaded scales (as the reference's export does)
    assert np.allclose(info2["epsilon"], info["epsilon"], rtol=1e-6)


def test_error_cases(tmp_path):
    good = open(os.path.join(GOLD, "ges_3d_deg3.ges"), "rb").read()
    bad = tmp_path / "bad.ges"
    bad.write_bytes(good[:10])
    with pytest.raises(GesFileError, match="truncated"):
        load_ges(bad)
    bad.write_bytes(b"XXXX" + good[4:])
    with pytest.raises(GesFileError, match="magic"):
        load_ges(bad)
    bad.write_bytes(good[:-4])
    with pytest.raises(GesFileError, match="size"):
        load_ges(bad)
    magic, ver, deg, flags, ns, ng = HEADER.unpack_from(good)
    bad.write_bytes(HEADER.pack(magic, ver, 4, flags, ns, ng) + good[HEADER.size:])
    with pytest.raises(GesFileError, match="degree"):
        load_ges(bad)
    bad.write_bytes(HEADER.pack(magic, 2, deg, flags, ns, ng) + good[HEADER.size:])
    with pytest.raises(GesFileError, match="version"):
        load_ges(bad)


def test_cli_export_roundtrip(tmp_path):
    """``export`` (cli.py:147-151) re-writes a model that loads to the same arrays."""
    from paper_2504_17545_b200 import cli
    src = os.path.join(GOLD, "ges_2d_rgb.ges")
    out = tmp_path / "re.ges"
    assert cli.main(["export", "--model", src, "--out", str(out)]) == 0
    a, ia = load_ges(src)
    b, ib = load_ges(out)
    assert ia["rgb_surfels"] == ib["rgb_surfels"]
    assert np.array_equal(a.surfels.pos, b.surfels.pos) and np.array_equal(a.gaussians.sh, b.gaussians.sh)
    assert cli.main(["export", "--model", str(tmp_path / "missing.ges"), "--out", str(out)]) == 1


def test_save_rejects_like_reference_export(tmp_path):
    """save_ges applies export_ges's checks (gesfile.py:44-47, :66-69)."""
    import copy
    from paper_2504_17545_b200.types import Scene, Stage
    scene, _ = load_ges(os.path.join(GOLD, "ges_3d_deg3.ges"))
    p = tmp_path / "x.ges"
    joint = Scene(scene.surfels, scene.gaussians, scene.sh_degree, Stage.JOINT)
    with pytest.raises(GesFileError, match="frozen"):
        save_ges(joint, p)
    s2 = copy.deepcopy(scene)
    s2.surfels.w = s2.surfels.w.copy()
    s2.surfels.w[0] = 128.0
    with pytest.raises(GesFileError, match="w = 255"):
        save_ges(s2, p)
    s3 = copy.deepcopy(scene)
    s3.surfels.pos = s3.surfels.pos.copy()
    s3.surfels.pos[0, 0] = np.nan
    with pytest.raises(GesFileError, match="non-finite surfel"):
        save_ges(s3, p)
    s4 = copy.deepcopy(scene)
    s4.gaussians.sh = s4.gaussians.sh.copy()
    s4.gaussians.sh[0, 0, 0] = np.inf
    with pytest.raises(GesFileError, match="non-finite gaussian"):
        save_ges(s4, p)
    assert not p.exists()
