"""Evaluation datasets in the reference's on-disk layout
(``/root/reference/pkg/src/ges/datasets.py:30-46, 152-176``): a directory with
``cameras.json`` (entries {fx, fy, cx, cy, width, height, w2c[16], image}),
the images it names (8-bit RGB, read as float64 in [0, 1]) and optionally
``points.ply``.  Only what ``metrics.evaluate`` / the ``eval`` command need:
the point cloud (training initialisation) is read when present and left
empty otherwise.  Errors raise ``DatasetError`` like the reference's.
"""

from __future__ import annotations

import json
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np

from .cli import camera_from_entry

TEST_EVERY_DEFAULT = 8   # datasets.py:22


class DatasetError(RuntimeError):
    pass


@dataclass
class Dataset:
    cameras: list
    images: list                      # (H, W, 3) float64 in [0, 1]
    points: np.ndarray = field(default_factory=lambda: np.zeros((0, 3)))
    point_colors: np.ndarray = field(default_factory=lambda: np.zeros((0, 3)))
    train_idx: list = field(default_factory=list)
    test_idx: list = field(default_factory=list)

    @property
    def train_cameras(self):
        return [self.cameras[i] for i in self.train_idx]

    def split(self, test_every: int):
        """Every ``test_every``-th view is a test view (datasets.py:42-46)."""
        n = len(self.cameras)
        self.test_idx = [i for i in range(n) if test_every > 0 and i % test_every == 0]
        test = set(self.test_idx)
        self.train_idx = [i for i in range(n) if i not in test]


def load_image(path) -> np.ndarray:
    from PIL import Image
    with Image.open(path) as im:
        return np.asarray(im.convert("RGB"), dtype=np.float64) / 255.0


def _points(path: Path):
    """x/y/z (+ red/green/blue) of a binary little-endian or ASCII PLY."""
    raw = path.read_bytes()
    marker = b"end_header\n"
    stop = raw.find(marker)
    if not raw.startswith(b"ply") or stop < 0:
        raise DatasetError(f"{path} is not a PLY file")
    lines = raw[:stop].decode("ascii", "replace").splitlines()
    fmt, count, props = None, None, []
    for ln in lines:
        w = ln.split()
        if w[:1] == ["format"]:
            fmt = w[1]
        elif w[:2] == ["element", "vertex"]:
            count = int(w[2])
        elif w[:1] == ["property"] and len(w) == 3:
            props.append((w[2], w[1]))
    names = [p for p, _ in props]
    if fmt is None or count is None or not {"x", "y", "z"} <= set(names):
        raise DatasetError(f"{path}: malformed PLY header")
    body = raw[stop + len(marker):]
    if fmt == "ascii":
        rows = np.array([[float(v) for v in ln.split()] for ln in body.decode().splitlines() if ln.strip()][:count],
                        dtype=np.float64).reshape(-1, len(names))
        col = {p: rows[:, k] for k, p in enumerate(names)}
    elif fmt == "binary_little_endian":
        kinds = {"float": "<f4", "float32": "<f4", "double": "<f8", "float64": "<f8", "uchar": "u1",
                 "uint8": "u1", "int": "<i4"}
        rec = np.frombuffer(body, dtype=np.dtype([(p, kinds[t]) for p, t in props]), count=count)
        col = {p: rec[p].astype(np.float64) for p in names}
    else:
        raise DatasetError(f"{path}: unsupported PLY format {fmt}")
    pts = np.stack([col["x"], col["y"], col["z"]], axis=1)
    rgb = (np.stack([col["red"], col["green"], col["blue"]], axis=1) / 255.0
           if {"red", "green", "blue"} <= set(names) else np.full((len(pts), 3), 0.5))
    return pts, rgb


def load_dataset(root, *, test_every: int = TEST_EVERY_DEFAULT) -> Dataset:
    """datasets.py:152-176 (point cloud optional)."""
    root = Path(root)
    cam_file = root / "cameras.json"
    if not cam_file.is_file():
        raise DatasetError(f"missing camera file {cam_file}")
    try:
        entries = json.loads(cam_file.read_text())
    except json.JSONDecodeError as e:
        raise DatasetError(f"corrupt camera file {cam_file}: {e}") from e
    cams, imgs = [], []
    for e in entries:
        cam = camera_from_entry(e)
        ip = root / e["image"]
        if not ip.is_file():
            raise DatasetError(f"camera references missing image {ip}")
        img = load_image(ip)
        if img.shape[:2] != (cam.height, cam.width):
            raise DatasetError(f"image size {img.shape[:2]} does not match camera {cam.width}x{cam.height}: {ip}")
        cams.append(cam)
        imgs.append(img)
    ds = Dataset(cams, imgs)
    ply = root / "points.ply"
    if ply.is_file():
        ds.points, ds.point_colors = _points(ply)
    ds.split(test_every)
    return ds
