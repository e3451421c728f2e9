"""B200-native (sm_100a) GES two-pass sorting-free forward renderer.

Drop-in for the reference render API ``ges.forward`` (forward.py:36-417):
``render``, ``rasterize_surfels``, ``accumulate_gaussians``, ``composite``,
``smooth_geometry``, ``RenderSettings`` and the buffer dataclasses.  The
device-native engine is :class:`Renderer` / :class:`DeviceScene`.
"""

from .forward import (GaussianBuffers, RenderResult, RenderSettings, SurfelBuffers,
                      accumulate_gaussians, composite, rasterize_surfels, render,
                      smooth_geometry)
from .renderer import SCENE_CACHE, DeviceScene, Frame, Renderer, default_renderer
from .types import (Camera, GaussianKind, GaussianSet, Scene, Stage, SurfelSet, look_at,
                    orbit_cameras)

__version__ = "0.1.0"


def invalidate(scene) -> None:
    """Forget the device copy of ``scene`` after editing its arrays in place
    (replaced arrays are detected automatically)."""
    SCENE_CACHE.invalidate(scene)

__all__ = ["render", "rasterize_surfels", "accumulate_gaussians", "composite",
           "smooth_geometry", "RenderSettings", "SurfelBuffers", "GaussianBuffers",
           "RenderResult", "Renderer", "DeviceScene", "Frame", "default_renderer",
           "Camera", "GaussianKind", "GaussianSet", "Scene", "Stage", "SurfelSet",
           "look_at", "orbit_cameras", "invalidate"]
