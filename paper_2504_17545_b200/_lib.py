"""ctypes binding of ``libges_b200.so`` (the C ABI in ``include/ges_b200.h``).

There is no CPU fallback: if the library is missing the import of the render
API raises, and calls on a machine without a CUDA device fail with the CUDA
error the library reports.
"""

from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# GES_B200_LIB overrides the library path (A/B runs of alternative builds)
LIB_PATH = os.environ.get("GES_B200_LIB") or os.path.join(HERE, "libges_b200.so")

ABI_VERSION = 3   # include/ges_b200.h GES_ABI_VERSION
GES_OK, GES_EINVAL, GES_EDEGREE, GES_EWORKSPACE, GES_ECUDA = 0, 1, 2, 3, 4
GES_IMAGE_F32_RGB, GES_IMAGE_RGBA8 = 0, 1
LAYERS = {"full": 0, "surfels_only": 1, "gaussians_only": 2}

# Every symbol include/ges_b200.h declares (checked by tests/test_abi.py).
EXPORTS = ("ges_abi_version", "ges_last_error", "ges_scene_bytes", "ges_scene_pack",
           "ges_workspace_bytes", "ges_render", "ges_render_profiled", "ges_rasterize_surfels",
           "ges_accumulate_gaussians", "ges_composite", "ges_smooth_geometry",
           "ges_render_views_host", "ges_debug_stats", "ges_surfel_colors",
           "ges_backward_scratch_bytes", "ges_backward_workspace_bytes", "ges_backward_gaussians",
           "ges_backward_surfels_frozen", "ges_gaussian_contributions",
           "ges_frozen_surfel_buffers", "ges_peer_alloc", "ges_peer_free", "ges_peer_open", "ges_peer_close",
           "ges_workspace_bytes_f64", "ges_render_f64", "ges_composite_f64", "ges_smooth_geometry_f64")


class Camera(C.Structure):
    _fields_ = [("fx", C.c_double), ("fy", C.c_double), ("cx", C.c_double), ("cy", C.c_double),
                ("width", C.c_int32), ("height", C.c_int32), ("w2c", C.c_double * 12)]


class Settings(C.Structure):
    _fields_ = [("supersample", C.c_int32), ("layers", C.c_int32), ("mip", C.c_int32),
                ("epsilon_mode", C.c_int32), ("with_geometry", C.c_int32), ("epsilon_value", C.c_double),
                ("background", C.c_double * 3), ("tile_mode", C.c_int32)]


class SceneSrc(C.Structure):
    _fields_ = [("n_surfels", C.c_int64), ("n_gaussians", C.c_int64), ("sh_degree", C.c_int32),
                ("gaussian_dim", C.c_int32)] + [
        (n, C.c_void_p) for n in ("s_pos", "s_quat", "s_log_scale", "s_sh", "g_pos",
                                  "g_raw_opacity", "g_quat", "g_log_scale", "g_sh", "g_filter3d",
                                  "s_order", "g_order")] + [("bounds", C.c_double * 7)]


class Scene(C.Structure):
    _fields_ = [("n_surfels", C.c_int64), ("n_gaussians", C.c_int64), ("sh_degree", C.c_int32),
                ("gaussian_dim", C.c_int32)] + [
        (n, C.c_void_p) for n in ("s_pos_s1", "s_quat", "s_s2", "s_sh", "s_id", "s_pack", "g_pos_op", "g_quat",
                                  "g_scale_eps", "g_sh")] + [("bounds", C.c_double * 7)]


class Outputs(C.Structure):
    _fields_ = [(n, C.c_void_p) for n in ("image", "s_color", "s_depth", "s_normal", "s_winner",
                                          "g_color", "g_weight", "g_depth", "g_normal",
                                          "image_rgba8")]


class OutputsF64(C.Structure):
    _fields_ = [(n, C.c_void_p) for n in ("image", "s_color", "s_depth", "s_normal", "s_winner",
                                          "g_color", "g_weight", "g_depth", "g_normal")]


class FrameStatus(C.Structure):
    _fields_ = [("surfel_pairs", C.c_int64), ("gaussian_pairs", C.c_int64),
                ("overflow", C.c_int32), ("pad", C.c_int32)]


class GaussGrads(C.Structure):
    _fields_ = [(n, C.c_void_p) for n in ("pos", "opacity", "quat", "scale", "sh", "screen")]


_lib = None


def lib():
    """Load the shared library once; raise loudly if it was not built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'`"
                          " (there is no CPU fallback)")
    L = C.CDLL(LIB_PATH)
    P = C.POINTER
    sig = {
        "ges_abi_version": (C.c_int, []),
        "ges_last_error": (C.c_char_p, []),
        "ges_scene_bytes": (C.c_size_t, [C.c_int64, C.c_int64, C.c_int32]),
        "ges_scene_pack": (C.c_int, [P(SceneSrc), C.c_void_p, C.c_size_t, P(Scene), C.c_void_p]),
        "ges_workspace_bytes": (C.c_size_t, [P(Scene), P(Camera), P(Settings), C.c_int64, C.c_int64]),
        "ges_render": (C.c_int, [P(Scene), P(Camera), P(Settings), P(Outputs), C.c_void_p, C.c_size_t,
                                 C.c_int64, C.c_int64, C.c_void_p, C.c_void_p]),
        "ges_render_profiled": (C.c_int, [P(Scene), P(Camera), P(Settings), P(Outputs), C.c_void_p,
                                          C.c_size_t, C.c_int64, C.c_int64, C.c_void_p, C.c_void_p,
                                          C.c_void_p]),
        "ges_rasterize_surfels": (C.c_int, [P(Scene), P(Camera), P(Settings), P(Outputs), C.c_void_p,
                                            C.c_size_t, C.c_int64, C.c_void_p, C.c_void_p]),
        "ges_accumulate_gaussians": (C.c_int, [P(Scene), P(Camera), C.c_void_p, P(Settings), P(Outputs),
                                               C.c_void_p, C.c_size_t, C.c_int64, C.c_void_p, C.c_void_p]),
        "ges_composite": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_float, C.c_void_p,
                                    C.c_int64, C.c_void_p]),
        "ges_smooth_geometry": (C.c_int, [C.c_void_p] * 7 + [C.c_int64, C.c_void_p]),
        "ges_render_views_host": (C.c_int, [P(Scene), P(Camera), C.c_int32, P(Settings), C.c_int32,
                                            C.c_void_p, C.c_int32, C.c_void_p, C.c_size_t, C.c_int64,
                                            C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    }
    sig["ges_debug_stats"] = (C.c_int, [C.POINTER(C.c_uint64)])
    sig["ges_surfel_colors"] = (C.c_int, [P(Scene), P(Camera), C.c_void_p, C.c_void_p])
    sig["ges_backward_scratch_bytes"] = (C.c_size_t, [C.c_int64])
    sig["ges_backward_workspace_bytes"] = (C.c_size_t, [P(Scene), P(Camera), P(Settings), C.c_int64])
    sig["ges_backward_gaussians"] = (C.c_int, [P(Scene), P(SceneSrc), C.c_int32, P(Camera), P(Settings)]
                                     + [C.c_void_p] * 5 + [P(GaussGrads), C.c_void_p, C.c_size_t,
                                                           C.c_void_p, C.c_size_t, C.c_int64, C.c_void_p,
                                                           C.c_void_p])
    sig["ges_backward_surfels_frozen"] = (C.c_int, [P(SceneSrc), P(Camera), C.c_int32] + [C.c_void_p] * 6)
    sig["ges_peer_alloc"] = (C.c_int, [C.c_size_t, C.POINTER(C.c_void_p), C.c_void_p])
    sig["ges_peer_free"] = (C.c_int, [C.c_void_p])
    sig["ges_peer_open"] = (C.c_int, [C.c_void_p, C.c_int32, C.POINTER(C.c_void_p)])
    sig["ges_peer_close"] = (C.c_int, [C.c_void_p])
    sig["ges_frozen_surfel_buffers"] = (C.c_int, [C.c_void_p] * 4 + [C.c_int32] * 3 + [C.c_void_p] * 6)
    sig["ges_gaussian_contributions"] = (C.c_int, [P(Scene), P(SceneSrc), P(Camera), P(Settings)] + [C.c_void_p] * 4
                                         + [C.c_size_t, C.c_int64, C.c_void_p, C.c_void_p])
    sig["ges_workspace_bytes_f64"] = (C.c_size_t, [P(Scene), P(Camera), P(Settings), C.c_int64, C.c_int64])
    sig["ges_render_f64"] = (C.c_int, [P(Scene), P(SceneSrc), P(Camera), P(Settings), C.c_int32, C.c_void_p,
                                       P(OutputsF64), C.c_void_p, C.c_size_t, C.c_int64, C.c_int64, C.c_void_p,
                                       C.c_void_p])
    sig["ges_composite_f64"] = (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_double, C.c_void_p,
                                          C.c_int64, C.c_void_p])
    sig["ges_smooth_geometry_f64"] = (C.c_int, [C.c_void_p] * 7 + [C.c_int64, C.c_void_p])
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    if L.ges_abi_version() != ABI_VERSION:
        raise ImportError("libges_b200.so ABI version mismatch")
    _lib = L
    return L


def check(rc: int, what: str):
    """Map a return code to the reference's exception types."""
    if rc == GES_OK:
        return
    msg = f"{what}: {lib().ges_last_error().decode(errors='replace')}"
    if rc in (GES_EINVAL, GES_EDEGREE):
        raise ValueError(msg)
    raise RuntimeError(msg)
