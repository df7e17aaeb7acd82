"""ctypes mirror of include/wt_gpu.h and the in-tree library loader.

The product path has no fallback: if libwt_gpu.so is missing or cannot be
loaded, importing a GPU entry point raises instead of silently computing on
the CPU.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

import numpy as np

LIB_PATH = Path(__file__).resolve().parent / "libwt_gpu.so"

ABI_VERSION = 2  # WT_ABI_VERSION, include/wt_gpu.h
WT_OK, WT_EINVAL, WT_ELENGTH, WT_ECUDA, WT_ENOMEM, WT_ENOTPD, WT_ENODEV, WT_ERANGE = range(8)
MODE_DYNAMIC, MODE_SHAPE_MATCH, MODE_SMOOTH_BIND, MODE_RIGID = range(4)
JOINT_HINGE, JOINT_PRISMATIC = 0, 1


class Intrinsics(C.Structure):
    _fields_ = [("fx", C.c_double), ("fy", C.c_double), ("cx", C.c_double), ("cy", C.c_double),
                ("width", C.c_int32), ("height", C.c_int32)]


class KinConfig(C.Structure):
    _fields_ = [("iterations", C.c_int32), ("assoc_refresh", C.c_int32),
                ("lambda_k", C.c_double), ("lambda_s", C.c_double),
                ("diag_floor", C.c_double), ("clamp_limits", C.c_int32), ("pad_", C.c_int32),
                ("limit", C.c_double)]


class ShapeConfig(C.Structure):
    _fields_ = [("iterations", C.c_int32), ("pad_", C.c_int32), ("lambda_phi", C.c_double),
                ("lambda_nbr", C.c_double), ("lambda_w", C.c_double), ("diag_floor", C.c_double)]


class AssocConfig(C.Structure):
    _fields_ = [("window_radius", C.c_int32), ("pad_", C.c_int32), ("cutoff", C.c_double)]


class TrackConfigC(C.Structure):
    _fields_ = [("mode", C.c_int32), ("threads", C.c_int32), ("kin", KinConfig),
                ("shape", ShapeConfig), ("assoc", AssocConfig), ("shape_stats", C.c_int32),
                ("pad_", C.c_int32)]


class KinIterStats(C.Structure):
    _fields_ = [("iteration", C.c_int32), ("associated", C.c_int32),
                ("residual_sum", C.c_double), ("step_norm", C.c_double),
                ("solver_skipped", C.c_int32), ("pad_", C.c_int32)]


class ShapeIterStats(C.Structure):
    _fields_ = [("iteration", C.c_int32), ("singular", C.c_int32), ("mean_phi", C.c_double),
                ("max_phi", C.c_double), ("mean_abs_r_before", C.c_double),
                ("mean_abs_r_after", C.c_double)]


class FrameStatsC(C.Structure):
    _fields_ = [("frame", C.c_int32), ("n_kin", C.c_int32), ("n_shape", C.c_int32),
                ("cap_kin", C.c_int32), ("cap_shape", C.c_int32), ("pad_", C.c_int32),
                ("kin", C.POINTER(KinIterStats)), ("shape", C.POINTER(ShapeIterStats))]


class Noise(C.Structure):
    _fields_ = [("sigma", C.c_double), ("dropout", C.c_double), ("quantization", C.c_double),
                ("seed", C.c_uint64)]


class ModelDesc(C.Structure):
    _fields_ = [("n_links", C.c_int32), ("n_vertices", C.c_int32), ("n_triangles", C.c_int32),
                ("pad_", C.c_int32),
                ("parent", C.POINTER(C.c_int32)), ("parent_offset", C.POINTER(C.c_double)),
                ("joint_kind", C.POINTER(C.c_int32)), ("joint_axis", C.POINTER(C.c_double)),
                ("theta_index", C.POINTER(C.c_int32)), ("v0", C.POINTER(C.c_double)),
                ("phi", C.POINTER(C.c_double)), ("weight_count", C.POINTER(C.c_int32)),
                ("weight_link", C.POINTER(C.c_int32)), ("weight", C.POINTER(C.c_double)),
                ("triangles", C.POINTER(C.c_int32)), ("vtri_offsets", C.POINTER(C.c_int32)),
                ("vtri_items", C.POINTER(C.c_int32)), ("nbr_offsets", C.POINTER(C.c_int32)),
                ("nbr_items", C.POINTER(C.c_int32))]


# Every symbol include/wt_gpu.h declares (checked by the CPU test suite).
EXPORTS = [
    "wt_gpu_abi_version", "wt_gpu_device_count", "wt_gpu_global_last_error", "wt_gpu_create",
    "wt_gpu_destroy", "wt_gpu_last_error", "wt_gpu_set_state", "wt_gpu_get_state",
    "wt_gpu_load_depth", "wt_gpu_load_cloud", "wt_gpu_track_loaded", "wt_gpu_track_frame",
    "wt_gpu_track_frame_cloud", "wt_gpu_optimize_pose", "wt_gpu_optimize_shape", "wt_gpu_skin",
    "wt_gpu_associate", "wt_gpu_associate_posed", "wt_gpu_normal_system", "wt_gpu_solve_step",
    "wt_gpu_solve_vertices", "wt_gpu_render_depth", "wt_gpu_stream", "wt_gpu_track_async", "wt_gpu_sync",
    "wt_gpu_profile_frame", "wt_gpu_bucket_count", "wt_gpu_mesh_subdivide", "wt_gpu_mesh_sizes",
    "wt_gpu_mesh_export", "wt_gpu_mesh_free", "wt_gpu_mesh_last_error", "wt_gpu_build_neighbors", "wt_gpu_host_alloc", "wt_gpu_host_free", "wt_gpu_track_sequence", "wt_gpu_joint_positions", "wt_gpu_recon_error",
    "wt_gpu_create_batch", "wt_gpu_batch_size", "wt_gpu_batch_set_state", "wt_gpu_batch_get_state",
    "wt_gpu_batch_load_depth", "wt_gpu_batch_track_async", "wt_gpu_batch_stats", "wt_gpu_batch_track",
]
KERNEL_KINDS = ["fk", "skin", "normals+bucket", "scatter", "search+average", "pose_system",
                "shape_step", "shape_stats", "pose_solve", "pixoff"]


class WarptrackError(RuntimeError):
    """Mirrors warptrack::Error (errors.hpp:9); .code carries the WT_* status."""

    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


class LengthMismatch(WarptrackError):
    pass


class NotPositiveDefinite(WarptrackError):
    pass


class ValidationError(WarptrackError):
    pass


_lib = None


def lib() -> C.CDLL:
    """Loads libwt_gpu.so (built in-tree by paper_1711_07999_b200.build)."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise WarptrackError(WT_ENODEV, f"CUDA library not built: {LIB_PATH} "
                                 "(run python -m paper_1711_07999_b200.build)")
        _lib = C.CDLL(str(LIB_PATH))
        _declare(_lib)
    return _lib


def _declare(L: C.CDLL) -> None:
    P = C.POINTER
    vp = C.c_void_p
    L.wt_gpu_global_last_error.restype = C.c_char_p
    L.wt_gpu_last_error.restype = C.c_char_p
    L.wt_gpu_last_error.argtypes = [vp]
    L.wt_gpu_create.argtypes = [C.c_int, P(ModelDesc), P(Intrinsics), P(vp)]
    L.wt_gpu_destroy.argtypes = [vp]
    L.wt_gpu_destroy.restype = None
    L.wt_gpu_set_state.argtypes = [vp, vp, vp, C.c_int32]
    L.wt_gpu_get_state.argtypes = [vp, vp, vp, P(C.c_int32)]
    L.wt_gpu_load_depth.argtypes = [vp, vp, C.c_double]
    L.wt_gpu_load_cloud.argtypes = [vp, vp, vp]
    L.wt_gpu_track_loaded.argtypes = [vp, P(TrackConfigC), P(FrameStatsC)]
    L.wt_gpu_track_frame.argtypes = [vp, vp, C.c_double, P(TrackConfigC), P(FrameStatsC)]
    L.wt_gpu_track_frame_cloud.argtypes = [vp, vp, vp, P(TrackConfigC), P(FrameStatsC)]
    L.wt_gpu_optimize_pose.argtypes = [vp, P(KinConfig), P(AssocConfig), P(KinIterStats), C.c_int32,
                                       P(C.c_int32)]
    L.wt_gpu_optimize_shape.argtypes = [vp, P(ShapeConfig), P(AssocConfig), C.c_int32,
                                        P(ShapeIterStats), C.c_int32, P(C.c_int32)]
    L.wt_gpu_skin.argtypes = [vp, vp, vp, vp, vp, vp]
    L.wt_gpu_associate.argtypes = [vp, C.c_int32, C.c_double, vp, vp, vp, vp]
    L.wt_gpu_associate_posed.argtypes = [C.c_int, P(Intrinsics), C.c_int32, vp, vp, vp, vp, vp,
                                         C.c_int32, C.c_double, vp, vp, vp, vp]
    L.wt_gpu_normal_system.argtypes = [vp, vp, P(KinConfig), vp, vp, vp, vp]
    L.wt_gpu_solve_step.argtypes = [C.c_int, C.c_int32, vp, vp, C.c_double, C.c_double, vp]
    L.wt_gpu_solve_vertices.argtypes = [C.c_int, C.c_int32, vp, vp, vp, vp, vp, P(ShapeConfig), vp,
                                        vp]
    L.wt_gpu_render_depth.argtypes = [vp, vp, vp, P(Noise), C.c_int32, vp, vp]
    L.wt_gpu_stream.argtypes = [vp]
    L.wt_gpu_stream.restype = vp
    L.wt_gpu_track_async.argtypes = [vp, P(TrackConfigC)]
    L.wt_gpu_sync.argtypes = [vp]
    L.wt_gpu_track_sequence.argtypes = [vp, vp, C.c_int32, C.c_double, P(TrackConfigC), vp, vp]
    L.wt_gpu_joint_positions.argtypes = [vp, vp]
    L.wt_gpu_recon_error.argtypes = [vp, vp, P(C.c_int32)]
    L.wt_gpu_bucket_count.argtypes = [vp, C.c_int32, P(C.c_int32)]
    L.wt_gpu_mesh_subdivide.argtypes = [C.c_int, C.c_int32, C.c_int32, vp, vp, vp, vp, vp, C.c_int32, vp, vp,
                                        C.c_int32, C.c_int32, P(vp)]
    L.wt_gpu_mesh_sizes.argtypes = [vp, P(C.c_int32), P(C.c_int32), P(C.c_int32), P(C.c_int32), P(C.c_int32)]
    L.wt_gpu_mesh_export.argtypes = [vp] + [vp] * 11
    L.wt_gpu_mesh_free.argtypes = [vp]
    L.wt_gpu_mesh_free.restype = None
    L.wt_gpu_mesh_last_error.restype = C.c_char_p
    L.wt_gpu_build_neighbors.argtypes = [C.c_int, C.c_int32, vp, C.c_int32, vp]
    L.wt_gpu_host_alloc.argtypes = [C.c_size_t, P(vp)]
    L.wt_gpu_host_free.argtypes = [vp]
    L.wt_gpu_host_free.restype = None
    L.wt_gpu_profile_frame.argtypes = [vp, P(TrackConfigC), vp, vp, C.c_int32, P(C.c_int32)]
    L.wt_gpu_create_batch.argtypes = [C.c_int, P(ModelDesc), P(Intrinsics), C.c_int32, P(vp)]
    L.wt_gpu_batch_size.argtypes = [vp]
    L.wt_gpu_batch_size.restype = C.c_int32
    L.wt_gpu_batch_set_state.argtypes = [vp, C.c_int32, vp, vp]
    L.wt_gpu_batch_get_state.argtypes = [vp, C.c_int32, vp, vp]
    L.wt_gpu_batch_load_depth.argtypes = [vp, vp, C.c_double]
    L.wt_gpu_batch_track_async.argtypes = [vp, P(TrackConfigC)]
    L.wt_gpu_batch_stats.argtypes = [vp, P(FrameStatsC)]
    L.wt_gpu_batch_track.argtypes = [vp, vp, C.c_double, P(TrackConfigC), P(FrameStatsC)]


def check(rc: int, ctx=None) -> None:
    if rc == WT_OK:
        return
    L = lib()
    msg = (L.wt_gpu_last_error(ctx) if ctx else L.wt_gpu_global_last_error()) or b""
    msg = msg.decode(errors="replace")
    cls = {WT_ELENGTH: LengthMismatch, WT_ENOTPD: NotPositiveDefinite,
           WT_EINVAL: ValidationError}.get(rc, WarptrackError)
    raise cls(rc, msg)


def ptr(a: np.ndarray | None):
    """Raw data pointer of a C-contiguous array (None -> NULL)."""
    if a is None:
        return None
    assert a.flags["C_CONTIGUOUS"], "array must be C-contiguous"
    return a.ctypes.data
