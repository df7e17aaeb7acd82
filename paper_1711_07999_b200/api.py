"""The reference's Python entry points for this path, with the same names,
arguments and results (python/src/bindings.cpp):

  track_sequence(bundle, sequence_path, init_theta=None, mode="dynamic", ...)
      bindings.cpp:241-303 -> run_tracking (tracker.cpp:70-100)
  skin_mesh(bundle, theta, phi=None)   bindings.cpp:185-202 -> skin

Both run on the GPU through libwt_gpu.so; `threads` is accepted for
signature compatibility and ignored (one context = one CUDA stream).
"""
from __future__ import annotations

import numpy as np

from .model import ModelBundle, rigidify
from .seqio import SequenceReader
from .tracker import (AssocConfig, Intrinsics, KinSolverConfig, ShapeSolverConfig, TrackConfig, Tracker,
                      parse_track_mode)

_K, _S, _A = KinSolverConfig(), ShapeSolverConfig(), AssocConfig()


def config_from_kwargs(mode="dynamic", iterations=_K.iterations, lambda_k=_K.lambda_k, lambda_s=_K.lambda_s,
                       shape_iterations=_S.iterations, lambda_phi=_S.lambda_phi, lambda_nbr=_S.lambda_nbr,
                       lambda_w=_S.lambda_w, window=_A.window_radius, cutoff=_A.cutoff, threads=0) -> TrackConfig:
    """config_from_kwargs (bindings.cpp:40-57)."""
    parse_track_mode(mode)
    return TrackConfig(mode=mode,
                       kin=KinSolverConfig(iterations=iterations, lambda_k=lambda_k, lambda_s=lambda_s),
                       shape=ShapeSolverConfig(iterations=shape_iterations, lambda_phi=lambda_phi,
                                               lambda_nbr=lambda_nbr, lambda_w=lambda_w),
                       assoc=AssocConfig(window_radius=window, cutoff=cutoff), threads=threads)


def track_sequence(bundle: ModelBundle, sequence_path, init_theta=None, mode: str = "dynamic",
                   iterations: int = _K.iterations, lambda_k: float = _K.lambda_k, lambda_s: float = _K.lambda_s,
                   shape_iterations: int = _S.iterations, lambda_phi: float = _S.lambda_phi,
                   lambda_nbr: float = _S.lambda_nbr, lambda_w: float = _S.lambda_w,
                   window: int = _A.window_radius, cutoff: float = _A.cutoff, threads: int = 0,
                   device: int = 0) -> dict:
    """Track a .wts sequence; returns {"theta" [F,L], "joints" [F,L,3],
    "final_phi" [V,3]} exactly as bindings.cpp:241-303 does."""
    cfg = config_from_kwargs(mode, iterations, lambda_k, lambda_s, shape_iterations, lambda_phi, lambda_nbr,
                             lambda_w, window, cutoff, threads)
    tracked = rigidify(bundle) if mode == "rigid" else bundle
    reader = SequenceReader(sequence_path)
    h = reader.header
    intr = Intrinsics(h.fx, h.fy, h.cx, h.cy, h.width, h.height)
    trk = Tracker(tracked, intr, init_theta, device=device)
    try:
        frames = reader.frames() if reader.frame_count() else np.zeros((0, h.height, h.width), np.float32)
        theta, joints = trk.track_sequence(frames, cfg, depth_scale=h.depth_scale)
        final_phi = trk.get_state()[1]
    finally:
        trk.close()
    return {"theta": theta, "joints": joints, "final_phi": final_phi}


def skin_mesh(bundle: ModelBundle, theta, phi=None, device: int = 0) -> dict:
    """skin_mesh (bindings.cpp:185-202): {"vertices", "normals", "valid"}."""
    trk = Tracker(bundle, Intrinsics(), device=device)
    try:
        v, n, valid = trk.skin(np.asarray(theta, float), phi)
    finally:
        trk.close()
    return {"vertices": v, "normals": n, "valid": valid}
