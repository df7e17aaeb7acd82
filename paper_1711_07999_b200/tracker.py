"""Host-side mirror of the reference tracker API over the C-ABI.

Names, defaults and semantics follow the reference:
  KinSolverConfig   kinopt.hpp:10-18      ShapeSolverConfig  shapeopt.hpp:9-15
  AssocConfig       tracker_state.hpp:11-14   TrackConfig   tracker.hpp:14-20
  Intrinsics        association.hpp:11-15
  Tracker           TrackerState (tracker_state.hpp:18-23) + make_tracker
                    (tracker.cpp:45-52) with the state resident on one GPU
  track_frame       tracker.cpp:54-68     optimize_pose  kinopt.cpp:132-171
  optimize_shape    shapeopt.cpp:50-130   solve_step     kinopt.cpp:121-130
  solve_vertex      shapeopt.cpp:25-48    associate      association.cpp:111-138
Every numeric call runs on the GPU; there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from ._lib import check, lib, ptr
from .model import ModelBundle

MODES = {"dynamic": _lib.MODE_DYNAMIC, "shape-match": _lib.MODE_SHAPE_MATCH,
         "smooth-bind": _lib.MODE_SMOOTH_BIND, "rigid": _lib.MODE_RIGID}


def parse_track_mode(name: str) -> int:
    """parse_track_mode (tracker.cpp:15-22)."""
    if name not in MODES:
        raise _lib.ValidationError(_lib.WT_EINVAL, f"unknown mode '{name}' "
                                   "(expected dynamic|shape-match|smooth-bind|rigid)")
    return MODES[name]


@dataclass
class Intrinsics:
    fx: float = 365.456
    fy: float = 365.456
    cx: float = 256.0
    cy: float = 212.0
    width: int = 512
    height: int = 424

    def c(self) -> _lib.Intrinsics:
        return _lib.Intrinsics(self.fx, self.fy, self.cx, self.cy, self.width, self.height)

    @staticmethod
    def scaled(width: int, height: int) -> "Intrinsics":
        """The benchmark intrinsics: fx = fy = 365.456 * W / 512, centre."""
        f = 365.456 * width / 512.0
        return Intrinsics(f, f, width / 2.0, height / 2.0, width, height)


@dataclass
class KinSolverConfig:
    iterations: int = 12
    lambda_k: float = 1e-2
    lambda_s: float = 1e-4
    diag_floor: float = 1e-9
    assoc_refresh: int = 1
    clamp_limits: bool = False
    limit: float = 0.0

    def c(self) -> _lib.KinConfig:
        return _lib.KinConfig(self.iterations, self.assoc_refresh, self.lambda_k, self.lambda_s,
                              self.diag_floor, int(self.clamp_limits), 0, self.limit)


@dataclass
class ShapeSolverConfig:
    iterations: int = 2
    lambda_phi: float = 0.05
    lambda_nbr: float = 0.5
    lambda_w: float = 1e-2
    diag_floor: float = 1e-9

    def c(self) -> _lib.ShapeConfig:
        return _lib.ShapeConfig(self.iterations, 0, self.lambda_phi, self.lambda_nbr, self.lambda_w,
                                self.diag_floor)


@dataclass
class AssocConfig:
    window_radius: int = 5
    cutoff: float = 0.10

    def c(self) -> _lib.AssocConfig:
        return _lib.AssocConfig(self.window_radius, 0, self.cutoff)


@dataclass
class TrackConfig:
    mode: str = "dynamic"
    kin: KinSolverConfig = field(default_factory=KinSolverConfig)
    shape: ShapeSolverConfig = field(default_factory=ShapeSolverConfig)
    assoc: AssocConfig = field(default_factory=AssocConfig)
    threads: int = 1
    shape_stats: bool = True  # track_frame always asks for shape stats (tracker.cpp:64)

    def c(self) -> _lib.TrackConfigC:
        return _lib.TrackConfigC(parse_track_mode(self.mode), self.threads, self.kin.c(),
                                 self.shape.c(), self.assoc.c(), int(self.shape_stats), 0)


@dataclass
class KinIterStats:
    iteration: int
    residual_sum: float
    step_norm: float
    associated: int
    solver_skipped: bool


@dataclass
class ShapeIterStats:
    iteration: int
    mean_phi: float
    max_phi: float
    mean_abs_r_before: float
    mean_abs_r_after: float
    singular: int


@dataclass
class FrameStats:
    frame: int
    kin: list
    shape: list


def _kin_list(arr, n) -> list:
    return [KinIterStats(arr[k].iteration, arr[k].residual_sum, arr[k].step_norm, arr[k].associated,
                         bool(arr[k].solver_skipped)) for k in range(n)]


def _shape_list(arr, n) -> list:
    return [ShapeIterStats(arr[k].iteration, arr[k].mean_phi, arr[k].max_phi, arr[k].mean_abs_r_before,
                           arr[k].mean_abs_r_after, arr[k].singular) for k in range(n)]


def _f64(a, shape=None) -> np.ndarray:
    a = np.ascontiguousarray(a, dtype=np.float64)
    if shape is not None and a.shape != shape:
        raise _lib.LengthMismatch(_lib.WT_ELENGTH, f"expected shape {shape}, got {a.shape}")
    return a


class Tracker:
    """TrackerState resident on one GPU: theta, Phi, frame index + the model.

    One Tracker = one tracking sequence = one CUDA stream (not thread-safe;
    distinct Trackers are independent)."""

    def __init__(self, bundle: ModelBundle, intr: Intrinsics, init_theta=None, device: int = 0):
        self.bundle = bundle
        self.intr = intr
        self._ctx = C.c_void_p()
        desc, keep = bundle.to_desc()
        check(lib().wt_gpu_create(device, C.byref(desc), C.byref(intr.c()), C.byref(self._ctx)))
        del keep
        L = bundle.link_count
        theta = np.zeros(L)
        if init_theta is not None and np.asarray(init_theta).size == L:  # make_tracker
            theta = np.asarray(init_theta, dtype=np.float64)
        self.set_state(theta=theta, frame_index=0)
        self._kin = (_lib.KinIterStats * 64)()
        self._shape = (_lib.ShapeIterStats * 64)()

    def _ensure_stats(self, n_kin: int, n_shape: int) -> None:
        """Stats arrays sized for the call's iteration counts (the reference
        has no iteration cap), before anything is launched."""
        if n_kin > len(self._kin):
            self._kin = (_lib.KinIterStats * n_kin)()
        if n_shape > len(self._shape):
            self._shape = (_lib.ShapeIterStats * n_shape)()

    # ---- state ---------------------------------------------------------------
    def close(self) -> None:
        if self._ctx:
            lib().wt_gpu_destroy(self._ctx)
            self._ctx = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_state(self, theta=None, phi=None, frame_index: int = 0) -> None:
        th = None if theta is None else _f64(theta, (self.bundle.link_count,))
        ph = None if phi is None else _f64(phi, (self.bundle.vertex_count, 3))
        check(lib().wt_gpu_set_state(self._ctx, ptr(th), ptr(ph), frame_index), self._ctx)

    def get_state(self, with_phi: bool = True):
        th = np.zeros(self.bundle.link_count)
        ph = np.zeros((self.bundle.vertex_count, 3)) if with_phi else None
        fi = C.c_int32()
        check(lib().wt_gpu_get_state(self._ctx, ptr(th), ptr(ph), C.byref(fi)), self._ctx)
        return th, ph, fi.value

    @property
    def theta(self) -> np.ndarray:
        return self.get_state(with_phi=False)[0]

    @property
    def phi(self) -> np.ndarray:
        return self.get_state()[1]

    @property
    def frame_index(self) -> int:
        return self.get_state(with_phi=False)[2]

    # ---- frames --------------------------------------------------------------
    def load_depth(self, depth, depth_scale: float = 1.0) -> None:
        d = np.ascontiguousarray(depth, dtype=np.float32).reshape(-1)
        if d.size != self.intr.width * self.intr.height:
            raise _lib.LengthMismatch(_lib.WT_ELENGTH, "depth image size differs from intrinsics grid")
        check(lib().wt_gpu_load_depth(self._ctx, ptr(d), depth_scale), self._ctx)

    def load_cloud(self, points, valid) -> None:
        P = self.intr.width * self.intr.height
        p = _f64(points).reshape(P, 3)
        v = np.ascontiguousarray(valid, dtype=np.uint8).reshape(P)
        check(lib().wt_gpu_load_cloud(self._ctx, ptr(p), ptr(v)), self._ctx)

    def _stats(self) -> _lib.FrameStatsC:
        return _lib.FrameStatsC(0, 0, 0, len(self._kin), len(self._shape), 0, self._kin, self._shape)

    def track_frame(self, cfg: TrackConfig, depth=None, depth_scale: float = 1.0, cloud=None,
                    stats: bool = True) -> FrameStats | None:
        """track_frame (tracker.cpp:54-68) on a depth image, an organized
        cloud (points, valid), or the frame already loaded."""
        self._ensure_stats(cfg.kin.iterations, cfg.shape.iterations)
        if depth is not None:
            self.load_depth(depth, depth_scale)
        elif cloud is not None:
            self.load_cloud(*cloud)
        st = self._stats() if stats else None
        check(lib().wt_gpu_track_loaded(self._ctx, C.byref(cfg.c()), C.byref(st) if st else None),
              self._ctx)
        if not st:
            return None
        return FrameStats(st.frame, _kin_list(self._kin, st.n_kin), _shape_list(self._shape, st.n_shape))

    def track_sequence(self, frames, cfg: TrackConfig, depth_scale: float = 1.0):
        """run_tracking (tracker.cpp:70-100) over depth frames [F,H,W] (host
        array, or a device address with n_frames given as frames=(ptr, F)):
        returns (theta [F,L], joints [F,L,3]). Uploads overlap the solves."""
        if isinstance(frames, tuple):
            addr, F = frames
        else:
            arr = np.ascontiguousarray(frames, dtype=np.float32)
            F = arr.shape[0] if arr.size else 0
            if arr.size and arr[0].size != self.intr.width * self.intr.height:
                raise _lib.LengthMismatch(_lib.WT_ELENGTH, "depth image size differs from intrinsics grid")
            addr = ptr(arr)
        L = self.bundle.link_count
        th, jt = np.zeros((F, L)), np.zeros((F, L, 3))
        check(lib().wt_gpu_track_sequence(self._ctx, addr, F, depth_scale, C.byref(cfg.c()), ptr(th), ptr(jt)),
              self._ctx)
        return th, jt

    def reconstruction_error(self, per_vertex: bool = False) -> np.ndarray:
        """reconstruction_error_frame (metrics.cpp:110-142) of the current
        state against the loaded frame: distances of the visible vertices in
        ascending vertex order (per_vertex=True: [V] with NaN where hidden)."""
        d = np.zeros(self.bundle.vertex_count)
        n = C.c_int32()
        check(lib().wt_gpu_recon_error(self._ctx, ptr(d), C.byref(n)), self._ctx)
        return d if per_vertex else d[~np.isnan(d)]

    def joint_positions(self) -> np.ndarray:
        """Link origins at the current theta (tracker.cpp:84-86), [L,3]."""
        out = np.zeros((self.bundle.link_count, 3))
        check(lib().wt_gpu_joint_positions(self._ctx, ptr(out)), self._ctx)
        return out

    def optimize_pose(self, kin: KinSolverConfig, assoc: AssocConfig = AssocConfig()) -> list:
        n = C.c_int32()
        self._ensure_stats(kin.iterations, 0)
        check(lib().wt_gpu_optimize_pose(self._ctx, C.byref(kin.c()), C.byref(assoc.c()), self._kin,
                                         len(self._kin), C.byref(n)), self._ctx)
        return _kin_list(self._kin, min(n.value, len(self._kin)))

    def optimize_shape(self, shape: ShapeSolverConfig, assoc: AssocConfig = AssocConfig(),
                       stats: bool = True) -> list:
        n = C.c_int32()
        self._ensure_stats(0, shape.iterations)
        check(lib().wt_gpu_optimize_shape(self._ctx, C.byref(shape.c()), C.byref(assoc.c()), int(stats),
                                          self._shape, len(self._shape), C.byref(n)), self._ctx)
        return _shape_list(self._shape, min(n.value, len(self._shape))) if stats else []

    # ---- stage hooks ---------------------------------------------------------
    def skin(self, theta, phi=None):
        """skin(mesh, link_offsets(theta), phi) -> (v, n, valid) (skinmesh.cpp:104-141)."""
        V = self.bundle.vertex_count
        th = _f64(theta, (self.bundle.link_count,))
        ph = None if phi is None else _f64(phi, (V, 3))
        v, n = np.zeros((V, 3)), np.zeros((V, 3))
        valid = np.zeros(V, dtype=np.uint8)
        check(lib().wt_gpu_skin(self._ctx, ptr(th), ptr(ph), ptr(v), ptr(n), ptr(valid)), self._ctx)
        return v, n, valid

    def associate(self, window_radius: int = 5, cutoff: float = 0.10) -> dict:
        """associate() of the last skinned mesh against the loaded frame."""
        V = self.bundle.vertex_count
        P = self.intr.width * self.intr.height
        out = dict(winners=np.zeros(P, np.int32), p_tilde=np.zeros((V, 3)), count=np.zeros(V, np.int32),
                   residual=np.zeros(V))
        check(lib().wt_gpu_associate(self._ctx, window_radius, cutoff, ptr(out["winners"]),
                                     ptr(out["p_tilde"]), ptr(out["count"]), ptr(out["residual"])),
              self._ctx)
        return out

    def normal_system(self, theta, kin: KinSolverConfig, count, residual):
        """accumulate_normal_system at theta for (count, residual)."""
        L, V = self.bundle.link_count, self.bundle.vertex_count
        th = _f64(theta, (L,))
        cnt = np.ascontiguousarray(count, dtype=np.int32).reshape(V)
        res = _f64(residual, (V,))
        jtj, jtr = np.zeros((L, L)), np.zeros(L)
        check(lib().wt_gpu_normal_system(self._ctx, ptr(th), C.byref(kin.c()), ptr(cnt), ptr(res), ptr(jtj),
                                         ptr(jtr)), self._ctx)
        return jtj, jtr

    def render_depth(self, theta, phi=None, sigma=0.0, dropout=0.0, quantization=0.0, seed=0,
                     frame: int = 0, out_ptr: int | None = None):
        """synthesize_frame (synth.cpp:229-270) on the GPU: (depth [H,W] f32, joint_visible [L]).
        With out_ptr (a device or host address of H*W floats) the depth is
        written there and None is returned in its place."""
        th = _f64(theta, (self.bundle.link_count,))
        ph = None if phi is None else _f64(phi, (self.bundle.vertex_count, 3))
        depth = None if out_ptr is not None else np.zeros((self.intr.height, self.intr.width), np.float32)
        vis = np.zeros(self.bundle.link_count, np.uint8)
        nz = _lib.Noise(sigma, dropout, quantization, seed)
        check(lib().wt_gpu_render_depth(self._ctx, ptr(th), ptr(ph), C.byref(nz), frame,
                                        out_ptr if out_ptr is not None else ptr(depth), ptr(vis)), self._ctx)
        return depth, vis


class BatchTracker:
    """B independent tracking sequences of one model, tracked in lockstep on
    one GPU (run_tracking, tracker.cpp:70-100, for B sequences at once).

    Each sequence has its own TrackerState (theta, Phi) and frame; a frame of
    the whole batch is one CUDA graph whose kernels carry the sequence index
    in blockIdx.y, so every launch covers B x the per-vertex / per-pixel
    work. The frame index and mode schedule are shared."""

    def __init__(self, bundle: ModelBundle, intr: Intrinsics, n_seq: int, init_theta=None,
                 device: int = 0):
        self.bundle = bundle
        self.intr = intr
        self.n_seq = n_seq
        self._ctx = C.c_void_p()
        desc, keep = bundle.to_desc()
        check(lib().wt_gpu_create_batch(device, C.byref(desc), C.byref(intr.c()), n_seq,
                                        C.byref(self._ctx)))
        del keep
        if init_theta is not None:
            th = np.asarray(init_theta, dtype=np.float64)
            for b in range(n_seq):
                self.set_state(b, theta=th if th.ndim == 1 else th[b])
        self._kin = [(_lib.KinIterStats * 64)() for _ in range(n_seq)]
        self._shape = [(_lib.ShapeIterStats * 32)() for _ in range(n_seq)]

    def close(self) -> None:
        if self._ctx:
            lib().wt_gpu_destroy(self._ctx)
            self._ctx = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_state(self, seq: int, theta=None, phi=None) -> None:
        th = None if theta is None else _f64(theta, (self.bundle.link_count,))
        ph = None if phi is None else _f64(phi, (self.bundle.vertex_count, 3))
        check(lib().wt_gpu_batch_set_state(self._ctx, seq, ptr(th), ptr(ph)), self._ctx)

    def get_state(self, seq: int, with_phi: bool = True):
        th = np.zeros(self.bundle.link_count)
        ph = np.zeros((self.bundle.vertex_count, 3)) if with_phi else None
        check(lib().wt_gpu_batch_get_state(self._ctx, seq, ptr(th), ptr(ph)), self._ctx)
        return th, ph

    def thetas(self) -> np.ndarray:
        return np.stack([self.get_state(b, with_phi=False)[0] for b in range(self.n_seq)])

    def load_depth(self, depth, depth_scale: float = 1.0) -> None:
        """depth [B, H, W] (host array) or (device address,) of the same layout."""
        if isinstance(depth, tuple):
            addr = depth[0]
        else:
            d = np.ascontiguousarray(depth, dtype=np.float32)
            if d.size != self.n_seq * self.intr.width * self.intr.height:
                raise _lib.LengthMismatch(_lib.WT_ELENGTH, "depth batch differs from B x intrinsics grid")
            addr = ptr(d)
        check(lib().wt_gpu_batch_load_depth(self._ctx, addr, depth_scale), self._ctx)

    def track_async(self, cfg: TrackConfig) -> None:
        check(lib().wt_gpu_batch_track_async(self._ctx, C.byref(cfg.c())), self._ctx)

    def sync(self) -> None:
        check(lib().wt_gpu_sync(self._ctx), self._ctx)

    def stats(self) -> list:
        arr = (_lib.FrameStatsC * self.n_seq)()
        for b in range(self.n_seq):
            arr[b] = _lib.FrameStatsC(0, 0, 0, 64, 32, 0, self._kin[b], self._shape[b])
        check(lib().wt_gpu_batch_stats(self._ctx, arr), self._ctx)
        return [FrameStats(arr[b].frame, _kin_list(self._kin[b], arr[b].n_kin),
                           _shape_list(self._shape[b], arr[b].n_shape)) for b in range(self.n_seq)]

    def track_frame(self, cfg: TrackConfig, depth=None, depth_scale: float = 1.0,
                    stats: bool = True) -> list | None:
        """track_frame (tracker.cpp:54-68) of every sequence on its own frame."""
        if depth is not None:
            self.load_depth(depth, depth_scale)
        self.track_async(cfg)
        out = self.stats() if stats else None
        self.sync()
        return out

    @property
    def stream(self) -> int:
        return lib().wt_gpu_stream(self._ctx) or 0


# ---- context-free stage functions ------------------------------------------------

def solve_step(jtj, jtr, cfg: KinSolverConfig, device: int = 0) -> np.ndarray:
    """solve_step (kinopt.cpp:121-130); raises NotPositiveDefinite."""
    a = _f64(jtj)
    b = _f64(jtr)
    n = b.shape[0]
    if a.shape != (n, n):
        raise _lib.LengthMismatch(_lib.WT_ELENGTH, "jtj/jtr size mismatch")
    x = np.zeros(n)
    check(lib().wt_gpu_solve_step(device, n, ptr(a), ptr(b), cfg.lambda_k, cfg.diag_floor, ptr(x)))
    return x


def solve_vertices(dr_dphi, r, phi, nbr_delta, nbr_count, cfg: ShapeSolverConfig, device: int = 0):
    """Batched solve_vertex (shapeopt.cpp:25-48): (delta [n,3], singular [n])."""
    dr = _f64(dr_dphi).reshape(-1, 3)
    n = dr.shape[0]
    rr = _f64(r).reshape(n)
    ph = _f64(phi).reshape(n, 3)
    nd = _f64(nbr_delta).reshape(n, 3)
    nc = np.ascontiguousarray(nbr_count, dtype=np.int32).reshape(n)
    delta = np.zeros((n, 3))
    sing = np.zeros(n, np.uint8)
    check(lib().wt_gpu_solve_vertices(device, n, ptr(dr), ptr(rr), ptr(ph), ptr(nd), ptr(nc),
                                      C.byref(cfg.c()), ptr(delta), ptr(sing)))
    return delta, sing.astype(bool)


def associate_posed(intr: Intrinsics, v, n, valid, points, point_valid, window_radius: int = 5,
                    cutoff: float = 0.10, device: int = 0) -> dict:
    """associate()/associate_winners() of explicit posed vertices (the
    reference's loose-vertex PosedMesh) against an organized cloud."""
    vv = _f64(v).reshape(-1, 3)
    nv = vv.shape[0]
    nn = _f64(n).reshape(nv, 3)
    va = np.ascontiguousarray(valid, dtype=np.uint8).reshape(nv)
    P = intr.width * intr.height
    pts = _f64(points).reshape(P, 3)
    pv = np.ascontiguousarray(point_valid, dtype=np.uint8).reshape(P)
    out = dict(winners=np.zeros(P, np.int32), p_tilde=np.zeros((nv, 3)), count=np.zeros(nv, np.int32),
               residual=np.zeros(nv))
    check(lib().wt_gpu_associate_posed(device, C.byref(intr.c()), nv, ptr(vv), ptr(nn), ptr(va), ptr(pts),
                                       ptr(pv), window_radius, cutoff, ptr(out["winners"]),
                                       ptr(out["p_tilde"]), ptr(out["count"]), ptr(out["residual"])))
    return out
