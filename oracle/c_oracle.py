"""ctypes access to the C restatement oracle (oracle/wt_oracle.c) -- TEST
INFRASTRUCTURE ONLY: the checker of tests/ and __graft_entry__.smoke(), and
bench.py's CPU-baseline fallback when oracle/_ref is absent. Never on the
product path.
"""
from __future__ import annotations

import ctypes as C
import subprocess
from pathlib import Path

import numpy as np

from paper_1711_07999_b200 import _lib as W
from paper_1711_07999_b200.model import ModelBundle

HERE = Path(__file__).resolve().parent
SRC = HERE / "wt_oracle.c"
LIB_PATH = HERE / "_build" / "libwtoracle.so"
_lib = None


def build(force: bool = False) -> Path:
    """gcc, -ffp-contract=off so products and sums round separately."""
    LIB_PATH.parent.mkdir(exist_ok=True)
    if LIB_PATH.exists() and not force and LIB_PATH.stat().st_mtime >= SRC.stat().st_mtime:
        return LIB_PATH
    tmp = LIB_PATH.with_suffix(".so.tmp")
    subprocess.run(["gcc", "-std=c11", "-O2", "-fPIC", "-shared", "-ffp-contract=off",
                    "-I", str(HERE.parent / "include"), str(SRC), "-o", str(tmp), "-lm"], check=True)
    tmp.replace(LIB_PATH)
    return LIB_PATH


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            build()
        _lib = C.CDLL(str(LIB_PATH))
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def project(intr: W.Intrinsics, p):
    u, v = C.c_int(), C.c_int()
    ok = lib().wto_project(C.byref(intr), _p(np.ascontiguousarray(p, float)), C.byref(u), C.byref(v))
    return (u.value, v.value) if ok else None


def associate(intr: W.Intrinsics, v, n, valid, points, point_valid, window=5, cutoff=0.10):
    nv = v.shape[0]
    P = intr.width * intr.height
    out = dict(winners=np.zeros(P, np.int32), p_tilde=np.zeros((nv, 3)), count=np.zeros(nv, np.int32),
               residual=np.zeros(nv))
    lib().wto_associate(C.byref(intr), nv, _p(np.ascontiguousarray(v, float)), _p(np.ascontiguousarray(n, float)),
                        _p(np.ascontiguousarray(valid, np.uint8)), _p(np.ascontiguousarray(points, float)),
                        _p(np.ascontiguousarray(point_valid, np.uint8)), window, C.c_double(cutoff),
                        _p(out["winners"]), _p(out["p_tilde"]), _p(out["count"]), _p(out["residual"]))
    return out


def bucket_occupancy(intr: W.Intrinsics, v, n, valid):
    nv = v.shape[0]
    off = np.zeros(intr.width * intr.height + 1, np.int32)
    items = np.zeros(max(nv, 1), np.int32)
    k = lib().wto_bucket_occupancy(C.byref(intr), nv, _p(np.ascontiguousarray(v, float)),
                                   _p(np.ascontiguousarray(n, float)), _p(np.ascontiguousarray(valid, np.uint8)),
                                   _p(off), _p(items))
    return off, items[:k]


def solve_step(jtj, jtr, lambda_k=1e-2, diag_floor=1e-9):
    n = jtr.shape[0]
    x = np.zeros(n)
    rc = lib().wto_solve_step(n, _p(np.ascontiguousarray(jtj, float)), _p(np.ascontiguousarray(jtr, float)),
                              C.c_double(lambda_k), C.c_double(diag_floor), _p(x))
    return (x if rc == 0 else None), rc


def solve_vertex(g, r, phi, nd, ncount, cfg: W.ShapeConfig):
    delta = np.zeros(3)
    sing = lib().wto_solve_vertex(_p(np.ascontiguousarray(g, float)), C.c_double(r),
                                  _p(np.ascontiguousarray(phi, float)), _p(np.ascontiguousarray(nd, float)),
                                  ncount, C.byref(cfg), _p(delta))
    return delta, bool(sing)


def d_normalized_transform(h8, u):
    D = np.zeros((3, 8))
    lib().wto_d_normalized_transform(_p(np.ascontiguousarray(h8, float)), _p(np.ascontiguousarray(u, float)), _p(D))
    return D


def depth_to_cloud(intr: W.Intrinsics, depth, scale=1.0):
    P = intr.width * intr.height
    pts, valid = np.zeros((P, 3)), np.zeros(P, np.uint8)
    lib().wto_depth_to_cloud(C.byref(intr), _p(np.ascontiguousarray(depth, np.float32)), C.c_double(scale),
                             _p(pts), _p(valid))
    return pts, valid


class OracleTracker:
    """TrackerState + track_frame / optimize_pose / optimize_shape of the C
    restatement (single-threaded, fp64)."""

    def __init__(self, bundle: ModelBundle, intr: W.Intrinsics, init_theta=None):
        self.bundle = bundle
        self.intr = intr
        self._desc, self._keep = bundle.to_desc()
        self.h = C.c_void_p()
        rc = lib().wto_create(C.byref(self._desc), C.byref(intr), C.byref(self.h))
        if rc != 0:
            raise W.ValidationError(rc, "oracle: invalid model")
        self.L, self.V = bundle.link_count, bundle.vertex_count
        th = np.zeros(self.L) if init_theta is None else np.ascontiguousarray(init_theta, float)
        self.set_state(th, None, 0)
        self._kin = (W.KinIterStats * 64)()
        self._shape = (W.ShapeIterStats * 64)()

    def __del__(self):
        if getattr(self, "h", None):
            lib().wto_destroy(self.h)
            self.h = None

    def set_state(self, theta, phi=None, frame_index=0):
        lib().wto_set_state(self.h, _p(np.ascontiguousarray(theta, float)),
                            _p(None if phi is None else np.ascontiguousarray(phi, float)), frame_index)

    def get_state(self):
        th, ph, fi = np.zeros(self.L), np.zeros((self.V, 3)), C.c_int()
        lib().wto_get_state(self.h, _p(th), _p(ph), C.byref(fi))
        return th, ph, fi.value

    def load_depth(self, depth, scale=1.0):
        lib().wto_load_depth(self.h, _p(np.ascontiguousarray(depth, np.float32)), C.c_double(scale))

    def load_cloud(self, points, valid):
        lib().wto_load_cloud(self.h, _p(np.ascontiguousarray(points, float)), _p(np.ascontiguousarray(valid, np.uint8)))

    def skin(self, theta, phi=None):
        v, n, valid = np.zeros((self.V, 3)), np.zeros((self.V, 3)), np.zeros(self.V, np.uint8)
        lib().wto_skin(self.h, _p(np.ascontiguousarray(theta, float)),
                       _p(None if phi is None else np.ascontiguousarray(phi, float)), _p(v), _p(n), _p(valid))
        return v, n, valid

    def track_loaded(self, cfg: W.TrackConfigC):
        st = W.FrameStatsC(0, 0, 0, 64, 64, 0, self._kin, self._shape)
        lib().wto_track_loaded(self.h, C.byref(cfg), C.byref(st))
        return st

    def optimize_pose(self, kin: W.KinConfig, assoc: W.AssocConfig):
        lib().wto_optimize_pose(self.h, C.byref(kin), C.byref(assoc), self._kin)
        return [self._kin[k] for k in range(kin.iterations)]

    def optimize_shape(self, shape: W.ShapeConfig, assoc: W.AssocConfig, stats=True):
        lib().wto_optimize_shape(self.h, C.byref(shape), C.byref(assoc), int(stats), self._shape)
        return [self._shape[k] for k in range(shape.iterations)]

    def normal_system(self, theta, kin: W.KinConfig, count, residual):
        jtj, jtr = np.zeros((self.L, self.L)), np.zeros(self.L)
        lib().wto_normal_system(self.h, _p(np.ascontiguousarray(theta, float)), C.byref(kin),
                                _p(np.ascontiguousarray(count, np.int32)), _p(np.ascontiguousarray(residual, float)),
                                _p(jtj), _p(jtr))
        return jtj, jtr

    def pose_derivatives(self, theta):
        L = self.L
        fk, off, dch = np.zeros((L, 8)), np.zeros((L, 8)), np.zeros((L, L, 8))
        lib().wto_pose_derivatives(self.h, _p(np.ascontiguousarray(theta, float)), _p(fk), _p(off), _p(dch))
        return fk, off, dch
