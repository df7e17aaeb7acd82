"""ctypes access to oracle/_ref/libwtref.so -- TEST INFRASTRUCTURE ONLY.

The library is the UNMODIFIED reference warptrack sources compiled by
oracle/ref/Makefile (see ref_driver.cpp for the entry points). Only tests/,
__graft_entry__.smoke() and bench.py's CPU-baseline leg may use this module,
and only as the checker / the timed reference arm -- never on the product
path.
"""
from __future__ import annotations

import ctypes as C
import subprocess
from pathlib import Path

import numpy as np

from paper_1711_07999_b200 import _lib as W
from paper_1711_07999_b200.model import ModelBundle

HERE = Path(__file__).resolve().parent
LIB_PATH = HERE / "_ref" / "libwtref.so"
REF_SRC = Path("/root/reference/proj")

_lib = None


def available() -> bool:
    return LIB_PATH.exists()


def build() -> bool:
    """Builds the checker when the reference sources are present (never on
    the GPU box, which only receives the prebuilt .so)."""
    if not REF_SRC.exists():
        return LIB_PATH.exists()
    subprocess.run(["make", "-s", "-j8", "-C", str(HERE / "ref"), "all", "adapter"], check=True)
    return LIB_PATH.exists()


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        _lib = C.CDLL(str(LIB_PATH))
        _lib.wtref_last_error.restype = C.c_char_p
    return _lib


def _p(a):
    # data_as keeps a reference to the array, so temporaries outlive the call
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _check(rc: int) -> None:
    if rc != 0:
        raise RuntimeError(f"reference error {rc}: {lib().wtref_last_error().decode()}")


class RefModel:
    """A reference ModelBundle handle."""

    def __init__(self, handle: C.c_void_p):
        self.h = handle

    def __del__(self):
        if self.h:
            lib().wtref_model_free(self.h)
            self.h = None

    @staticmethod
    def from_bundle(b: ModelBundle) -> "RefModel":
        desc, keep = b.to_desc()
        h = C.c_void_p()
        _check(lib().wtref_model_from_desc(C.byref(desc), C.byref(h)))
        del keep
        return RefModel(h)

    @staticmethod
    def rig(name: str) -> "RefModel":
        h = C.c_void_p()
        _check(lib().wtref_make_rig(name.encode(), C.byref(h)))
        return RefModel(h)

    def subdivide(self, iterations: int) -> "RefModel":
        h = C.c_void_p()
        _check(lib().wtref_subdivide(self.h, iterations, C.byref(h)))
        return RefModel(h)

    def rigidify(self) -> "RefModel":
        h = C.c_void_p()
        _check(lib().wtref_rigidify(self.h, C.byref(h)))
        return RefModel(h)

    def sizes(self):
        v = [C.c_int() for _ in range(7)]
        lib().wtref_model_sizes(self.h, *[C.byref(x) for x in v])
        return [x.value for x in v]

    def to_bundle(self) -> ModelBundle:
        """Exports the reference bundle (rig, subdivision, finalize, kNN all
        computed by the reference) as the arrays the GPU consumes."""
        L, V, T, nvt, nnb, npoly, npi = self.sizes()
        a = dict(parent=np.zeros(L, np.int32), parent_offset=np.zeros((L, 8)), joint_kind=np.zeros(L, np.int32),
                 joint_axis=np.zeros((L, 3)), theta_index=np.zeros(L, np.int32), v0=np.zeros((V, 3)),
                 phi=np.zeros((V, 3)), weight_count=np.zeros(V, np.int32), weight_link=np.zeros((V, 4), np.int32),
                 weight=np.zeros((V, 4)), triangles=np.zeros((T, 3), np.int32),
                 vtri_offsets=np.zeros(V + 1, np.int32), vtri_items=np.zeros(nvt, np.int32),
                 nbr_offsets=np.zeros(V + 1, np.int32), nbr_items=np.zeros(nnb, np.int32))
        poff = np.zeros(npoly + 1, np.int32)
        pitems = np.zeros(npi, np.int32)
        order = ["parent", "parent_offset", "joint_kind", "joint_axis", "theta_index", "v0", "phi",
                 "weight_count", "weight_link", "weight", "triangles", "vtri_offsets", "vtri_items",
                 "nbr_offsets", "nbr_items"]
        _check(lib().wtref_model_export(self.h, *[_p(a[k]) for k in order], _p(poff), _p(pitems)))
        polys = [pitems[poff[f]:poff[f + 1]].tolist() for f in range(npoly)]
        return ModelBundle(parent=a["parent"], parent_offset=a["parent_offset"], joint_kind=a["joint_kind"],
                           joint_axis=a["joint_axis"], theta_index=a["theta_index"], v0=a["v0"],
                           weight_count=a["weight_count"], weight_link=a["weight_link"], weight=a["weight"],
                           polys=polys, phi=a["phi"], triangles=a["triangles"], vtri_offsets=a["vtri_offsets"],
                           vtri_items=a["vtri_items"], nbr_offsets=a["nbr_offsets"], nbr_items=a["nbr_items"])

    # ---- stages ---------------------------------------------------------------
    def fk(self, theta):
        L = self.sizes()[0]
        fk, off = np.zeros((L, 8)), np.zeros((L, 8))
        _check(lib().wtref_fk(self.h, _p(np.ascontiguousarray(theta, float)), _p(fk), _p(off)))
        return fk, off

    def pose_derivatives(self, theta):
        L = self.sizes()[0]
        d = np.zeros((L, L, 8))
        _check(lib().wtref_pose_derivatives(self.h, _p(np.ascontiguousarray(theta, float)), _p(d)))
        return d

    def skin(self, theta, phi=None, threads: int = 1):
        V = self.sizes()[1]
        v, n, valid = np.zeros((V, 3)), np.zeros((V, 3)), np.zeros(V, np.uint8)
        ph = None if phi is None else np.ascontiguousarray(phi, float)
        _check(lib().wtref_skin(self.h, _p(np.ascontiguousarray(theta, float)), _p(ph), threads, _p(v), _p(n),
                                _p(valid)))
        return v, n, valid

    def influence_counts(self):
        s = np.zeros(self.sizes()[0])
        _check(lib().wtref_influence_counts(self.h, _p(s)))
        return s

    def vertex_jacobian(self, theta, i: int):
        row = np.zeros(self.sizes()[0])
        _check(lib().wtref_vertex_jacobian(self.h, _p(np.ascontiguousarray(theta, float)), i, _p(row)))
        return row

    def normal_system(self, theta, kin: W.KinConfig, count, residual, threads: int = 1):
        L = self.sizes()[0]
        jtj, jtr = np.zeros((L, L)), np.zeros(L)
        _check(lib().wtref_normal_system(self.h, _p(np.ascontiguousarray(theta, float)), C.byref(kin),
                                         _p(np.ascontiguousarray(count, np.int32)),
                                         _p(np.ascontiguousarray(residual, float)), threads, _p(jtj), _p(jtr)))
        return jtj, jtr

    def render_depth(self, theta, intr: W.Intrinsics, phi=None, noise: W.Noise | None = None, frame: int = 0):
        d = np.zeros((intr.height, intr.width), np.float32)
        vis = np.zeros(self.sizes()[0], np.uint8)
        ph = None if phi is None else np.ascontiguousarray(phi, float)
        _check(lib().wtref_render_depth(self.h, _p(np.ascontiguousarray(theta, float)), _p(ph), C.byref(intr),
                                        C.byref(noise) if noise else None, frame, _p(d), _p(vis)))
        return d, vis

    def rasterize(self, theta, intr: W.Intrinsics, phi=None):
        P = intr.width * intr.height
        depth, tri = np.zeros(P), np.zeros(P, np.int32)
        ph = None if phi is None else np.ascontiguousarray(phi, float)
        _check(lib().wtref_rasterize(self.h, _p(np.ascontiguousarray(theta, float)), _p(ph), C.byref(intr),
                                     _p(depth), _p(tri)))
        return depth, tri


def depth_to_cloud(intr: W.Intrinsics, depth, scale: float = 1.0):
    P = intr.width * intr.height
    pts, valid = np.zeros((P, 3)), np.zeros(P, np.uint8)
    _check(lib().wtref_depth_to_cloud(C.byref(intr), _p(np.ascontiguousarray(depth, np.float32)), C.c_double(scale),
                                      _p(pts), _p(valid)))
    return pts, valid


def project(intr: W.Intrinsics, p):
    u, v = C.c_int(), C.c_int()
    ok = lib().wtref_project(C.byref(intr), C.c_double(p[0]), C.c_double(p[1]), C.c_double(p[2]),
                             C.byref(u), C.byref(v))
    return (u.value, v.value) if ok else None


def associate(intr: W.Intrinsics, v, n, valid, points, point_valid, window=5, cutoff=0.10, threads=1):
    nv = v.shape[0]
    P = intr.width * intr.height
    out = dict(winners=np.zeros(P, np.int32), p_tilde=np.zeros((nv, 3)), count=np.zeros(nv, np.int32),
               residual=np.zeros(nv))
    _check(lib().wtref_associate(C.byref(intr), nv, _p(np.ascontiguousarray(v, float)),
                                 _p(np.ascontiguousarray(n, float)), _p(np.ascontiguousarray(valid, np.uint8)),
                                 _p(np.ascontiguousarray(points, float)),
                                 _p(np.ascontiguousarray(point_valid, np.uint8)), window, C.c_double(cutoff),
                                 threads, _p(out["winners"]), _p(out["p_tilde"]), _p(out["count"]),
                                 _p(out["residual"])))
    return out


def bucket_occupancy(intr: W.Intrinsics, v, n, valid):
    nv = v.shape[0]
    P = intr.width * intr.height
    off, items, ni = np.zeros(P + 1, np.int32), np.zeros(max(nv, 1), np.int32), C.c_int()
    _check(lib().wtref_bucket_occupancy(C.byref(intr), nv, _p(np.ascontiguousarray(v, float)),
                                        _p(np.ascontiguousarray(n, float)),
                                        _p(np.ascontiguousarray(valid, np.uint8)), _p(off), _p(items), C.byref(ni)))
    return off, items[:ni.value]


def solve_step(jtj, jtr, lambda_k=1e-2, diag_floor=1e-9):
    n = jtr.shape[0]
    x = np.zeros(n)
    rc = lib().wtref_solve_step(n, _p(np.ascontiguousarray(jtj, float)), _p(np.ascontiguousarray(jtr, float)),
                                C.c_double(lambda_k), C.c_double(diag_floor), _p(x))
    return (x if rc == 0 else None), rc


def solve_vertex(dr, r, phi, nd, ncount, cfg: W.ShapeConfig):
    delta = np.zeros(3)
    sing = C.c_int()
    _check(lib().wtref_solve_vertex(_p(np.ascontiguousarray(dr, float)), C.c_double(r),
                                    _p(np.ascontiguousarray(phi, float)), _p(np.ascontiguousarray(nd, float)),
                                    ncount, C.byref(cfg), _p(delta), C.byref(sing)))
    return delta, bool(sing.value)


def build_neighbors(v0, k):
    nv = v0.shape[0]
    items, counts = np.zeros(nv * k, np.int32), np.zeros(nv, np.int32)
    _check(lib().wtref_build_neighbors(nv, _p(np.ascontiguousarray(v0, float)), k, _p(items), _p(counts)))
    return items.reshape(nv, k), counts


def finalize(v0, polys):
    nv = v0.shape[0]
    poff = np.zeros(len(polys) + 1, np.int32)
    poff[1:] = np.cumsum([len(p) for p in polys])
    pitems = np.ascontiguousarray(np.concatenate([np.asarray(p, np.int32) for p in polys]) if polys
                                  else np.zeros(0, np.int32), np.int32)
    nt = C.c_int()
    _check(lib().wtref_finalize(nv, _p(np.ascontiguousarray(v0, float)), len(polys), _p(poff), _p(pitems),
                                C.byref(nt), None, None, None))
    tri = np.zeros((nt.value, 3), np.int32)
    off = np.zeros(nv + 1, np.int32)
    items = np.zeros(3 * nt.value, np.int32)
    _check(lib().wtref_finalize(nv, _p(np.ascontiguousarray(v0, float)), len(polys), _p(poff), _p(pitems),
                                C.byref(nt), _p(tri), _p(off), _p(items)))
    return tri, off, items


class RefTracker:
    """make_tracker + track_frame / optimize_pose / optimize_shape of the
    reference on its own CPU threads."""

    def __init__(self, model: RefModel, init_theta=None):
        self.model = model
        self.h = C.c_void_p()
        th = None if init_theta is None else np.ascontiguousarray(init_theta, float)
        _check(lib().wtref_tracker_create(model.h, _p(th), C.byref(self.h)))
        self.L, self.V = model.sizes()[:2]
        self._kin = (W.KinIterStats * 64)()
        self._shape = (W.ShapeIterStats * 64)()

    def __del__(self):
        if self.h:
            lib().wtref_tracker_free(self.h)
            self.h = None

    def get_state(self):
        th, ph, fi = np.zeros(self.L), np.zeros((self.V, 3)), C.c_int()
        lib().wtref_tracker_get(self.h, _p(th), _p(ph), C.byref(fi))
        return th, ph, fi.value

    def set_state(self, theta, phi=None, frame_index=0):
        lib().wtref_tracker_set(self.h, _p(np.ascontiguousarray(theta, float)),
                                _p(None if phi is None else np.ascontiguousarray(phi, float)), frame_index)

    def _fs(self):
        return W.FrameStatsC(0, 0, 0, 64, 64, 0, self._kin, self._shape)

    def track_frame_depth(self, intr: W.Intrinsics, depth, cfg: W.TrackConfigC, scale=1.0):
        st = self._fs()
        _check(lib().wtref_track_frame_depth(self.h, C.byref(intr), _p(np.ascontiguousarray(depth, np.float32)),
                                             C.c_double(scale), C.byref(cfg), C.byref(st)))
        return st

    def track_frame_cloud(self, intr: W.Intrinsics, points, valid, cfg: W.TrackConfigC):
        st = self._fs()
        _check(lib().wtref_track_frame_cloud(self.h, C.byref(intr), _p(np.ascontiguousarray(points, float)),
                                             _p(np.ascontiguousarray(valid, np.uint8)), C.byref(cfg), C.byref(st)))
        return st

    def optimize_pose(self, intr, points, valid, kin: W.KinConfig, assoc: W.AssocConfig, threads=1):
        n = C.c_int()
        _check(lib().wtref_optimize_pose(self.h, C.byref(intr), _p(np.ascontiguousarray(points, float)),
                                         _p(np.ascontiguousarray(valid, np.uint8)), C.byref(kin), C.byref(assoc),
                                         threads, self._kin, 64, C.byref(n)))
        return [self._kin[k] for k in range(n.value)]

    def optimize_shape(self, intr, points, valid, shape: W.ShapeConfig, assoc: W.AssocConfig, threads=1,
                       stats=True):
        n = C.c_int()
        _check(lib().wtref_optimize_shape(self.h, C.byref(intr), _p(np.ascontiguousarray(points, float)),
                                          _p(np.ascontiguousarray(valid, np.uint8)), C.byref(shape), C.byref(assoc),
                                          threads, int(stats), self._shape, 64, C.byref(n)))
        return [self._shape[k] for k in range(n.value)]


def hardware_threads() -> int:
    return lib().wtref_hardware_threads()


def write_sequence(path, intr: W.Intrinsics, frames, depth_scale: float = 1.0) -> None:
    """SequenceWriter (seqio.cpp:493-535)."""
    fr = np.ascontiguousarray(frames, np.float32)
    _check(lib().wtref_write_sequence(str(path).encode(), C.byref(intr), C.c_double(depth_scale), _p(fr),
                                      fr.shape[0]))


def read_depth(path, frame: int):
    """SequenceReader::read_depth (seqio.cpp:476-487) -> (intr, scale, count, depth)."""
    intr, scale, n = W.Intrinsics(), C.c_double(), C.c_int()
    _check(lib().wtref_read_depth(str(path).encode(), frame, C.byref(intr), C.byref(scale), C.byref(n), None))
    d = np.zeros((intr.height, intr.width), np.float32)
    _check(lib().wtref_read_depth(str(path).encode(), frame, None, None, None, _p(d)))
    return intr, scale.value, n.value, d


def run_tracking(model: RefModel, path, cfg: W.TrackConfigC, init_theta=None):
    """run_tracking (tracker.cpp:70-100) over a .wts: {theta, joints, final_phi}."""
    L, V = model.sizes()[:2]
    F = read_depth(path, 0)[2]
    th, jt, ph = np.zeros((F, L)), np.zeros((F, L, 3)), np.zeros((V, 3))
    init = None if init_theta is None else np.ascontiguousarray(init_theta, float)
    _check(lib().wtref_run_tracking(model.h, str(path).encode(), C.byref(cfg), _p(init), _p(th), _p(jt), _p(ph)))
    return dict(theta=th, joints=jt, final_phi=ph)


def recon_error(model: RefModel, theta, intr: W.Intrinsics, points, valid, phi=None, threads: int = 0):
    """reconstruction_error_frame (metrics.cpp:110-142): visible-vertex distances."""
    V = model.sizes()[1]
    d = np.zeros(V)
    n = C.c_int()
    _check(lib().wtref_recon_error(model.h, _p(np.ascontiguousarray(theta, float)),
                                   _p(None if phi is None else np.ascontiguousarray(phi, float)), C.byref(intr),
                                   _p(np.ascontiguousarray(points, float)), _p(np.ascontiguousarray(valid, np.uint8)),
                                   threads, _p(d), C.byref(n)))
    return d[:n.value]
