"""Model bundles as flat arrays: the skeleton + skinned template mesh that the
GPU context uploads once (wt_model_desc in include/wt_gpu.h).

Mirrors warptrack::ModelBundle {Skeleton (skeleton.hpp:14-63), SkinnedMesh
(skinmesh.hpp:31-48)}. The derived fields follow the reference exactly:
  * finalize(): quads split along the shorter diagonal, n-gons fanned, the
    vertex->triangle CSR in triangle order (skinmesh.cpp:13-58);
  * build_neighbors(v0, k): exact k nearest template vertices, ties to the
    lower index (skinmesh.cpp:196-247), k = 4 as load_model uses (seqio.cpp:25);
  * rigidify(): dominant link at weight one, phi zeroed (tracker.cpp:24-43).
Model preprocessing is host-side and out of the GPU hot path (SURVEY.md §2
rows 4 and 12).
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field, replace

import numpy as np

from . import _lib

HINGE, PRISMATIC = _lib.JOINT_HINGE, _lib.JOINT_PRISMATIC


@dataclass
class ModelBundle:
    # skeleton (links topologically sorted, one root)
    parent: np.ndarray          # [L] int32
    parent_offset: np.ndarray   # [L,8] float64 canonical DQ
    joint_kind: np.ndarray      # [L] int32
    joint_axis: np.ndarray      # [L,3] float64 unit
    theta_index: np.ndarray     # [L] int32
    # mesh
    v0: np.ndarray              # [V,3] float64
    weight_count: np.ndarray    # [V] int32
    weight_link: np.ndarray     # [V,4] int32 (-1 padded)
    weight: np.ndarray          # [V,4] float64
    polys: list = field(default_factory=list)
    phi: np.ndarray | None = None
    # derived by finalize / build_neighbors
    triangles: np.ndarray | None = None
    vtri_offsets: np.ndarray | None = None
    vtri_items: np.ndarray | None = None
    nbr_offsets: np.ndarray | None = None
    nbr_items: np.ndarray | None = None
    link_names: list = field(default_factory=list)
    name: str = ""

    @property
    def link_count(self) -> int:
        return int(self.parent.shape[0])

    joint_count = link_count

    @property
    def vertex_count(self) -> int:
        return int(self.v0.shape[0])

    @property
    def triangle_count(self) -> int:
        return 0 if self.triangles is None else int(self.triangles.shape[0])

    def zero_pose(self) -> np.ndarray:
        return np.zeros(self.link_count)

    def finalize(self) -> "ModelBundle":
        self.triangles, self.vtri_offsets, self.vtri_items = finalize(self.v0, self.polys)
        if self.phi is None or self.phi.shape != self.v0.shape:
            self.phi = np.zeros_like(self.v0)
        return self

    def with_neighbors(self, k: int = 4) -> "ModelBundle":
        self.nbr_offsets, self.nbr_items = build_neighbors(self.v0, k)
        return self

    def to_desc(self):
        """(wt_model_desc, keepalive) for the C-ABI."""
        keep = []

        def arr(a, dt):
            a = np.ascontiguousarray(a, dtype=dt)
            keep.append(a)
            return a.ctypes.data_as(C.POINTER(C.c_int32 if dt == np.int32 else C.c_double))

        assert self.triangles is not None and self.nbr_offsets is not None, "finalize + neighbours first"
        d = _lib.ModelDesc()
        d.n_links = self.link_count
        d.n_vertices = self.vertex_count
        d.n_triangles = self.triangle_count
        d.parent = arr(self.parent, np.int32)
        d.parent_offset = arr(self.parent_offset, np.float64)
        d.joint_kind = arr(self.joint_kind, np.int32)
        d.joint_axis = arr(self.joint_axis, np.float64)
        d.theta_index = arr(self.theta_index, np.int32)
        d.v0 = arr(self.v0, np.float64)
        d.phi = arr(self.phi if self.phi is not None else np.zeros_like(self.v0), np.float64)
        d.weight_count = arr(self.weight_count, np.int32)
        d.weight_link = arr(self.weight_link, np.int32)
        d.weight = arr(self.weight, np.float64)
        d.triangles = arr(self.triangles.reshape(-1, 3) if self.triangle_count else np.zeros((1, 3)),
                          np.int32)
        d.vtri_offsets = arr(self.vtri_offsets, np.int32)
        d.vtri_items = arr(self.vtri_items if self.vtri_items.size else np.zeros(1), np.int32)
        d.nbr_offsets = arr(self.nbr_offsets, np.int32)
        d.nbr_items = arr(self.nbr_items if self.nbr_items.size else np.zeros(1), np.int32)
        return d, keep

    def copy(self) -> "ModelBundle":
        return replace(self, **{k: (v.copy() if isinstance(v, np.ndarray) else v)
                                for k, v in self.__dict__.items()})


# ---------------------------------------------------------------------------
# derived topology

def finalize(v0: np.ndarray, polys) -> tuple[np.ndarray, np.ndarray, np.ndarray]:
    """SkinnedMesh::finalize (skinmesh.cpp:13-58): triangles in poly order
    (quads split along the shorter diagonal, d02 <= d13 keeps 0-2, n-gons
    fanned, out-of-range polys skipped) + the vertex->triangle CSR."""
    nv = v0.shape[0]
    sizes = np.fromiter((len(p) for p in polys), dtype=np.int64, count=len(polys))
    if sizes.size and np.all((sizes == 3) | (sizes == 4)):
        pad = np.full((len(polys), 4), -1, dtype=np.int64)
        for k, p in enumerate(polys):
            pad[k, :len(p)] = p
        ok = np.all((pad < nv) & ((pad >= 0) | (np.arange(4)[None, :] >= sizes[:, None])), axis=1)
        pad, sizes = pad[ok], sizes[ok]
        quad = sizes == 4
        q = np.where(quad[:, None], pad, 0)
        d02 = v0[q[:, 0]] - v0[q[:, 2]]
        d13 = v0[q[:, 1]] - v0[q[:, 3]]
        s02 = (d02[:, 0] * d02[:, 0] + d02[:, 1] * d02[:, 1]) + d02[:, 2] * d02[:, 2]
        s13 = (d13[:, 0] * d13[:, 0] + d13[:, 1] * d13[:, 1]) + d13[:, 2] * d13[:, 2]
        keep02 = s02 <= s13
        t1 = np.where(keep02[:, None], pad[:, [0, 1, 2]], pad[:, [0, 1, 3]])
        t2 = np.where(keep02[:, None], pad[:, [0, 2, 3]], pad[:, [1, 2, 3]])
        t1 = np.where(quad[:, None], t1, pad[:, [0, 1, 2]])
        both = np.stack([t1, t2], axis=1)                      # [n, 2, 3]
        take = np.stack([np.ones_like(quad), quad], axis=1)    # second only for quads
        tri = both[take].astype(np.int32).reshape(-1, 3)
    else:
        tris = []
        for poly in polys:
            if any(vi < 0 or vi >= nv for vi in poly):
                continue
            if len(poly) == 4:
                p0, p1, p2, p3 = poly
                d02 = v0[p0] - v0[p2]
                d13 = v0[p1] - v0[p3]
                s02 = (d02[0] * d02[0] + d02[1] * d02[1]) + d02[2] * d02[2]
                s13 = (d13[0] * d13[0] + d13[1] * d13[1]) + d13[2] * d13[2]
                tris += [(p0, p1, p2), (p0, p2, p3)] if s02 <= s13 else [(p0, p1, p3), (p1, p2, p3)]
            else:
                for i in range(1, len(poly) - 1):
                    tris.append((poly[0], poly[i], poly[i + 1]))
        tri = np.asarray(tris, dtype=np.int32).reshape(-1, 3)
    return tri, *_vertex_tri_csr(nv, tri)


def _vertex_tri_csr(nv: int, tri: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
    flat = tri.reshape(-1)
    order = np.argsort(flat, kind="stable")
    items = (order // 3).astype(np.int32)
    counts = np.bincount(flat, minlength=nv)
    offsets = np.zeros(nv + 1, dtype=np.int32)
    np.cumsum(counts, out=offsets[1:])
    return offsets, items


def build_neighbors(v0: np.ndarray, k: int) -> tuple[np.ndarray, np.ndarray]:
    """build_neighbors (skinmesh.cpp:196-247): the k nearest distinct template
    vertices, squared distance computed as ((dx^2 + dy^2) + dz^2) in fp64,
    ties broken toward the lower index. Returns CSR (offsets, items)."""
    from scipy.spatial import cKDTree

    nv = v0.shape[0]
    offsets = np.zeros(nv + 1, dtype=np.int32)
    if nv <= 1 or k < 1:
        return offsets, np.zeros(0, dtype=np.int32)
    want = min(k, nv - 1)
    tree = cKDTree(v0)
    out = np.empty((nv, want), dtype=np.int32)
    extra = 6
    todo = np.arange(nv)
    while todo.size:
        q = min(want + 1 + extra, nv)
        _, idx = tree.query(v0[todo], k=q)
        idx = idx.reshape(len(todo), q)
        d = v0[idx] - v0[todo][:, None, :]
        d2 = (d[..., 0] * d[..., 0] + d[..., 1] * d[..., 1]) + d[..., 2] * d[..., 2]
        d2 = np.where(idx == todo[:, None], np.inf, d2)  # exclude self
        order = np.lexsort((idx, d2), axis=-1)
        d2s = np.take_along_axis(d2, order, -1)
        ids = np.take_along_axis(idx, order, -1)
        out[todo] = ids[:, :want]
        # exact only if the furthest fetched candidate is strictly beyond the
        # k-th (the tree's own metric may differ from ours in the last ulp)
        kth = d2s[:, want - 1]
        far = np.max(np.where(np.isinf(d2), -np.inf, d2), axis=-1)
        unsure = (far <= kth * (1 + 1e-9) + 1e-300) & (q < nv)
        todo = todo[unsure]
        extra = extra * 4
    np.cumsum(np.full(nv, want), out=offsets[1:])
    return offsets, out.reshape(-1).astype(np.int32)


def dominant_links(b: ModelBundle) -> np.ndarray:
    dom = np.full(b.vertex_count, -1, dtype=np.int32)
    for i in range(b.vertex_count):
        best = -1.0
        for s in range(int(b.weight_count[i])):
            e, l = b.weight[i, s], b.weight_link[i, s]
            if e > best or (e == best and l < dom[i]):
                best, dom[i] = e, l
    return dom


def rigidify(b: ModelBundle) -> ModelBundle:
    """rigidify (tracker.cpp:24-43): every weight row becomes its dominant
    link at weight one (ties to the lower link) and phi is zeroed."""
    out = b.copy()
    w = b.weight.copy()
    links = b.weight_link
    cnt = b.weight_count
    valid = np.arange(4)[None, :] < cnt[:, None]
    w_masked = np.where(valid, w, -1.0)
    best = w_masked.max(axis=1)
    cand = valid & (w_masked == best[:, None])
    big = np.where(cand, links, np.iinfo(np.int32).max)
    dom = big.min(axis=1)
    out.weight_count = np.where(cnt > 0, 1, 1).astype(np.int32)
    out.weight_link = np.full_like(links, -1)
    out.weight = np.zeros_like(w)
    has = cnt > 0
    out.weight_link[:, 0] = np.where(has, dom, 0)
    out.weight[:, 0] = 1.0
    out.phi = np.zeros_like(b.v0)
    return out


# ---------------------------------------------------------------------------
# parametric rigs (synthetic inputs; the tracked human model of the original
# system is licensed, so all data comes from generated rigs)

def _translation(t) -> np.ndarray:
    return np.array([1.0, 0.0, 0.0, 0.0, 0.0, t[0] * 0.5, t[1] * 0.5, t[2] * 0.5])


def _smooth01(t: np.ndarray) -> np.ndarray:
    t = np.clip(t, 0.0, 1.0)
    return t * t * (3.0 - 2.0 * t)


def _capsule(p0, axis, length, r0, r1, h, vbase):
    """Tapered capsule (hemispherical caps r0/r1 joined by a frustum) around
    the segment p0 -> p0 + axis*length, in the layout of append_capsule
    (synth.cpp:365-422): a pole, rings, a pole; quads between rings and pole
    fans. Segments ~ 2 pi r / h (8..24), caps and body rings chosen for
    near-square quads. Returns (positions [n,3], height-along-axis [n], polys)."""
    a = np.asarray(axis, float)
    a = a / np.linalg.norm(a)
    ref = np.array([1.0, 0, 0]) if abs(a[0]) < 0.9 else np.array([0, 0, 1.0])
    b = np.cross(a, ref)
    b /= np.linalg.norm(b)
    c = np.cross(b, a)
    rmax = max(r0, r1)
    seg = int(min(24, max(8, round(2 * math.pi * rmax / h))))
    step = 2 * math.pi * rmax / seg
    caps = max(2, int(round(seg / 4)))
    body = max(1, int(round(length / step)))
    rings = []
    for i in range(1, caps + 1):
        ang = -math.pi / 2 + (math.pi / 2) * i / caps
        rings.append((r0 * math.sin(ang), r0 * math.cos(ang)))
    for j in range(1, body + 1):
        t = j / body
        rings.append((length * t, r0 + (r1 - r0) * t))
    for i in range(1, caps):
        ang = (math.pi / 2) * i / caps
        rings.append((length + r1 * math.sin(ang), r1 * math.cos(ang)))
    nr = len(rings)
    ang = 2 * math.pi * np.arange(seg) / seg
    pos = [p0 + a * (-r0)]
    hgt = [-r0]
    for (y, r) in rings:
        ring = p0[None, :] + b[None, :] * (r * np.cos(ang))[:, None] + a[None, :] * y + \
            c[None, :] * (r * np.sin(ang))[:, None]
        pos.extend(ring)
        hgt.extend([y] * seg)
    pos.append(p0 + a * (length + r1))
    hgt.append(length + r1)
    top = vbase + 1 + nr * seg

    def rv(i, s):
        return vbase + 1 + i * seg + (s % seg)

    polys = [[vbase, rv(0, s), rv(0, s + 1)] for s in range(seg)]
    for i in range(nr - 1):
        for s in range(seg):
            polys.append([rv(i, s), rv(i + 1, s), rv(i + 1, s + 1), rv(i, s + 1)])
    polys += [[top, rv(nr - 1, s + 1), rv(nr - 1, s)] for s in range(seg)]
    return np.asarray(pos), np.asarray(hgt), polys


# (name, parent, offset from parent origin, kind, axis, capsule dir, length, r0, r1)
_HUMANOID = [
    ("pelvis", -1, (0.0, 0.0, 0.0), PRISMATIC, (0, 0, 1), (0, -1, 0), 0.12, 0.140, 0.130),
    ("abdomen", 0, (0.0, -0.10, 0.0), HINGE, (1, 0, 0), (0, -1, 0), 0.12, 0.130, 0.135),
    ("chest", 1, (0.0, -0.12, 0.0), HINGE, (0, 0, 1), (0, -1, 0), 0.14, 0.145, 0.150),
    ("upper_chest", 2, (0.0, -0.14, 0.0), HINGE, (0, 1, 0), (0, -1, 0), 0.10, 0.150, 0.130),
    ("neck", 3, (0.0, -0.12, 0.0), HINGE, (1, 0, 0), (0, -1, 0), 0.06, 0.050, 0.050),
    ("head", 4, (0.0, -0.07, 0.0), HINGE, (0, 1, 0), (0, -1, 0), 0.15, 0.090, 0.080),
    ("l_clavicle", 3, (0.05, -0.06, 0.0), HINGE, (0, 1, 0), (1, 0, 0), 0.13, 0.055, 0.050),
    ("l_uparm", 6, (0.15, 0.0, 0.0), HINGE, (0, 0, 1), (1, 0.35, 0), 0.27, 0.050, 0.042),
    ("l_forearm", 7, None, HINGE, (0, 0, 1), (1, 0.35, 0), 0.24, 0.040, 0.032),
    ("l_hand", 8, None, HINGE, (1, 0, 0), (1, 0.35, 0), 0.11, 0.034, 0.028),
    ("r_clavicle", 3, (-0.05, -0.06, 0.0), HINGE, (0, 1, 0), (-1, 0, 0), 0.13, 0.055, 0.050),
    ("r_uparm", 10, (-0.15, 0.0, 0.0), HINGE, (0, 0, 1), (-1, 0.35, 0), 0.27, 0.050, 0.042),
    ("r_forearm", 11, None, HINGE, (0, 0, 1), (-1, 0.35, 0), 0.24, 0.040, 0.032),
    ("r_hand", 12, None, HINGE, (1, 0, 0), (-1, 0.35, 0), 0.11, 0.034, 0.028),
    ("l_thigh", 0, (0.09, 0.06, 0.0), HINGE, (1, 0, 0), (0, 1, 0), 0.40, 0.075, 0.055),
    ("l_shin", 14, (0.0, 0.40, 0.0), HINGE, (1, 0, 0), (0, 1, 0), 0.38, 0.052, 0.040),
    ("l_foot", 15, (0.0, 0.40, 0.0), HINGE, (0, 1, 0), (0, 0.15, -1), 0.14, 0.040, 0.034),
    ("r_thigh", 0, (-0.09, 0.06, 0.0), HINGE, (1, 0, 0), (0, 1, 0), 0.40, 0.075, 0.055),
    ("r_shin", 17, (0.0, 0.40, 0.0), HINGE, (1, 0, 0), (0, 1, 0), 0.38, 0.052, 0.040),
    ("r_foot", 18, (0.0, 0.40, 0.0), HINGE, (0, 1, 0), (0, 0.15, -1), 0.14, 0.040, 0.034),
]


def _humanoid_at(h: float, depth: float) -> ModelBundle:
    L = len(_HUMANOID)
    parent = np.array([b[1] for b in _HUMANOID], dtype=np.int32)
    origins, offsets = [], []
    for j, (name, par, off, kind, axis, d, length, r0, r1) in enumerate(_HUMANOID):
        if off is None:  # continue along the parent's capsule
            pb = _HUMANOID[par]
            pd = np.asarray(pb[5], float)
            off = tuple(pd / np.linalg.norm(pd) * pb[6])
        off = np.asarray(off, float)
        if par < 0:
            off = off + np.array([0.03, 0.0, depth])
            origins.append(off)
        else:
            origins.append(origins[par] + off)
        offsets.append(_translation(off))
    v0, hts, polys, wc, wl, ww = [], [], [], [], [], []
    nvert = 0
    for j, (name, par, off, kind, axis, d, length, r0, r1) in enumerate(_HUMANOID):
        d = np.asarray(d, float)
        d /= np.linalg.norm(d)
        start = origins[j] - d * (length * 0.5) if par < 0 else origins[j]
        pos, hgt, pl = _capsule(start, d, length, r0, r1, h, nvert)
        v0.append(pos)
        polys.extend(pl)
        nvert += pos.shape[0]
        # weights: self, parent, grandparent, blended near the link origin
        # (the scheme of make_biped_rig, synth.cpp:548-562, plus a third entry)
        n = pos.shape[0]
        wpar = 0.5 * (1.0 - _smooth01(hgt / 0.08)) if par >= 0 else np.zeros(n)
        gp = parent[par] if par >= 0 else -1
        wgp = 0.25 * wpar if gp >= 0 else np.zeros(n)
        links = np.full((n, 4), -1, dtype=np.int32)
        wts = np.zeros((n, 4))
        cnt = np.ones(n, dtype=np.int32)
        links[:, 0] = j
        wts[:, 0] = 1.0
        blend = wpar > 1e-9
        wself = 1.0 - wpar - wgp
        wts[blend, 0] = wself[blend]
        links[blend, 1] = par
        wts[blend, 1] = wpar[blend]
        cnt[blend] = 2
        if gp >= 0:
            links[blend, 2] = gp
            wts[blend, 2] = wgp[blend]
            cnt[blend] = 3
        wc.append(cnt)
        wl.append(links)
        ww.append(wts)
    axes = np.array([np.asarray(b[4], float) / np.linalg.norm(b[4]) for b in _HUMANOID])
    return ModelBundle(
        parent=parent, parent_offset=np.array(offsets), joint_kind=np.array([b[3] for b in _HUMANOID], np.int32),
        joint_axis=axes, theta_index=np.arange(L, dtype=np.int32), v0=np.concatenate(v0),
        weight_count=np.concatenate(wc), weight_link=np.concatenate(wl), weight=np.concatenate(ww),
        polys=polys, link_names=[b[0] for b in _HUMANOID], name="humanoid20")


def make_humanoid(target_vertices: int = 100_000, depth: float = 2.2, neighbors: int = 4,
                  levels: int | None = None, device: int | None = None) -> ModelBundle:
    """20-link humanoid (one prismatic root, hinges about x/y/z axes): a coarse
    capsule rig refined by `levels` Catmull-Clark subdivisions (the reference
    tracks subdivided templates, acceptance.cpp:543-548), with the coarse
    spacing solved so the result has ~target_vertices (within ~3%). Placed
    `depth` metres in front of the camera, head up in the image, 3 cm off the
    optical axis. Finalized, with k-NN neighbour sets. With a device the
    subdivision, finalize and neighbour search run on that GPU (same bits)."""
    if levels is None:
        levels = 1 if target_vertices < 20_000 else (2 if target_vertices <= 200_000 else 3)
    base_target = target_vertices / (4.0 ** levels)
    lo, hi = 1e-3, 0.5
    best = None
    for _ in range(60):
        mid = math.sqrt(lo * hi)
        n = _humanoid_at(mid, depth).vertex_count
        if best is None or abs(n - base_target) < abs(best[1] - base_target):
            best = (mid, n)
        if n > base_target:
            lo = mid
        else:
            hi = mid
    b = _humanoid_at(best[0], depth)
    if device is not None:
        return subdivide_on_device(b, levels, neighbors, device)
    b.finalize()
    return subdivide(b, levels, neighbors) if levels > 0 else b.with_neighbors(neighbors)


def humanoid_trajectory(L: int, frame: int, fps: float = 30.0, phase_offset: float = 0.0) -> np.ndarray:
    """Sinusoidal joint curves in the style of the reference's closed-loop
    biped test (acceptance.cpp:105-137): <= 0.35 rad on hinges and a 2 cm
    prismatic bob on the root."""
    t = frame / fps
    rng = np.random.default_rng(1234)
    amp = rng.uniform(0.08, 0.30, size=L)
    freq = rng.uniform(0.2, 0.5, size=L)
    ph = rng.uniform(0, 2 * math.pi, size=L) + phase_offset
    theta = amp * np.sin(2 * math.pi * freq * t + ph)
    theta[0] = 0.02 * math.sin(2 * math.pi * 0.3 * t + phase_offset)
    return theta


# ---------------------------------------------------------------------------
# Catmull-Clark subdivision (subdivide, skinmesh.cpp:249-511): positions, phi
# and skin weights follow the position scheme; weights are then truncated to
# the four largest entries (ties to the lower link) and renormalised. Sums are
# accumulated in the reference's order so results agree to the last bit.

def _cc_once(pos, phi, W, faces):
    nv = pos.shape[0]
    nf = len(faces)
    # edges in order of first appearance (face order, side order)
    edge_index = {}
    ea, eb, ef0, ef1, nfe = [], [], [], [], []
    face_edges = []
    for f, poly in enumerate(faces):
        fe = []
        n = len(poly)
        for s in range(n):
            a, b = poly[s], poly[(s + 1) % n]
            key = (a, b) if a < b else (b, a)
            e = edge_index.get(key)
            if e is None:
                e = len(ea)
                edge_index[key] = e
                ea.append(key[0])
                eb.append(key[1])
                ef0.append(f)
                ef1.append(-1)
                nfe.append(1)
            else:
                if nfe[e] >= 2:
                    raise ValueError(f"edge ({key[0]}, {key[1]}) has more than two incident faces")
                ef1[e] = f
                nfe[e] += 1
            fe.append(e)
        face_edges.append(fe)
    ne = len(ea)
    ea, eb, ef0, ef1, nfe = map(np.asarray, (ea, eb, ef0, ef1, nfe))
    sizes = np.fromiter((len(p) for p in faces), dtype=np.int64, count=nf)
    maxn = int(sizes.max()) if nf else 0
    pad = np.zeros((nf, maxn), dtype=np.int64)
    for f, p in enumerate(faces):
        pad[f, :len(p)] = p
    face_base, edge_base = nv + ne, nv

    # face points: sum of pos * (1/n) in vertex order
    c = 1.0 / sizes.astype(np.float64)
    fp = np.zeros((nf, 3))
    fph = np.zeros((nf, 3))
    fw = np.zeros((nf, W.shape[1]))
    for k in range(maxn):
        m = k < sizes
        idx = pad[m, k]
        fp[m] += pos[idx] * c[m, None]
        fph[m] += phi[idx] * c[m, None]
        fw[m] += W[idx] * c[m, None]

    # edge points
    two = nfe == 2
    epos = np.empty((ne, 3))
    ephi = np.empty((ne, 3))
    ew = np.empty((ne, W.shape[1]))
    f0, f1 = ef0, np.where(two, ef1, 0)
    epos[two] = (((pos[ea[two]] + pos[eb[two]]) + fp[f0[two]]) + fp[f1[two]]) * 0.25
    ephi[two] = (((phi[ea[two]] + phi[eb[two]]) + fph[f0[two]]) + fph[f1[two]]) * 0.25
    ew[two] = (((0.25 * W[ea[two]] + 0.25 * W[eb[two]]) + 0.25 * fw[f0[two]]) + 0.25 * fw[f1[two]])
    bd = ~two
    epos[bd] = (pos[ea[bd]] + pos[eb[bd]]) * 0.5
    ephi[bd] = (phi[ea[bd]] + phi[eb[bd]]) * 0.5
    ew[bd] = 0.5 * W[ea[bd]] + 0.5 * W[eb[bd]]

    # vertex points
    vdeg = np.bincount(np.concatenate([ea, eb]), minlength=nv)
    # (vertex, edge) pairs in edge order, (vertex, face) pairs in face order
    pv_e = np.empty(2 * ne, dtype=np.int64)
    pv_e[0::2], pv_e[1::2] = ea, eb
    pe = np.repeat(np.arange(ne), 2)
    order = np.argsort(pv_e, kind="stable")  # per vertex: ascending edge index
    ve_v, ve_e = pv_e[order], pe[order]
    fl = pad[sizes[:, None] > np.arange(maxn)[None, :]]
    ff = np.repeat(np.arange(nf), sizes)
    order = np.argsort(fl, kind="stable")
    vf_v, vf_f = fl[order], ff[order]
    vnf = np.bincount(vf_v, minlength=nv)
    boundary = np.zeros(nv, bool)
    boundary[ve_v[nfe[ve_e] < 2]] = True
    npos, nphi, nw = pos.copy(), phi.copy(), W.copy()
    inter = (vdeg > 0) & ~boundary
    # interior rule (F + 2R + (n-3)P)/n
    favg = np.zeros((nv, 3))
    fphi = np.zeros((nv, 3))
    np.add.at(favg, vf_v, fp[vf_f])
    np.add.at(fphi, vf_v, fph[vf_f])
    fwv = np.zeros_like(W)
    cf = 1.0 / np.maximum(vnf, 1).astype(np.float64)
    np.add.at(fwv, vf_v, fw[vf_f] * cf[vf_v][:, None])
    favg /= np.maximum(vnf, 1)[:, None]
    fphi /= np.maximum(vnf, 1)[:, None]
    rsum = np.zeros((nv, 3))
    rphi = np.zeros((nv, 3))
    np.add.at(rsum, ve_v, (pos[ea[ve_e]] + pos[eb[ve_e]]) * 0.5)
    np.add.at(rphi, ve_v, (phi[ea[ve_e]] + phi[eb[ve_e]]) * 0.5)
    nn = np.maximum(vdeg, 1).astype(np.float64)
    rsum /= nn[:, None]
    rphi /= nn[:, None]
    rw = np.zeros_like(W)
    seq_v = np.repeat(ve_v, 2)
    seq_src = np.empty(2 * len(ve_e), dtype=np.int64)
    seq_src[0::2], seq_src[1::2] = ea[ve_e], eb[ve_e]
    np.add.at(rw, seq_v, W[seq_src] * (0.5 / nn[seq_v])[:, None])
    i = np.where(inter)[0]
    n_i = nn[i][:, None]
    npos[i] = (favg[i] + 2.0 * rsum[i] + (n_i - 3.0) * pos[i]) / n_i
    nphi[i] = (fphi[i] + 2.0 * rphi[i] + (n_i - 3.0) * phi[i]) / n_i
    nw[i] = ((fwv[i] * (1.0 / n_i)) + rw[i] * (2.0 / n_i)) + W[i] * ((n_i - 3.0) / n_i)
    # boundary (crease) rule (m1 + 6P + m2)/8, rarely used by our rigs
    for v in np.where(boundary)[0]:
        p = np.zeros(3)
        ph = np.zeros(3)
        wm = np.zeros(W.shape[1])
        for e in ve_e[ve_v == v]:
            if nfe[e] < 2:
                other = eb[e] if ea[e] == v else ea[e]
                p += (pos[v] + pos[other]) * 0.5
                ph += (phi[v] + phi[other]) * 0.5
                wm += (0.5 / 8.0) * W[v]
                wm += (0.5 / 8.0) * W[other]
        npos[v] = p / 8.0 + pos[v] * (6.0 / 8.0)
        nphi[v] = ph / 8.0 + phi[v] * (6.0 / 8.0)
        nw[v] = wm + (6.0 / 8.0) * W[v]

    out_pos = np.concatenate([npos, epos, fp])
    out_phi = np.concatenate([nphi, ephi, fph])
    out_w = np.concatenate([nw, ew, fw])
    new_faces = []
    for f, poly in enumerate(faces):
        n = len(poly)
        fe = face_edges[f]
        for s in range(n):
            new_faces.append([poly[s], edge_base + fe[s], face_base + f, edge_base + fe[(s + n - 1) % n]])
    return out_pos, out_phi, out_w, new_faces


def _truncate_weights(W: np.ndarray):
    """truncate_weights (skinmesh.cpp:274-289): four largest (ties to the lower
    link), summed in that order, re-sorted by link, zeros dropped, renormalised."""
    nv, L = W.shape
    order = np.argsort(-W, axis=1, kind="stable")[:, :4]
    top = np.take_along_axis(W, order, axis=1)
    s = np.zeros(nv)
    for k in range(min(4, L)):
        s = s + top[:, k]
    by_link = np.sort(order, axis=1)
    wl = np.take_along_axis(W, by_link, axis=1)
    keep = wl > 0.0
    cnt = keep.sum(axis=1).astype(np.int32)
    links = np.full((nv, 4), -1, np.int32)
    wts = np.zeros((nv, 4))
    rank = np.cumsum(keep, axis=1) - 1
    rows = np.repeat(np.arange(nv), keep.sum(axis=1))
    links[rows, rank[keep]] = by_link[keep]
    wts[rows, rank[keep]] = (wl / s[:, None])[keep]
    if L < 4:
        links, wts = links[:, :4], wts[:, :4]
    return cnt, links, wts


def _mesh_check(rc: int) -> None:
    if rc != _lib.WT_OK:
        msg = (_lib.lib().wt_gpu_mesh_last_error() or b"").decode(errors="replace")
        cls = {_lib.WT_EINVAL: _lib.ValidationError, _lib.WT_ELENGTH: _lib.LengthMismatch}.get(rc, _lib.WarptrackError)
        raise cls(rc, msg)


def subdivide_on_device(b: ModelBundle, iterations: int, neighbors: int = 4, device: int = 0) -> ModelBundle:
    """subdivide + finalize + build_neighbors on the GPU (wt_gpu_mesh_subdivide,
    wt_model.cu): bitwise the reference's (skinmesh.cpp:13-58,145-511) and the
    host path below. iterations == 0 only finalizes and builds neighbours."""
    import ctypes as C
    L = _lib.lib()
    V = b.vertex_count
    sizes = [len(p) for p in b.polys]
    poff = np.zeros(len(sizes) + 1, np.int32)
    poff[1:] = np.cumsum(sizes)
    pitems = np.ascontiguousarray(np.concatenate([np.asarray(p, np.int32) for p in b.polys])
                                  if b.polys else np.zeros(0, np.int32), np.int32)
    v0 = np.ascontiguousarray(b.v0, np.float64)
    phi = None if b.phi is None or b.phi.shape != b.v0.shape else np.ascontiguousarray(b.phi, np.float64)
    wc = np.ascontiguousarray(b.weight_count, np.int32)
    wl = np.ascontiguousarray(b.weight_link, np.int32)
    ww = np.ascontiguousarray(b.weight, np.float64)
    h = C.c_void_p()
    _mesh_check(L.wt_gpu_mesh_subdivide(device, V, b.link_count, _lib.ptr(v0), _lib.ptr(phi), _lib.ptr(wc),
                                        _lib.ptr(wl), _lib.ptr(ww), len(sizes), _lib.ptr(poff), _lib.ptr(pitems),
                                        iterations, neighbors, C.byref(h)))
    try:
        n = [C.c_int32() for _ in range(5)]
        _mesh_check(L.wt_gpu_mesh_sizes(h, *[C.byref(x) for x in n]))
        nv, nf, ni, nt, k = (x.value for x in n)
        o = dict(v0=np.zeros((nv, 3)), phi=np.zeros((nv, 3)), weight_count=np.zeros(nv, np.int32),
                 weight_link=np.zeros((nv, 4), np.int32), weight=np.zeros((nv, 4)),
                 poff=np.zeros(nf + 1, np.int32), pitems=np.zeros(ni, np.int32), triangles=np.zeros((nt, 3), np.int32),
                 vtri_offsets=np.zeros(nv + 1, np.int32), vtri_items=np.zeros(3 * nt, np.int32),
                 nbr=np.zeros((nv, k), np.int32))
        _mesh_check(L.wt_gpu_mesh_export(h, *[_lib.ptr(o[x]) for x in (
            "v0", "phi", "weight_count", "weight_link", "weight", "poff", "pitems", "triangles", "vtri_offsets",
            "vtri_items", "nbr")]))
    finally:
        L.wt_gpu_mesh_free(h)
    polys = np.split(o["pitems"], o["poff"][1:-1]) if nf else []
    out = replace(b, v0=o["v0"], phi=o["phi"], weight_count=o["weight_count"], weight_link=o["weight_link"],
                  weight=o["weight"], polys=[p.tolist() for p in polys], triangles=o["triangles"],
                  vtri_offsets=o["vtri_offsets"], vtri_items=o["vtri_items"])
    if neighbors > 0:
        out.nbr_offsets = np.arange(nv + 1, dtype=np.int32) * k
        out.nbr_items = o["nbr"].reshape(-1)
    else:
        out.nbr_offsets, out.nbr_items = None, None
    return out


def build_neighbors_on_device(v0: np.ndarray, k: int, device: int = 0) -> tuple[np.ndarray, np.ndarray]:
    """build_neighbors (skinmesh.cpp:196-247) on the GPU (wt_gpu_build_neighbors):
    CSR (offsets, items) as build_neighbors below."""
    nv = v0.shape[0]
    want = max(0, min(k, nv - 1))
    out = np.zeros((nv, want), np.int32)
    _mesh_check(_lib.lib().wt_gpu_build_neighbors(device, nv, _lib.ptr(np.ascontiguousarray(v0, np.float64)), k,
                                                  _lib.ptr(out)))
    return np.arange(nv + 1, dtype=np.int32) * want, out.reshape(-1)


def subdivide(b: ModelBundle, iterations: int, neighbors: int = 4) -> ModelBundle:
    """subdivide (skinmesh.cpp:490-511) + build_neighbors(v0, 4), as the
    reference's Python binding subdivide_model does (bindings.cpp:154-161).
    Host restatement (numpy); subdivide_on_device is the GPU path."""
    L = b.link_count
    W = np.zeros((b.vertex_count, L))
    for s in range(4):
        m = s < b.weight_count
        np.add.at(W, (np.where(m)[0], b.weight_link[m, s]), b.weight[m, s] * 1.0)
    pos = b.v0.copy()
    phi = b.phi.copy() if b.phi is not None and b.phi.shape == b.v0.shape else np.zeros_like(b.v0)
    faces = [list(p) for p in b.polys]
    for _ in range(iterations):
        pos, phi, W, faces = _cc_once(pos, phi, W, faces)
    cnt, links, wts = _truncate_weights(W)
    out = replace(b, v0=pos, phi=phi, weight_count=cnt, weight_link=links, weight=wts, polys=faces,
                  triangles=None, vtri_offsets=None, vtri_items=None, nbr_offsets=None, nbr_items=None)
    out.finalize()
    out.with_neighbors(neighbors)
    return out
