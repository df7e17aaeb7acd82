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
    the segment p0 -> p0 + axis*length, tessellated at spacing ~h. Returns
    (positions [n,3], height-along-axis [n], polys)."""
    a = np.asarray(axis, float)
    a = a / np.linalg.norm(a)
    ref = np.array([1.0, 0, 0]) if abs(a[0]) < 0.9 else np.array([0, 0, 1.0])
    b = np.cross(a, ref)
    b /= np.linalg.norm(b)
    c = np.cross(b, a)
    seg = max(8, int(round(2 * math.pi * max(r0, r1) / h)))
    caps = max(2, int(round(0.5 * math.pi * max(r0, r1) / h)))
    body = max(1, int(round(length / h)))
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
            off = off + np.array([0.0, 0.0, depth])
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


def make_humanoid(target_vertices: int = 100_000, depth: float = 2.2, neighbors: int = 4) -> ModelBundle:
    """20-link humanoid (one prismatic root, hinges on x/y/z axes) over tapered
    capsules with near-uniform vertex spacing solved to hit target_vertices
    (within ~2%). Placed `depth` metres in front of the camera, head up in
    the image. Finalized, with k-NN neighbour sets."""
    lo, hi = 1e-3, 0.2
    for _ in range(40):
        mid = math.sqrt(lo * hi)
        n = _humanoid_at(mid, depth).vertex_count
        if n > target_vertices:
            lo = mid
        else:
            hi = mid
        if abs(n - target_vertices) <= 0.01 * target_vertices:
            break
    b = _humanoid_at(mid, depth)
    b.finalize()
    b.with_neighbors(neighbors)
    return b


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
