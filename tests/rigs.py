"""Small rigs and scenes of the reference's unit tests, restated as numpy
model bundles (the reference builds them inline in its doctest suites):
  slider plates      test_kinopt.cpp:88-112, 170-206, 271-358
  random chain rigs  test_kinopt.cpp:29-74 (numpy RNG, same distributions)
  loose vertices     test_association.cpp:24-47
  dents / curves     synth.cpp:16-64 (PhiAnimation / JointCurve)
"""
from __future__ import annotations

import numpy as np

from paper_1711_07999_b200 import _lib as W
from paper_1711_07999_b200.model import ModelBundle, build_neighbors
from paper_1711_07999_b200.tracker import Intrinsics

IDENTITY_DQ = np.array([1.0, 0, 0, 0, 0, 0, 0, 0])


def translation(x, y, z) -> np.ndarray:
    return np.array([1.0, 0, 0, 0, 0, 0.5 * x, 0.5 * y, 0.5 * z])


def no_neighbors(b: ModelBundle) -> ModelBundle:
    b.nbr_offsets = np.zeros(b.vertex_count + 1, np.int32)
    b.nbr_items = np.zeros(0, np.int32)
    return b


def slider(v0, polys, neighbors: int = 0) -> ModelBundle:
    """One prismatic link along +z, every vertex rigidly bound to it."""
    v0 = np.asarray(v0, float)
    V = v0.shape[0]
    b = ModelBundle(parent=np.array([-1], np.int32), parent_offset=IDENTITY_DQ[None].copy(),
                    joint_kind=np.array([W.JOINT_PRISMATIC], np.int32), joint_axis=np.array([[0.0, 0, 1]]),
                    theta_index=np.array([0], np.int32), v0=v0, weight_count=np.ones(V, np.int32),
                    weight_link=np.tile(np.array([0, -1, -1, -1], np.int32), (V, 1)),
                    weight=np.tile([1.0, 0, 0, 0], (V, 1)), polys=[list(p) for p in polys]).finalize()
    return b.with_neighbors(neighbors) if neighbors else no_neighbors(b)


def slider_triangle() -> ModelBundle:
    """test_kinopt.cpp:91-101: three vertices at z = 1, normal (0,0,1)."""
    return slider([[0, 0, 1], [0.1, 0, 1], [0, 0.1, 1]], [[0, 1, 2]])


def slider_grid() -> ModelBundle:
    """test_kinopt.cpp:275-289: 4x4 plate at z = 1."""
    v = [[0.05 * x, 0.05 * y, 1.0] for y in range(4) for x in range(4)]
    polys = [[y * 4 + x, y * 4 + x + 1, y * 4 + x + 5, y * 4 + x + 4] for y in range(3) for x in range(3)]
    return slider(v, polys)


def camera_plate(n: int = 24, z: float = 1.2) -> ModelBundle:
    """test_kinopt.cpp:324-340: n x n plate facing the camera, kNN k = 4."""
    v = [[-0.3 + 0.6 * x / (n - 1), -0.3 + 0.6 * y / (n - 1), z] for y in range(n) for x in range(n)]
    polys = [[y * n + x, (y + 1) * n + x, (y + 1) * n + x + 1, y * n + x + 1]
             for y in range(n - 1) for x in range(n - 1)]
    return slider(v, polys, neighbors=4)


def random_rig(rng: np.random.Generator, links: int, vertices: int):
    """make_random_rig (test_kinopt.cpp:29-74): a chain with random offsets and
    axes (1 in 4 prismatic), 1-3 distinct weighted links per vertex, triangles
    over consecutive vertices, kNN k = 2, a random pose in [-0.4, 0.4]."""
    uni = lambda *s: rng.uniform(-1.0, 1.0, *s)  # noqa: E731
    off = np.zeros((links, 8))
    axis = np.zeros((links, 3))
    kind = np.zeros(links, np.int32)
    for j in range(links):
        off[j] = translation(0.3 + 0.1 * uni(), 0.1 * uni(), 0.1 * uni())
        ax = uni(3)
        while np.linalg.norm(ax) < 1e-3:
            ax = uni(3)
        axis[j] = ax / np.linalg.norm(ax)
        kind[j] = W.JOINT_PRISMATIC if rng.integers(4) == 0 else W.JOINT_HINGE
    v0 = np.stack([uni(vertices) * 2, uni(vertices), uni(vertices) + 1.5], 1)
    wc = np.zeros(vertices, np.int32)
    wl = np.full((vertices, 4), -1, np.int32)
    w = np.zeros((vertices, 4))
    for i in range(vertices):
        nw = 1 + int(rng.integers(3))
        used = rng.choice(links, size=nw, replace=False)
        vals = 0.2 + 0.8 * np.abs(uni(nw))
        wc[i], wl[i, :nw], w[i, :nw] = nw, used, vals / vals.sum()
    polys = [[i, i + 1, i + 2] for i in range(0, vertices - 2, 3)]
    b = ModelBundle(parent=np.arange(-1, links - 1, dtype=np.int32), parent_offset=off, joint_kind=kind,
                    joint_axis=axis, theta_index=np.arange(links, dtype=np.int32), v0=v0, weight_count=wc,
                    weight_link=wl, weight=w, polys=polys).finalize().with_neighbors(2)
    return b, 0.4 * uni(links)


def arm_curves(L: int, frame: int, fps: float = 30.0) -> np.ndarray:
    """The two sine curves of test_kinopt.cpp:389-401 (JointCurve::eval,
    synth.cpp:16-38)."""
    t = frame / fps
    th = np.zeros(L)
    th[1] = 0.3 * np.sin(2.0 * np.pi * 0.9 * t)
    th[2] = 0.25 * np.sin(2.0 * np.pi * 1.3 * t)
    return th


def dent_phi(v0: np.ndarray, direction=(0.0, 0.0, -1.0), amplitude=0.02, width=0.5) -> np.ndarray:
    """PhiAnimation::eval with one dent and no ramp (synth.cpp:41-64)."""
    c = v0.mean(axis=0)
    d = v0 - c
    ln = np.linalg.norm(d, axis=1)
    dirs = d / np.maximum(ln, 1e-300)[:, None]
    u = np.asarray(direction, float) / np.linalg.norm(direction)
    ang = np.arccos(np.clip(dirs @ u, -1.0, 1.0))
    depth = amplitude * np.exp(-(ang * ang) / (width * width))
    phi = -dirs * depth[:, None]
    phi[ln < 1e-9] = 0.0
    return phi


def kinect() -> Intrinsics:
    """Intrinsics defaults (association.hpp:11-15)."""
    return Intrinsics()


def small_intr() -> Intrinsics:
    """small_intr (test_association.cpp:13-21)."""
    return Intrinsics(500.0, 500.0, 256.0, 212.0, 512, 424)


def project(intr: Intrinsics, p):
    """project (association.cpp:29-37): lround is half away from zero."""
    x, y, z = p
    if not z > 0:
        return None
    fu = intr.fx * x / z + intr.cx
    fv = intr.fy * y / z + intr.cy
    u = int(np.sign(fu) * np.floor(abs(fu) + 0.5))
    v = int(np.sign(fv) * np.floor(abs(fv) + 0.5))
    if u < 0 or v < 0 or u >= intr.width or v >= intr.height:
        return None
    return u, v


def frame_from_points(intr: Intrinsics, pts):
    """frame_from_points (test_association.cpp:32-47): one point per pixel."""
    P = intr.width * intr.height
    points = np.zeros((P, 3))
    valid = np.zeros(P, np.uint8)
    for p in pts:
        pc = project(intr, p)
        if pc is None:
            continue
        i = pc[1] * intr.width + pc[0]
        if valid[i]:
            continue
        points[i], valid[i] = p, 1
    return points, valid


def loose(verts, normals=None):
    """loose_vertices (test_association.cpp:24-30): camera-facing normals."""
    v = np.asarray(verts, float).reshape(-1, 3)
    n = np.tile([0.0, 0.0, -1.0], (v.shape[0], 1)) if normals is None else np.asarray(normals, float)
    return v, n, np.ones(v.shape[0], np.uint8)


def empty_frame(intr: Intrinsics):
    P = intr.width * intr.height
    return np.zeros((P, 3)), np.zeros(P, np.uint8)
