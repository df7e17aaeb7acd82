"""Depth-frame ingest formats on the boundary.

.wts sequence (seqio.cpp:22,439-535): 8-byte magic "WTRKSEQ\\0", u32 version,
u32 width, u32 height, f64 fx, fy, cx, cy, u32 frame_count, f64 depth_scale
(64-byte header), then row-major little-endian float32 frames, 0 = invalid.
Ground-truth / estimate CSV (seqio.cpp:537-602): frame, theta_k...,
<joint>_x/_y/_z/_vis. depth_to_cloud is done on the GPU (k_ingest); the
numpy version here exists for tooling only.
"""
from __future__ import annotations

import struct
from dataclasses import dataclass
from pathlib import Path

import numpy as np

from ._lib import WT_EINVAL, WT_ELENGTH, LengthMismatch, ValidationError
from .tracker import Intrinsics

MAGIC = b"WTRKSEQ\x00"
_HDR = struct.Struct("<8sIII4dId")
assert _HDR.size == 64


@dataclass
class SequenceHeader:
    width: int
    height: int
    fx: float
    fy: float
    cx: float
    cy: float
    frame_count: int
    depth_scale: float = 1.0
    version: int = 1

    def intrinsics(self) -> Intrinsics:
        return Intrinsics(self.fx, self.fy, self.cx, self.cy, self.width, self.height)


class SequenceReader:
    """SequenceReader (seqio.cpp:439-491); frames decode lazily via memmap."""

    def __init__(self, path):
        self.path = Path(path)
        raw = self.path.read_bytes()[:64] if self.path.exists() else b""
        if len(raw) < 8 or raw[:8] != MAGIC:
            raise ValidationError(WT_EINVAL, f"sequence {self.path}: bad magic")
        if len(raw) < 64:
            raise ValidationError(WT_EINVAL, f"sequence {self.path}: truncated header")
        magic, ver, w, h, fx, fy, cx, cy, n, scale = _HDR.unpack(raw)
        if ver != 1:
            raise ValidationError(WT_EINVAL, f"sequence {self.path}: unsupported version {ver}")
        if w == 0 or h == 0:
            raise ValidationError(WT_EINVAL, f"sequence {self.path}: empty grid")
        self.header = SequenceHeader(w, h, fx, fy, cx, cy, n, scale, ver)
        size = self.path.stat().st_size - 64
        if size < w * h * 4 * n:
            raise ValidationError(WT_EINVAL, f"sequence {self.path}: frame {size // (w * h * 4)} of {n} "
                                  "is incomplete")
        self._mm = np.memmap(self.path, dtype="<f4", mode="r", offset=64, shape=(n, h, w))

    def frame_count(self) -> int:
        return self.header.frame_count

    def read_depth(self, frame: int) -> np.ndarray:
        if frame < 0 or frame >= self.header.frame_count:
            raise ValidationError(WT_EINVAL, f"sequence {self.path}: frame {frame} out of range")
        return np.array(self._mm[frame], dtype=np.float32)

    def frames(self) -> np.ndarray:
        """All frames [F,H,W] float32 (one read; the GPU driver stages them)."""
        return np.array(self._mm, dtype=np.float32)


class SequenceWriter:
    """SequenceWriter (seqio.cpp:493-535)."""

    def __init__(self, path, header: SequenceHeader):
        self.path = Path(path)
        self.header = header
        self._f = open(self.path, "wb")
        self._f.write(_HDR.pack(MAGIC, 1, header.width, header.height, header.fx, header.fy, header.cx,
                                header.cy, header.frame_count, header.depth_scale))
        self.written = 0

    def write_depth(self, depth) -> None:
        d = np.ascontiguousarray(depth, dtype="<f4").reshape(-1)
        if d.size != self.header.width * self.header.height:
            raise LengthMismatch(WT_ELENGTH, "depth frame size differs from header grid")
        self._f.write(d.tobytes())
        self.written += 1

    def close(self) -> None:
        if self._f.closed:
            return
        self._f.close()
        if self.written != self.header.frame_count:
            raise ValidationError(WT_EINVAL, f"sequence {self.path}: wrote {self.written} frames, header "
                                  f"declares {self.header.frame_count}")


def depth_to_cloud(intr: Intrinsics, depth, scale: float = 1.0):
    """depth_to_cloud (seqio.cpp:419-437) in numpy: (points [P,3], valid [P])."""
    d = np.asarray(depth, dtype=np.float32).reshape(intr.height, intr.width)
    valid = (d > 0) & np.isfinite(d)
    z = np.where(valid, d.astype(np.float64) * scale, 0.0)
    u = np.arange(intr.width, dtype=np.float64)[None, :]
    v = np.arange(intr.height, dtype=np.float64)[:, None]
    x = np.where(valid, (u - intr.cx) / intr.fx * z, 0.0)
    y = np.where(valid, (v - intr.cy) / intr.fy * z, 0.0)
    pts = np.stack([x, y, z], axis=-1).reshape(-1, 3)
    return pts, valid.reshape(-1).astype(np.uint8)


def format_double(x: float) -> str:
    """Shortest round-trip decimal (seqio.cpp:14-18)."""
    return repr(float(x))


def save_ground_truth(path, joint_names, theta, joints, visible) -> None:
    """save_ground_truth (seqio.cpp:537-561)."""
    theta = np.asarray(theta)
    nt = theta.shape[1] if theta.size else 0
    cols = ["frame"] + [f"theta_{k}" for k in range(nt)]
    for n in joint_names:
        cols += [f"{n}_x", f"{n}_y", f"{n}_z", f"{n}_vis"]
    lines = [",".join(cols)]
    for f in range(theta.shape[0]):
        row = [str(f)] + [format_double(t) for t in theta[f]]
        for j in range(len(joint_names)):
            row += [format_double(c) for c in joints[f][j]] + [str(int(visible[f][j]))]
        lines.append(",".join(row))
    Path(path).write_text("\n".join(lines) + "\n")


def load_ground_truth(path) -> dict:
    """load_ground_truth (seqio.cpp:563-602) -> dict of arrays."""
    text = Path(path).read_text().splitlines()
    header = text[0].split(",")
    if header[0] != "frame":
        raise ValidationError(WT_EINVAL, f"ground truth {path}: first column must be 'frame'")
    nt = sum(1 for c in header[1:] if c.startswith("theta_"))
    names = [c[:-2] for c in header[1 + nt::4]]
    theta, joints, vis = [], [], []
    for line in text[1:]:
        if not line:
            continue
        tok = line.split(",")
        if len(tok) != len(header):
            raise ValidationError(WT_EINVAL, f"ground truth {path}: bad row")
        theta.append([float(t) for t in tok[1:1 + nt]])
        j = np.array([float(t) for t in tok[1 + nt:]]).reshape(-1, 4)
        joints.append(j[:, :3])
        vis.append(j[:, 3].astype(np.uint8))
    return dict(joint_names=names, theta=np.array(theta), joints=np.array(joints), visible=np.array(vis))
