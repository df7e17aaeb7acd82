"""Shared fixtures for the parity tests: seeded models, frames and configs."""
from __future__ import annotations

import functools

import numpy as np

from paper_1711_07999_b200 import _lib as W
from paper_1711_07999_b200.model import humanoid_trajectory, make_humanoid
from paper_1711_07999_b200.tracker import (AssocConfig, Intrinsics, KinSolverConfig, ShapeSolverConfig,
                                           TrackConfig)


@functools.lru_cache(maxsize=None)
def humanoid(n: int):
    return make_humanoid(n)


def intr640() -> Intrinsics:
    return Intrinsics.scaled(640, 480)


def intr320() -> Intrinsics:
    return Intrinsics.scaled(320, 240)


def theta_at(b, frame: int, phase: float = 0.0) -> np.ndarray:
    return humanoid_trajectory(b.link_count, frame, phase_offset=phase)


def cfg(mode="dynamic", kin_its=5, shape_its=2, **kw) -> TrackConfig:
    c = TrackConfig(mode=mode, kin=KinSolverConfig(iterations=kin_its), shape=ShapeSolverConfig(iterations=shape_its),
                    assoc=AssocConfig())
    for k, v in kw.items():
        setattr(c, k, v)
    return c


def cmp_winners(a: np.ndarray, b: np.ndarray) -> float:
    """Fraction of pixels whose winning vertex agrees."""
    return float(np.mean(a == b))
