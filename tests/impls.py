"""One interface over the two implementations the KAT suite runs against:
  "oracle"  the C restatement (oracle/wt_oracle.c) on the CPU -- the checker;
  "gpu"     the product: libwt_gpu.so through its C-ABI on cuda:0.
The test bodies are written once, in the style of the reference's own unit
tests, and each runs on both (the "gpu" arm carries @pytest.mark.gpu)."""
from __future__ import annotations

import numpy as np
import pytest

from oracle import c_oracle
from paper_1711_07999_b200 import _lib as W
from paper_1711_07999_b200 import tracker as T
from paper_1711_07999_b200.model import ModelBundle


class OracleTrackerAdapter:
    def __init__(self, bundle: ModelBundle, intr: T.Intrinsics, theta=None):
        self.bundle, self.intr = bundle, intr
        self.t = c_oracle.OracleTracker(bundle, intr.c(), theta)

    def set_state(self, theta=None, phi=None, frame_index=0):
        th = self.get_state()[0] if theta is None else theta
        self.t.set_state(th, phi, frame_index)

    def get_state(self):
        return self.t.get_state()

    def load_depth(self, depth, scale=1.0):
        self.t.load_depth(depth, scale)

    def load_cloud(self, points, valid):
        self.t.load_cloud(points, valid)

    def skin(self, theta, phi=None):
        return self.t.skin(theta, phi)

    def optimize_pose(self, kin: T.KinSolverConfig, assoc: T.AssocConfig = T.AssocConfig()):
        return self.t.optimize_pose(kin.c(), assoc.c())

    def optimize_shape(self, shape: T.ShapeSolverConfig, assoc: T.AssocConfig = T.AssocConfig(), stats=True):
        return self.t.optimize_shape(shape.c(), assoc.c(), stats)

    def normal_system(self, theta, kin: T.KinSolverConfig, count, residual):
        return self.t.normal_system(theta, kin.c(), count, residual)

    def track_frame(self, cfg: T.TrackConfig):
        st = self.t.track_loaded(cfg.c())
        return T.FrameStats(st.frame, T._kin_list(st.kin, st.n_kin), T._shape_list(st.shape, st.n_shape))

    def close(self):
        pass


class GpuTrackerAdapter(T.Tracker):
    pass


class OracleImpl:
    name = "oracle"

    def tracker(self, bundle, intr, theta=None):
        return OracleTrackerAdapter(bundle, intr, theta)

    def associate(self, intr: T.Intrinsics, v, n, valid, points, pvalid, window=5, cutoff=0.10):
        return c_oracle.associate(intr.c(), v, n, valid, points, pvalid, window, cutoff)

    def solve_step(self, jtj, jtr, cfg: T.KinSolverConfig):
        x, rc = c_oracle.solve_step(jtj, jtr, cfg.lambda_k, cfg.diag_floor)
        if rc != 0:
            raise W.NotPositiveDefinite(W.WT_ENOTPD, "normal system not positive definite")
        return x

    def solve_vertices(self, g, r, phi, nd, ncount, cfg: T.ShapeSolverConfig):
        g = np.asarray(g, float).reshape(-1, 3)
        out = [c_oracle.solve_vertex(g[i], float(np.ravel(r)[i]), np.asarray(phi, float).reshape(-1, 3)[i],
                                     np.asarray(nd, float).reshape(-1, 3)[i], int(np.ravel(ncount)[i]), cfg.c())
               for i in range(g.shape[0])]
        return np.array([d for d, _ in out]).reshape(-1, 3), np.array([s for _, s in out], bool)


class GpuImpl:
    name = "gpu"

    def tracker(self, bundle, intr, theta=None):
        return GpuTrackerAdapter(bundle, intr, theta)

    def associate(self, intr, v, n, valid, points, pvalid, window=5, cutoff=0.10):
        return T.associate_posed(intr, v, n, valid, points, pvalid, window, cutoff)

    def solve_step(self, jtj, jtr, cfg):
        return T.solve_step(jtj, jtr, cfg)

    def solve_vertices(self, g, r, phi, nd, ncount, cfg):
        return T.solve_vertices(g, r, phi, nd, ncount, cfg)


IMPLS = [pytest.param(OracleImpl(), id="oracle"), pytest.param(GpuImpl(), id="gpu", marks=pytest.mark.gpu)]
