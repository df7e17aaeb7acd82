"""Small tracking run for compute-sanitizer (memcheck / racecheck / synccheck /
initcheck): a 7k-vertex humanoid at 320x240 through every entry point --
track_frame from pageable and from page-locked host frames (the overlapped
upload graph), the stage hooks, the reconstruction error, the sequence driver,
and a 16-sequence batch (the narrow 3x3-core search, the multi-vertex skin /
normals, the batch pose and shape grids).

    compute-sanitizer --tool memcheck python tools/sanitize_run.py
"""
import ctypes as C
import sys

sys.path.insert(0, ".")
import numpy as np

from paper_1711_07999_b200 import _lib as W
from paper_1711_07999_b200.model import humanoid_trajectory, make_humanoid
from paper_1711_07999_b200.tracker import (AssocConfig, BatchTracker, Intrinsics, KinSolverConfig,
                                           ShapeSolverConfig, TrackConfig, Tracker)

b = make_humanoid(7000)
intr = Intrinsics.scaled(320, 240)
cfg = TrackConfig(mode="dynamic", kin=KinSolverConfig(iterations=3), shape=ShapeSolverConfig(iterations=2),
                  assoc=AssocConfig())
trk = Tracker(b, intr, humanoid_trajectory(b.link_count, 0))
frames = []
for f in (1, 2, 3):
    d, _ = trk.render_depth(humanoid_trajectory(b.link_count, f), frame=f)
    frames.append(d)
trk.track_frame(cfg, depth=frames[0])
# page-locked host frame: the upload is forked inside the frame graph
P = intr.width * intr.height
p = C.c_void_p()
W.check(W.lib().wt_gpu_host_alloc(4 * P, C.byref(p)))
pinned = np.ctypeslib.as_array(C.cast(p, C.POINTER(C.c_float)), shape=(P,))
pinned[:] = frames[1].reshape(-1)
st = trk._stats()
W.check(W.lib().wt_gpu_track_frame(trk._ctx, p, 1.0, C.byref(cfg.c()), C.byref(st)), trk._ctx)
trk.skin(humanoid_trajectory(b.link_count, 2))
trk.associate(5, 0.1)
trk.normal_system(humanoid_trajectory(b.link_count, 2), KinSolverConfig(), np.ones(b.vertex_count, np.int32),
                  np.full(b.vertex_count, 1e-3))
trk.reconstruction_error()
th, jt = trk.track_sequence(np.stack(frames[1:]), cfg)
trk.optimize_pose(KinSolverConfig(iterations=2))
trk.optimize_shape(ShapeSolverConfig(iterations=1))
trk.close()
W.lib().wt_gpu_host_free(p)
B = 16
bt = BatchTracker(b, intr, B, init_theta=np.stack([humanoid_trajectory(b.link_count, 0, phase_offset=0.7 * s) for s in range(B)]))
batch = np.stack([np.roll(frames[1], s, axis=1) for s in range(B)])
for f in range(2):
    bt.track_frame(cfg, depth=batch)
print("ok", th[-1][:3], bt.get_state(3)[0][:3])
bt.close()
