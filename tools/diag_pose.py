import os, sys, ctypes as C
os.environ["WT_DEBUG_POSE"] = "1"
sys.path.insert(0, '.')
import numpy as np
from bench import make_workload, trajectory
from paper_1711_07999_b200.tracker import Tracker
from paper_1711_07999_b200 import _lib as W
bundle, intr, cfg = make_workload("c3")
trk = Tracker(bundle, intr, trajectory(bundle, 0, 0))
L = W.lib(); L.wt_gpu_debug_pose.argtypes = [C.c_void_p, C.c_void_p]
buf = np.zeros(8, np.int64)
for f in range(1, 5):
    d, _ = trk.render_depth(trajectory(bundle, f, 0), frame=f)
    trk.track_frame(cfg, depth=d)
    L.wt_gpu_debug_pose(trk._ctx, buf.ctypes.data)
    print("frame", f, "main", buf[0], "atomics+wait", buf[1], "assemble", buf[2], "cholesky", buf[3], "update+fk", buf[4])
