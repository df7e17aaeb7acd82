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
buf = np.zeros(8 + 8 * 296, np.int64)
for f in range(1, 5):
    d, _ = trk.render_depth(trajectory(bundle, f, 0), frame=f)
    trk.track_frame(cfg, depth=d)
    L.wt_gpu_debug_pose(trk._ctx, buf.ctypes.data)
    print("frame", f, "main", buf[0], "atomics+wait", buf[1], "assemble", buf[2], "cholesky", buf[3], "update+fk", buf[4], "(fk: local", buf[5], "levels", buf[6], ")")

rec = buf[8:8 + 3 * 296].reshape(296, 3)
st = buf[8 + 3 * 296: 8 + 4 * 296]
t0 = st.min()
print("start spread us", (st.max() - t0) / 1e3)
print("main end (us from first start): median", np.median(rec[:, 0] - t0) / 1e3, "max", (rec[:, 0].max() - t0) / 1e3)
print("atomics end: median", np.median(rec[:, 1] - t0) / 1e3, "max", (rec[:, 1].max() - t0) / 1e3)
print("main cycles: median", np.median(rec[:, 2]), "max", rec[:, 2].max(), "argmax", rec[:, 2].argmax())
print("atomic phase us: median", np.median(rec[:, 1] - rec[:, 0]) / 1e3, "max", (rec[:, 1] - rec[:, 0]).max() / 1e3)
sec = buf[8 + 4 * 296: 8 + 8 * 296].reshape(296, 4)
for j, n in enumerate(["stage", "scan", "rows", "outer"]):
    print(f"{n} cycles (thread 0 of each CTA slot): median {np.median(sec[:, j]):.0f} max {sec[:, j].max()}")
