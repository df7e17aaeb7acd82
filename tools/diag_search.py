import os, sys, ctypes as C
os.environ["WT_DEBUG_SEARCH"] = "1"
sys.path.insert(0, '.')
import numpy as np
from bench import make_workload, trajectory
from paper_1711_07999_b200.tracker import Tracker
from paper_1711_07999_b200 import _lib as W
bundle, intr, cfg = make_workload("c3")
trk = Tracker(bundle, intr, trajectory(bundle, 0, 0))
d, _ = trk.render_depth(trajectory(bundle, 1, 0), frame=1)
trk.track_frame(cfg, depth=d)
L = W.lib(); L.wt_gpu_debug_search.argtypes = [C.c_void_p, C.c_void_p, C.c_int]
buf = np.zeros((1200, 8), np.int64)
n = L.wt_gpu_debug_search(trk._ctx, buf.ctypes.data, 1200)
rec = buf[buf[:, 3] > 0]
print("active tiles", len(rec), "cycles: median", np.median(rec[:, 3]), "max", rec[:, 3].max())
order = np.argsort(-rec[:, 3])
for r in rec[order[:12]]:
    t = r[0]; print("tile", t, "tx,ty", t % 40, t // 40, "cand", r[1], "cycles", r[3], "prefix", r[2], "loads", r[7], "stage", r[4], "scan", r[5], "exact", r[6])
print("cand: median", np.median(rec[:, 1]), "max", rec[:, 1].max())
# second association on the same posed mesh: warm caches / TLB
for rep in range(2):
    trk.associate(5, 0.10)
    n = L.wt_gpu_debug_search(trk._ctx, buf.ctypes.data, 1200)
    rec = buf[buf[:, 3] > 0]
    print(f"rep {rep}: median cycles", np.median(rec[:, 3]), "max", rec[:, 3].max(), "median pass1", np.median(rec[:, 2]), "max pass1", rec[:, 2].max())
