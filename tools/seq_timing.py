import sys, time
sys.path.insert(0, '.')
import numpy as np, torch
from bench import make_workload, trajectory
from paper_1711_07999_b200.tracker import Tracker
bundle, intr, cfg = make_workload("c3")
trk = Tracker(bundle, intr, trajectory(bundle, 0, 0))
F = 40
frames = np.stack([trk.render_depth(trajectory(bundle, f, 0), frame=f)[0] for f in range(F + 1)])
pinned = torch.from_numpy(frames).pin_memory()
dev = torch.from_numpy(frames).cuda()
for name, src in [("numpy", frames[1:]), ("pinned", (pinned[1:].data_ptr(), F)), ("device", (dev[1:].data_ptr(), F))]:
    for rep in range(2):
        trk.set_state(theta=trajectory(bundle, 0, 0), phi=np.zeros((bundle.vertex_count, 3)), frame_index=0)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        trk.track_sequence(src, cfg)
        dt = time.perf_counter() - t0
        print(name, rep, f"{F / dt:.0f} fps")
t0 = time.perf_counter()
for f in range(1, F + 1):
    trk.track_frame(cfg, depth=frames[f], stats=False)
print("track_frame loop", f"{F / (time.perf_counter() - t0):.0f} fps")
