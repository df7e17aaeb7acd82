"""Runs a few C3 frames for ncu captures (one tracker, device-resident frames)."""
import sys
sys.path.insert(0, '.')
import numpy as np
from bench import make_workload, trajectory
from paper_1711_07999_b200.tracker import Tracker

cfg_name = sys.argv[1] if len(sys.argv) > 1 else "c3"
nframes = int(sys.argv[2]) if len(sys.argv) > 2 else 2
bundle, intr, cfg = make_workload(cfg_name)
trk = Tracker(bundle, intr, trajectory(bundle, 0, 0))
frames = [trk.render_depth(trajectory(bundle, f, 0), frame=f)[0] for f in range(nframes + 1)]
for f in range(1, nframes + 1):
    st = trk.track_frame(cfg, depth=frames[f])
print("ok", st.kin[-1].associated, trk.theta[:3])
