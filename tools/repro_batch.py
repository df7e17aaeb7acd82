"""Repeat the C5 batch-vs-lone comparison to catch intermittent differences:
python tools/repro_batch.py [reps] [nseq]"""
import sys
sys.path.insert(0, '.')
import numpy as np
from paper_1711_07999_b200.tracker import BatchTracker, Intrinsics, Tracker
from tests.helpers import bench_humanoid, cfg, theta_at

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
nseq = int(sys.argv[2]) if len(sys.argv) > 2 else 16
b = bench_humanoid(100_000)
intr = Intrinsics.scaled(640, 480)
c = cfg("dynamic")
renderer = Tracker(b, intr)
frames = np.zeros((2, nseq, intr.height, intr.width), np.float32)
for f in range(2):
    for s in range(nseq):
        frames[f, s] = renderer.render_depth(theta_at(b, f + 1, 0.7 * s), frame=f + 1)[0]
renderer.close()
th0 = np.stack([theta_at(b, 0, 0.7 * s) for s in range(nseq)])
lone = []
for s in range(nseq):
    t = Tracker(b, intr, th0[s])
    for f in range(2):
        t.track_frame(c, depth=frames[f, s])
    lone.append(t.get_state()[0])
    t.close()
for r in range(reps):
    bt = BatchTracker(b, intr, nseq, init_theta=th0)
    for f in range(2):
        bt.track_frame(c, depth=frames[f])
    d = [float(np.abs(bt.get_state(s)[0] - lone[s]).max()) for s in range(nseq)]
    bt.close()
    worst = max(d)
    print(f"rep {r}: max dtheta {worst:.3g} at seq {int(np.argmax(d))}", "BAD" if worst > 1e-8 else "ok", flush=True)
    # and a fresh lone run of the worst sequence
    s = int(np.argmax(d))
    t = Tracker(b, intr, th0[s])
    for f in range(2):
        t.track_frame(c, depth=frames[f, s])
    print(f"   lone rerun seq {s}: {float(np.abs(t.get_state()[0] - lone[s]).max()):.3g}", flush=True)
    t.close()
