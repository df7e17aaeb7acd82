"""Small tracking run for compute-sanitizer (memcheck / racecheck / synccheck):
a 7k-vertex humanoid at 320x240, two dynamic frames, the stage hooks and the
reconstruction error."""
import sys

sys.path.insert(0, ".")
import numpy as np

from paper_1711_07999_b200.model import humanoid_trajectory, make_humanoid
from paper_1711_07999_b200.tracker import (AssocConfig, Intrinsics, KinSolverConfig, ShapeSolverConfig,
                                           TrackConfig, Tracker)

b = make_humanoid(7000)
intr = Intrinsics.scaled(320, 240)
cfg = TrackConfig(mode="dynamic", kin=KinSolverConfig(iterations=3), shape=ShapeSolverConfig(iterations=2),
                  assoc=AssocConfig())
trk = Tracker(b, intr, humanoid_trajectory(b.link_count, 0))
for f in (1, 2):
    d, _ = trk.render_depth(humanoid_trajectory(b.link_count, f), frame=f)
    trk.track_frame(cfg, depth=d)
trk.skin(humanoid_trajectory(b.link_count, 2))
trk.associate(5, 0.1)
trk.reconstruction_error()
th, jt = trk.track_sequence(np.stack([d, d]), cfg)
print("ok", th[-1][:3])
