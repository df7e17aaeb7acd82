"""Classifies GPU vs reference winner-map disagreements (diagnostic)."""
import sys
sys.path.insert(0, '.')
import numpy as np
from oracle import ref
from tests.helpers import humanoid, intr640, theta_at
from paper_1711_07999_b200.tracker import Tracker

b = humanoid(25000); intr = intr640(); rm = ref.RefModel.from_bundle(b); trk = Tracker(b, intr)
depth, _ = rm.render_depth(theta_at(b, 5), intr.c())
th = theta_at(b, 4)
trk.load_depth(depth)
gv, gn, gval = trk.skin(th)
g = trk.associate(5, 0.10)
rv, rn, rvalid = rm.skin(th)
pts, pvalid = ref.depth_to_cloud(intr.c(), depth)
r = ref.associate(intr.c(), rv, rn, rvalid, pts, pvalid, 5, 0.10)
off, items = ref.bucket_occupancy(intr.c(), rv, rn, rvalid)
rb = np.zeros(b.vertex_count, bool); rb[items] = True
# GPU-side bucket emulation from the gpu's own fp32 v/n
gb = gval.astype(bool) & ~((gn * gv).sum(1) > 0)
print("bucketed ref", rb.sum(), "gpu-emul", gb.sum(), "differ", (rb != gb).sum())
bad = np.where(pvalid.astype(bool) & (g["winners"] != r["winners"]))[0]
print("valid px", pvalid.sum(), "disagree", len(bad))
cls = dict(tie=0, gpu_none=0, ref_none=0, bucket=0, other=0)
for p in bad[:2000]:
    wg, wr = g["winners"][p], r["winners"][p]
    if wg < 0: cls["gpu_none"] += 1; continue
    if wr < 0: cls["ref_none"] += 1; continue
    if rb[wg] != gb[wg] or rb[wr] != gb[wr]: cls["bucket"] += 1; continue
    dg = np.sum((rv[wg] - pts[p])**2); dr = np.sum((rv[wr] - pts[p])**2)
    if abs(dg - dr) <= 1e-4 * dr: cls["tie"] += 1
    else:
        cls["other"] += 1
        if cls["other"] < 6: print("other", p, wg, wr, dg, dr, gv[wg]-rv[wg])
print(cls)
rel = []
for p in bad[:60]:
    wg, wr = g["winners"][p], r["winners"][p]
    dg = np.sum((rv[wg] - pts[p])**2); dr = np.sum((rv[wr] - pts[p])**2)
    rel.append((dg - dr) / dr)
    if len(rel) < 8:
        print(p, wg, wr, dg, dr, (dg-dr)/dr, "gv-rv", np.abs(gv[wg]-rv[wg]).max(), np.abs(gv[wr]-rv[wr]).max())
rel = np.array(rel); print("rel gaps: exact-tie", np.sum(rel == 0), "max", np.abs(rel).max(), "median", np.median(np.abs(rel)))
