import faulthandler, sys; faulthandler.enable()
sys.path.insert(0, '.')
import numpy as np
from paper_1711_07999_b200.model import make_humanoid
for n in (7000, 100000):
    a = make_humanoid(n, depth=1.6, device=0); print(n, a.vertex_count, flush=True)
    b = make_humanoid(n, depth=1.6); print("host", b.vertex_count, all(np.array_equal(getattr(a,k), getattr(b,k)) for k in ["v0","weight","triangles","nbr_items"]), flush=True)
