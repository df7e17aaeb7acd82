"""Batched-sequence throughput (BatchTracker) vs batch size at C3, plus the
per-kernel device times of one batched frame (wt_gpu_profile_frame).

    python tools/batch_timing.py [B ...]
"""
import ctypes as C
import sys
import time

sys.path.insert(0, '.')
import numpy as np
import torch

from bench import alg_bytes, make_workload, trajectory
from paper_1711_07999_b200 import _lib as W
from paper_1711_07999_b200.tracker import BatchTracker, Tracker

bundle, intr, cfg = make_workload("c3")
ccfg = cfg.c()
r = Tracker(bundle, intr)
F = 6
Bs = [int(x) for x in sys.argv[1:]] or [1, 8, 32, 64]
Bmax = max(Bs)
P = intr.width * intr.height
frames = torch.empty((F, Bmax, intr.height, intr.width), dtype=torch.float32, device="cuda")
for f in range(F):
    for s in range(Bmax):
        r.render_depth(trajectory(bundle, f, s), frame=f, out_ptr=frames[f, s].data_ptr())
torch.cuda.synchronize()
L = W.lib()
for B in Bs:
    bt = BatchTracker(bundle, intr, B, init_theta=np.stack([trajectory(bundle, 0, s) for s in range(B)]))
    fr = frames[:, :B].contiguous()
    for f in range(2):
        bt.load_depth((fr[f].data_ptr(),))
        bt.track_async(cfg)
    bt.sync()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    n = 0
    for f in range(2, F):
        bt.load_depth((fr[f].data_ptr(),))
        bt.track_async(cfg)
        n += 1
    bt.sync()
    dt = time.perf_counter() - t0
    print(f"B={B:3d}: {n * B / dt:8.0f} frames/s  ({1e3 * dt / n:.2f} ms per batch frame)", flush=True)
    if B == Bmax:
        kinds = (C.c_int32 * 512)()
        ms = (C.c_float * 512)()
        nk = C.c_int32()
        bt.load_depth((fr[F - 1].data_ptr(),))
        W.check(L.wt_gpu_profile_frame(bt._ctx, C.byref(ccfg), kinds, ms, 512, C.byref(nk)), bt._ctx)
        per = {}
        for k in range(nk.value):
            d = per.setdefault(W.KERNEL_KINDS[kinds[k]], [0.0, 0])
            d[0] += ms[k]
            d[1] += 1
        tot = sum(v[0] for v in per.values())
        A = bundle.vertex_count // 6
        for name, (t, c) in sorted(per.items(), key=lambda kv: -kv[1][0]):
            b = alg_bytes(name, bundle.vertex_count, P, A, bundle.vertex_count // 2) * B
            print(f"  {name:16s} {c:3d} launches {1e3 * t / c:9.1f} us avg  {100 * t / tot:5.1f}%  "
                  f"{b / (t / c * 1e-3) / 1e9:8.0f} GB/s alg")
        print(f"  total {1e3 * tot:.0f} us (events between kernels)")
    bt.close()
