#!/usr/bin/env python
"""Per-frame tracking throughput of the warptrack hot path on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config c1|c2|c3|c4|c5] [--sequences S] [--streams]

A step is one track_frame (tracker.cpp:54-68) on one synthetic depth frame:
5 pose Gauss-Newton iterations + 2 surface iterations + optimize_shape's
closing stats pass (dynamic mode), the BASELINE.json headline configuration
C3 (640x480 depth, ~100k-vertex 20-link humanoid 1.6 m from the camera,
~42k valid pixels) unless --config says otherwise. Frames are rendered on the
GPU (synthesize_frame semantics, no noise) from a sinusoidal joint trajectory
before timing.

value: frames/s over all ranks with the depth frames already resident in
HBM, each frame = device copy into the tracker + one graph launch, timed
with CUDA events on the tracker's stream; L2 is flushed (256 MiB write)
between frames, outside the timed spans. e2e: the same metric through the
public per-frame C-ABI call (wt_gpu_track_frame with a pinned host depth
frame, stats + theta read back), timed with the HOST clock around each call.

--gpus N > 1 without torchrun re-launches itself under torch.distributed.run
(one process per GPU). Each rank tracks its own sequence (C3 weak scaling, no
collective in the loop; time = max over ranks), and the north_star
multi-sequence case C5 (64 sequences per job, 64/N per rank as one batch)
is reported beside it as `batch_c5`.
--impl reference times the unmodified reference CPU implementation
(oracle/_ref, all host threads) on rank 0 on the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

CONFIGS = {
    # name: (width, height, target vertices, mode, pose its, shape its)
    "c1": (320, 240, 7_000, "smooth-bind", 12, 0),
    "c2": (640, 480, 25_000, "dynamic", 5, 2),
    "c3": (640, 480, 100_000, "dynamic", 5, 2),
    "c4": (1920, 1080, 400_000, "dynamic", 5, 2),
    # C5: 64 independent C3 sequences per job, sharded over the GPUs; the
    # sequences of a rank are one batch (BatchTracker: one frame graph whose
    # kernels carry the sequence in blockIdx.y)
    "c5": (640, 480, 100_000, "dynamic", 5, 2),
}
C5_SEQUENCES = 64
HOST_LEAD_CYCLES = 400_000  # ~0.2 ms spin before each device-timed frame (host enqueue lead)
METRIC = "frames/s at 640×480 depth, pose+surface, 100k-vert mesh; % of HBM roofline"


# SURVEY.md §8(d) algorithmic bytes (fp32, unpadded) attributed to the kernel
# that does the work here: V vertices, P pixels, A associated vertices, Vvis
# bucketed (visible, front-facing, in-frame) vertices. K5's per-vertex
# finalize (p~ = sum / count, r = n.(p~ - v), 72 B/V) runs inside each
# consumer of an association (pose system, shape step, stats pass).
def alg_bytes(kind: str, V: int, P: int, A: int, Vvis: int) -> float:
    return {
        "skin": 56 * V,                          # K1
        "normals+bucket": 77 * V + 37 * V,       # K2 + K3's per-vertex histogram
        "pixoff": 16 * P,                        # K3's per-pixel CSR scan
        "scatter": 8 * Vvis,                     # K3's scatter into pixel order
        "search+average": 12 * P + 16 * Vvis + 8 * P,  # K4 + K5's per-pixel accumulation
        "pose_system": 4 * V + 61 * A + 72 * V,  # K6 + K5 finalize
        "pose_solve": 0,                         # K7 (+K0 FK): one CTA, latency only
        "shape_step": 81 * V + 72 * V,           # K8 + K5 finalize
        "shape_stats": 72 * V,                   # K5 finalize + mean |r|
        "fk": 0,
    }[kind]


def ncu_traffic(config: str, kernel: str):
    """DRAM bytes (read + write) per launch of `kernel` from the committed
    `ncu --set full` capture summarised in profiles/traffic.json (None if absent)."""
    p = ROOT / "profiles" / "traffic.json"
    try:
        return json.loads(p.read_text())[config][kernel]["dram_bytes_per_launch"]
    except Exception:
        return None


def env_int(name, default):
    try:
        return int(os.environ.get(name, default))
    except ValueError:
        return default


def peak_hbm():
    p = ROOT / "MEASURED_PEAKS.json"
    peaks = json.loads(p.read_text()) if p.exists() else {}
    if "hbm_gbs" in peaks:
        return float(peaks["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """SM clocks + throttle reasons sampled during the timed region: NVML
    every 2 ms (nvidia-smi every 0.2 s where NVML is unavailable)."""

    REASONS = {  # NVML clocks-event bit -> name
        0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown", 0x4: "sw_power_cap"}

    def __init__(self, index: int):
        self.index = index
        self.samples = []  # (sm_mhz, max_mhz, [reasons])
        self._stop = threading.Event()
        self._t = None

    def _nvml_sample(self, nv, h, mx):
        sm = float(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM))
        bits = (nv.nvmlDeviceGetCurrentClocksEventReasons(h) if hasattr(nv, "nvmlDeviceGetCurrentClocksEventReasons")
                else nv.nvmlDeviceGetCurrentClocksThrottleReasons(h))
        self.samples.append((sm, mx, [n for b, n in self.REASONS.items() if bits & b]))

    def _run_nvml(self, nv, h, mx):
        while not self._stop.is_set():
            try:
                self._nvml_sample(nv, h, mx)
            except Exception:
                pass
            self._stop.wait(0.002)

    def _run_smi(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                f = [x.strip() for x in out.split(",")]
                if len(f) >= 6 and f[0].replace(".", "").isdigit():
                    self.samples.append((float(f[0]), float(f[1]),
                                         [names[k] for k in range(4) if f[2 + k].lower() == "active"]))
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        try:  # NVML initialised and sampled once before the timed region starts
            import pynvml as nv
            nv.nvmlInit()
            h = nv.nvmlDeviceGetHandleByIndex(self.index)
            mx = float(nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM))
            self._nvml_sample(nv, h, mx)
            target = lambda: self._run_nvml(nv, h, mx)  # noqa: E731
        except Exception:
            target = self._run_smi
        self._t = threading.Thread(target=target, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self) -> dict:
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [s[0] for s in self.samples]
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": max(s[1] for s in self.samples),
                "reasons": sorted({r for s in self.samples for r in s[2]}), "samples": len(self.samples)}


# the humanoid 1.6 m from the camera: ~42k valid pixels per 640x480 frame
# (acceptance.cpp:694-700 brings its biped closer the same way)
SUBJECT_DEPTH = 1.6


def make_workload(cfg_name: str, device: int | None = None):
    """The config's model, intrinsics and TrackConfig. With a device the model
    is subdivided / finalized / k-NN'd on that GPU (subdivide_on_device, the
    same bits as the host path the reference arm uses)."""
    from paper_1711_07999_b200.model import make_humanoid
    from paper_1711_07999_b200.tracker import AssocConfig, Intrinsics, KinSolverConfig, ShapeSolverConfig, TrackConfig
    W, H, nv, mode, kits, sits = CONFIGS[cfg_name]
    bundle = make_humanoid(nv, depth=SUBJECT_DEPTH, device=device)
    intr = Intrinsics.scaled(W, H)
    cfg = TrackConfig(mode=mode, kin=KinSolverConfig(iterations=kits), shape=ShapeSolverConfig(iterations=max(sits, 1)),
                      assoc=AssocConfig())
    return bundle, intr, cfg


def trajectory(bundle, frame: int, seq: int) -> np.ndarray:
    from paper_1711_07999_b200.model import humanoid_trajectory
    return humanoid_trajectory(bundle.link_count, frame, phase_offset=0.7 * seq)


def cpu_port(bundle, intr, cfg, frames_host, seconds: float, theta0):
    """Fallback when oracle/_ref was not built: the C restatement
    (oracle/wt_oracle.c, single thread) over a bounded sample."""
    from oracle import c_oracle
    ot = c_oracle.OracleTracker(bundle, intr.c(), theta0)
    c = cfg.c()
    ot.load_depth(frames_host[0])
    ot.track_loaded(c)
    thetas = [ot.get_state()[0]]
    n, t0 = 0, time.perf_counter()
    while n + 1 < len(frames_host):
        ot.load_depth(frames_host[n + 1])
        ot.track_loaded(c)
        n += 1
        if n < 3:
            thetas.append(ot.get_state()[0])
        if time.perf_counter() - t0 > seconds:
            break
    dt = time.perf_counter() - t0
    return {"value": n / dt, "unit": "frames/s", "cores": 1, "kind": "port",
            "sample": f"{n} frames of the same workload after 1 warm-up frame, C restatement of the reference "
                      f"(oracle/wt_oracle.c, 1 thread), {dt:.1f} s"}, thetas


def cpu_reference(bundle, intr, cfg, frames_host, seconds: float, theta0):
    """The reference's own track_frame (oracle/_ref) on all host threads over a
    bounded sample of the same frames. Also returns theta after each of the
    first frames (for the bench line's parity check)."""
    from oracle import ref
    if not ref.available():
        return cpu_port(bundle, intr, cfg, frames_host, seconds, theta0)
    rm = ref.RefModel.from_bundle(bundle)
    rt = ref.RefTracker(rm, theta0)
    c = cfg.c()
    c.threads = 0  # resolve_threads(0) = all hardware threads (parallel.hpp:17-21)
    rt.track_frame_depth(intr.c(), frames_host[0], c)  # warm-up frame
    thetas = [rt.get_state()[0]]
    n, t0 = 0, time.perf_counter()
    while n + 1 < len(frames_host):
        rt.track_frame_depth(intr.c(), frames_host[n + 1], c)
        n += 1
        if n < 3:
            thetas.append(rt.get_state()[0])
        if time.perf_counter() - t0 > seconds:
            break
    dt = time.perf_counter() - t0
    return {"value": n / dt, "unit": "frames/s", "cores": ref.hardware_threads(), "kind": "reference",
            "sample": f"{n} frames of the same workload after 1 warm-up frame, track_frame threads=0 "
                      f"(oracle/_ref, reference sources compiled unmodified), {dt:.1f} s"}, thetas


def parity_line(bundle, intr, cfg, frames_host, theta0, ref_thetas, device: int) -> dict:
    """Max |theta_gpu - theta_ref| after each of the first frames the CPU
    baseline tracked, the GPU tracking the same frames from the same start."""
    from paper_1711_07999_b200.tracker import Tracker
    trk = Tracker(bundle, intr, theta0, device=device)
    worst = 0.0
    try:
        for f, rth in enumerate(ref_thetas):
            trk.track_frame(cfg, depth=frames_host[f])
            worst = max(worst, float(np.abs(trk.theta - rth).max()))
    finally:
        trk.close()
    return {"max_abs_dtheta": worst, "frames": len(ref_thetas), "tolerance": 1e-6,
            "vs": "the cpu_baseline leg (the reference on the host) on the same frames from the same start"}


def write_desc(bundle, path) -> None:
    """A raw wt_model_desc dump (tests/cpp/adapter_bench.cpp reads it)."""
    L, V, T = bundle.link_count, bundle.vertex_count, bundle.triangle_count
    with open(path, "wb") as f:
        np.array([L, V, T, bundle.vtri_items.size, bundle.nbr_items.size], np.int32).tofile(f)
        for a, dt in ((bundle.parent, np.int32), (bundle.parent_offset, np.float64), (bundle.joint_kind, np.int32),
                      (bundle.joint_axis, np.float64), (bundle.theta_index, np.int32), (bundle.v0, np.float64),
                      (bundle.phi if bundle.phi is not None else np.zeros_like(bundle.v0), np.float64),
                      (bundle.weight_count, np.int32), (bundle.weight_link, np.int32), (bundle.weight, np.float64),
                      (bundle.triangles, np.int32), (bundle.vtri_offsets, np.int32), (bundle.vtri_items, np.int32),
                      (bundle.nbr_offsets, np.int32), (bundle.nbr_items, np.int32)):
            np.ascontiguousarray(a, dt).tofile(f)


def reference_api_e2e(bundle, intr, frames_host, steps: int):
    """The reference's own C++ API on the GPU: oracle/_ref/adapter_bench is the
    reference library with adapter/warptrack_gpu.cpp linked in, as
    INTEGRATION.md integrates it. It builds the reference ModelBundle of this
    model, reads the frames with the reference's SequenceReader, and times
    warptrack::gpu::track_frame on the reference's CloudFrames and
    warptrack::gpu::run_tracking over the .wts. None where not built."""
    import tempfile
    exe = ROOT / "oracle" / "_ref" / "adapter_bench"
    from oracle import ref
    if not exe.exists() or not ref.available():
        return None
    with tempfile.TemporaryDirectory() as td:
        write_desc(bundle, Path(td) / "model.desc")
        fr = np.stack([np.asarray(f) for f in frames_host])
        ref.write_sequence(Path(td) / "seq.wts", intr.c(), fr)
        warm = 3
        n = min(steps, fr.shape[0] - warm)
        out = subprocess.run([str(exe), str(Path(td) / "model.desc"), str(Path(td) / "seq.wts"), str(warm), str(n)],
                             capture_output=True, text=True, timeout=600)
    if out.returncode != 0:
        return {"error": out.stderr.strip()[-300:]}
    try:
        return json.loads(out.stdout.strip().splitlines()[-1])
    except Exception:
        return {"error": out.stdout.strip()[-300:]}


def workload_config(args, bundle, intr, cfg) -> dict:
    """The workload only (identical on both arms): no measured statistics."""
    W, H, nv, mode, kits, sits = CONFIGS[args.config]
    names = {"c1": "C1", "c2": "C2", "c3": "C3 (headline)", "c4": "C4", "c5": "C5 (64 sequences per job)"}
    return {"workload": f"{names[args.config]}: {W}x{H} depth, {bundle.vertex_count}-vertex "
                        f"{bundle.link_count}-link humanoid at {SUBJECT_DEPTH} m, {mode} ({kits} pose + {sits} "
                        f"surface GN iterations{' + stats pass' if sits else ''})",
            "vertices": bundle.vertex_count, "triangles": bundle.triangle_count, "links": bundle.link_count,
            "width": W, "height": H, "mode": mode, "pose_iterations": kits, "shape_iterations": sits,
            "window_radius": cfg.assoc.window_radius, "cutoff": cfg.assoc.cutoff,
            "l2": "flushed between timed frames (256 MiB write, outside the timed spans)"}


def run_reference(args, rank: int, world: int) -> None:
    if rank != 0:
        return
    from oracle import ref
    bundle, intr, cfg = make_workload(args.config)
    rm = ref.RefModel.from_bundle(bundle)
    nframes = args.warmup + args.steps + 1
    frames = [rm.render_depth(trajectory(bundle, f, 0), intr.c(), frame=f)[0] for f in range(nframes)]
    rt = ref.RefTracker(rm, trajectory(bundle, 0, 0))
    c = cfg.c()
    c.threads = 0
    for f in range(args.warmup):
        rt.track_frame_depth(intr.c(), frames[f + 1], c)
    t0 = time.perf_counter()
    for f in range(args.steps):
        rt.track_frame_depth(intr.c(), frames[args.warmup + f + 1], c)
    dt = time.perf_counter() - t0
    v = args.steps / dt
    kits, sits = CONFIGS[args.config][4], CONFIGS[args.config][5]
    line = {"metric": METRIC, "value": v, "unit": "frames/s", "impl": "reference", "n_gpus": 0,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (reference synthesize_frame renders of a sinusoidal trajectory, no noise)",
            "config": workload_config(args, bundle, intr, cfg),
            "gn_iterations_per_s": v * (kits + sits),
            "cpu_baseline": {"value": v, "unit": "frames/s", "cores": ref.hardware_threads(), "kind": "reference",
                             "sample": f"{args.steps} frames after {args.warmup} warm-up frames, "
                                       "track_frame threads=0, wall clock"},
            "e2e": {"value": v, "unit": "frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def profile_kernels(L, ctx, ccfg, load, nprof: int, nseq: int, bundle, P, A, Vvis, peak, config):
    """Per-kernel device times inside the real frame graph (an event after
    every kernel, wt_gpu_profile_frame) over nprof frames, with the §8(d)
    algorithmic bytes (times nseq for a batch) and the DRAM-measured traffic."""
    import ctypes as C

    from paper_1711_07999_b200 import _lib as W
    kinds = (C.c_int32 * 1024)()
    ms = (C.c_float * 1024)()
    n = C.c_int32()
    per_kind = {}
    nker = 0
    for rep in range(nprof):
        load(rep)
        W.check(L.wt_gpu_profile_frame(ctx, C.byref(ccfg), kinds, ms, 1024, C.byref(n)), ctx)
        nker = n.value
        for k in range(n.value):
            d = per_kind.setdefault(W.KERNEL_KINDS[kinds[k]], [0.0, 0])
            d[0] += ms[k]
            d[1] += 1
    kernels = {}
    for name, (tot, cnt) in per_kind.items():
        avg_ms = tot / cnt
        b = alg_bytes(name, bundle.vertex_count, P, A, Vvis) * nseq
        gbs = b / (avg_ms * 1e-3) / 1e9 if avg_ms > 0 else None
        tr = ncu_traffic(config, name)
        kernels[name] = {"launches_per_frame": cnt / nprof, "avg_us": 1e3 * avg_ms,
                         "us_per_frame": 1e3 * tot / nprof, "alg_bytes": b, "achieved_gbs": gbs,
                         "frac": (gbs or 0.0) / peak,
                         "dram_bytes_per_launch": tr,
                         "dram_frac": (tr / (avg_ms * 1e-3) / 1e9 / peak) if (tr and avg_ms > 0) else None}
    return kernels, nker


def roofline_of(kernels, peak, peak_src, config):
    # the dominant kernel among those that move data (the one-CTA solve is pure latency)
    dominant = max((k for k in kernels if kernels[k]["alg_bytes"] > 0), key=lambda k: kernels[k]["us_per_frame"])
    dk = kernels[dominant]
    frame_bytes = sum(kernels[nm]["alg_bytes"] * kernels[nm]["launches_per_frame"] for nm in kernels)
    frame_us = sum(kernels[nm]["us_per_frame"] for nm in kernels)
    roof = {"bound": "hbm", "kernel": dominant, "achieved": dk["achieved_gbs"], "peak": peak,
            "peak_source": peak_src, "unit": "GB/s", "frac": dk["achieved_gbs"] / peak,
            "traffic": ncu_traffic(config, dominant), "alg_bytes_per_launch": dk["alg_bytes"],
            "avg_launch_us": dk["avg_us"], "dram_frac": dk["dram_frac"]}
    frame = {"alg_bytes_per_frame": frame_bytes, "kernel_us_per_frame": frame_us,
             "achieved": frame_bytes / (frame_us * 1e-6) / 1e9, "frac": frame_bytes / (frame_us * 1e-6) / 1e9 / peak}
    return roof, frame


def run_ours(args, rank: int, world: int, local_rank: int, emit: bool = True):
    import ctypes as C

    import torch
    import torch.distributed as dist

    from paper_1711_07999_b200 import _lib as W
    from paper_1711_07999_b200.tracker import Tracker

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    bundle, intr, cfg = make_workload(args.config, device=local_rank)
    S = args.sequences
    trackers = [Tracker(bundle, intr, trajectory(bundle, 0, rank * S + s), device=local_rank) for s in range(S)]
    L = W.lib()
    ccfg = cfg.c()
    nprof = 3  # profiled frames (per-kernel event timing) after the timed ones
    nframes = args.warmup + max(args.steps, nprof + 1) + 1
    P = intr.width * intr.height
    # frames rendered on the GPU straight into HBM, plus pinned host copies
    frames_dev = [torch.empty((nframes, intr.height, intr.width), dtype=torch.float32, device=dev) for _ in range(S)]
    for s, trk in enumerate(trackers):
        for f in range(nframes):
            trk.render_depth(trajectory(bundle, f, rank * S + s), frame=f, out_ptr=frames_dev[s][f].data_ptr())
    torch.cuda.synchronize()
    frames_host = [t.cpu().pin_memory() for t in frames_dev]
    valid_px = float((frames_dev[0][1:] > 0).float().sum().item() / (nframes - 1))
    streams = [torch.cuda.ExternalStream(L.wt_gpu_stream(t._ctx), device=dev) for t in trackers]
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    def reset():
        for s, trk in enumerate(trackers):
            trk.set_state(theta=trajectory(bundle, 0, rank * S + s), phi=np.zeros((bundle.vertex_count, 3)),
                          frame_index=0)

    def frame_dev(s, f):
        W.check(L.wt_gpu_load_depth(trackers[s]._ctx, frames_dev[s][f].data_ptr(), 1.0), trackers[s]._ctx)
        W.check(L.wt_gpu_track_async(trackers[s]._ctx, C.byref(ccfg)), trackers[s]._ctx)

    # ---- device-resident timing (value) ----
    reset()
    for f in range(1, args.warmup + 1):
        for s in range(S):
            frame_dev(s, f)
    for t in trackers:
        W.check(L.wt_gpu_sync(t._ctx))
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    st0 = streams[0]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local_rank) as clk:
        for k in range(args.steps):
            f = args.warmup + 1 + k
            with torch.cuda.stream(st0):
                flush.zero_()
                # a short device-side delay: the host enqueues the frame while it
                # runs, so the timed span holds device work only, not launch latency
                torch.cuda._sleep(HOST_LEAD_CYCLES)
                starts[k].record(st0)
            for s in range(S):
                if s > 0:
                    streams[s].wait_event(starts[k])
                frame_dev(s, f)
            for s in range(1, S):
                e = torch.cuda.Event()
                e.record(streams[s])
                st0.wait_event(e)
            ends[k].record(st0)
        torch.cuda.synchronize()
    dev_ms = sum(starts[k].elapsed_time(ends[k]) for k in range(args.steps))
    if world > 1:
        dist.barrier()

    # ---- end-to-end through the public per-frame C-ABI call (e2e), host clock ----
    # every step: the pinned host frame goes up, the frame is tracked, the
    # stats and theta come back (wt_gpu_track_frame + wt_gpu_get_state)
    reset()
    for f in range(1, args.warmup + 1):
        for s in range(S):
            trackers[s].track_frame(cfg, depth=frames_host[s][f].numpy())
    from concurrent.futures import ThreadPoolExecutor
    nthr = min(S, 16)
    bufs = [(W.FrameStatsC(0, 0, 0, 64, 64, 0, t._kin, t._shape), np.zeros(bundle.link_count)) for t in trackers]

    def drive(f, lo):
        for s in range(lo, S, nthr):
            t = trackers[s]
            sb, th = bufs[s]
            W.check(L.wt_gpu_track_frame(t._ctx, frames_host[s][f].data_ptr(), 1.0, C.byref(ccfg), C.byref(sb)),
                    t._ctx)
            W.check(L.wt_gpu_get_state(t._ctx, th.ctypes.data, None, None), t._ctx)

    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e2e_s = 0.0
    with ThreadPoolExecutor(max_workers=nthr) as pool:
        for k in range(args.steps):
            f = args.warmup + 1 + k
            with torch.cuda.stream(st0):
                flush.zero_()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            if S == 1:
                drive(f, 0)
            else:  # one host thread per sequence slice (the C-ABI calls release the GIL)
                list(pool.map(lambda lo: drive(f, lo), range(nthr)))
            e2e_s += time.perf_counter() - t0
    e2e_ms = 1e3 * e2e_s

    # ---- the sequence driver: all K frames in one call from pinned host memory ----
    reset()
    warm = frames_host[0][1: args.warmup + 1]
    W.check(L.wt_gpu_track_sequence(trackers[0]._ctx, warm.data_ptr(), args.warmup, 1.0, C.byref(ccfg), None,
                                    None), trackers[0]._ctx)
    seq_frames = frames_host[0][args.warmup + 1: args.warmup + 1 + args.steps]
    th_out = np.zeros((args.steps, bundle.link_count))
    jt_out = np.zeros((args.steps, bundle.link_count, 3))
    trackers[0].set_state(theta=trajectory(bundle, args.warmup, rank * S), frame_index=args.warmup)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    W.check(L.wt_gpu_track_sequence(trackers[0]._ctx, seq_frames.data_ptr(), args.steps, 1.0, C.byref(ccfg),
                                    th_out.ctypes.data, jt_out.ctypes.data), trackers[0]._ctx)
    seq_s = time.perf_counter() - t0

    # ---- association statistics of the workload: bucketed and associated vertices ----
    trackers[0].set_state(theta=trajectory(bundle, args.warmup, rank * S), phi=np.zeros((bundle.vertex_count, 3)),
                          frame_index=1)
    st = trackers[0].track_frame(cfg, depth=frames_host[0][args.warmup + 1].numpy())
    nb = C.c_int32()
    W.check(L.wt_gpu_bucket_count(trackers[0]._ctx, 0, C.byref(nb)), trackers[0]._ctx)
    A = int(np.mean([k.associated for k in st.kin]))
    Vvis = int(nb.value)

    # ---- per-kernel device times inside the real frame (events between kernels) ----
    peak, peak_src = peak_hbm()
    trackers[0].set_state(theta=trajectory(bundle, args.warmup, rank * S), phi=np.zeros((bundle.vertex_count, 3)),
                          frame_index=1)

    def load(rep):
        f = args.warmup + 1 + rep
        W.check(L.wt_gpu_load_depth(trackers[0]._ctx, frames_dev[0][f].data_ptr(), 1.0), trackers[0]._ctx)

    kernels, nker = profile_kernels(L, trackers[0]._ctx, ccfg, load, nprof, 1, bundle, P, A, Vvis, peak,
                                    args.config)

    # ---- aggregate over ranks (max time) ----
    t = torch.tensor([dev_ms, e2e_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    dev_ms, e2e_ms = t.tolist()
    total_frames = args.steps * S * world
    value = total_frames / (dev_ms * 1e-3)
    e2e = total_frames / (e2e_ms * 1e-3)
    batch = None
    bargs = None
    if args.config == "c3" and not args.no_batch:
        # C5, the north_star multi-sequence case: 64 sequences per job, 64/N
        # per rank as one batch -- where the per-vertex / per-pixel kernels
        # become HBM-bound, so their roofline fraction is meaningful
        bargs = argparse.Namespace(**{**vars(args), "config": "c5", "sequences": max(1, C5_SEQUENCES // world),
                                      "steps": 10, "warmup": 3})
        batch = run_batched(bargs, rank, world, local_rank, emit=False)
    if rank != 0:
        for t_ in trackers:
            t_.close()
        return None
    roof, frame = roofline_of(kernels, peak, peak_src, args.config)
    kits, sits = CONFIGS[args.config][4], CONFIGS[args.config][5]
    line = {
        "metric": METRIC, "value": value, "unit": "frames/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": dev_ms / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None,
        "dtype": "f64 (geometry, distances, normal equations; normals stored f32)",
        "data": "synthetic (GPU synthesize_frame renders of a sinusoidal joint trajectory, no noise)",
        "config": {**workload_config(args, bundle, intr, cfg), "sequences_per_gpu": S},
        "workload_stats": {"valid_pixels_mean": valid_px, "bucketed_vertices": Vvis, "associated_vertices_mean": A},
        "gn_iterations_per_s": value * (kits + sits),
        "e2e": {"value": e2e, "unit": "frames/s", "h2d_bytes_per_step": 4 * P * S,
                "d2h_bytes_per_step": S * (8 * bundle.link_count + 32 * (kits + sits)),
                "api": "wt_gpu_track_frame (pinned host depth frame, FrameStats) + wt_gpu_get_state (theta), "
                       "host clock around the calls"},
        "e2e_sequence": {"value": args.steps / seq_s, "unit": "frames/s",
                         "api": "wt_gpu_track_sequence (one call, K pinned host frames, uploads overlapped, "
                                "theta + joints read back), host clock", "h2d_bytes_per_step": 4 * P,
                         "d2h_bytes_per_step": 32 * bundle.link_count, "l2": "not flushed inside the sequence"},
        "roofline": roof,
        "frame_roofline": {**frame, "aggregate_achieved": frame["alg_bytes_per_frame"] * value / world / 1e9,
                           "aggregate_frac": frame["alg_bytes_per_frame"] * value / world / 1e9 / peak,
                           "note": "per-kernel times from one sequence's frame graph (events between kernels); "
                                   "aggregate = algorithmic bytes per frame x frames/s per GPU"},
        "kernels": kernels,
        "gpu_launches": args.steps * S * (nker + 1),
        "clocks": clk.summary(),
    }
    if getattr(args, "oversubscribed", False):
        line["oversubscribed"] = "more ranks than GPUs: a functional check of the N>1 path, not a scaling number"
    if batch is not None:
        line["batch_c5"] = {
            "workload": batch["config"]["workload"], "value": batch["value"], "unit": "frames/s",
            "n_gpus": world, "sequences_per_gpu": bargs.sequences, "scaling": "strong",
            "ms_per_step": batch["ms_per_step"], "steps": bargs.steps, "step": batch["step"],
            "gn_iterations_per_s": batch["gn_iterations_per_s"], "workload_stats": batch["workload_stats"],
            "e2e": batch["e2e"], "roofline": batch["roofline"], "frame_roofline": batch["frame_roofline"],
            "kernels": {k: {kk: v[kk] for kk in ("avg_us", "us_per_frame", "achieved_gbs", "frac",
                                                 "dram_bytes_per_launch", "dram_frac")}
                        for k, v in batch["kernels"].items()},
            "gpu_launches": batch["gpu_launches"], "clocks": batch["clocks"]}
    if world == 1 and not args.no_cpu_baseline:
        # a bounded CPU sample of the same workload: enough frames of the same
        # trajectory for ~cpu_seconds of reference work (rendered on the GPU)
        ncpu = int(args.cpu_seconds * 40) + 2
        cpu_frames = [trackers[0].render_depth(trajectory(bundle, f, 0), frame=f)[0] for f in range(ncpu)]
        line["cpu_baseline"], ref_thetas = cpu_reference(bundle, intr, cfg, cpu_frames, args.cpu_seconds,
                                                         trajectory(bundle, 0, 0))
        line["parity"] = parity_line(bundle, intr, cfg, cpu_frames, trajectory(bundle, 0, 0), ref_thetas,
                                     local_rank)
        api = reference_api_e2e(bundle, intr, [f.numpy() for f in frames_host[0]], args.steps)
        if api is not None:
            line["e2e_reference_api"] = api
    for t_ in trackers:
        t_.close()
    if world == 1 and args.config == "c3" and not args.no_batch:
        # C4, the 1920x1080 / 409k-vertex stress configuration, one sequence
        cargs = argparse.Namespace(**{**vars(args), "config": "c4", "sequences": 1, "steps": 10, "warmup": 3,
                                      "no_batch": True, "no_cpu_baseline": True})
        c4 = run_ours(cargs, rank, world, local_rank, emit=False)
        line["c4"] = {k: c4[k] for k in ("value", "unit", "ms_per_step", "steps", "gn_iterations_per_s",
                                         "workload_stats", "e2e", "roofline", "frame_roofline", "gpu_launches",
                                         "clocks")}
        line["c4"]["workload"] = c4["config"]["workload"]
        line["c4"]["kernels"] = {k: {kk: v[kk] for kk in ("avg_us", "us_per_frame", "achieved_gbs", "frac",
                                                          "dram_bytes_per_launch", "dram_frac")}
                                 for k, v in c4["kernels"].items()}
    if emit:
        print(json.dumps(line), flush=True)
    return line


def run_batched(args, rank: int, world: int, local_rank: int, emit: bool = True):
    """C5: the rank's sequences tracked as one batch (wt_gpu_create_batch).
    Prints the JSON line (emit) or returns it (rank 0; None elsewhere)."""
    import ctypes as C

    import torch
    import torch.distributed as dist

    from paper_1711_07999_b200 import _lib as W
    from paper_1711_07999_b200.tracker import BatchTracker, Tracker

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    bundle, intr, cfg = make_workload(args.config, device=local_rank)
    S = args.sequences
    seqs = [rank * S + s for s in range(S)]
    th0 = np.stack([trajectory(bundle, 0, q) for q in seqs])
    bt = BatchTracker(bundle, intr, S, init_theta=th0, device=local_rank)
    L = W.lib()
    ccfg = cfg.c()
    P = intr.width * intr.height
    nframes = args.warmup + args.steps + 2
    renderer = Tracker(bundle, intr, device=local_rank)
    frames_dev = torch.empty((nframes, S, intr.height, intr.width), dtype=torch.float32, device=dev)
    for f in range(nframes):
        for s, q in enumerate(seqs):
            renderer.render_depth(trajectory(bundle, f, q), frame=f, out_ptr=frames_dev[f, s].data_ptr())
    torch.cuda.synchronize()
    frames_host = frames_dev.cpu().pin_memory()
    valid_px = float((frames_dev[1:] > 0).float().sum().item() / ((nframes - 1) * S))
    st0 = torch.cuda.ExternalStream(bt.stream, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    def reset():
        for s in range(S):
            bt.set_state(s, theta=th0[s], phi=np.zeros((bundle.vertex_count, 3)))

    def frame_dev(f):
        W.check(L.wt_gpu_batch_load_depth(bt._ctx, frames_dev[f].data_ptr(), 1.0), bt._ctx)
        W.check(L.wt_gpu_batch_track_async(bt._ctx, C.byref(ccfg)), bt._ctx)

    # ---- device-resident timing (value) ----
    reset()
    for f in range(1, args.warmup + 1):
        frame_dev(f)
    bt.sync()
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local_rank) as clk:
        for k in range(args.steps):
            with torch.cuda.stream(st0):
                flush.zero_()
                torch.cuda._sleep(HOST_LEAD_CYCLES)  # see run_ours
                starts[k].record(st0)
            frame_dev(args.warmup + 1 + k)
            ends[k].record(st0)
        torch.cuda.synchronize()
    dev_ms = sum(starts[k].elapsed_time(ends[k]) for k in range(args.steps))
    if world > 1:
        dist.barrier()

    # ---- end to end: pinned host frames in, stats + every theta out, host clock ----
    reset()
    kin = [(W.KinIterStats * 64)() for _ in range(S)]
    shp = [(W.ShapeIterStats * 32)() for _ in range(S)]
    stats = (W.FrameStatsC * S)(*[W.FrameStatsC(0, 0, 0, 64, 32, 0, kin[s], shp[s]) for s in range(S)])
    theta = np.zeros(bundle.link_count)

    def frame_e2e(f):
        W.check(L.wt_gpu_batch_track(bt._ctx, frames_host[f].data_ptr(), 1.0, C.byref(ccfg), stats), bt._ctx)
        for s in range(S):
            W.check(L.wt_gpu_batch_get_state(bt._ctx, s, theta.ctypes.data, None), bt._ctx)

    for f in range(1, args.warmup + 1):
        frame_e2e(f)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e2e_s = 0.0
    for k in range(args.steps):
        with torch.cuda.stream(st0):
            flush.zero_()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        frame_e2e(args.warmup + 1 + k)
        e2e_s += time.perf_counter() - t0
    e2e_ms = 1e3 * e2e_s
    A = int(np.mean([np.mean([kin[s][k].associated for k in range(stats[s].n_kin)]) for s in range(S)]))
    nb = C.c_int32()
    W.check(L.wt_gpu_bucket_count(bt._ctx, 0, C.byref(nb)), bt._ctx)
    Vvis = int(nb.value)

    # ---- per-kernel device times of one batch frame (events between kernels) ----
    peak, peak_src = peak_hbm()

    def load(rep):
        W.check(L.wt_gpu_batch_load_depth(bt._ctx, frames_dev[args.warmup + args.steps + 1].data_ptr(), 1.0),
                bt._ctx)

    kernels, nker = profile_kernels(L, bt._ctx, ccfg, load, 1, S, bundle, P, A, Vvis, peak, "c5")

    t = torch.tensor([dev_ms, e2e_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    dev_ms, e2e_ms = t.tolist()
    total_frames = args.steps * S * world
    value = total_frames / (dev_ms * 1e-3)
    e2e = total_frames / (e2e_ms * 1e-3)
    bt.close()
    renderer.close()
    if rank != 0:
        return None
    roof, frame = roofline_of(kernels, peak, peak_src, "c5")
    kits, sits = CONFIGS[args.config][4], CONFIGS[args.config][5]
    line = {
        "metric": METRIC, "value": value, "unit": "frames/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": dev_ms / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None,
        "dtype": "f64 (geometry, distances, normal equations; normals stored f32)",
        "data": "synthetic (GPU synthesize_frame renders of sinusoidal joint trajectories, one phase per sequence)",
        "config": {**workload_config(args, bundle, intr, cfg), "sequences_per_gpu": S, "batched": True},
        "step": f"one frame of every sequence of the rank's batch ({S} frames per rank per step)",
        "workload_stats": {"valid_pixels_mean": valid_px, "bucketed_vertices": Vvis, "associated_vertices_mean": A},
        "gn_iterations_per_s": value * (kits + sits),
        "e2e": {"value": e2e, "unit": "frames/s", "h2d_bytes_per_step": 4 * P * S,
                "d2h_bytes_per_step": S * (8 * bundle.link_count + 32 * 64 + 40 * 32),
                "api": "wt_gpu_batch_track (pinned host frames of the batch, stats) + wt_gpu_batch_get_state "
                       "theta of every sequence, host clock"},
        "roofline": roof,
        "frame_roofline": {**frame, "note": "one batch frame of the rank's sequences, events between kernels"},
        "kernels": kernels,
        "gpu_launches": args.steps * (nker + 1),
        "clocks": clk.summary(),
    }
    if emit:
        print(json.dumps(line), flush=True)
    return line


def plumbing_check(args, rank: int, world: int) -> None:
    """--plumbing-check (CPU, gloo): the multi-rank host path of the bench
    without device work -- each rank's C5 shard, the barrier, the max over
    ranks and rank 0's single JSON line."""
    import torch.distributed as dist

    from paper_1711_07999_b200 import shard
    r = shard.Rank(rank, world, rank)
    if world > 1:
        dist.init_process_group("gloo")
    mine = list(shard.shard(C5_SEQUENCES, r))
    shard.barrier(r)
    ms = shard.max_over_ranks([1.0 + rank], r)
    got = shard.gather_to_root({"rank": rank, "pid": os.getpid(), "sequences": mine}, r)
    if rank == 0:
        print(json.dumps({"metric": METRIC, "n_gpus": world, "plumbing_check": True, "max_ms": float(ms[0]),
                          "shards": got}), flush=True)
    if world > 1:
        dist.destroy_process_group()


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def main() -> None:
    import faulthandler
    faulthandler.enable()  # a crash in native code still names the Python frame
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=sorted(CONFIGS), default="c3")
    ap.add_argument("--sequences", type=int, default=1)
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-batch", action="store_true",
                    help="c3: skip the C5 batch sub-measurement (batch_c5)")
    ap.add_argument("--streams", action="store_true",
                    help="c5: one Tracker + stream per sequence instead of one batch")
    ap.add_argument("--plumbing-check", action="store_true", help=argparse.SUPPRESS)
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: re-launch under torch.distributed.run
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", f"--master-port={_free_port()}", str(Path(__file__).resolve())]
        sys.exit(subprocess.call(cmd + sys.argv[1:]))
    rank, world, local_rank = env_int("RANK", 0), env_int("WORLD_SIZE", 1), env_int("LOCAL_RANK", 0)
    if args.plumbing_check:
        plumbing_check(args, rank, world)
        return
    if args.config == "c5":  # 64 sequences per job, strong-scaled over the ranks
        args.sequences = max(1, C5_SEQUENCES // world)
    oversubscribed = False
    if world > 1 and args.impl == "ours":
        import torch
        import torch.distributed as dist
        ngpu = torch.cuda.device_count()
        if ngpu < world:
            # more ranks than GPUs (a functional check of the N > 1 path on a
            # smaller box): ranks share devices, gloo carries the barriers and
            # the max over ranks; the numbers are not a scaling measurement
            oversubscribed = True
            local_rank = local_rank % max(ngpu, 1)
            torch.cuda.set_device(local_rank)
            dist.init_process_group("gloo")
        else:
            torch.cuda.set_device(local_rank)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    args.oversubscribed = oversubscribed
    if args.impl == "reference":
        run_reference(args, rank, world)
    elif args.config == "c5" and not args.streams:
        run_batched(args, rank, world, local_rank)
    else:
        run_ours(args, rank, world, local_rank)
    if world > 1 and args.impl == "ours":
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
