"""bench.py's contract pieces that do not need a GPU: the reference arm runs
on the host cores and prints one JSON line with the required keys; the
algorithmic byte model matches SURVEY.md §8(d); the committed ncu traffic
table is read back per kernel; the clock sampler degrades to 'unsampled'."""
import json
import subprocess
import sys

import pytest

import bench
from .conftest import ROOT


def test_alg_bytes_match_survey_8d():
    """SURVEY §8(d)'s per-kernel bytes, each attributed to the kernel that
    does the work: K3 splits into the per-vertex histogram (normals), the
    per-pixel scan (pixoff) and the scatter; K5's per-pixel accumulation sits
    in the search and its per-vertex finalize (72 B/V) in every consumer."""
    V, P, A, Vv = 102392, 640 * 480, 16000, 51196
    assert bench.alg_bytes("skin", V, P, A, Vv) == 56 * V                          # K1
    assert bench.alg_bytes("normals+bucket", V, P, A, Vv) == 77 * V + 37 * V      # K2 + K3 (per vertex)
    assert bench.alg_bytes("pixoff", V, P, A, Vv) == 16 * P                        # K3 (per pixel)
    assert bench.alg_bytes("scatter", V, P, A, Vv) == 8 * Vv                       # K3 (scatter)
    assert bench.alg_bytes("search+average", V, P, A, Vv) == 12 * P + 16 * Vv + 8 * P  # K4 + K5 (per pixel)
    assert bench.alg_bytes("pose_system", V, P, A, Vv) == 4 * V + 61 * A + 72 * V  # K6 + K5 finalize
    assert bench.alg_bytes("shape_step", V, P, A, Vv) == 81 * V + 72 * V           # K8 + K5 finalize
    assert bench.alg_bytes("pose_solve", V, P, A, Vv) == 0
    # the per-frame total is SURVEY's pose iteration (254 V + 61 A + 36 P) x 5
    # + shape iteration (331 V + 36 P) x 2, plus the stats pass's association
    per_frame = (5 * sum(bench.alg_bytes(k, V, P, A, Vv) for k in
                         ("skin", "normals+bucket", "pixoff", "scatter", "search+average", "pose_system")) +
                 2 * sum(bench.alg_bytes(k, V, P, A, Vv) for k in
                         ("skin", "normals+bucket", "pixoff", "scatter", "search+average", "shape_step")))
    assert per_frame == 5 * (254 * V + 61 * A + 36 * P + 8 * Vv + 16 * Vv - 8 * V) + \
        2 * (331 * V + 36 * P + 8 * Vv + 16 * Vv - 8 * V)


@pytest.mark.timeout(300)
def test_multi_gpu_spawn_path_with_gloo():
    """--gpus 2 without torchrun re-launches bench.py as two ranks (one
    process per GPU) that shard C5's 64 sequences; the plumbing check runs
    that path on CPU over gloo: n_gpus == 2, two distinct processes, each
    rank its 32 sequences, rank 0 alone prints."""
    out = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--plumbing-check"], cwd=ROOT,
                         capture_output=True, text=True, timeout=280)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.strip().splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["max_ms"] == 2.0
    assert [s["sequences"] for s in d["shards"]] == [list(range(32)), list(range(32, 64))]
    assert len({s["pid"] for s in d["shards"]}) == 2


def test_ncu_traffic_table():
    t = json.loads((ROOT / "profiles" / "traffic.json").read_text())
    for cfg in ("c3", "c5"):
        for kind in ("skin", "normals+bucket", "search+average", "pose_system"):
            assert bench.ncu_traffic(cfg, kind) == t[cfg][kind]["dram_bytes_per_launch"] > 0
    assert bench.ncu_traffic("c3", "no-such-kernel") is None


def test_clock_sampler_without_samples():
    c = bench.ClockSampler(0)
    assert c.summary()["reasons"] == ["unsampled"]


@pytest.mark.ref
def test_reference_arm_prints_the_contract_line():
    out = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--config", "c1", "--steps", "2",
                          "--warmup", "3"], cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    d = json.loads(out.stdout.strip().splitlines()[-1])
    for k in ("metric", "value", "unit", "steps", "warmup", "ms_per_step", "higher_is_better", "config",
              "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["steps"] == 2
    assert d["cpu_baseline"]["kind"] == "reference" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
