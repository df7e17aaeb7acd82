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
    V, P, A, Vv = 102392, 640 * 480, 16000, 51196
    assert bench.alg_bytes("skin", V, P, A, Vv) == 56 * V                          # K1
    assert bench.alg_bytes("normals+bucket", V, P, A, Vv) == 77 * V + 37 * V + 16 * P  # K2 + K3
    assert bench.alg_bytes("search+average", V, P, A, Vv) == 12 * P + 16 * Vv + 8 * P + 72 * V  # K4 + K5
    assert bench.alg_bytes("pose_system", V, P, A, Vv) == 4 * V + 61 * A           # K6
    assert bench.alg_bytes("shape_step", V, P, A, Vv) == 81 * V                    # K8
    assert bench.alg_bytes("pose_solve", V, P, A, Vv) == 0


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
