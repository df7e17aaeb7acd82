"""The reference's own C++ API (track_frame, optimize_pose, optimize_shape,
run_tracking) executed through the GPU adapter (adapter/warptrack_gpu.*)
against the unmodified reference CPU implementation: tests/cpp/adapter_check.cpp,
built by `make -C oracle/ref adapter` next to oracle/_ref/libwtref.so."""
import subprocess
from pathlib import Path

import pytest

EXE = Path(__file__).resolve().parents[1] / "oracle" / "_ref" / "adapter_check"

pytestmark = [pytest.mark.gpu, pytest.mark.ref]


def test_reference_api_through_gpu_adapter(tmp_path):
    if not EXE.exists():
        pytest.skip("adapter_check not built (make -C oracle/ref adapter)")
    r = subprocess.run([str(EXE), str(tmp_path)], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "FAIL" not in r.stdout


ACC = Path(__file__).resolve().parents[1] / "oracle" / "_ref" / "acceptance_gpu"


@pytest.mark.timeout(1800)
def test_reference_acceptance_suite_through_gpu_adapter(tmp_path):
    """The reference's own acceptance suite (proj/tests/acceptance.cpp, compiled
    unmodified) with its tracking calls -- :165 and :724 track_frame, :541
    optimize_pose, :647 run_tracking -- routed to warptrack::gpu by a
    force-included header (tests/cpp/route_to_gpu.hpp): all 9 criteria,
    including criterion 9's throughput bars, must PASS on the GPU path."""
    if not ACC.exists():
        pytest.skip("acceptance_gpu not built (make -C oracle/ref adapter)")
    env = dict(__import__("os").environ, TMPDIR=str(tmp_path))
    r = subprocess.run([str(ACC)], capture_output=True, text=True, timeout=1700, env=env)
    print(r.stdout)
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith(("PASS", "FAIL"))]
    assert len(lines) == 9, r.stdout + r.stderr
    assert r.returncode == 0 and all(ln.startswith("PASS") for ln in lines), r.stdout + r.stderr
