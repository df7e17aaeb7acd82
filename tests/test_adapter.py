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
