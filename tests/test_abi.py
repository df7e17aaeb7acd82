"""The drop-in boundary on CPU: libwt_gpu.so loads, exports every entry point
include/wt_gpu.h declares, its struct layouts agree with the ctypes mirror,
and without a GPU the product path fails loudly (no CPU fallback)."""
import ctypes as C
import re
import subprocess
from pathlib import Path

import numpy as np
import pytest

from paper_1711_07999_b200 import _lib as W

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "wt_gpu.h"


def declared():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    text = re.sub(r"//[^\n]*", "", text)
    return sorted(set(re.findall(r"\b(wt_gpu_\w+)\s*\(", text)))


def test_header_declares_the_surface():
    names = declared()
    for must in ("wt_gpu_create", "wt_gpu_destroy", "wt_gpu_set_state", "wt_gpu_get_state", "wt_gpu_track_frame",
                 "wt_gpu_optimize_pose", "wt_gpu_optimize_shape", "wt_gpu_skin", "wt_gpu_associate",
                 "wt_gpu_normal_system", "wt_gpu_solve_step", "wt_gpu_last_error"):
        assert must in names


def test_library_exports_every_declared_symbol():
    lib = C.CDLL(str(W.LIB_PATH))
    missing = [n for n in declared() if not hasattr(lib, n)]
    assert not missing, missing
    assert set(W.EXPORTS) <= set(declared())


def test_nm_shows_c_linkage():
    out = subprocess.run(["nm", "-D", "--defined-only", str(W.LIB_PATH)], capture_output=True, text=True,
                         check=True).stdout
    syms = {ln.split()[-1] for ln in out.splitlines() if ln.strip()}
    assert set(declared()) <= syms  # unmangled: extern "C"


STRUCTS = {
    "wt_intrinsics": W.Intrinsics, "wt_kin_config": W.KinConfig, "wt_shape_config": W.ShapeConfig,
    "wt_assoc_config": W.AssocConfig, "wt_track_config": W.TrackConfigC, "wt_kin_iter_stats": W.KinIterStats,
    "wt_shape_iter_stats": W.ShapeIterStats, "wt_frame_stats": W.FrameStatsC, "wt_noise": W.Noise,
    "wt_model_desc": W.ModelDesc,
}


def test_struct_layouts_match_ctypes(tmp_path):
    src = ['#include <stdio.h>', '#include <stddef.h>', '#include "wt_gpu.h"', "int main(void) {"]
    for cname, py in STRUCTS.items():
        src.append(f'  printf("{cname} size %zu\\n", sizeof({cname}));')
        for fname, _ in py._fields_:
            src.append(f'  printf("{cname} {fname} %zu\\n", offsetof({cname}, {fname}));')
    src.append("  return 0; }")
    c = tmp_path / "layout.c"
    c.write_text("\n".join(src))
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-std=c11", "-I", str(ROOT / "include"), str(c), "-o", str(exe)], check=True)
    got = {}
    for ln in subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.splitlines():
        s, f, v = ln.split()
        got[(s, f)] = int(v)
    for cname, py in STRUCTS.items():
        assert got[(cname, "size")] == C.sizeof(py), cname
        for fname, _ in py._fields_:
            assert got[(cname, fname)] == getattr(py, fname).offset, (cname, fname)


def test_abi_version_and_no_fallback_without_gpu():
    lib = W.lib()
    assert lib.wt_gpu_abi_version() == W.ABI_VERSION
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    assert lib.wt_gpu_device_count() == 0
    from paper_1711_07999_b200.tracker import Intrinsics, Tracker
    from tests.rigs import slider_triangle
    with pytest.raises(W.WarptrackError):
        Tracker(slider_triangle(), Intrinsics())


def test_null_and_invalid_arguments_are_rejected():
    lib = W.lib()
    assert lib.wt_gpu_set_state(None, None, None, 0) == W.WT_EINVAL
    assert lib.wt_gpu_track_loaded(None, None, None) == W.WT_EINVAL
    ctx = C.c_void_p()
    assert lib.wt_gpu_create(0, None, None, C.byref(ctx)) == W.WT_EINVAL
    assert not ctx.value
    assert lib.wt_gpu_solve_step(0, -1, None, None, 0.0, 0.0, None) in (W.WT_EINVAL, W.WT_ELENGTH)
    assert isinstance(lib.wt_gpu_global_last_error(), bytes)


def test_model_validation_before_device_use():
    """Invalid descriptors are rejected with WT_EINVAL/WT_ELENGTH regardless
    of the device (validate_model mirrors Skeleton::build / finalize checks)."""
    from tests.rigs import slider_triangle
    b = slider_triangle()
    b.parent = np.array([3], np.int32)  # parent out of range
    desc, keep = b.to_desc()
    ctx = C.c_void_p()
    rc = W.lib().wt_gpu_create(0, C.byref(desc), C.byref(W.Intrinsics(1, 1, 0, 0, 4, 4)), C.byref(ctx))
    assert rc in (W.WT_EINVAL, W.WT_ELENGTH)
    assert b"parent" in W.lib().wt_gpu_global_last_error()
