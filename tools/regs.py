"""Registers / spills / smem per kernel from ptxas -v (no GPU needed).

    python tools/regs.py [repo_root] [unit.cu ...]
"""
import os
import re
import subprocess
import sys
from pathlib import Path

root = Path(sys.argv[1]) if len(sys.argv) > 1 else Path(__file__).resolve().parents[1]
units = sys.argv[2:] or ["wt_gpu.cu", "wt_exact.cu"]
for u in units:
    cmd = ["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17",
           "-I", str(root / "include"), "-I", str(root / "paper_1711_07999_b200/csrc"), "--expt-relaxed-constexpr",
           *os.environ.get("WT_NVCC_FLAGS", "").split(), "-Xptxas", "-v", "-c", str(root / "paper_1711_07999_b200/csrc" / u), "-o", "/dev/null"]
    if u != "wt_gpu.cu":
        cmd.insert(-4, "-fmad=false")
    out = subprocess.run(cmd, capture_output=True, text=True).stderr
    name = None
    for line in out.splitlines():
        m = re.search(r"Compiling entry function '(\S+)'", line)
        if m:
            name = subprocess.run(["c++filt"], input=m.group(1), capture_output=True, text=True).stdout.strip()
            name = re.sub(r"\(.*", "", name).replace("wt::", "")
            spill = ""
        m2 = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
        if m2 and (m2.group(1) != "0" or m2.group(2) != "0"):
            spill = f" spill {m2.group(1)}/{m2.group(2)}"
        m3 = re.search(r"Used (\d+) registers", line)
        if m3 and name:
            print(f"{name:50s} {m3.group(1):>4s} regs{spill}")
            name = None
