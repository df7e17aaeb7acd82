"""profiles/r02_sass_counts.md: per-kernel SASS instruction counts of the built
objects (cuobjdump -sass): 256-bit loads / stores, fp64 ops, MUFU, shuffles,
RED / ATOM. Run after `python -m paper_1711_07999_b200.build`."""
import collections
import re
import subprocess
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
KERNELS = ("k_skin", "k_normals", "k_search", "k_scatter", "k_pixoff", "k_pose_system", "k_pose_solve", "k_shape",
           "k_ingest", "k_fk")
out = ["# SASS evidence (cuobjdump -sass of the built objects, sm_100a)", "",
       "Per kernel: 256-bit global loads/stores (`LDG.E.ENL2.256` / `STG.E.ENL2.256`, the `ld256`/`st256`",
       "helpers of wt_kernels.cuh), all global loads/stores, fp64 FMA/MUL/ADD, MUFU (rcp64h/rsq64h), shuffles,",
       "fire-and-forget reductions (`RED`/`REDG`) and returning atomics (`ATOM`; `ATOMS` = the shared-memory",
       "CAS fallback a generic atomic carries). Regenerate: `python tools/sass_counts.py`.", "",
       "| kernel | LDG.256 | STG.256 | LDG all | STG all | DFMA | DMUL | DADD | MUFU | SHFL | RED | ATOM | ATOMS | instructions |",
       "|---|---|---|---|---|---|---|---|---|---|---|---|---|---|"]
for obj in ("wt_gpu.o", "wt_exact.o"):
    txt = subprocess.run(["cuobjdump", "-sass", str(ROOT / "paper_1711_07999_b200/_build" / obj)], capture_output=True,
                         text=True).stdout
    for m in re.finditer(r"Function : (\S+)\n(.*?)(?=\n\s*Function : |\Z)", txt, re.S):
        dem = subprocess.run(["c++filt", m.group(1)], capture_output=True, text=True).stdout.strip()
        dem = re.sub(r"\(.*", "", dem).replace("wt::", "").replace("void ", "")
        if not any(k in dem for k in KERNELS):
            continue
        c = collections.Counter()
        for ins in re.findall(r"/\*[0-9a-f]{4}\*/\s+([^;]*);", m.group(2)):
            t = ins.split()
            op = t[1] if t and t[0].startswith("@") else (t[0] if t else "")
            c["all"] += 1
            if op.startswith("LDG"):
                c["ldg"] += 1
                c["ldg256"] += ".256" in op
            if op.startswith("STG"):
                c["stg"] += 1
                c["stg256"] += ".256" in op
            for k in ("DFMA", "DMUL", "DADD", "MUFU", "SHFL"):
                c[k] += op.startswith(k)
            c["RED"] += op.startswith("RED")
            c["ATOMS"] += op.startswith("ATOMS")
            c["ATOM"] += op.startswith("ATOM") and not op.startswith("ATOMS")
        out.append(f"| {dem} | {c['ldg256']} | {c['stg256']} | {c['ldg']} | {c['stg']} | {c['DFMA']} | {c['DMUL']} | "
                   f"{c['DADD']} | {c['MUFU']} | {c['SHFL']} | {c['RED']} | {c['ATOM']} | {c['ATOMS']} | {c['all']} |")
(ROOT / "profiles" / "r02_sass_counts.md").write_text("\n".join(out) + "\n")
print("\n".join(out))
