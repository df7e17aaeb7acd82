"""Warp-stall samples aggregated per CUDA source line from
`ncu -i rep --page source --csv --print-source cuda,sass` output (needs -lineinfo).

    ncu -i rep --page source --csv --print-source cuda,sass -k regex:k_pose > /tmp/x.csv
    python tools/ncu_lines.py /tmp/x.csv [top]
"""
import csv
import sys
from collections import defaultdict


def main(path, top=30):
    rows = list(csv.reader(open(path)))
    agg = defaultdict(lambda: [0.0, defaultdict(float), ""])
    fname = "?"
    line = None
    src = ""
    hdr = None
    for r in rows:
        if len(r) >= 2 and r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if len(r) > 3 and r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or len(r) < 5:
            continue
        if r[0]:  # a source line row
            line, src = r[0], r[1]
            continue
        # sass row under the current line
        try:
            v = float(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
        except (ValueError, IndexError):
            continue
        key = (fname, line)
        agg[key][0] += v
        agg[key][2] = src
        for i, h in enumerate(hdr):
            if h.startswith("stall_") and "Not Issued" not in h and i < len(r) and r[i] not in ("", "0"):
                try:
                    agg[key][1][h] += float(r[i])
                except ValueError:
                    pass
    tot = sum(a[0] for a in agg.values()) or 1.0
    print(f"total samples {tot:.0f}")
    for (f, l), (v, st, s) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
        stalls = sorted(st.items(), key=lambda kv: -kv[1])[:2]
        st_s = " ".join(f"{k[6:]}={100 * x / v:.0f}%" for k, x in stalls) if v else ""
        print(f"{100 * v / tot:5.1f}%  {f}:{l:<5} {s.strip()[:70]:70s} {st_s}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30)
