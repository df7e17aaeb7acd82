"""Top SASS instructions by warp-stall samples from an ncu source-page CSV."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ia, isrc, iss = hdr.index("Address"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_")]
data = []
for r in rows[2:]:
    try:
        data.append((float(r[iss] or 0), r[ia], r[isrc], {hdr[i]: r[i] for i in stall_cols if r[i] not in ("", "0")}))
    except (ValueError, IndexError):
        pass
tot = sum(d[0] for d in data)
print("total samples", tot)
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
for s, a, src, st in sorted(data, key=lambda d: -d[0])[:n]:
    top = sorted(st.items(), key=lambda kv: -float(kv[1]))[:3]
    print(f"{100*s/tot:5.1f}% {a} {src[:60]:60s} {top}")
