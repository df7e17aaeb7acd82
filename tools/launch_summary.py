"""Per-kernel share of device time from an ncu launch list
(--metrics gpu__time_duration.sum --csv). Launches are cold-cache and
serialised under ncu, so compare SHARES with the in-graph event timing of
bench.py, not absolutes.

    python tools/launch_summary.py gpurun_out/r01b/launches.csv > profiles/r01_launches.md
"""
import collections
import csv
import sys

SCALE = {"ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3}
TRACK = ("k_fk", "k_ingest", "k_skin<", "k_skin(", "k_normals", "k_pixoff", "k_scatter", "k_search", "k_pose_system",
         "k_pose_solve", "k_shape<", "k_shape(", "k_shape_after", "k_record")


def main(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ik, iv, im, iu = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Name"), h.index("Metric Unit")
    agg = collections.OrderedDict()
    for r in rows[hi + 1:]:
        if len(r) <= iv or r[im] != "gpu__time_duration.sum":
            continue
        name = r[ik].split("(")[0].replace("wt::", "").replace("void ", "")
        full = r[ik]
        us = float(r[iv].replace(",", "")) * SCALE.get(r[iu], 1.0)
        tracked = any(t in full for t in TRACK)
        a = agg.setdefault(name, [0, 0.0, tracked])
        a[0] += 1
        a[1] += us
    tot = sum(a[1] for a in agg.values() if a[2])
    print(f"Launch list: `{path}` (ncu --metrics gpu__time_duration.sum, --clock-control none).")
    print("Tracking kernels only in the share column; renderer / torch kernels listed for completeness.\n")
    print("| kernel | launches | total us | mean us | share of tracking time |")
    print("|---|---|---|---|---|")
    for name, (n, us, tracked) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        share = f"{100 * us / tot:.1f} %" if tracked else "-"
        print(f"| {name} | {n} | {us:.1f} | {us / n:.2f} | {share} |")


if __name__ == "__main__":
    main(sys.argv[1])
