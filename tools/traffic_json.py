"""profiles/traffic.json from ncu `--set full` frame captures summarised by
tools/ncu_summary.py: DRAM bytes (read + write) per launch of each bench
kernel kind, averaged over the captured launches.

    python tools/traffic_json.py c3=profiles/r01_ncu_c3_frame.md c5=profiles/r01_ncu_c5_frame.md > profiles/traffic.json
"""
import collections
import json
import sys

KIND = {"k_skin": "skin", "k_normals": "normals+bucket", "k_pixoff": "pixoff", "k_scatter": "scatter",
        "k_search": "search+average", "k_pose_system": "pose_system", "k_pose_solve": "pose_solve",
        "k_shape": "shape_step", "k_shape_after": "shape_stats", "k_fk": "fk", "k_ingest": "ingest"}


def parse(path):
    rows = [l.strip().strip("|").split("|") for l in open(path) if l.startswith("|")]
    hdr = [h.strip() for h in rows[0]]
    ik, ird, iwr = hdr.index("kernel"), hdr.index("dram rd MB"), hdr.index("dram wr MB")
    acc = collections.defaultdict(lambda: [0.0, 0])
    for r in rows[2:]:
        name = r[ik].strip().replace("void ", "").split("<")[0]
        kind = KIND.get(name)
        if not kind:
            continue
        a = acc[kind]
        a[0] += (float(r[ird]) + float(r[iwr])) * 1e6
        a[1] += 1
    return {k: {"dram_bytes_per_launch": v[0] / v[1], "launches_captured": v[1]} for k, v in acc.items()}


def main():
    out = {"source": "ncu --set full --clock-control none (default cache control: caches flushed before "
                     "every replayed launch, so these are cold-cache DRAM bytes)"}
    for arg in sys.argv[1:]:
        cfg, path = arg.split("=", 1)
        out[cfg] = parse(path)
        out[cfg]["_file"] = path
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
