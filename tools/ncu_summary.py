"""Markdown summary of ncu --set full reports (one row per captured launch).

    python tools/ncu_summary.py gpurun_out/r01/full_*.ncu-rep > profiles/r01_ncu_full.md
"""
import csv
import io
import subprocess
import sys

COLS = [
    ("kernel", "Kernel Name", None),
    ("grid", "launch__grid_size", None),
    ("block", "launch__block_size", None),
    ("regs", "launch__registers_per_thread", None),
    ("time us", "gpu__time_duration.sum", "us"),
    ("dram rd MB", "dram__bytes_read.sum", "MB"),
    ("dram wr MB", "dram__bytes_write.sum", "MB"),
    ("L2 hit %", "lts__t_sector_hit_rate.pct", None),
    ("L2 req", "lts__t_requests_srcunit_tex.sum", None),
    ("atom sectors", "l1tex__m_xbar2l1tex_read_sectors_mem_global_op_atom.sum", None),
    ("red sectors", "l1tex__m_l1tex2xbar_write_sectors_mem_global_op_red.sum", None),
    ("L2 atomic busy %", "lts__d_atomic_input_cycles_active.avg.pct_of_peak_sustained_elapsed", None),
    ("warps active %", "sm__warps_active.avg.pct_of_peak_sustained_active", None),
    ("SM thru %", "sm__throughput.avg.pct_of_peak_sustained_elapsed", None),
    ("mem thru %", "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", None),
]
SCALE = {("us", "usecond"): 1, ("us", "us"): 1, ("us", "msecond"): 1e3, ("us", "nsecond"): 1e-3, ("MB", "byte"): 1e-6,
         ("MB", "Kbyte"): 1e-3, ("MB", "Mbyte"): 1, ("MB", "Gbyte"): 1e3}


def rows_of(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    hdr, units = r[0], r[1]
    for row in r[2:]:
        d = {}
        for name, metric, unit in COLS:
            if metric not in hdr:
                d[name] = "n/a"
                continue
            i = hdr.index(metric)
            v = row[i]
            if unit:
                try:
                    v = f"{float(v.replace(',', '')) * SCALE[(unit, units[i])]:.3f}"
                except (ValueError, KeyError):
                    v = f"{v} {units[i]}"
            elif name == "kernel":
                v = v.split("(")[0]
            d[name] = v
        yield d


def main():
    print("| " + " | ".join(c[0] for c in COLS) + " |")
    print("|" + "---|" * len(COLS))
    for rep in sys.argv[1:]:
        for d in rows_of(rep):
            print("| " + " | ".join(str(d[c[0]]) for c in COLS) + " |")


if __name__ == "__main__":
    main()
