"""Compact text summary of ncu reports (for profiles/).

    python tools/ncu_summary.py gpurun_out/prof_*.ncu-rep > profiles/ncu_<round>.txt
"""
import csv
import io
import subprocess
import sys

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram % of peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM % of peak"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__shared_mem_per_block_dynamic", "dyn smem/block"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("smsp__average_warp_latency_per_inst_issued.ratio", "cycles/issued inst"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("lts__t_sector_hit_rate.pct", "L2 hit %"),
]


def summarize(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        return f"{path}: no data\n"
    h, u = rows[0], rows[1]
    s = []
    for v in rows[2:]:
        name = v[h.index("Kernel Name")].split("(")[0]
        s.append(f"== {path}\n   kernel: {name}")
        for m, label in METRICS:
            if m in h:
                i = h.index(m)
                s.append(f"   {label:24s} {v[i]} {u[i]}")
        rd = wr = None
        for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            if m in h:
                i = h.index(m)
                scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u[i], 1)
                val = float(v[i]) * scale
                rd, wr = (val, wr) if m.endswith("read.sum") else (rd, val)
        if rd is not None and wr is not None:
            s.append(f"   {'traffic (r+w) bytes':24s} {rd + wr:.0f}")
    return "\n".join(s) + "\n"


if __name__ == "__main__":
    for p in sys.argv[1:]:
        sys.stdout.write(summarize(p))
