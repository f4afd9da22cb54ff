"""Summarise an ncu --set full report: per kernel time, DRAM bytes, throughput
and occupancy counters.   python tools/ncu_summary.py <report.ncu-rep>"""
import csv
import io
import subprocess
import sys

WANT = [
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "dram_rd"),
    ("dram__bytes_write.sum", "dram_wr"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram%"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm%"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "l1%"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "l2%"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64%"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps%"),
    ("launch__registers_per_thread", "regs"),
    ("launch__block_size", "block"),
    ("launch__grid_size", "grid"),
    ("launch__shared_mem_per_block_dynamic", "smem"),
]

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, units = rows[0], rows[1]
print("| kernel | " + " | ".join(s for _, s in WANT) + " |")
print("|---" * (len(WANT) + 1) + "|")
for r in rows[2:]:
    name = r[hdr.index("Kernel Name")].split("(")[0].replace("void ", "")
    cells = []
    for m, _ in WANT:
        if m in hdr:
            i = hdr.index(m)
            cells.append(f"{r[i]} {units[i]}".strip())
        else:
            cells.append("-")
    print(f"| {name} | " + " | ".join(cells) + " |")
