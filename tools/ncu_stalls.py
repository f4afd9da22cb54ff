"""Top warp-stall reasons and a few pipe counters per kernel of an ncu report."""
import csv
import io
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[0]
for r in rows[2:]:
    name = r[hdr.index("Kernel Name")][:60]
    st = [(hdr[i].replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""), float(r[i]))
          for i in range(len(hdr)) if hdr[i].startswith("smsp__average_warps_issue_stalled_")
          and hdr[i].endswith("_per_issue_active.ratio") and r[i] not in ("", "n/a")]
    st.sort(key=lambda t: -t[1])
    print(name)
    print("  stalls: " + " ".join(f"{a}={b:.2f}" for a, b in st[:8]))
    for m in ["gpu__time_duration.sum", "smsp__inst_executed.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
              "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
              "l1tex__throughput.avg.pct_of_peak_sustained_active", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
              "dram__bytes_read.sum", "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct",
              "launch__registers_per_thread", "launch__occupancy_limit_registers"]:
        if m in hdr:
            print(f"  {m} = {r[hdr.index(m)]}")
