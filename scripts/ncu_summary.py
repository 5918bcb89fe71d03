"""Summarise an ncu report (raw page): per-kernel time, DRAM bytes, issue, stalls."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "smsp__thread_inst_executed_per_inst_executed.ratio",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "l1tex__t_sector_hit_rate.pct", "launch__grid_size", "launch__block_size"]
for r in rows[2:]:
    name = r[hdr.index("Kernel Name")]
    print(f"== {name[:60]}")
    for w in want:
        if w in hdr:
            i = hdr.index(w)
            print(f"   {w} = {r[i]} {units[i]}")
    st = []
    for i, h in enumerate(hdr):
        if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
            try:
                st.append((h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")], float(r[i])))
            except ValueError:
                pass
    st.sort(key=lambda x: -x[1])
    print("   stalls/issue: " + ", ".join(f"{k} {v:.2f}" for k, v in st[:8]))
