"""Summarise an ncu report (raw page) for the hot kernels: duration, DRAM
bytes, throughput, occupancy and the top stall reasons."""
import csv
import subprocess
import sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr, units = rows[0], rows[1]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "launch__registers_per_thread", "launch__grid_size", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "lts__t_bytes.sum", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum"]
stall_cols = [i for i, h in enumerate(hdr) if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued")]
for r in rows[2:]:
    name = r[hdr.index("Kernel Name")].split("(")[0][-40:]
    print(f"== {name}")
    for w in want:
        if w in hdr:
            i = hdr.index(w)
            print(f"   {w:60s} {r[i]:>14s} {units[i]}")
    st = []
    for i in stall_cols:
        try:
            st.append((float(r[i]), hdr[i].replace("smsp__pcsamp_warps_issue_stalled_", "")))
        except ValueError:
            pass
    st.sort(reverse=True)
    tot = sum(v for v, _ in st) or 1.0
    print("   stall samples:", ", ".join(f"{n}={100 * v / tot:.0f}%" for v, n in st[:7]))
