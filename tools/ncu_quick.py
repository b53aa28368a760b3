"""Summary of one ncu report: headline metrics, top stalled SASS lines, and
the mbarrier wait loops. Usage: python tools/ncu_quick.py report.ncu-rep"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, vals = rows[0], rows[1], rows[2]
want = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed', 'sm__warps_active.avg.pct_of_peak_sustained_active',
        'launch__registers_per_thread', 'launch__grid_size', 'launch__block_size', 'smsp__inst_executed.sum',
        'smsp__issue_active.avg.pct_of_peak_sustained_active', 'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum',
        'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum', 'sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active',
        'l1tex__throughput.avg.pct_of_peak_sustained_active', 'lts__t_bytes.sum']
for w in want:
    if w in hdr:
        i = hdr.index(w)
        print(f"{w:60s} {vals[i]} {units[i]}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
srows = list(csv.reader(io.StringIO(src)))
h = srows[1]
data = srows[2:]
ia, isrc, iss = h.index("Instructions Executed"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
tot = sum(float(r[ia] or 0) for r in data)
stall = sum(float(r[iss] or 0) for r in data)
print(f"sass instructions executed {tot:.4g}, stall samples {stall:.4g}")
for r in sorted(data, key=lambda r: -float(r[iss] or 0))[:int(sys.argv[2]) if len(sys.argv) > 2 else 12]:
    print(f"  {r[iss]:>7s} {r[ia]:>10s} {r[isrc]}")
for k, r in enumerate(data):
    if 'TRYWAIT' in r[isrc]:
        print("  wait", k, r[ia], r[iss], r[isrc])
