"""Print the device timeline (timed launches, csv from sdr_debug_timeline)
around its largest gaps: kernel, start / end (us from the first launch), gap
before. Usage: python tools/timeline_window.py gpurun_out/timeline_c3.csv [--around 3] [--before 6 --after 8]"""
import argparse

ap = argparse.ArgumentParser()
ap.add_argument("csv")
ap.add_argument("--around", type=int, default=3, help="windows around the N largest gaps")
ap.add_argument("--before", type=int, default=6)
ap.add_argument("--after", type=int, default=10)
args = ap.parse_args()
rows = []
with open(args.csv) as fh:
    next(fh)
    for ln in fh:
        n, a, e = ln.strip().split(",")
        rows.append((n, float(a), float(e)))
rows.sort(key=lambda r: r[1])
t0 = rows[0][1]
gaps = sorted(((rows[i][1] - rows[i - 1][2], i) for i in range(1, len(rows))), reverse=True)[: args.around]
for g, i in sorted(gaps, key=lambda x: x[1]):
    print(f"--- gap {g:.1f} us before launch {i}")
    for k in range(max(0, i - args.before), min(len(rows), i + args.after)):
        n, a, e = rows[k]
        gb = a - rows[k - 1][2] if k else 0.0
        print(f"  {n:16s} start {a - t0:10.1f} end {e - t0:10.1f} dur {e - a:8.1f} gap_before {gb:8.1f}")
