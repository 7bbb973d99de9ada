"""Per-CUDA-source-line instruction and stall-sample totals from an ncu report
(ncu -i REP --page source --csv --print-source cuda,sass).

  python tools/ncu_lines.py REP [per-unit divisor] [top N] [kernel-name regex]
"""
import csv, io, subprocess, sys

rep = sys.argv[1]
div = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
kfilt = ["-k", "regex:" + sys.argv[4]] if len(sys.argv) > 4 else []
out = subprocess.run(["ncu", "-i", rep] + kfilt + ["--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
fname, cur, hdr = None, None, None
agg = {}
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if not hdr or len(r) != len(hdr):
        continue
    if r[0]:
        cur = (fname, r[0], r[1][:90])
        continue
    d = dict(zip(hdr[2:], r[2:]))
    try:
        n = float(d["Instructions Executed"] or 0)
        s = float(d["Warp Stall Sampling (All Samples)"] or 0)
    except (KeyError, ValueError):
        continue
    a = agg.setdefault(cur, [0.0, 0.0])
    a[0] += n
    a[1] += s
tn = sum(v[0] for v in agg.values()) or 1
ts = sum(v[1] for v in agg.values()) or 1
print(f"total instructions / unit: {tn / div:.0f}")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{v[0] / div:8.0f} {100 * v[0] / tn:5.1f}% inst {100 * v[1] / ts:5.1f}% stall  {k[0]}:{k[1]}  {k[2]}")
