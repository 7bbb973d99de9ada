"""DRAM bytes per fit step with the L2 left warm between kernels, from an ncu
metrics CSV of consecutive fit-step launches taken with --cache-control none:

  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
      --cache-control none --clock-control none -k <fit-step kernels> -s S -c C --csv \
      --log-file warm.csv python tools/step_probe.py 3 1
  python tools/warm_dram.py warm.csv LAUNCHES_PER_STEP "command" > profiles/r2_warm_dram.json

LAUNCHES_PER_STEP = launches of each kernel class per fit step (2 in the split
step: one per half of the group).  Per step = the per-launch average x that, so
the window need not cover whole steps.  Also writes the design's inherent bytes
per step (cfg2) for comparison."""
import collections
import csv
import json
import sys

path, lps, cmd = sys.argv[1], float(sys.argv[2]), sys.argv[3]
rows = [r for r in csv.reader(open(path)) if r]
hdr = next(r for r in rows if r[0] == "ID")
per = collections.OrderedDict()
for r in rows[rows.index(hdr) + 1:]:
    if len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    name = d["Kernel Name"].split("(")[0].replace("void ", "").replace("inr::", "")
    key = (d["ID"], name)
    v = float(d["Metric Value"].replace(",", ""))
    unit = d["Metric Unit"]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "nsecond": 1e-3, "us": 1.0,
             "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(unit, 1.0)
    per.setdefault(key, {})[d["Metric Name"]] = v * scale
agg = collections.OrderedDict()
for (i, name), m in per.items():
    a = agg.setdefault(name, {"launches": 0, "dram_read_bytes": 0.0, "dram_write_bytes": 0.0, "us": 0.0})
    a["launches"] += 1
    a["dram_read_bytes"] += m.get("dram__bytes_read.sum", 0.0)
    a["dram_write_bytes"] += m.get("dram__bytes_write.sum", 0.0)
    a["us"] += m.get("gpu__time_duration.sum", 0.0)
total = sum((a["dram_read_bytes"] + a["dram_write_bytes"]) / a["launches"] * lps for a in agg.values())
# cfg2: 8 blocks of 12 177 491 parameters (inr_param_count) and 81 920 coordinates per block-step
P, nb, coords = 12177491, 8, 81920
design = {"adam_28B_per_param": 28.0 * P * nb, "gradient_zeroing_4B": 4.0 * P * nb,
          "encode_table_reads_4B": 4.0 * P * nb, "scatter_gradient_rmw_8B": 8.0 * P * nb,
          "texels_feature_tiles_samples": 167772160}
design["total"] = sum(design.values())
design["note"] = ("the traffic this design needs when the 1.56 GB per-GPU working set cannot stay in the 126 MB L2 "
                  "across kernels (parameters re-read by the next encode, gradients zeroed, scattered and read once "
                  "each)")
out = {"command": cmd, "launches_per_step": lps,
       "per_launch": {k: {"launches_seen": a["launches"], "dram_read_bytes": a["dram_read_bytes"] / a["launches"],
                          "dram_write_bytes": a["dram_write_bytes"] / a["launches"], "us": a["us"] / a["launches"]}
                      for k, a in agg.items()},
       "dram_bytes_per_step": total, "design_bytes_per_step": design,
       "dram_over_design": total / design["total"],
       "dram_over_strict_algorithmic": total / (32.0 * P * nb + 32.0 * coords * nb)}
print(json.dumps(out, indent=1))
