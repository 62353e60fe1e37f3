"""Print the launches of the last decomposition step from an ncu --metrics
gpu__time_duration.sum --csv launch list (tkb kernels only): python tools/step_launches.py FILE [passes]"""
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if r]
npass = int(sys.argv[2]) if len(sys.argv) > 2 else 3
hdr, data = None, []
for r in rows:
    if r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d["Metric Name"] == "gpu__time_duration.sum":
            name = d["Kernel Name"].split("(")[0].replace("void ", "").replace("tkb::<unnamed>::", "")
            data.append((name, d["Grid Size"], float(d["Metric Value"].replace(",", ""))))
ours = [x for x in data if not x[0].startswith("at::")]
big = [i for i, x in enumerate(ours) if x[2] > 300000]
start = big[-npass] - 3 if len(big) >= npass else 0
tot = 0.0
for name, grid, ns in ours[start:]:
    tot += ns
    print(f"{ns / 1000:9.1f} us  {grid:>16}  {name[:70]}")
print(f"total {tot / 1000:.1f} us (serialised, ncu)")
