"""Summarise an ncu --metrics gpu__time_duration.sum launch list: per-kernel time of the
last `--steps` decomposition steps (identified by the Y-streaming TTM launches)."""
import collections
import csv
import sys

path = sys.argv[1]
nsteps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
rows = [r for r in csv.reader(open(path)) if r]
hdr = None
data = []
for r in rows:
    if r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d["Metric Name"] == "gpu__time_duration.sum":
            data.append((d["Kernel Name"], d["Grid Size"], float(d["Metric Value"].replace(",", ""))))
# tkb kernels only, last nsteps * (launches per step)
tk = [x for x in data if "tkb::" in x[0]]
thr = float(sys.argv[4]) if len(sys.argv) > 4 else 200000.0  # ns: a launch at least this long is a Y pass
big = [i for i, x in enumerate(tk) if ("ttm_mmajor" in x[0] or "ttm_tc" in x[0] or "ttm_stream" in x[0]) and x[2] > thr]
per_step = int(sys.argv[3]) if len(sys.argv) > 3 else 3  # Y passes per decomposition (grouped)
start = big[-per_step * nsteps] if len(big) >= per_step * nsteps else 0
win = tk[start:]
tot = collections.defaultdict(float)
cnt = collections.Counter()
for name, grid, v in win:
    short = name.split("(")[0].replace("void ", "").replace("tkb::<unnamed>::", "")
    tot[short] += v
    cnt[short] += 1
s = sum(tot.values())
for n, v in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"{v / 1e6 / nsteps:9.4f} ms/step {100 * v / s:5.1f}%  x{cnt[n] / nsteps:5.1f}/step  {n}")
print(f"total {s / 1e6 / nsteps:.4f} ms/step (serialised, cold-cache ncu timings)")
