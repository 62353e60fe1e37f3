#!/bin/bash
# One-pass-per-step mode (the reference's structure) with and without the persistent TTM.
for v in 1 0; do
  TENKIT_TC_PERSIST=$v python bench.py --one-pass-per-step --steps 20 --no-e2e --no-cpu 2>/dev/null | tail -1 > /tmp/opps_$v.json
  python - "$v" <<'PY'
import json, sys
d = json.load(open(f"/tmp/opps_{sys.argv[1]}.json"))
print("persist", sys.argv[1], d["ms_per_step"], d["config"]["passes_per_step"], d["roofline"]["frac"])
PY
done
