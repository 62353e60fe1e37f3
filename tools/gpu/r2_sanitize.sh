#!/bin/bash
# compute-sanitizer over the round-2 code paths: blocked tall QR, two-q tiles, host-input landing
mkdir -p gpurun_out
cat > /tmp/san_case.py <<'PY'
import os, sys
import numpy as np
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import paper_1412_1885_b200 as P
from oracle import pyoracle as O
O.build()
which = sys.argv[1]
if which == "tall":
    z = O.gaussian_matrix(7000, 60, (1, 2))
    u, mg = P.orthonormal_basis(z, with_margins=True)
    ur = O.fix_column_signs(O.orthonormal_basis(z))
    print("tall max diff", float(np.max(np.abs(u - ur))), mg)
elif which == "bq":
    t = O.gaussian_matrix(640 * 64 * 301, 1, (5, 1)).reshape((640, 64, 301), order="F").astype(np.float32)
    m = O.gaussian_matrix(40, 64, (6, 1))
    ctx = P.Context.default(); ctx.set_ttm_path("stream")
    got = P.ttm(P.DenseTensor.from_numpy(t, np.float32), m, 1)
    ref = O.ttm(t.astype(np.float64), m, 1)
    print("bq rel", float(np.linalg.norm(got - ref) / np.linalg.norm(ref)))
elif which == "land":
    y = O.add_noise(O.gen_tucker((416, 400, 208), (10, 10, 10), (8, 3)), 20.0, (8, 4)).astype(np.float32)
    m = P.rand_tucker_2i(P.DenseTensor.from_numpy(y, np.float32), (12, 12, 12), 8, (7, 4), sync_ranks=False, out="host")
    print("land passes", m.stats["passes"], "launches", m.stats["kernel_launches"])
PY
for c in tall bq land; do
  for tool in memcheck racecheck; do
    timeout 900 compute-sanitizer --tool $tool --kernel-regex kns=tall,kns=ttm_stream,kns=qr_colpiv python /tmp/san_case.py $c > gpurun_out/san_${c}_$tool.log 2>&1
    echo "$c $tool rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/san_${c}_$tool.log | tail -1) | $(grep -E 'max diff|rel |passes' gpurun_out/san_${c}_$tool.log | tail -1 | cut -c1-120)"
  done
done
