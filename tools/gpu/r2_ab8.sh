#!/bin/bash
# blocked (TSQR) QR path forced for sketches above N rows (TENKIT_QR_TALL_ABOVE) vs the cluster QR:
# parity, per-launch time at 2400x40 / 4000x60, cfg5slab and cfg3 steps
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo "build rc=$?"
TENKIT_QR_TALL_ABOVE=1500 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_qr_margins.py -m gpu -q > gpurun_out/tall_tests.log 2>&1; echo "tests (tall above 1500) rc=$?"; grep -E "^E |passed|failed|^FAILED" gpurun_out/tall_tests.log | head -20
for v in 0 1500 3000; do echo "TALL_ABOVE=$v"; TENKIT_QR_TALL_ABOVE=$v timeout 120 ./tools/qr_trace 2>&1 | grep -E "per launch"; done
for C in cfg5slab cfg3; do
  for v in 0 1500; do
    TENKIT_QR_TALL_ABOVE=$v timeout 600 python tools/phase_bench.py $C 2>&1 | grep "tenkit phases" | tail -1 | sed "s/^/$C tall_above=$v /"
  done
done
