#!/bin/bash
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -1
for v in 2 1; do echo "ROWPAR=$v"; TENKIT_QR_ROWPAR=$v timeout 120 ./tools/qr_trace 2>&1 | grep -E "1000x30"; done
for v in 2 1 2 1; do echo "ROWPAR=$v"; TENKIT_QR_ROWPAR=$v python tools/phase_bench.py 2>&1 | grep phases | tail -1; done
