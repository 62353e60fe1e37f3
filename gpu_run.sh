#!/bin/bash
for t in 64 128 256 512; do echo "target $t"; TENKIT_QR_TARGET_ROWS=$t timeout 120 python tools/qr_bench.py | head -3; done
