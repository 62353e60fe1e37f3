#!/bin/bash
for g in 148 96 64 32 16; do echo "grid $g"; TENKIT_FFCP_GRID=$g timeout 120 python tools/ffcp_bench.py 200 2>&1 | grep -E "persistent" | grep -v max; done
