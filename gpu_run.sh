#!/bin/bash
timeout 60 ./tools/qr_trace_new | grep -E "fast"
timeout 120 python tools/qr_bench.py
timeout 400 python -m pytest tests -m gpu -q -x -k "qr or basis or golden or parity or dist or edge" 2>&1 | tail -2
