#!/bin/bash
timeout 120 python tools/ffcp_exp.py 2>&1 | grep -E "mode-step|ldlt cycles"
timeout 120 python tools/ffcp_bench.py 200 2>&1 | grep -E "persistent|max"
timeout 300 python -m pytest tests -m gpu -q -x -k "ffcp or golden or cpp or fit" 2>&1 | tail -1
