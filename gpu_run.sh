#!/bin/bash
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k repeated 2>&1 | tail -2
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -1
