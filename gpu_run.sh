#!/bin/bash
timeout 300 python tools/alg2_bench.py
timeout 400 python -m pytest tests -m gpu -q -x -k "rand_tucker or alg2 or config1 or golden" 2>&1 | tail -2
