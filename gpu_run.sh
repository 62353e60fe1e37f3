#!/bin/bash
timeout 400 python -m pytest tests/test_gpu_dist.py -q -x 2>&1 | tail -3
timeout 400 python -m pytest tests -m gpu -q -x -k "rand_tucker or alg2 or config1 or golden" 2>&1 | tail -2
