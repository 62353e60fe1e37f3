#!/bin/bash
timeout 400 python -m pytest tests/test_gpu_parity.py -q -k "edge or limit" 2>&1 | tail -15
