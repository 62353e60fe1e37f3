#!/bin/bash
# full-size oracle parity at seeds other than the tests' seed 0
mkdir -p gpurun_out
rm -f gpurun_out/parity_seeds.jsonl
export TENKIT_PARITY_LOG=gpurun_out/parity_seeds.jsonl
timeout 1500 python tools/parity_seeds.py cfg3 1 2 3 2>&1 | grep parity_seeds | cut -c1-400
timeout 900 python tools/parity_seeds.py cfg4 1 2 2>&1 | grep parity_seeds | cut -c1-400
timeout 900 python tools/parity_seeds.py cfg5slab 1 2>&1 | grep parity_seeds | cut -c1-400
