#!/bin/bash
# the final stream kernel: stream / tc / qr tests, full-size parity (all R~ columns, logged), bench cfg3
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo "build rc=$?"
timeout 900 python -m pytest tests/test_gpu_stream.py tests/test_gpu_tc.py tests/test_gpu_qr_margins.py -m gpu -q -x > gpurun_out/kern_tests.log 2>&1; echo "kernel tests rc=$?"; grep -E "^E |passed|failed" gpurun_out/kern_tests.log | head -8
rm -f gpurun_out/parity_final.jsonl
TENKIT_PARITY_LOG=gpurun_out/parity_final.jsonl timeout 1500 python -m pytest tests/test_gpu_fullsize.py -m gpu -q -x -s > gpurun_out/fullsize.log 2>&1; echo "fullsize rc=$?"; grep -E "^E |passed|failed|margin|worst" gpurun_out/fullsize.log | head -20
timeout 900 python bench.py > gpurun_out/bench_cfg3.log 2> gpurun_out/bench_cfg3.err; echo "bench rc=$?"; tail -c 3000 gpurun_out/bench_cfg3.log
