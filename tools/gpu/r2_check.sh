#!/bin/bash
mkdir -p gpurun_out
export TENKIT_PARITY_LOG=$PWD/gpurun_out/parity7.jsonl
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_stream.py tests/test_gpu_qr_margins.py -m gpu -q > gpurun_out/stream_tests.log 2>&1; echo "stream tests rc=$?"; grep -E "^E |passed|failed" gpurun_out/stream_tests.log | head -12
timeout 900 python bench.py --config cfg5slab --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_cfg5slab.log 2> gpurun_out/bench_cfg5slab.err; echo "cfg5slab rc=$?"; tail -c 600 gpurun_out/bench_cfg5slab.log
timeout 2400 python -m pytest tests/test_gpu_fullsize.py -m gpu -q -s > gpurun_out/fs.log 2>&1; echo "fullsize rc=$?"; grep -E "^E |passed|failed" gpurun_out/fs.log | head
