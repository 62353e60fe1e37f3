#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1500 python tools/diag_cfg3_parity.py cfg3 > gpurun_out/diag_cfg3.log 2>&1; echo "diag rc=$?"; cat gpurun_out/diag_cfg3.log | tail -30
timeout 900 python -m pytest tests/test_gpu_nccl.py tests/test_gpu_ref_fixtures.py -m gpu -q > gpurun_out/nccl_ref.log 2>&1; echo "nccl+ref rc=$?"; grep -E "^E |passed|failed" gpurun_out/nccl_ref.log | head -20
timeout 1200 python -m pytest tests/test_gpu_bench_dist.py -m gpu -q > gpurun_out/bench_dist.log 2>&1; echo "bench dist rc=$?"; grep -E "^E |passed|failed" gpurun_out/bench_dist.log | head -20
