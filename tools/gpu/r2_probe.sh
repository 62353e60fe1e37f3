#!/bin/bash
# Round-2 first call: host probe, cfg3 bench line, phase timing, ncu of cfg3's Y passes.
mkdir -p gpurun_out
{ nproc; lscpu | head -25; free -g; nvidia-smi -L; } > gpurun_out/host.txt 2>&1
python - > gpurun_out/dgemm.txt 2>&1 <<'PY'
import time, numpy as np, os
a = np.random.rand(40, 2400); b = np.random.rand(2400, 2400*16)
for _ in range(2):
    t = time.perf_counter(); c = a @ b; dt = time.perf_counter() - t
print("dgemm 40x2400x38400 GF/s", 2*40*2400*38400/dt/1e9, "threads", os.cpu_count())
PY
timeout 900 python bench.py --config cfg3 --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_cfg3.log 2> gpurun_out/bench_cfg3.err; echo "cfg3 bench rc=$?"
TENKIT_PHASE_TIMING=1 timeout 600 python tools/phase_bench.py cfg3 > gpurun_out/phase_cfg3.log 2>&1; echo "phase rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:ttm_tc_kernel' --launch-count 12 -o gpurun_out/r2_cfg3_tc python tools/one_decomp.py cfg3 > gpurun_out/ncu_cfg3.log 2>&1; echo "ncu rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launches_cfg3.csv python tools/one_decomp.py cfg3 > gpurun_out/ncu_list_cfg3.log 2>&1; echo "ncu list rc=$?"
ls -la gpurun_out
