#!/bin/bash
timeout 600 python -m pytest tests/test_gpu_dist.py tests/test_gpu_workload.py -q -x 2>&1 | tail -3
TENKIT_BENCH_GLOO=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_n2.log 2> gpurun_out/bench_n2.err; echo "n2 rc=$?"
tail -1 gpurun_out/bench_n2.log | python -c "import json,sys; d=json.load(sys.stdin); print(d['n_gpus'], d['config']['dims'], d['fit_model'])"
