"""bench.py's multi-GPU partitions as code paths on one GPU: `TENKIT_BENCH_GLOO=1 torchrun
--nproc-per-node N bench.py --gpus N` runs N ranks sharing cuda:0 over gloo (host-staged
all-reduce, so no kernel waits on another rank) on BASELINE's partitions at reduced size
(--scale): cfg3 mode-3 slabs at 2 and 4 ranks, cfg5's 2 x 2 x 2 block grid at 8 ranks. The
distributed model must equal the single-process one of the same tensor (its fit and core
norm). Not scaling numbers: the real multi-GPU runs use the native NCCL communicator."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _bench(args, nproc=1):
    env = dict(os.environ, TENKIT_BENCH_GLOO="1")
    base = [sys.executable]
    if nproc > 1:
        base += ["-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}", "--master-addr", "127.0.0.1",
                 "--master-port", str(_free_port())]
    r = subprocess.run(base + ["bench.py", "--gpus", str(nproc), "--steps", "2", "--warmup", "3", "--no-e2e", "--no-cpu"]
                       + args, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    return json.loads(r.stdout.strip().splitlines()[-1])


@pytest.fixture(scope="module")
def gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")


@pytest.mark.parametrize("config,scale,nprocs", [("cfg3", 10, (2, 4)), ("cfg5", 10, (8,))])
def test_bench_partitions_equal_single_process(gpu, config, scale, nprocs):
    one = _bench(["--config", config, "--scale", str(scale)])
    for n in nprocs:
        d = _bench(["--config", config, "--scale", str(scale)], nproc=n)
        assert d["n_gpus"] == n and d["config"]["dims"] == one["config"]["dims"]
        grid = [2, 2, 2] if (config == "cfg5" and n == 8) else [1, 1, n]
        assert d["config"]["parallelism"].startswith("grid" + "x".join(map(str, grid)))
        assert abs(d["fit_model"] - one["fit_model"]) < 1e-5
        assert abs(d["core_norm"] - one["core_norm"]) <= 1e-5 * one["core_norm"]
