"""CPU checks of bench.py: every name a function reads is bound somewhere (catches a
renamed local that only the GPU run would hit), the reference arm runs on the host, and
the JSON line keeps the driver's contract keys."""
import ast
import builtins
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BENCH = os.path.join(ROOT, "bench.py")


def _bound_names(fn: ast.AST) -> set:
    out = set()
    for node in ast.walk(fn):
        if isinstance(node, (ast.FunctionDef, ast.AsyncFunctionDef, ast.Lambda)):
            a = node.args
            for x in a.args + a.kwonlyargs + a.posonlyargs:
                out.add(x.arg)
            if a.vararg:
                out.add(a.vararg.arg)
            if a.kwarg:
                out.add(a.kwarg.arg)
            if not isinstance(node, ast.Lambda):
                out.add(node.name)
        elif isinstance(node, ast.ClassDef):
            out.add(node.name)
        elif isinstance(node, ast.Name) and isinstance(node.ctx, (ast.Store, ast.Del)):
            out.add(node.id)
        elif isinstance(node, (ast.Import, ast.ImportFrom)):
            for al in node.names:
                out.add((al.asname or al.name).split(".")[0])
        elif isinstance(node, ast.ExceptHandler) and node.name:
            out.add(node.name)
        elif isinstance(node, ast.comprehension):
            for n in ast.walk(node.target):
                if isinstance(n, ast.Name):
                    out.add(n.id)
    return out


def test_bench_functions_read_only_bound_names():
    tree = ast.parse(open(BENCH).read())
    module_names = _bound_names(tree)
    known = module_names | set(dir(builtins))
    for fn in [n for n in tree.body if isinstance(n, ast.FunctionDef)]:
        local = _bound_names(fn)
        for node in ast.walk(fn):
            if isinstance(node, ast.Name) and isinstance(node.ctx, ast.Load):
                assert node.id in local or node.id in known, f"bench.py:{node.lineno} {fn.name}: unbound '{node.id}'"


def test_reference_arm_runs_on_the_host():
    r = subprocess.run([sys.executable, BENCH, "--impl", "reference", "--config", "cfg2", "--steps", "1", "--warmup",
                        "0", "--cpu-slabs", "4"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "impl", "e2e", "cpu_baseline"):
        assert k in line, k
    assert line["impl"] == "reference" and line["config"]["workload"] == "cfg2"
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["cpu_baseline"]["kind"] == "port"
    # the reference arm generates its sample with the oracle: the product library is never loaded
    assert line["repo_library_loaded"] is False and line["config"]["sample_dims"] == [1000, 1000, 4]
    assert line["host"]["nproc"] == os.cpu_count()


def test_bench_partitions_follow_baseline():
    """BASELINE's partitions: cfg3 mode-3 slabs at every N, cfg5 slabs at 2/4 and 2x2x2 at 8."""
    sys.path.insert(0, ROOT)
    import bench
    assert bench.bench_grid("cfg3", 3, 1, "strong") == [1, 1, 1]
    assert bench.bench_grid("cfg3", 3, 8, "strong") == [1, 1, 8]
    assert bench.bench_grid("cfg4", 4, 4, "strong") == [1, 1, 1, 4]
    assert bench.bench_grid("cfg5", 3, 2, "strong") == [1, 1, 2]
    assert bench.bench_grid("cfg5", 3, 4, "strong") == [1, 1, 4]
    assert bench.bench_grid("cfg5", 3, 8, "strong") == [2, 2, 2]
    assert bench.bench_grid("cfg2", 3, 8, "weak") == [2, 2, 2]
    assert bench.sample_dims(bench.CONFIGS["cfg3"]) == [2400, 2400, 40]
    assert bench.sample_dims(bench.CONFIGS["cfg1"]) == [200, 200, 200]
