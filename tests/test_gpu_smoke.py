"""GPU: the driver's smoke() entry point (toy step vs the reference golden, U-Net step
vs the fp64 oracle) runs clean."""
import pytest

pytestmark = pytest.mark.gpu


def test_graft_entry_smoke():
    import __graft_entry__
    __graft_entry__.smoke()


def test_bench_line_contract():
    """bench.py's JSON line (the driver's contract) on the configs[1] patch workload: the
    required keys, a device-timed value, e2e through the public API with host copies, the
    roofline / clocks objects and a nonzero kernel-launch count."""
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "bench.py", "--config", "p128-b2", "--steps", "3",
                        "--warmup", "3", "--no-cpu-baseline"], cwd=root, capture_output=True,
                       text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-2000:]
    d = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
              "roofline", "e2e", "gpu_launches", "clocks"):
        assert k in d, k
    assert d["value"] > 0 and d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] >= 3
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["value"] > 0
    assert d["gpu_launches"] > 0 and d["roofline"]["bound"] == "tensor"
    assert 0 < d["roofline"]["frac"] < 1.5
