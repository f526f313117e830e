"""CPU checks: the C-ABI library loads and exports every symbol include/unetswap.h
declares; the oracle restatements are pinned (toy executor == reference fixtures
bit-for-bit; fp64 real-op step == finite differences)."""
import ctypes
import os

import numpy as np
import pytest

from paper_1812_07816_b200 import _native
from paper_1812_07816_b200.rewrite import apply_rewrite, resolve_preset
from paper_1812_07816_b200.training import expand_training_graph

from golden_configs import GOLDEN, build, load


def test_library_exports_every_declared_symbol():
    lib = _native.load_library()
    declared = _native.exported_symbols()
    assert len(declared) >= 20
    raw = ctypes.CDLL(_native.LIB_PATH)
    missing = [s for s in declared if not hasattr(raw, s)]
    assert not missing, missing
    assert lib.us_abi_version() == 1


def test_workspace_query_without_a_device():
    op = _native.OP
    n = _native.workspace_bytes(op["US_OP_BN_BWD"], [192 ** 3, 64])
    assert n >= 2 * 64 * 4
    n = _native.workspace_bytes(op["US_OP_CONV_WGRAD"],
                                [1, 192, 192, 192, 64, 64, 0, _native.ALGO_TCGEN05])
    assert n > 0


def test_context_creation_fails_loudly_without_gpu():
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("a GPU is present")
    except ImportError:
        pass
    with pytest.raises(_native.EngineError):
        _native.Engine(0, 1 << 20)


@pytest.mark.parametrize("row", load("numeric_index.json"),
                         ids=lambda r: f"{r['graph']}-{r['preset']}-s{r['seed']}")
def test_toy_oracle_pinned_to_reference(row):
    from oracle.toy_numeric import run_numeric
    tg = expand_training_graph(build(row["graph"]))
    plan = None
    if row["preset"]:
        tg, plan = apply_rewrite(tg, resolve_preset(row["preset"]))
    loss, grads = run_numeric(tg, plan, row["seed"])
    gold = np.load(os.path.join(GOLDEN, row["file"]))
    assert loss == float(gold["loss"])
    for tid in row["grads"]:
        assert np.array_equal(grads[tid], gold[tid.replace(":", "__")])


def test_unet_oracle_gradients_match_finite_differences():
    import torch
    from oracle.unet_fp64 import forward_loss, reference_step
    from paper_1812_07816_b200.unet import TrainConfig, UNetTrainer
    cfg = TrainConfig(dims=(8, 8, 8), base_filters=4, depth=2, dtype="f32", preset=None)
    tr = UNetTrainer(cfg, device_engine=False)
    x, y = tr.synthetic_batch(seed=2)
    p = {k: v.astype(np.float64) for k, v in tr.initial_params().items()}
    ref = reference_step(cfg, p, x, y)

    def loss_at(pp):
        with torch.no_grad():
            return float(forward_loss(tr.graph, pp, x, y, cfg.n_classes)[0])

    eps = 1e-6
    for name, idx in [("head.b", (1,)), ("analysis/l0/conv1.w", (2, 13, 1)),
                      ("analysis/l1/norm1.gamma", (3,)), ("synthesis/l0/upsample.w", (1, 5, 2))]:
        hi = {k: v.copy() for k, v in p.items()}
        lo = {k: v.copy() for k, v in p.items()}
        hi[name][idx] += eps
        lo[name][idx] -= eps
        fd = (loss_at(hi) - loss_at(lo)) / (2 * eps)
        an = ref["grads"][name][idx]
        assert abs(fd - an) <= 1e-5 * max(abs(fd), 1e-8) + 1e-9, (name, fd, an)


def test_smoke_golden_fixture_has_the_keys_smoke_reads():
    import os
    g = np.load(os.path.join(os.path.dirname(__file__), "golden",
                             "numeric_toy8_paper-c1_s1.npz"))
    assert {"loss", "source__0"} <= set(g.files)


def test_oracle_init_matches_the_engine_layout():
    """The CPU baseline builds parameters and inputs without the CUDA library; they must
    be exactly the engine's (fp32 layout, no padded input channels)."""
    from oracle.unet_fp64 import init_params, synthetic_batch
    from paper_1812_07816_b200.unet import TrainConfig, UNetTrainer
    cfg = TrainConfig(dims=(32, 32, 32), base_filters=16, depth=3, dtype="f32", seed=5)
    tr = UNetTrainer(cfg, device_engine=False)
    a, b = tr.initial_params(), init_params(tr.graph, cfg.seed, cfg.n_classes)
    assert set(a) == set(b)
    assert all(np.array_equal(a[k], b[k]) for k in a)
    x0, y0 = tr.synthetic_batch(seed=2)
    x1, y1 = synthetic_batch(cfg.dims, cfg.batch, cfg.in_channels, cfg.n_classes, seed=2)
    assert np.array_equal(x0, x1) and np.array_equal(y0, y1)


def test_bench_reference_arm_runs_on_cpu_without_the_cuda_library():
    """`bench.py --impl reference` (the driver's reference arm) is CPU-only: one JSON line
    with impl, value, e2e and cpu_baseline, and libunetswap.so never mapped."""
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = ("import runpy, sys\n"
            "sys.argv = ['bench.py', '--impl', 'reference', '--steps', '1', '--warmup', '3']\n"
            "try:\n"
            "    runpy.run_path('bench.py', run_name='__main__')\n"
            "finally:\n"
            "    maps = open('/proc/self/maps').read()\n"
            "    print('UNETSWAP_MAPPED' if 'libunetswap' in maps else 'UNETSWAP_NOT_MAPPED')\n")
    r = subprocess.run([sys.executable, "-c", code], cwd=root, capture_output=True, text=True,
                       timeout=900, env=dict(os.environ, OMP_NUM_THREADS="4"))
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["value"] > 0 and d["e2e"]["value"] == d["value"]
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["cores"] >= 1
    assert "UNETSWAP_NOT_MAPPED" in r.stdout
