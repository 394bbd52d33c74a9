"""bench.py on the GPU: the JSON line the driver reads, at small configs (C1 fp32 SIMT path, C3
bf16 tensor-core path, and the peer-memory EP path on a 1-rank group), checked for the keys and
for internal consistency (value = tokens / time, roofline fraction = achieved / peak, e2e copies
counted, the library's kernels launched)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _bench(*extra):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--steps", "3", "--warmup", "3",
                        "--cpu-tokens", "64", *extra], capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.strip().splitlines() if ln.strip()]
    assert len(lines) == 1, r.stdout[-2000:]
    return json.loads(lines[0])


def _check(d, workload, bound="tensor"):
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e", "gpu_launches", "clocks"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] == 3 and d["higher_is_better"] is True
    assert d["config"]["workload"].startswith(workload)
    T = d["config"]["tokens_per_gpu"]
    assert abs(d["value"] - T / (d["ms_per_step"] / 1e3)) <= 1e-6 * d["value"]
    r = d["roofline"]
    assert r["bound"] == bound and r["unit"] == "TFLOP/s" and 0 < r["frac"] < 1.2
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert d["gpu_launches"] > 0
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["value"] > 0


@pytest.mark.gpu
@pytest.mark.parametrize("cfg,bound", [("C1", "alu"), ("C3", "tensor")])
def test_bench_line_single_gpu(cfg, bound):
    _check(_bench("--config", cfg), cfg, bound)


@pytest.mark.gpu
def test_bench_line_ep_path_one_rank():
    d = _bench("--config", "C3", "--ep", "p2p")
    _check(d, "C3")
    assert str(d["config"].get("ep_path", "")).startswith("p2p")
