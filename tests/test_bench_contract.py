"""bench.py's output contract, checked on the CPU through the reference arm (the oracle): one JSON
line on stdout whatever else the run prints, with the keys the driver reads.  The GPU arm's line is
produced by the same printer (bench.py main)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_prints_one_json_line():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "2",
                        "--warmup", "0", "--ref-tokens", "32", "--config", "C1"],
                       capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = r.stdout.strip().splitlines()
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["steps"] == 2 and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]


def test_reference_arm_other_ranks_print_nothing():
    env = dict(os.environ, RANK="1", WORLD_SIZE="2")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                        "--warmup", "0", "--ref-tokens", "16", "--config", "C1"],
                       capture_output=True, text=True, timeout=300, cwd=ROOT, env=env)
    assert r.returncode == 0 and r.stdout.strip() == ""


def test_gemm_mixed_roofline():
    """The per-GEMM max(tensor, HBM) roofline: closed forms at two shapes (tensor peak 1000 TF/s,
    1000 GB/s of HBM so that times are FLOPs / 1e15 and bytes / 1e12)."""
    sys.path.insert(0, ROOT)
    from bench import gemm_roofline_us
    pk = {"bf16_tflops": 1000.0, "hbm_gbs": 1000.0}
    # tiny R, big weights: every GEMM is bound by its bytes (weights dominate)
    R, d, f, E = 128, 256, 512, 8
    w = 2 * E * d * f
    byts = [2 * R * d + w + 4 * R * f, 2 * R * f + w + 2 * R * d, 2 * R * d + w + 4 * R * f,
            2 * R * f + w + 2 * R * d, 2 * R * d + 2 * R * f + 2 * w, 2 * R * f + 2 * R * d + 2 * w]
    us, n_hbm = gemm_roofline_us(R, d, f, E, pk)
    assert n_hbm == 6 and abs(us - sum(byts) / 1e12 * 1e6) < 1e-9
    # huge R: FLOPs dominate (6 x 2 R d f at the tensor peak), no GEMM is HBM-bound
    R, d, f, E = 1 << 20, 4096, 16384, 1
    us, n_hbm = gemm_roofline_us(R, d, f, E, pk)
    assert n_hbm == 0 and abs(us - 6 * 2.0 * R * d * f / 1e15 * 1e6) < 1e-6 * us
