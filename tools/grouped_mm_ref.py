"""Same-box comparison point for the expert GEMMs (not in the path): PyTorch's
grouped GEMM (torch._grouped_mm, cuBLAS/CUTLASS inside) on the same ragged per-expert row
offsets as our routing of a config, forward GEMM1 / GEMM2 shapes without the fused bias /
GELU epilogues, plus the dense cuBLAS GEMM of the same total size.  Dev tool.

    python tools/grouped_mm_ref.py [C2|C4|C5:S]     (C5:S = the C5 schedule's step S)
"""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from harness import configs, inputs  # noqa: E402


def timed(fn, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    e.synchronize()
    return s.elapsed_time(e) / reps


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "C2"
    cfg = configs.get(name.split(":")[0])
    tau, c = float(np.float32(cfg.tau)), float(np.float32(cfg.threshold))
    u = inputs.make_inputs(cfg).u
    if ":" in name:
        step = int(name.split(":")[1])
        tau, c = (float(np.float32(v)) for v in cfg.schedule[step])
        u = inputs.uniform_u(cfg.T, cfg.E, step=step)
    from paper_2112_14397_b200.layer import DTSMoELayer
    dev = torch.device("cuda", 0)
    li = inputs.make_inputs(cfg)
    layer = DTSMoELayer(cfg.T, cfg.d_model, cfg.d_ff, cfg.E, dtype=torch.bfloat16, device=dev)
    layer.set_gate(li.Wg.to(dev))
    layer.spawn(*(t.to(dev) for t in (li.W1s, li.b1s, li.W2s, li.b2s, li.M1bits, li.M2bits)))
    layer.forward(li.x.to(dev), u.to(dev), tau, c)
    torch.cuda.synchronize()
    counts = layer.state.counts.cpu().numpy()
    R = int(counts.sum())
    d, f, E = cfg.d_model, cfg.d_ff, cfg.E
    offs = torch.tensor(np.cumsum(counts), dtype=torch.int32, device=dev)
    x = torch.randn(R, d, device=dev, dtype=torch.bfloat16)
    h = torch.randn(R, f, device=dev, dtype=torch.bfloat16)
    w1t = layer.W1.transpose(1, 2).contiguous().transpose(1, 2)      # [E, d, f] view of W1^T (column-major)
    w1t = layer.W1.transpose(1, 2)
    w2t = layer.W2.transpose(1, 2)
    out = {"config": name, "rows_R": R}
    fl1 = 2.0 * R * d * f
    try:
        ms1 = timed(lambda: torch._grouped_mm(x, w1t, offs=offs))
        ms2 = timed(lambda: torch._grouped_mm(h, w2t, offs=offs))
        out["grouped_mm_gemm1_ms"], out["grouped_mm_gemm1_tflops"] = ms1, fl1 / ms1 / 1e9
        out["grouped_mm_gemm2_ms"], out["grouped_mm_gemm2_tflops"] = ms2, fl1 / ms2 / 1e9
    except Exception as ex:  # noqa: BLE001
        out["grouped_mm_error"] = str(ex)[:200]
    a = torch.randn(R, d, device=dev, dtype=torch.bfloat16)
    b = torch.randn(d, f, device=dev, dtype=torch.bfloat16)
    b2 = torch.randn(f, d, device=dev, dtype=torch.bfloat16)
    ms3 = timed(lambda: a @ b)
    ms4 = timed(lambda: h @ b2)
    out["dense_cublas_gemm1_shape_tflops"], out["dense_cublas_gemm1_ms"] = fl1 / ms3 / 1e9, ms3
    out["dense_cublas_gemm2_shape_tflops"], out["dense_cublas_gemm2_ms"] = fl1 / ms4 / 1e9, ms4
    print(json.dumps(out))


if __name__ == "__main__":
    main()
