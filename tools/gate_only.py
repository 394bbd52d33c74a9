"""Time the forward gate call alone (moe_dts_gate: W_g transpose, fused tcgen05 gate, fp64
refine) on a config's inputs, per-kernel device times via CUPTI.  Dev tool, not product.

    python tools/gate_only.py C4
"""
import sys

import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, ".")
from harness import configs, inputs  # noqa: E402
from paper_2112_14397_b200 import _lib as L  # noqa: E402

cfg = getattr(configs, sys.argv[1] if len(sys.argv) > 1 else "C4")
li = inputs.make_inputs(cfg)
dev = torch.device("cuda", 0)
T, d, E = li.x.shape[0], cfg.d_model, cfg.E
ctx = L.moe_create(T, d, cfg.d_ff, E, L.MOE_BF16)
ws = torch.empty(L.moe_workspace_bytes(ctx), dtype=torch.uint8, device=dev)
L.moe_set_workspace(ctx, ws)
x, Wg, u = li.x.to(dev), li.Wg.to(dev), li.u.to(dev)
probs = torch.empty(T, E, device=dev)
slot = torch.empty(T, E, dtype=torch.int32, device=dev)
counts = torch.empty(E, dtype=torch.int32, device=dev)
near = torch.empty(1, dtype=torch.int32, device=dev)
tau, c = float(np.float32(cfg.tau)), float(np.float32(cfg.threshold))
for _ in range(5):
    L.moe_dts_gate(ctx, x, Wg, u, tau, c, False, probs, slot, counts, near)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(20):
        L.moe_dts_gate(ctx, x, Wg, u, tau, c, False, probs, slot, counts, near)
    torch.cuda.synchronize()
for e in prof.key_averages():
    if "gate" in e.key or "wg_" in e.key:
        print(round(e.device_time_total / e.count, 1), "us", e.count, e.key[:70])
L.moe_destroy(ctx)
