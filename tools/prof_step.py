"""Run a few eager fwd+bwd steps of one config through DTSMoELayer (profiling driver).

    python tools/prof_step.py [--config C2] [--steps 3] [--kernel-times]

Under ncu use `-k regex:tc_gemm -s <7 * (steps-1)> -c 7` to capture the last step's GEMMs.
With --kernel-times, per-kernel device times of the last steps are collected with
torch.profiler (CUPTI activity records; warm, back-to-back, no replay) and printed as
JSON lines: {"kernel", "calls", "us_per_step"}.
"""
from __future__ import annotations

import argparse
import collections
import json
import re
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from harness import configs, inputs  # noqa: E402
from paper_2112_14397_b200.layer import DTSMoELayer  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C2")
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--kernel-times", action="store_true")
    ap.add_argument("--step", type=int, default=None, help="C5 schedule step (tau, c and noise of that step)")
    a = ap.parse_args()
    cfg = configs.get(a.config)
    if a.step is not None:
        cfg = cfg.at_step(a.step)
    dev = torch.device("cuda", 0)
    li = inputs.make_inputs(cfg, step=a.step or 0)
    dt = inputs.TORCH_DTYPE[cfg.dtype]
    tau, c = float(np.float32(cfg.tau)), float(np.float32(cfg.threshold))
    layer = DTSMoELayer(cfg.T, cfg.d_model, cfg.d_ff, cfg.E, dtype=dt, device=dev)
    layer.set_gate(li.Wg.to(dev))
    layer.spawn(*(t.to(dev) for t in (li.W1s, li.b1s, li.W2s, li.b2s, li.M1bits, li.M2bits)))
    x, u, dy = li.x.to(dev), li.u.to(dev), li.dy.to(dev)

    def step():
        layer.forward(x, u, tau, c)
        layer.backward(dy)

    if not a.kernel_times:
        for _ in range(a.steps):
            step()
        torch.cuda.synchronize()
        layer.check()
        print("ok", a.config, "R =", int(layer.state.offsets[-1].item()))
        return
    for _ in range(3):
        step()
    torch.cuda.synchronize()
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(a.steps):
            step()
        torch.cuda.synchronize()
    layer.check()
    agg = collections.OrderedDict()
    for e in prof.events():
        if e.device_type.name != "CUDA":
            continue
        k = e.name.replace("(anonymous namespace)::", "").replace("void ", "")
        k = re.sub(r"\(CUtensorMap.*|\((const |float|int|__nv|moe::).*", "", k)[:90]
        n, t = agg.get(k, (0, 0.0))
        agg[k] = (n + 1, t + e.device_time)
    tot = 0.0
    for k, (n, t) in agg.items():
        tot += t / a.steps
        print(json.dumps({"kernel": k, "calls": n // a.steps, "us_per_step": round(t / a.steps, 1)}))
    print(json.dumps({"kernel": "TOTAL", "us_per_step": round(tot, 1)}))


if __name__ == "__main__":
    main()
