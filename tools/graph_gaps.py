"""Idle time between consecutive kernels inside one replayed CUDA-graph step (CUPTI via
torch.profiler): how much a step loses to launch gaps / kernel tails.  Dev tool.

    python tools/graph_gaps.py [--config C2] [--step S] [--timeline]

--step S takes tau / threshold and the Gumbel draw of C5's schedule step S; --timeline also
prints every kernel of the step (start offset, duration, gap before it) as JSON lines.
"""
import argparse
import json
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
    ap.add_argument("--step", type=int, default=None)
    ap.add_argument("--timeline", action="store_true")
    a = ap.parse_args()
    cfg = configs.get(a.config)
    dev = torch.device("cuda", 0)
    li = inputs.make_inputs(cfg)
    layer = DTSMoELayer(cfg.T, cfg.d_model, cfg.d_ff, cfg.E, dtype=inputs.TORCH_DTYPE[cfg.dtype], device=dev)
    layer.set_gate(li.Wg.to(dev))
    layer.spawn(*(t.to(dev) for t in (li.W1s, li.b1s, li.W2s, li.b2s, li.M1bits, li.M2bits)))
    x, u, dy = li.x.to(dev), li.u.to(dev), li.dy.to(dev)
    tau, c = float(np.float32(cfg.tau)), float(np.float32(cfg.threshold))
    if a.step is not None:
        tau, c = (float(np.float32(v)) for v in cfg.schedule[a.step])
        u = inputs.uniform_u(cfg.T, cfg.E, step=a.step).to(dev)
    for _ in range(3):
        layer.forward(x, u, tau, c)
        layer.backward(dy)
    torch.cuda.synchronize()
    R = layer.state.R_cap
    layer.forward(x, u, tau, c, R_cap=R)
    layer.backward(dy)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        layer.forward(x, u, tau, c, R_cap=R)
        layer.backward(dy)
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        g.replay()
        torch.cuda.synchronize()
    ev = sorted([e for e in prof.events() if e.device_type.name == "CUDA"], key=lambda e: e.time_range.start)
    def short(n):
        return n.replace("(anonymous namespace)::", "").replace("void ", "").split("(")[0][-48:]

    spans = [(e.time_range.start, e.time_range.end, short(e.name)) for e in ev]
    busy = sum(e1 - s1 for s1, e1, _ in spans)
    wall = spans[-1][1] - spans[0][0]
    gaps = [(spans[i + 1][0] - spans[i][1], spans[i][2], spans[i + 1][2]) for i in range(len(spans) - 1)]
    if a.timeline:
        t0 = spans[0][0]
        prev = t0
        for s0, s1, nm in spans:
            print(json.dumps({"k": nm, "at_us": round(s0 - t0, 2), "us": round(s1 - s0, 2), "gap_us": round(s0 - prev, 2)}))
            prev = s1
    print(json.dumps({"config": a.config, "step": a.step, "kernels": len(spans), "wall_us": wall, "busy_us": busy,
                      "idle_us": wall - busy, "largest_gaps": sorted(gaps, reverse=True)[:6]}))


if __name__ == "__main__":
    main()
