"""Per-kernel device times of the peer-memory EP step (moe_ep2_*) on a 1-rank group, next to the
single-GPU layer's, to see what the EP path adds at W = 1.  Dev tool.

    python tools/ep_kernel_times.py [--config C4] [--steps 3] [--dedup]
"""
import argparse
import collections
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from harness import configs, inputs  # noqa: E402


def times(fn, steps):
    from torch.profiler import ProfilerActivity, profile
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(steps):
            fn()
        torch.cuda.synchronize()
    acc = collections.defaultdict(lambda: [0, 0.0])
    for e in prof.events():
        if e.device_type.name != "CUDA":
            continue
        k = e.name.replace("(anonymous namespace)::", "").replace("void ", "").split("(")[0]
        acc[k][0] += 1
        acc[k][1] += e.time_range.end - e.time_range.start
    return {k: (n / steps, us / steps) for k, (n, us) in acc.items()}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C4")
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--dedup", action="store_true")
    a = ap.parse_args()
    rank, world, _ = bench.dist_setup(force_pg=True)
    import torch.distributed as dist
    from paper_2112_14397_b200.ep2 import EP2Rank, SymmetricBuffers
    from paper_2112_14397_b200.layer import DTSMoELayer, make_nccl_comm
    cfg = configs.get(a.config)
    dev = torch.device("cuda", torch.cuda.current_device())
    li = inputs.make_inputs(cfg)
    x, u, dy = li.x.to(dev), li.u.to(dev), li.dy.to(dev)
    tau, c = float(np.float32(cfg.tau)), float(np.float32(cfg.threshold))
    comm = make_nccl_comm(rank, world)
    syms = SymmetricBuffers(world, dev, mode="symm_mem", group=dist.group.WORLD)
    r = EP2Rank(cfg.T, cfg.d_model, cfg.d_ff, cfg.E, inputs.TORCH_DTYPE[cfg.dtype], dev, rank, world, syms,
                comm=comm, dedup=a.dedup)
    r.set_gate(li.Wg.to(dev))
    r.spawn(*(t.to(dev) for t in (li.W1s, li.b1s, li.W2s, li.b2s, li.M1bits, li.M2bits)))
    dyb = r.dy_buffer()
    dyb.copy_(dy)
    r.step(x, u, dyb, tau, c, cfg.top1)
    r.prepare()

    def ep_step():
        r.forward(x, u, tau, c, cfg.top1)
        r.backward(dyb)

    layer = DTSMoELayer(cfg.T, cfg.d_model, cfg.d_ff, cfg.E, dtype=inputs.TORCH_DTYPE[cfg.dtype], device=dev)
    layer.set_gate(li.Wg.to(dev))
    layer.spawn(*(t.to(dev) for t in (li.W1s, li.b1s, li.W2s, li.b2s, li.M1bits, li.M2bits)))

    def single_step():
        layer.forward(x, u, tau, c)
        layer.backward(dy)

    te, ts = times(ep_step, a.steps), times(single_step, a.steps)
    for name, t in (("ep2" + ("d" if a.dedup else ""), te), ("single", ts)):
        tot = sum(us for _, us in t.values())
        for k, (n, us) in sorted(t.items(), key=lambda kv: -kv[1][1]):
            print(json.dumps({"path": name, "kernel": k[-60:], "calls": n, "us_per_step": round(us, 1)}))
        print(json.dumps({"path": name, "kernel": "TOTAL", "us_per_step": round(tot, 1)}))
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
