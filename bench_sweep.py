"""bench_sweep.py -- the dense-to-sparse schedule sweep (BASELINE.json configs[4], C5):
T=16384 tokens/GPU, d=512, d_ff=2048, E=32; tau 2.0 -> 0.05 geometric and c 0 -> 0.3 linear
over 20 steps with fresh Gumbel noise per step (harness seed +5+step).  Prints one JSON line
per schedule step (tokens/s, mean active experts/token, rows, expert-GEMM TFLOP/s) and an
aggregate line (sum tokens / sum time).  Each step is replayed as a CUDA graph captured for that
step (static row capacity for the dense phase); --no-graph launches eagerly.

    python bench_sweep.py [--reps 5] [--warmup 2]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from harness import configs, inputs  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=2)
    ap.add_argument("--no-graph", dest="graph", action="store_false", help="eager launches (host sync per step)")
    args = ap.parse_args()
    from paper_2112_14397_b200.layer import DTSMoELayer
    cfg = configs.C5
    dev = torch.device("cuda", 0)
    li = inputs.make_inputs(cfg)
    layer = DTSMoELayer(cfg.T, cfg.d_model, cfg.d_ff, cfg.E, dtype=torch.bfloat16, device=dev)
    layer.set_gate(li.Wg.to(dev))
    layer.spawn(*(t.to(dev) for t in (li.W1s, li.b1s, li.W2s, li.b2s, li.M1bits, li.M2bits)))
    x, dy = li.x.to(dev), li.dy.to(dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    gev = lambda: torch.cuda.Event(enable_timing=True, external=True)  # noqa: E731  (recorded inside graphs)
    tot_tokens, tot_ms, tot_flops = 0, 0.0, 0.0
    # CUDA-graph mode (default): the step's launches replayed as one graph with a static row
    # capacity covering the dense phase (every token to every expert), as bench.py does; the
    # graph is captured per schedule step (tau and c are launch arguments), outside the timing.
    R_static = (cfg.T * cfg.E + 127 * cfg.E + 127) // 128 * 128
    u_static = torch.empty(cfg.T, cfg.E, dtype=torch.float32, device=dev)
    for s, (tau, c) in enumerate(cfg.schedule):
        u = inputs.uniform_u(cfg.T, cfg.E, step=s).to(dev)
        tau32, c32 = float(np.float32(tau)), float(np.float32(c))
        for _ in range(args.warmup):
            layer.forward(x, u, tau32, c32)
            layer.backward(dy)
        torch.cuda.synchronize()
        graph = None
        g_f, g_b = (gev(), gev()), (gev(), gev())
        if args.graph:
            u_static.copy_(u)
            layer.forward(x, u_static, tau32, c32, R_cap=R_static)
            layer.backward(dy)
            torch.cuda.synchronize()
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph):
                layer.forward(x, u_static, tau32, c32, R_cap=R_static, events=g_f)
                layer.backward(dy, events=g_b)
            for _ in range(2):
                graph.replay()
            torch.cuda.synchronize()
        ms, gms = [], []
        for _ in range(args.reps):
            flush.fill_(1)
            e0, e1 = ev(), ev()
            f_ev, b_ev = (ev(), ev()), (ev(), ev())
            e0.record()
            if graph is not None:
                graph.replay()
                f_ev, b_ev = g_f, g_b
            else:
                layer.forward(x, u, tau32, c32, events=f_ev)
                layer.backward(dy, events=b_ev)
            e1.record()
            e1.synchronize()
            ms.append(e0.elapsed_time(e1))
            gms.append(f_ev[0].elapsed_time(f_ev[1]) + b_ev[0].elapsed_time(b_ev[1]))
        layer.check()
        R = int(layer.state.offsets[-1].item())
        counts = layer.state.counts.cpu().numpy()
        t_ms = float(np.median(ms))
        flops = 12.0 * int(counts.sum()) * cfg.d_model * cfg.d_ff
        line = {"step": s, "tau": tau, "threshold": c, "tokens_per_s": cfg.T / (t_ms / 1e3), "ms": t_ms,
                "mean_experts_per_token": float(counts.sum()) / cfg.T, "rows_R_pad": R,
                "max_over_mean_load": float(counts.max() / max(1e-9, counts.mean())),
                "near_band": int(layer.state.near_band.item()),
                "rows_R": int(counts.sum()),
                # algorithmic FLOPs of the realised rows (pad rows excluded), VERDICT r1 weak #3
                "expert_gemm_tflops": flops / (float(np.median(gms)) / 1e3) / 1e12,
                "expert_gemm_tflops_incl_pad_rows": 12.0 * R * cfg.d_model * cfg.d_ff / (float(np.median(gms)) / 1e3) / 1e12}
        print(json.dumps(line), flush=True)
        tot_tokens += cfg.T
        tot_ms += t_ms
        tot_flops += flops
    print(json.dumps({"aggregate": "C5 schedule, 20 steps", "tokens_per_s": tot_tokens / (tot_ms / 1e3),
                      "ms_total": tot_ms, "useful_tflops": tot_flops / (tot_ms / 1e3) / 1e12}))


if __name__ == "__main__":
    main()
