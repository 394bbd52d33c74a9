"""Is the e2e gap a copy bubble or the power state?  Alternates device-timed graph replays
(L2 flushed), bench.run_e2e (pipelined host copies) and back-to-back replays in one process.
Dev tool.    python tools/e2e_probe.py
"""
import sys, os, time, json
sys.path.insert(0, '.')
import numpy as np, torch
import bench
from harness import configs, inputs
from paper_2112_14397_b200.layer import DTSMoELayer
cfg = configs.C2
dev = torch.device("cuda", 0); torch.cuda.set_device(0)
li = inputs.make_inputs(cfg)
layer = DTSMoELayer(cfg.T, cfg.d_model, cfg.d_ff, cfg.E, dtype=torch.bfloat16, device=dev)
layer.set_gate(li.Wg.to(dev)); layer.spawn(*(t.to(dev) for t in (li.W1s, li.b1s, li.W2s, li.b2s, li.M1bits, li.M2bits)))
x, u, dy = li.x.to(dev), li.u.to(dev), li.dy.to(dev)
tau, c = float(np.float32(cfg.tau)), float(np.float32(cfg.threshold))
for _ in range(3):
    layer.forward(x, u, tau, c); layer.backward(dy)
torch.cuda.synchronize()
R = layer.state.R_cap
g = torch.cuda.CUDAGraph()
layer.forward(x, u, tau, c, R_cap=R); layer.backward(dy); torch.cuda.synchronize()
with torch.cuda.graph(g):
    layer.forward(x, u, tau, c, R_cap=R); layer.backward(dy)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
class A: steps = 30
def dev_time(n=30, with_flush=True):
    ms = []
    for _ in range(n):
        if with_flush: flush.fill_(1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); g.replay(); e1.record(); e1.synchronize(); ms.append(e0.elapsed_time(e1))
    return sum(ms)/len(ms)
def back_to_back(n=30):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n): g.replay()
    e1.record(); e1.synchronize(); return e0.elapsed_time(e1)/n
for rnd in range(2):
    d1 = dev_time()
    e = bench.run_e2e(A, layer, li, tau, c, 1, (g, x, u, dy))
    d2 = dev_time()
    b = back_to_back()
    print(json.dumps({"dev_flush_ms": round(d1,3), "e2e_ms": round(e["ms_per_step"],3), "dev_flush_ms_after": round(d2,3), "back_to_back_ms": round(b,3)}))
