"""Host link bandwidth of this box, for the e2e bound: pinned host <-> device copies of the C4
step's byte counts (570 MB in, 537 MB out), each direction alone and both at once on two
streams (the pipelined e2e overlaps them).  Dev tool.   python tools/pcie_probe.py
"""
import json

import torch


def timed(fn, reps=5):
    best = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        best.append(e0.elapsed_time(e1))
    return sorted(best)[len(best) // 2]


def main():
    dev = torch.device("cuda", 0)
    bi, bo = 570425344, 536870912
    hin = torch.empty(bi, dtype=torch.uint8).pin_memory()
    hout = torch.empty(bo, dtype=torch.uint8).pin_memory()
    din = torch.empty(bi, dtype=torch.uint8, device=dev)
    dout = torch.empty(bo, dtype=torch.uint8, device=dev)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    cur = torch.cuda.current_stream()

    def h2d():
        din.copy_(hin, non_blocking=True)

    def d2h():
        hout.copy_(dout, non_blocking=True)

    def both():
        s1.wait_stream(cur)
        s2.wait_stream(cur)
        with torch.cuda.stream(s1):
            din.copy_(hin, non_blocking=True)
        with torch.cuda.stream(s2):
            hout.copy_(dout, non_blocking=True)
        cur.wait_stream(s1)
        cur.wait_stream(s2)

    t_in, t_out, t_both = timed(h2d), timed(d2h), timed(both)
    print(json.dumps({"h2d_GBs": bi / t_in / 1e6, "d2h_GBs": bo / t_out / 1e6,
                      "h2d_ms": t_in, "d2h_ms": t_out, "both_ms": t_both,
                      "both_GBs_total": (bi + bo) / t_both / 1e6}))


if __name__ == "__main__":
    main()
