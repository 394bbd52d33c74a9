"""bench.py -- DTS-Gate MoE layer forward+backward throughput on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C2] [--impl ours|reference]

One "step" = one pass of the whole hot path over one batch of synthetic tokens:
moe_dts_gate -> moe_dispatch -> moe_expert_ffn -> moe_combine -> moe_combine_bwd ->
moe_expert_ffn_bwd -> moe_dts_gate_bwd -> moe_dispatch_bwd (all through the C ABI).
The spawn runs once before timing (it is an initialisation step, Alg. 1 lines 4-5).

Workload: BASELINE.json configs[1] (C2, GPT-small-shaped, T=8192 tokens per GPU,
d=768, d_ff=3072, E=16, tau=2.0, c=0.001), synthetic seeded data (harness/inputs.py).
Under torchrun (N > 1) each rank runs its own T tokens (weak scaling).

Timing: W untimed warm-up steps; then K steps, each bracketed by CUDA events on the
launching stream, with an L2 flush (write of a 256 MiB buffer) between steps outside
the events; barrier + synchronize on both sides; the max over ranks is reported.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from harness import configs, inputs  # noqa: E402

METRIC = "MoE-layer fwd+bwd tokens/sec at 1/2/4/8 B200; % bf16 tensor peak"


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return d, "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


# ------------------------------------------------------------------ clocks sampler
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        sm, smax, reasons = [], [], set()
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
            for n, v in zip(names, parts[4:8]):
                if v.lower() in ("active", "1"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------------ distributed plumbing
def dist_setup(n_gpus: int, force_pg: bool = False):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if force_pg and world == 1 and "MASTER_ADDR" not in os.environ:
        # single process without torchrun: a 1-rank group (the peer-memory path's symmetric
        # allocations rendezvous through it)
        import socket
        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK="0", WORLD_SIZE="1")
    if world > 1 or force_pg:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    return rank, world, local


def barrier(world):
    import torch.distributed as dist
    if world > 1 or (dist.is_available() and dist.is_initialized()):
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(v: float, world: int) -> float:
    if world == 1:
        return v
    import torch.distributed as dist
    t = torch.tensor([v], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# ------------------------------------------------------------------ CPU baseline (oracle)
def oracle_sample(cfg, T_sub: int, step: int = 0):
    """Time the fp64 oracle (as it stands) on T_sub tokens of the workload, fwd+bwd."""
    from oracle import dts_moe as O
    li = inputs.make_inputs(cfg, T=T_sub, step=step)
    ex = O.spawn(inputs.to_f64(li.W1s), inputs.to_f64(li.b1s), inputs.to_f64(li.W2s), inputs.to_f64(li.b2s),
                 inputs.bits_u32(li.M1bits), inputs.bits_u32(li.M2bits))
    x, Wg, u, dy = (inputs.to_f64(t) for t in (li.x, li.Wg, li.u, li.dy))
    t0 = time.perf_counter()
    fw = O.forward(x, Wg, u, float(np.float32(cfg.tau)), float(np.float32(cfg.threshold)), ex, top1=cfg.top1)
    O.backward(fw, dy)
    dt = time.perf_counter() - t0
    return dt


def cpu_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


# ------------------------------------------------------------------ our arm
def run_ours(args, rank, world):
    from paper_2112_14397_b200 import _lib as L
    from paper_2112_14397_b200.layer import DTSMoELayer

    cfg = configs.get(args.config)
    dev = torch.device("cuda", torch.cuda.current_device())
    li = inputs.make_inputs(cfg, rank=rank)
    dt = inputs.TORCH_DTYPE[cfg.dtype]
    tau, c = float(np.float32(cfg.tau)), float(np.float32(cfg.threshold))
    comm = 0
    if world > 1:
        from paper_2112_14397_b200.layer import make_nccl_comm
        comm = make_nccl_comm(rank, world)
    layer = DTSMoELayer(cfg.T, cfg.d_model, cfg.d_ff, cfg.E, dtype=dt, device=dev, rank=rank, world=world,
                        nccl_comm=comm)
    layer.set_gate(li.Wg.to(dev))
    layer.spawn(*(t.to(dev) for t in (li.W1s, li.b1s, li.W2s, li.b2s, li.M1bits, li.M2bits)))
    x, u, dy = li.x.to(dev), li.u.to(dev), li.dy.to(dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream()

    ev = lambda: torch.cuda.Event(enable_timing=True, external=True)  # noqa: E731  (usable inside graphs)

    # --- one step = the 8 C-ABI calls (DTSMoELayer.forward + backward), with events around the
    # expert GEMM calls on the launching stream.
    def full_step(timed: bool, R_cap=None):
        ev_ffn = (ev(), ev())
        ev_bwd = (ev(), ev())
        layer.forward(x, u, tau, c, R_cap=R_cap, events=ev_ffn if timed else None)
        layer.backward(dy, events=ev_bwd if timed else None)
        return ev_ffn, ev_bwd

    for _ in range(args.warmup):
        full_step(False)
    torch.cuda.synchronize()
    layer.check()
    R = int(layer.state.offsets[-1].item())
    counts = layer.state.counts.cpu().numpy()

    # --- CUDA graph of the whole step (single GPU): the row capacity is fixed to the routed
    # rows seen in warm-up (static capacity; an overflow would raise MOE_ECAPACITY at the
    # check after the timed region), so the step has no host synchronisation and is replayed
    # as one graph launch.
    graph = None
    n_launch0 = L.moe_kernel_launch_count()
    launches = None
    stage_ev = {}
    if args.graph and world == 1:
        R_static = layer.state.R_cap
        full_step(False, R_cap=R_static)
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        g_ffn, g_bwd = (ev(), ev()), (ev(), ev())
        n0 = L.moe_kernel_launch_count()
        with torch.cuda.graph(graph):
            layer.forward(x, u, tau, c, R_cap=R_static, events=g_ffn, stage_events=stage_ev)
            layer.backward(dy, events=g_bwd, stage_events=stage_ev)
        launches = L.moe_kernel_launch_count() - n0
        for _ in range(max(1, args.warmup)):
            graph.replay()
        torch.cuda.synchronize()
        layer.check()

    clocks = ClockSampler(torch.cuda.current_device())
    clocks.start()
    barrier(world)
    torch.cuda.synchronize()
    n_launch1 = L.moe_kernel_launch_count()
    step_ms, ffn_ms, bwd_ms = [], [], []
    stage_ms = {k: [] for k in stage_ev}
    t_wall = time.perf_counter()
    for _ in range(args.steps):
        flush.fill_(1)                       # L2 flush outside the timed events
        s0, s1 = ev(), ev()
        s0.record(stream)
        if graph is not None:
            graph.replay()
            e_f, e_b = g_ffn, g_bwd
        else:
            e_f, e_b = full_step(True)
        s1.record(stream)
        s1.synchronize()
        step_ms.append(s0.elapsed_time(s1))
        ffn_ms.append(e_f[0].elapsed_time(e_f[1]))
        bwd_ms.append(e_b[0].elapsed_time(e_b[1]))
        for k, (a, b) in stage_ev.items():
            stage_ms[k].append(a.elapsed_time(b))
    torch.cuda.synchronize()
    barrier(world)
    wall = time.perf_counter() - t_wall
    clk = clocks.stop()
    if launches is None:
        launches = (L.moe_kernel_launch_count() - n_launch1) // max(1, args.steps)
    layer.check()

    ms_step = max_over_ranks(sum(step_ms) / len(step_ms), world)
    tokens = cfg.T * world
    value = tokens / (ms_step / 1e3)

    # roofline: expert GEMMs (12 R d d_ff FLOPs per step: 2 fwd + 4 bwd GEMMs)
    peaks, peak_src = _peaks()
    flops = 12.0 * R * cfg.d_model * cfg.d_ff
    gemm_ms = (sum(ffn_ms) + sum(bwd_ms)) / len(ffn_ms)
    achieved = flops / (gemm_ms / 1e3) / 1e12
    peak = float(peaks.get("bf16_tflops_sustained", peaks.get("bf16_tflops")))
    step_flops = flops + 6.0 * cfg.T * cfg.d_model * cfg.E

    # e2e through the public API with host buffers
    e2e = run_e2e(args, layer, li, tau, c, world, (graph, x, u, dy) if graph is not None else None) \
        if args.e2e else None

    out = {
        "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "bf16" if cfg.dtype == "bf16" else "f32",
        "data": "synthetic (seeded N(0,1) tokens, N(0,1/d) gate, N(0,0.02) shared expert, Bernoulli(0.8) masks)",
        "config": {"workload": f"{cfg.name}: T={cfg.T}/GPU d_model={cfg.d_model} d_ff={cfg.d_ff} E={cfg.E} "
                               f"tau={cfg.tau} c={cfg.threshold}",
                   "tokens_per_gpu": cfg.T, "global_tokens": tokens, "rows_R": R,
                   "mean_experts_per_token": R / cfg.T if cfg.T else 0.0,
                   "max_over_mean_load": float(counts.max() / max(1e-9, counts.mean())),
                   "parallelism": f"ep{world} (E/{world} experts per GPU, NCCL all-to-all-v over NVLink)"
                   if world > 1 else "single",
                   "l2": "flushed between steps (256 MiB write, outside the events)",
                   "launch": "cuda-graph replay, static row capacity" if graph is not None else "eager",
                   "wall_s_timed_region": wall},
        "roofline": {"bound": "tensor", "kernel": "expert grouped GEMMs (moe_expert_ffn + moe_expert_ffn_bwd)",
                     "achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
                     "peak_source": f"{peak_src} bf16_tflops_sustained",
                     "frac_of_burst": achieved / float(peaks.get("bf16_tflops", peak)),
                     "gemm_ms_per_step": gemm_ms, "flops_per_step": flops,
                     "algorithmic_bytes_per_step": R * (12 * cfg.d_model + 16 * cfg.d_ff) * (1 if cfg.dtype == "bf16" else 2)
                     + cfg.E * cfg.d_model * cfg.d_ff * (4 * (2 if cfg.dtype == "bf16" else 4) + 2 * 4),
                     **_traffic(cfg.name, world)},
        "step_tflops": step_flops / (ms_step / 1e3) / 1e12,
        "stages": _stages(cfg, layer, counts, {k: sum(v) / len(v) for k, v in stage_ms.items() if v}),
        "gpu_launches": int(launches),
        "clocks": clk,
    }
    if e2e:
        out["e2e"] = e2e
    if rank == 0 and world == 1 and args.cpu_baseline:
        T_sub = args.cpu_tokens
        dt_cpu = oracle_sample(cfg, T_sub)
        out["cpu_baseline"] = {"value": T_sub / dt_cpu, "unit": "tokens/s", "cores": cpu_cores(), "kind": "oracle",
                               "sample": f"{T_sub} tokens of {cfg.name} (same d/d_ff/E/tau/c), fwd+bwd, fp64 NumPy, "
                                         f"{dt_cpu:.2f} s"}
    return out


def _stages(cfg, layer, counts, ms):
    """Per C-ABI stage: mean ms inside the replayed step and achieved GB/s of the stage's
    algorithmic HBM bytes (SURVEY §8d terms; GEMM operand traffic excluded) or TFLOP/s."""
    if not ms:
        return None
    b = 2 if cfg.dtype == "bf16" else 4
    T, d, f, E = cfg.T, cfg.d_model, cfg.d_ff, cfg.E
    R = int(counts.sum())
    Rp = int(layer.state.offsets[-1].item())
    Ep = (E + 15) // 16 * 16
    Kp = (2 * Ep + 63) // 64 * 64
    byts = {
        "gate": T * d * b + 3 * T * E * 4,
        "dispatch": 2 * T * E * 4 + T * d * b + Rp * (d * b + 8),
        "combine": R * d * b + T * d * b + T * E * 4 + R * 4,
        "combine_bwd": T * d * b + 2 * Rp * d * b + Rp * 12,
        "gate_bwd": R * 4 + 3 * T * E * 4 + T * Kp * 2 + T * d * b,
        "dispatch_bwd": T * E * 4 + R * d * b + 2 * T * d * 2 + T * d * b + T * Kp * 2,
    }
    flops = {"expert_ffn": 4.0 * Rp * d * f, "expert_ffn_bwd": 8.0 * Rp * d * f}
    out = {}
    for k, v in ms.items():
        o = {"ms": v}
        if k in byts:
            o["GB/s"] = byts[k] / (v / 1e3) / 1e9
            o["algorithmic_bytes"] = byts[k]
        if k in flops:
            o["TFLOP/s"] = flops[k] / (v / 1e3) / 1e12
        out[k] = o
    return out


def _traffic(name, world):
    """roofline.traffic: dram__bytes_read.sum + dram__bytes_write.sum of the expert GEMM set per
    step (the six tc_gemm_kernel launches that `achieved` covers), from the committed
    `ncu --set full` capture summary profiles/<round>/ncu_gemm_<workload>.json (null if none)."""
    import glob
    if world != 1:
        return {"traffic": None}
    hits = sorted(glob.glob(os.path.join(ROOT, "profiles", "r*", f"ncu_gemm_{name}.json")))
    if not hits:
        return {"traffic": None}
    with open(hits[-1]) as f:
        s = json.load(f)["expert_gemm_set"]
    return {"traffic": s["dram_bytes"], "traffic_unit": "bytes per step (6 launches)",
            "traffic_source": os.path.relpath(hits[-1], ROOT)}


def run_ours_p2p(args, rank, world):
    """The fused peer-memory EP path (paper_2112_14397_b200.ep2, moe_ep2_*): token rows are
    stored straight into the owners' expert-side layouts and gathered back over NVLink peer
    pointers inside the routing kernels (torch symmetric memory), no NCCL all-to-all.  Eager
    phases with stream-ordered NCCL barriers between them; the step and its expert-GEMM part
    are timed with CUDA events, max over ranks."""
    import torch.distributed as dist
    from paper_2112_14397_b200 import _lib as L
    from paper_2112_14397_b200.ep2 import EP2Rank, SymmetricBuffers
    from paper_2112_14397_b200.layer import make_nccl_comm

    cfg = configs.get(args.config)
    if cfg.dtype != "bf16":
        raise SystemExit("--ep p2p: bf16 configs only")
    dev = torch.device("cuda", torch.cuda.current_device())
    li = inputs.make_inputs(cfg, rank=rank)
    tau, c = float(np.float32(cfg.tau)), float(np.float32(cfg.threshold))
    comm = make_nccl_comm(rank, world)
    syms = SymmetricBuffers(world, dev, mode="symm_mem", group=dist.group.WORLD)
    r = EP2Rank(cfg.T, cfg.d_model, cfg.d_ff, cfg.E, torch.bfloat16, dev, rank, world, syms, comm=comm,
                dedup=args.ep == "p2p-dedup")
    r.set_gate(li.Wg.to(dev))
    r.spawn(*(t.to(dev) for t in (li.W1s, li.b1s, li.W2s, li.b2s, li.M1bits, li.M2bits)))
    x, u, dy = li.x.to(dev), li.u.to(dev), li.dy.to(dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream()
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731

    def step():
        r.forward(x, u, tau, c)
        return r.backward(dy)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    r.check()
    # rows of my experts (all ranks' tokens), for the GEMM FLOPs
    ca = r._sym("counts_all", (world, cfg.E), torch.int32)[0].cpu().numpy()
    R_mine = int(ca[:, rank * r.El:(rank + 1) * r.El].sum())

    clocks = ClockSampler(torch.cuda.current_device())
    clocks.start()
    barrier(world)
    torch.cuda.synchronize()
    n_launch0 = L.moe_kernel_launch_count()
    step_ms, gemm_ms = [], []
    t_wall = time.perf_counter()
    for _ in range(args.steps):
        flush.fill_(1)
        r.events = {"experts_fwd": (ev(), ev()), "experts_bwd": (ev(), ev())}
        s0, s1 = ev(), ev()
        s0.record(stream)
        step()
        s1.record(stream)
        s1.synchronize()
        step_ms.append(s0.elapsed_time(s1))
        gemm_ms.append(sum(a.elapsed_time(b) for a, b in r.events.values()))
    torch.cuda.synchronize()
    wall = time.perf_counter() - t_wall
    launches = (L.moe_kernel_launch_count() - n_launch0) // max(1, args.steps)
    r.events = None
    barrier(world)
    clk = clocks.stop()
    r.check()
    ms_step = max_over_ranks(sum(step_ms) / len(step_ms), world)
    g_ms = max_over_ranks(sum(gemm_ms) / len(gemm_ms), world)
    flops = 12.0 * R_mine * cfg.d_model * cfg.d_ff
    t = torch.tensor([flops], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t)
    flops_per_gpu = float(t.item()) / world
    peaks, peak_src = _peaks()
    peak = float(peaks.get("bf16_tflops_sustained", peaks.get("bf16_tflops")))
    achieved = flops_per_gpu / (g_ms / 1e3) / 1e12

    e2e = None
    if args.e2e:
        hx, hu, hdy = (tt.pin_memory() for tt in (li.x, li.u, li.dy))
        hy, hdx = torch.empty_like(li.x).pin_memory(), torch.empty_like(li.x).pin_memory()

        def step_host():
            x.copy_(hx, non_blocking=True)
            u.copy_(hu, non_blocking=True)
            dy.copy_(hdy, non_blocking=True)
            y = r.forward(x, u, tau, c)
            g = r.backward(dy)
            hy.copy_(y, non_blocking=True)
            hdx.copy_(g["dx"], non_blocking=True)

        step_host()
        torch.cuda.synchronize()
        barrier(world)
        e0, e1 = ev(), ev()
        e0.record(stream)
        for _ in range(args.steps):
            step_host()
        e1.record(stream)
        e1.synchronize()
        ms = max_over_ranks(e0.elapsed_time(e1) / args.steps, world)
        bi = sum(tt.numel() * tt.element_size() for tt in (hx, hu, hdy))
        bo = 2 * hy.numel() * hy.element_size()
        e2e = {"value": cfg.T * world / (ms / 1e3), "unit": "tokens/s", "ms_per_step": ms,
               "h2d_bytes_per_step": bi, "d2h_bytes_per_step": bo, "pipelined": False}
        r.check()

    out = {
        "metric": METRIC, "value": cfg.T * world / (ms_step / 1e3), "unit": "tokens/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (seeded N(0,1) tokens, N(0,1/d) gate, N(0,0.02) shared expert, Bernoulli(0.8) masks)",
        "config": {"workload": f"{cfg.name}: T={cfg.T}/GPU d_model={cfg.d_model} d_ff={cfg.d_ff} E={cfg.E} "
                               f"tau={cfg.tau} c={cfg.threshold}",
                   "tokens_per_gpu": cfg.T, "global_tokens": cfg.T * world, "rows_R_rank0": R_mine,
                   "parallelism": f"ep{world} (E/{world} experts per GPU, fused NVLink peer-memory dispatch / "
                                  f"combine, " + ("one row per (token, owner), moe_ep2d_*)" if r.dedup
                                                  else "moe_ep2_*)"),
                   "l2": "flushed between steps (256 MiB write, outside the events)", "launch": "eager phases",
                   "wall_s_timed_region": wall},
        "roofline": {"bound": "tensor", "kernel": "expert grouped GEMMs (moe_expert_ffn + moe_expert_ffn_bwd)",
                     "achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
                     "peak_source": f"{peak_src} bf16_tflops_sustained", "gemm_ms_per_step": g_ms,
                     "flops_per_step_per_gpu": flops_per_gpu, "traffic": None},
        "gpu_launches": int(launches),
        "clocks": clk,
    }
    if e2e:
        out["e2e"] = e2e
    return out


def run_e2e(args, layer, li, tau, c, world, graphed=None):
    """Same metric through the public API with host (pinned) buffers: every step copies x, u,
    dy host->device and reads y and dx back device->host.

    Graph mode pipelines the copies with compute: two captured replicas of the step (each with
    its own device input buffers) alternate; step i+1's H2D runs on a copy stream while step i
    computes, step i's D2H runs on a third stream.  Every byte of every step is still copied
    inside the timed region (first H2D start .. last D2H end)."""
    dev = layer.device
    hx, hu, hdy = (t.pin_memory() for t in (li.x, li.u, li.dy))
    hy = torch.empty_like(li.x).pin_memory()
    hdx = torch.empty_like(li.x).pin_memory()
    comp = torch.cuda.current_stream()
    bi = sum(t.numel() * t.element_size() for t in (hx, hu, hdy))
    bo = sum(t.numel() * t.element_size() for t in (hy, hdx))

    if graphed is None:
        def step():
            x = hx.to(dev, non_blocking=True)
            u = hu.to(dev, non_blocking=True)
            dy = hdy.to(dev, non_blocking=True)
            y = layer.forward(x, u, tau, c)
            g = layer.backward(dy)
            hy.copy_(y, non_blocking=True)
            hdx.copy_(g["dx"], non_blocking=True)

        for _ in range(2):
            step()
        torch.cuda.synchronize()
        barrier(world)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(comp)
        for _ in range(args.steps):
            step()
        e1.record(comp)
        e1.synchronize()
        ms = max_over_ranks(e0.elapsed_time(e1) / args.steps, world)
        return {"value": layer.T * world / (ms / 1e3), "unit": "tokens/s", "ms_per_step": ms,
                "h2d_bytes_per_step": bi, "d2h_bytes_per_step": bo, "pipelined": False}

    # ---- two graph replicas with their own static inputs, copies overlapped with compute
    R_static = layer.state.R_cap
    reps = []
    for k in range(2):
        X = torch.empty_like(li.x, device=dev)
        U = torch.empty_like(li.u, device=dev)
        DY = torch.empty_like(li.dy, device=dev)
        X.copy_(hx); U.copy_(hu); DY.copy_(hdy)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            Y = layer.forward(X, U, tau, c, R_cap=R_static)
            DX = layer.backward(DY)["dx"]
        reps.append((g, X, U, DY, Y, DX))
    torch.cuda.synchronize()
    s_h2d, s_d2h = torch.cuda.Stream(), torch.cuda.Stream()
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    in_free = [ev(), ev()]     # replica k finished reading its inputs (compute done)
    h2d_done = [ev(), ev()]
    comp_done = [ev(), ev()]
    out_free = [ev(), ev()]    # replica k's outputs copied to the host
    for k in range(2):
        in_free[k].record(comp)
        out_free[k].record(comp)

    def run(n):
        t0, t1 = ev(), ev()
        t0.record(s_h2d)
        for i in range(n):
            k = i % 2
            g, X, U, DY, Y, DX = reps[k]
            with torch.cuda.stream(s_h2d):
                s_h2d.wait_event(in_free[k])
                X.copy_(hx, non_blocking=True)
                U.copy_(hu, non_blocking=True)
                DY.copy_(hdy, non_blocking=True)
                h2d_done[k].record(s_h2d)
            comp.wait_event(h2d_done[k])
            comp.wait_event(out_free[k])
            g.replay()
            comp_done[k].record(comp)
            in_free[k].record(comp)
            with torch.cuda.stream(s_d2h):
                s_d2h.wait_event(comp_done[k])
                hy.copy_(Y, non_blocking=True)
                hdx.copy_(DX, non_blocking=True)
                out_free[k].record(s_d2h)
        t1.record(s_d2h)
        t1.synchronize()
        return t0.elapsed_time(t1)

    run(4)
    torch.cuda.synchronize()
    barrier(world)
    ms = max_over_ranks(run(args.steps) / args.steps, world)
    layer.check()
    return {"value": layer.T * world / (ms / 1e3), "unit": "tokens/s", "ms_per_step": ms,
            "h2d_bytes_per_step": bi, "d2h_bytes_per_step": bo, "pipelined": True}


# ------------------------------------------------------------------ reference arm (the oracle)
def run_reference(args, rank, world):
    if rank != 0:
        return None
    cfg = configs.get(args.config)
    T_sub = args.ref_tokens
    for _ in range(args.warmup):
        oracle_sample(cfg, T_sub)
    times = [oracle_sample(cfg, T_sub) for _ in range(args.steps)]
    ms = 1e3 * sum(times) / len(times)
    value = T_sub / (ms / 1e3)
    return {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{cfg.name}: T={cfg.T}/GPU d_model={cfg.d_model} d_ff={cfg.d_ff} E={cfg.E} "
                               f"tau={cfg.tau} c={cfg.threshold}", "sample_tokens_per_step": T_sub},
        "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": cpu_cores(), "kind": "oracle",
                         "sample": f"{T_sub} tokens of {cfg.name} per step, fwd+bwd, fp64 NumPy oracle"},
        "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="C2")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", dest="e2e", action="store_false")
    ap.add_argument("--no-cpu-baseline", dest="cpu_baseline", action="store_false")
    ap.add_argument("--cpu-tokens", type=int, default=1024)
    ap.add_argument("--ref-tokens", type=int, default=256)
    ap.add_argument("--no-graph", dest="graph", action="store_false",
                    help="launch the step eagerly instead of replaying a CUDA graph")
    ap.add_argument("--ep", default="nccl", choices=["nccl", "p2p", "p2p-dedup"],
                    help="expert-parallel exchange: NCCL grouped send/recv (default), the fused NVLink "
                         "peer-memory path (moe_ep2_*, torch symmetric memory), or the same with one row "
                         "per (token, owner) each way (moe_ep2d_*)")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        print("warning: fewer than 3 warm-up steps", file=sys.stderr)
    if args.impl == "reference":
        rank = int(os.environ.get("RANK", "0"))
        world = int(os.environ.get("WORLD_SIZE", "1"))
        out = run_reference(args, rank, world)
        if out is not None:
            print(json.dumps(out))
        return 0
    p2p = args.ep.startswith("p2p")
    rank, world, local = dist_setup(args.gpus, force_pg=p2p)
    out = run_ours_p2p(args, rank, world) if p2p else run_ours(args, rank, world)
    if rank == 0:
        print(json.dumps(out))
    import torch.distributed as dist
    if dist.is_initialized():
        import torch.distributed as dist
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
