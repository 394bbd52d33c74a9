"""bench.py -- DTS-Gate MoE layer forward+backward throughput on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C4] [--impl ours|reference]
                    [--ep p2p|p2p-dedup|nccl]

One "step" = one pass of the whole hot path over one batch of synthetic tokens:
moe_dts_gate -> moe_dispatch -> moe_expert_ffn -> moe_combine -> moe_combine_bwd ->
moe_expert_ffn_bwd -> moe_dts_gate_bwd -> moe_dispatch_bwd (all through the C ABI; under EP
the exchanges are fused into the routing kernels as NVLink peer loads / stores).  The spawn
runs once before timing (an initialisation step, Alg. 1 lines 4-5) and is timed on its own.

Workload: BASELINE.json configs[3] (C4: T=131072 tokens per GPU, d=1024, d_ff=4096, E=64,
tau=0.1, c=0.2), the one config the metric names at 1/2/4/8 GPUs, so the N=1 line and the
N>1 lines of the scaling run measure the same per-GPU work (weak scaling).  --config C2 (the
GPT-small "1 GPU" config) etc. select another.  Synthetic seeded data (harness/inputs.py);
every timed step draws its Gumbel noise from a pool of 4 different resident u tensors, so the
routing changes from step to step as in training.

N > 1: `python bench.py --gpus N` re-launches itself under torch.distributed.run (one rank per
GPU) when WORLD_SIZE is not set; NCCL_DEBUG=INFO lines go to stderr.  Each rank holds T tokens
and E/N experts; the default exchange is the fused peer-memory path (ep2, torch symmetric
memory) captured as one CUDA graph per step; --ep nccl selects the NCCL send/recv path.

Timing: W untimed warm-up steps; then K steps, each bracketed by CUDA events on the launching
stream, with an L2 flush (write of a 256 MiB buffer) and the copy of the next u between steps,
outside the events; barrier + synchronize on both sides; the max over ranks is reported.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import socket
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
DEFAULT_CONFIG = "C4"
U_POOL = 4
DATASHEET_BF16_TFLOPS = 2250.0
NVLINK_GBS = 900.0      # NVLink 5 per direction per GPU (task statement; not measured here)


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            return json.load(f), "MEASURED_PEAKS.json"
    except Exception:
        # /opt/skills/guides/B200_PROFILING.md fallback figures
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, \
            "fallback (B200_PROFILING.md)"


def pick_peak(peaks, wall_s: float, clk: dict):
    """Burst peak for a short timed window at full clocks, sustained peak for a long one or a
    power-capped one (the 67 ms C2 window ran at burst clocks, so its denominator
    is the burst figure)."""
    burst = float(peaks.get("bf16_tflops"))
    sust = float(peaks.get("bf16_tflops_sustained", burst))
    sm, smax = clk.get("sm_mhz"), clk.get("sm_max_mhz") or peaks.get("sm_max_mhz")
    capped = bool(sm and smax and sm < 0.9 * smax)
    if wall_s < 1.0 and not capped:
        return burst, "bf16_tflops (burst: timed window < 1 s at full clocks)"
    return sust, ("bf16_tflops_sustained (" + ("SM clock median %.0f of %.0f MHz" % (sm, smax) if capped
                                               else "timed window %.1f s" % wall_s) + ")")


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
def relaunch_under_torchrun(args, out_stream) -> int:
    """`python bench.py --gpus N` with no WORLD_SIZE: run N ranks (one per GPU) under
    torch.distributed.run on this node; rank 0's JSON line comes through our stdout."""
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    env = dict(os.environ)
    print(f"bench.py: launching {args.gpus} ranks: {' '.join(cmd)}", file=sys.stderr, flush=True)
    return subprocess.call(cmd, env=env, stdout=out_stream)


def dist_setup(force_pg: bool = False):
    """force_pg: a 1-rank NCCL process group for --ep at N = 1 (the EP code path, its symmetric
    allocations and barriers, on one GPU)."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if force_pg and world == 1 and "MASTER_ADDR" not in os.environ:
        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK="0", WORLD_SIZE="1")
    if world > 1 or force_pg:
        import torch.distributed as dist
        if torch.cuda.device_count() <= local:
            raise SystemExit(f"bench.py: rank {rank} needs GPU {local}, only {torch.cuda.device_count()} visible")
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    return rank, world, local


def barrier(world):
    import torch.distributed as dist
    if world > 1 or dist.is_initialized():
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(v: float, world: int) -> float:
    if world == 1:
        return v
    import torch.distributed as dist
    t = torch.tensor([v], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(v: float, world: int) -> float:
    if world == 1:
        return v
    import torch.distributed as dist
    t = torch.tensor([v], dtype=torch.float64, device="cuda")
    dist.all_reduce(t)
    return float(t.item())


# ------------------------------------------------------------------ CPU baseline (oracle)
def oracle_sample(cfg, T_sub: int, step: int = 0, gpu_slot=None):
    """Time the fp64 oracle (as it stands) on the first T_sub tokens of the workload, fwd+bwd.
    With gpu_slot (the GPU's slot rows of those tokens) also count the selection flips against
    the oracle's mask (flips are allowed only inside the 1e-6 band)."""
    from oracle import dts_moe as O
    li = inputs.make_inputs(cfg, T=T_sub, step=step)
    ex = O.spawn(inputs.to_f64(li.W1s), inputs.to_f64(li.b1s), inputs.to_f64(li.W2s), inputs.to_f64(li.b2s),
                 inputs.bits_u32(li.M1bits), inputs.bits_u32(li.M2bits))
    x, Wg, u, dy = (inputs.to_f64(t) for t in (li.x, li.Wg, li.u, li.dy))
    t0 = time.perf_counter()
    fw = O.forward(x, Wg, u, float(np.float32(cfg.tau)), float(np.float32(cfg.threshold)), ex, top1=cfg.top1)
    O.backward(fw, dy)
    dt = time.perf_counter() - t0
    flips = None
    if gpu_slot is not None:
        flips = int(np.any(fw.m != (gpu_slot >= 0), axis=1).sum())
    return dt, flips


def cpu_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


# ------------------------------------------------------------------ shared helpers
def _u_pool(cfg, rank, dev):
    """U_POOL different Gumbel-noise inputs (harness steps 0..3), resident in HBM."""
    return [inputs.uniform_u(cfg.T, cfg.E, step=s, rank=rank).to(dev) for s in range(U_POOL)]


def spawn_timing(L, ctx, li, dev, cfg, El, reps=5):
    """moe_dts_spawn (Alg. 1 l.4-5) timed alone: GB/s of its algorithmic bytes (read W1s/W2s and
    the packed masks of the local experts once, write E_local masked copies + biases)."""
    b = 2 if cfg.dtype == "bf16" else 4
    d, f = cfg.d_model, cfg.d_ff
    srcs = [t.to(dev) for t in (li.W1s, li.b1s, li.W2s, li.b2s, li.M1bits, li.M2bits)]
    kw = dict(dtype=inputs.TORCH_DTYPE[cfg.dtype], device=dev)
    outs = [torch.empty(El, f, d, **kw), torch.empty(El, f, **kw), torch.empty(El, d, f, **kw), torch.empty(El, d, **kw)]
    L.moe_dts_spawn(ctx, *srcs, *outs)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        L.moe_dts_spawn(ctx, *srcs, *outs)
    e1.record()
    e1.synchronize()
    ms = e0.elapsed_time(e1) / reps
    words = (d * f + 31) // 32
    byts = 2 * d * f * b + (d + f) * b + El * 2 * words * 4 + El * (2 * d * f + d + f) * b
    return {"ms": ms, "algorithmic_bytes": byts, "GB/s": byts / (ms / 1e3) / 1e9,
            "what": f"{El} local experts: W1/W2 masked copies + biases"}


def _stages(cfg, R, Rp, ms):
    """Per C-ABI stage: mean ms inside the replayed step and achieved GB/s of the stage's
    algorithmic HBM bytes (SURVEY §8d terms; GEMM operand traffic excluded) or TFLOP/s."""
    if not ms:
        return None
    b = 2 if cfg.dtype == "bf16" else 4
    T, d, f, E = cfg.T, cfg.d_model, cfg.d_ff, cfg.E
    Ep = (E + 15) // 16 * 16
    Kp = (2 * Ep + 63) // 64 * 64
    byts = {
        "gate": T * d * b + 3 * T * E * 4,
        "dispatch": 2 * T * E * 4 + T * d * b + Rp * (d * b + 8),
        "combine": R * d * b + T * d * b + T * E * 4 + R * 4,
        "combine_bwd": T * d * b + 2 * Rp * d * b + Rp * 12,
        "gate_bwd": R * 4 + 3 * T * E * 4 + T * Kp * 2 + 2 * T * d * b,
        "dispatch_bwd": T * E * 4 + R * d * b + 2 * T * d * b,
    }
    flops = {"expert_ffn": 4.0 * R * d * f, "expert_ffn_bwd": 8.0 * R * d * f}
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



def gemm_roofline_us(R, d, f, E, peaks):
    """Roofline of the six expert GEMMs of one fwd+bwd over R realised rows (E experts with rows,
    bf16 activations and weights, fp32 weight gradients): per GEMM max(tensor time at the burst
    bf16 peak, HBM time of its algorithmic bytes at the measured copy bandwidth).  At the sparse
    end the weights (read four times) and the fp32 weight gradients dominate the bytes, so the
    late steps are HBM-bound, not tensor-bound."""
    fl = 2.0 * R * d * f
    w = 2.0 * E * d * f
    byts = [2 * R * d + w + 4 * R * f,          # GEMM1: x_perm, W1 -> h, GELU'(a)
            2 * R * f + w + 2 * R * d,          # GEMM2: h, W2 -> e_out
            2 * R * d + w + 4 * R * f,          # dgrad2: d_eout, W2, GELU'(a) -> da
            2 * R * f + w + 2 * R * d,          # dgrad1: da, W1 -> dx_perm
            2 * R * d + 2 * R * f + 2 * w,      # dW1: x_perm, da -> fp32 dW1
            2 * R * f + 2 * R * d + 2 * w]      # dW2: h, d_eout -> fp32 dW2
    t_tc = fl / (peaks["bf16_tflops"] * 1e12) * 1e6
    parts = [max(t_tc, b / (peaks["hbm_gbs"] * 1e9) * 1e6) for b in byts]
    return sum(parts), sum(1 for b in byts if b / (peaks["hbm_gbs"] * 1e9) * 1e6 > t_tc)


FP32_FMA_LANES_PER_SM = 128      # fp32 FMA lanes per SM per clock (measured: profiles/r02/ab_epilogue_math.txt)


def _roofline(cfg, flops_per_gpu, gemm_ms, wall, clk, world, R_pad):
    peaks, src = _peaks()
    peak, which = pick_peak(peaks, wall, clk)
    bound = "tensor"
    if cfg.dtype != "bf16":
        # the fp32 configuration (C1) runs its expert GEMMs on the CUDA cores (FFMA): bound by plain
        # ALU arithmetic, against SMs x 128 FMA lanes x 2 FLOP x the SM clock
        sms = torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count
        mhz = float(clk.get("sm_mhz") or peaks.get("sm_max_mhz") or 1965.0)
        peak = sms * FP32_FMA_LANES_PER_SM * 2 * mhz * 1e6 / 1e12
        bound, src, which = "alu", "derived", (f"fp32 FFMA: {sms} SMs x {FP32_FMA_LANES_PER_SM} lanes x 2 FLOP x "
                                               f"{mhz:.0f} MHz (median SM clock of the timed region)")
    achieved = flops_per_gpu / (gemm_ms / 1e3) / 1e12
    b = 2 if cfg.dtype == "bf16" else 4
    d, f, E = cfg.d_model, cfg.d_ff, cfg.E // world
    R = flops_per_gpu / (12.0 * d * f)
    return {"bound": bound, "kernel": "expert grouped GEMMs (moe_expert_ffn + moe_expert_ffn_bwd)",
            "achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
            "peak_source": f"{src} {which}",
            "frac_of_burst": achieved / float(peaks["bf16_tflops"]),
            "frac_of_sustained": achieved / float(peaks.get("bf16_tflops_sustained", peaks["bf16_tflops"])),
            "pct_peak_datasheet": 100.0 * achieved / DATASHEET_BF16_TFLOPS,
            "gemm_ms_per_step": gemm_ms, "flops_per_step": flops_per_gpu,
            "flops_rows": "realised (token, expert) rows = sum of counts (pad rows excluded)",
            "rows_R_pad": R_pad,
            "algorithmic_bytes_per_step": R * (12 * d + 16 * f) * (b // 2)
            + E * d * f * (4 * b + 2 * 4),
            **_gemm_mixed(R, d, f, E, peaks, gemm_ms),
            **_traffic(cfg.name, world)}


def _gemm_mixed(R, d, f, E, peaks, gemm_ms):
    roof_us, n_hbm = gemm_roofline_us(R, d, f, E, peaks)
    return {"gemm_roofline_ms_max_tensor_hbm": roof_us / 1e3, "gemm_frac_of_max_tensor_hbm": roof_us / 1e3 / gemm_ms,
            "gemms_hbm_bound": n_hbm}


def _config(cfg, world, extra):
    c = {"workload": f"{cfg.name}: T={cfg.T}/GPU d_model={cfg.d_model} d_ff={cfg.d_ff} E={cfg.E} "
                     f"tau={cfg.tau} c={cfg.threshold}",
         "tokens_per_gpu": cfg.T, "global_tokens": cfg.T * world,
         "l2": "flushed between steps (256 MiB write, outside the events)",
         "noise": f"fresh Gumbel u every step (pool of {U_POOL} resident u tensors, copied in outside the events)"}
    c.update(extra)
    return c


def _base_line(cfg, world, args, ms_step, value):
    return {"metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "bf16" if cfg.dtype == "bf16" else "f32",
            "data": "synthetic (seeded N(0,1) tokens, N(0,v) gate, N(0,0.02) shared expert, Bernoulli(0.8) masks; "
                    "random-init weights)"}


# ------------------------------------------------------------------ N = 1: the single-GPU layer
def run_single(args):
    from paper_2112_14397_b200 import _lib as L
    from paper_2112_14397_b200.layer import DTSMoELayer, padded_rows

    cfg = configs.get(args.config)
    dev = torch.device("cuda", torch.cuda.current_device())
    li = inputs.make_inputs(cfg)
    dt = inputs.TORCH_DTYPE[cfg.dtype]
    tau, c = float(np.float32(cfg.tau)), float(np.float32(cfg.threshold))
    layer = DTSMoELayer(cfg.T, cfg.d_model, cfg.d_ff, cfg.E, dtype=dt, device=dev)
    layer.set_gate(li.Wg.to(dev))
    layer.spawn(*(t.to(dev) for t in (li.W1s, li.b1s, li.W2s, li.b2s, li.M1bits, li.M2bits)))
    spawn = spawn_timing(L, layer.ctx, li, dev, cfg, cfg.E)
    x, dy = li.x.to(dev), li.dy.to(dev)
    upool = _u_pool(cfg, 0, dev)
    u = upool[0].clone()                      # the static noise input the graph reads
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream()
    ev = lambda: torch.cuda.Event(enable_timing=True, external=True)  # noqa: E731  (usable inside graphs)

    # warm-up (eager; sizes the row buffers from the counts) over the whole noise pool: the static
    # row capacity of the graph covers every pool member's routing
    rpad = []
    for i in range(max(args.warmup, U_POOL)):
        u.copy_(upool[i % U_POOL])
        layer.forward(x, u, tau, c)
        layer.backward(dy)
        rpad.append(padded_rows(layer.state.counts.cpu().tolist()))
    torch.cuda.synchronize()
    layer.check()
    R_static = max(rpad)

    graph, launches, stage_ev = None, None, {}
    g_ffn, g_bwd = (ev(), ev()), (ev(), ev())
    if args.graph:
        layer.forward(x, u, tau, c, R_cap=R_static)
        layer.backward(dy)
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        n0 = L.moe_kernel_launch_count()
        with torch.cuda.graph(graph):
            layer.forward(x, u, tau, c, R_cap=R_static, events=g_ffn, stage_events=stage_ev)
            layer.backward(dy, events=g_bwd, stage_events=stage_ev)
        launches = L.moe_kernel_launch_count() - n0
        for i in range(max(1, args.warmup)):
            u.copy_(upool[i % U_POOL])
            graph.replay()
        torch.cuda.synchronize()
        layer.check()

    clocks = ClockSampler(torch.cuda.current_device())
    clocks.start()
    torch.cuda.synchronize()
    n_launch1 = L.moe_kernel_launch_count()
    step_ms, gemm_ms, rows, band = [], [], [], []
    stage_ms = {k: [] for k in stage_ev}
    t_wall = time.perf_counter()
    for i in range(args.steps):
        flush.fill_(1)                       # L2 flush and the next step's noise, outside the events
        u.copy_(upool[i % U_POOL])
        s0, s1 = ev(), ev()
        s0.record(stream)
        if graph is not None:
            graph.replay()
            e_f, e_b = g_ffn, g_bwd
        else:
            e_f, e_b = (ev(), ev()), (ev(), ev())
            layer.forward(x, u, tau, c, events=e_f)
            layer.backward(dy, events=e_b)
        s1.record(stream)
        s1.synchronize()
        step_ms.append(s0.elapsed_time(s1))
        gemm_ms.append(e_f[0].elapsed_time(e_f[1]) + e_b[0].elapsed_time(e_b[1]))
        for k, (a, b) in stage_ev.items():
            stage_ms[k].append(a.elapsed_time(b))
        rows.append(int(layer.state.counts.sum().item()))          # realised rows (outside the events)
        band.append(int(layer.state.near_band.item()))
    torch.cuda.synchronize()
    wall = time.perf_counter() - t_wall
    clk = clocks.stop()
    if launches is None:
        launches = (L.moe_kernel_launch_count() - n_launch1) // max(1, args.steps)
    layer.check()                            # MOE_ECAPACITY here would mean the static capacity was short
    counts = layer.state.counts.cpu().numpy()

    ms_step = sum(step_ms) / len(step_ms)
    value = cfg.T / (ms_step / 1e3)
    R_mean = sum(rows) / len(rows)
    flops = 12.0 * R_mean * cfg.d_model * cfg.d_ff
    g_ms = sum(gemm_ms) / len(gemm_ms)
    out = _base_line(cfg, 1, args, ms_step, value)
    out["config"] = _config(cfg, 1, {
        "rows_R_mean": R_mean, "rows_R_pad_static": R_static, "mean_experts_per_token": R_mean / cfg.T,
        "max_over_mean_load": float(counts.max() / max(1e-9, counts.mean())),
        "band_tokens": {"mean_per_step": sum(band) / len(band), "max": max(band),
                        "what": "tokens with an fp32 p within 1e-6 of c (or top-2 gap < 1e-6 when argmax-decided)"},
        "parallelism": "single GPU (E experts local, no exchange)",
        "launch": "cuda-graph replay, static row capacity" if graph is not None else "eager",
        "wall_s_timed_region": wall})
    out["roofline"] = _roofline(cfg, flops, g_ms, wall, clk, 1, R_static)
    out["step_tflops"] = (flops + 6.0 * cfg.T * cfg.d_model * cfg.E) / (ms_step / 1e3) / 1e12
    out["stages"] = _stages(cfg, int(round(R_mean)), R_static,
                            {k: sum(v) / len(v) for k, v in stage_ms.items() if v})
    out["spawn"] = spawn
    out["gpu_launches"] = int(launches)
    out["clocks"] = clk
    if args.e2e:
        def capture(X, U, DY):
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                Y = layer.forward(X, U, tau, c, R_cap=R_static)
                DX = layer.backward(DY)["dx"]
            return g, Y, DX

        def eager_step(x_, u_, dy_):
            y_ = layer.forward(x_, u_, tau, c)
            return y_, layer.backward(dy_)["dx"]
        out["e2e"] = run_e2e(args, li, upool, cfg.T, 1, eager_step, capture if graph is not None else None,
                             layer.check)
    if args.cpu_baseline:
        T_sub = args.cpu_tokens
        # the GPU's routing of the sample tokens (pool member 0 = harness step 0, as the oracle draws)
        u.copy_(upool[0])
        layer.forward(x, u, tau, c)
        slot0 = layer.state.slot[:T_sub].cpu().numpy()
        band0 = int(layer.state.near_band.item())
        dt_cpu, flips = oracle_sample(cfg, T_sub, gpu_slot=slot0)
        out["cpu_baseline"] = {"value": T_sub / dt_cpu, "unit": "tokens/s", "cores": cpu_cores(), "kind": "oracle",
                               "sample": f"first {T_sub} tokens of {cfg.name} (same d/d_ff/E/tau/c), fwd+bwd, "
                                         f"fp64 NumPy, {dt_cpu:.2f} s"}
        out["config"]["mask_flips"] = {"sample_tokens": T_sub, "flips": flips,
                                       "band_tokens_all": band0,
                                       "what": "tokens of the oracle sample whose GPU selection differs from the "
                                               "fp64 oracle's (allowed only inside the band)"}
    return out


def run_e2e(args, li, upool, T_all, world, eager_step, capture, check):
    """Same metric through the public API with host (pinned) buffers: every step copies x, u,
    dy host->device and reads y and dx back device->host.

    capture(X, U, DY) -> (graph, Y, DX): one step captured as a CUDA graph on the given device
    inputs (None: no graph mode, then eager_step(x, u, dy) -> (y, dx) runs each step).
    Graph mode pipelines the copies with compute: two captured replicas of the step (each with
    its own device input buffers) alternate; step i+1's H2D runs on a copy stream while step i
    computes, step i's D2H runs on a third stream.  Every byte of every step is still copied
    inside the timed region (first H2D start .. last D2H end); max over ranks."""
    dev = torch.device("cuda", torch.cuda.current_device())
    hx, hdy = li.x.pin_memory(), li.dy.pin_memory()
    hus = [u.cpu().pin_memory() for u in upool]
    hy = torch.empty_like(li.x).pin_memory()
    hdx = torch.empty_like(li.x).pin_memory()
    comp = torch.cuda.current_stream()
    bi = sum(t.numel() * t.element_size() for t in (hx, hus[0], hdy))
    bo = sum(t.numel() * t.element_size() for t in (hy, hdx))

    if capture is None:
        def step(i):
            x = hx.to(dev, non_blocking=True)
            u = hus[i % U_POOL].to(dev, non_blocking=True)
            dy = hdy.to(dev, non_blocking=True)
            y, dx = eager_step(x, u, dy)
            hy.copy_(y, non_blocking=True)
            hdx.copy_(dx, non_blocking=True)

        for i in range(2):
            step(i)
        torch.cuda.synchronize()
        barrier(world)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(comp)
        for i in range(args.steps):
            step(i)
        e1.record(comp)
        e1.synchronize()
        ms = max_over_ranks(e0.elapsed_time(e1) / args.steps, world)
        check()
        return {"value": T_all / (ms / 1e3), "unit": "tokens/s", "ms_per_step": ms,
                "h2d_bytes_per_step": bi, "d2h_bytes_per_step": bo, "pipelined": False}

    reps = []
    for k in range(2):
        X = torch.empty_like(li.x, device=dev)
        U = torch.empty_like(hus[0], device=dev)
        DY = torch.empty_like(li.dy, device=dev)
        X.copy_(hx); U.copy_(hus[0]); DY.copy_(hdy)
        g, Y, DX = capture(X, U, DY)
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
                U.copy_(hus[i % U_POOL], non_blocking=True)
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

    def copies_only(n):
        """The same per-step copies on the same streams with no compute: the host-link bound."""
        g, X, U, DY, Y, DX = reps[0]
        t0, t1, t2 = ev(), ev(), ev()
        t0.record(comp)
        s_h2d.wait_stream(comp)
        s_d2h.wait_stream(comp)
        for i in range(n):
            with torch.cuda.stream(s_h2d):
                X.copy_(hx, non_blocking=True)
                U.copy_(hus[i % U_POOL], non_blocking=True)
                DY.copy_(hdy, non_blocking=True)
            with torch.cuda.stream(s_d2h):
                hy.copy_(Y, non_blocking=True)
                hdx.copy_(DX, non_blocking=True)
        t1.record(s_h2d)
        t2.record(s_d2h)
        t1.synchronize()
        t2.synchronize()
        return max(t0.elapsed_time(t1), t0.elapsed_time(t2))

    run(4)
    torch.cuda.synchronize()
    barrier(world)
    ms = max_over_ranks(run(args.steps) / args.steps, world)
    check()
    n_link = max(2, min(args.steps, 5))
    # the faster of two probes (PCIe throughput varies run to run; the bound is the best case)
    link_ms = max_over_ranks(min(copies_only(n_link), copies_only(n_link)) / n_link, world)
    return {"value": T_all / (ms / 1e3), "unit": "tokens/s", "ms_per_step": ms,
            "h2d_bytes_per_step": bi, "d2h_bytes_per_step": bo, "pipelined": True,
            "link_bound": {"ms_per_step": link_ms, "tokens_per_s": T_all / (link_ms / 1e3),
                           "frac": link_ms / ms, "GB/s_both_directions": (bi + bo) / link_ms / 1e6,
                           "what": "the step's host<->device copies alone, both directions at once on the "
                                   "same streams (pinned host memory); frac = link-bound time / e2e time"}}


# ------------------------------------------------------------------ N > 1: expert parallelism
def _nvlink_bytes(cfg, counts_all, rank, world):
    """Algorithmic NVLink bytes this rank moves per step on the peer-memory path (no dedup):
    its rows to / from remote owners (x out, e_out back, dy read by the owner, dx_perm back:
    4 rows of d elements each) plus the owners reading this rank's remote rows' metadata
    (SURVEY §8(d) B_NVL = (4 b d + 12) R_remote)."""
    b = 2 if cfg.dtype == "bf16" else 4
    El = cfg.E // world
    mine = counts_all[rank]
    remote = int(sum(mine[e] for e in range(cfg.E) if e // El != rank))
    return remote * (4 * b * cfg.d_model + 12)


def run_ep(args, rank, world):
    """Expert-parallel step on `world` GPUs (E/world experts per GPU, T tokens per GPU)."""
    import torch.distributed as dist
    from paper_2112_14397_b200 import _lib as L
    from paper_2112_14397_b200.layer import make_nccl_comm

    cfg = configs.get(args.config)
    dev = torch.device("cuda", torch.cuda.current_device())
    li = inputs.make_inputs(cfg, rank=rank)
    dt = inputs.TORCH_DTYPE[cfg.dtype]
    tau, c = float(np.float32(cfg.tau)), float(np.float32(cfg.threshold))
    comm = make_nccl_comm(rank, world)
    x, dy = li.x.to(dev), li.dy.to(dev)
    upool = _u_pool(cfg, rank, dev)
    u = upool[0].clone()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream()
    ev = lambda: torch.cuda.Event(enable_timing=True, external=True)  # noqa: E731
    El = cfg.E // world
    path, note = args.ep, None
    runner = None
    if path.startswith("p2p"):
        try:
            from paper_2112_14397_b200.ep2 import EP2Rank, SymmetricBuffers
            syms = SymmetricBuffers(world, dev, mode="symm_mem", group=dist.group.WORLD)
            r = EP2Rank(cfg.T, cfg.d_model, cfg.d_ff, cfg.E, dt, dev, rank, world, syms, comm=comm,
                        dedup=path == "p2p-dedup", overlap=not args.no_overlap)
            r.set_gate(li.Wg.to(dev))
            r.spawn(*(t.to(dev) for t in (li.W1s, li.b1s, li.W2s, li.b2s, li.M1bits, li.M2bits)))
            dyb = r.dy_buffer()
            dyb.copy_(dy)
            runner = r
        except Exception as e:   # symmetric memory unavailable: the NCCL exchange path instead
            note = f"peer-memory path unavailable ({type(e).__name__}: {e}); NCCL exchange used"
            print("bench.py: " + note, file=sys.stderr, flush=True)
            path = "nccl"
    if path == "nccl":
        from paper_2112_14397_b200.layer import DTSMoELayer
        layer = DTSMoELayer(cfg.T, cfg.d_model, cfg.d_ff, cfg.E, dtype=dt, device=dev, rank=rank, world=world,
                            nccl_comm=comm)
        layer.set_gate(li.Wg.to(dev))
        layer.spawn(*(t.to(dev) for t in (li.W1s, li.b1s, li.W2s, li.b2s, li.M1bits, li.M2bits)))
        spawn = spawn_timing(L, layer.ctx, li, dev, cfg, El)

        def step(events=None):
            layer.forward(x, u, tau, c, events=events[0] if events else None)
            return layer.backward(dy, events=events[1] if events else None)

        def counts_now():
            return L.moe_ep_exchange_counts(layer.ctx, layer.state.counts, world, cfg.E)
        check = layer.check
    else:
        r = runner
        spawn = spawn_timing(L, r.ctx, li, dev, cfg, El)

        def step(events=None):
            r.events = {"experts_fwd": events[0], "experts_bwd": events[1]} if events else None
            r.forward(x, u, tau, c, cfg.top1)
            return r.backward(dyb)

        def counts_now():
            return r.counts_all_host()
        check = r.check

    # warm-up over the noise pool (eager; the first step sizes the peer-memory capacity, and any
    # overflow of a later pool member grows it before the capture)
    for i in range(max(args.warmup, U_POOL)):
        u.copy_(upool[i % U_POOL])
        if path == "nccl":
            step()
            check()
        else:
            r.step(x, u, dyb, tau, c, cfg.top1)
    torch.cuda.synchronize()
    counts_all = counts_now()
    graph = None
    g_ev = ((ev(), ev()), (ev(), ev()))
    stage_ev = {}
    n0 = L.moe_kernel_launch_count()
    if path != "nccl" and args.graph:
        r.prepare()
        s = torch.cuda.Stream()
        s.wait_stream(stream)
        with torch.cuda.stream(s):
            step()
        stream.wait_stream(s)
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        n0 = L.moe_kernel_launch_count()
        r.stage_events = stage_ev
        with torch.cuda.graph(graph):
            step(g_ev)
        r.stage_events = None
        launches = L.moe_kernel_launch_count() - n0
        for i in range(max(1, args.warmup)):
            u.copy_(upool[i % U_POOL])
            graph.replay()
        torch.cuda.synchronize()
        check()

    clocks = ClockSampler(torch.cuda.current_device())
    clocks.start()
    barrier(world)
    torch.cuda.synchronize()
    n1 = L.moe_kernel_launch_count()
    step_ms, gemm_ms = [], []
    stage_ms = {}
    t_wall = time.perf_counter()
    for i in range(args.steps):
        flush.fill_(1)
        u.copy_(upool[i % U_POOL])
        s0, s1 = ev(), ev()
        s0.record(stream)
        if graph is not None:
            graph.replay()
            e = g_ev
        else:
            e = ((ev(), ev()), (ev(), ev()))
            step(e)
        s1.record(stream)
        s1.synchronize()
        step_ms.append(s0.elapsed_time(s1))
        gemm_ms.append(e[0][0].elapsed_time(e[0][1]) + e[1][0].elapsed_time(e[1][1]))
        for k, (a, b) in stage_ev.items():
            stage_ms.setdefault(k, []).append(a.elapsed_time(b))
    torch.cuda.synchronize()
    barrier(world)
    wall = time.perf_counter() - t_wall
    clk = clocks.stop()
    if graph is None:
        launches = (L.moe_kernel_launch_count() - n1) // max(1, args.steps)
    check()
    counts_all = counts_now()

    ms_step = max_over_ranks(sum(step_ms) / len(step_ms), world)
    g_ms = max_over_ranks(sum(gemm_ms) / len(gemm_ms), world)
    R_mine = int(counts_all[:, rank * El:(rank + 1) * El].sum())
    flops_per_gpu = sum_over_ranks(12.0 * R_mine * cfg.d_model * cfg.d_ff, world) / world
    nvl = sum_over_ranks(_nvlink_bytes(cfg, counts_all, rank, world), world) / world
    value = cfg.T * world / (ms_step / 1e3)
    out = _base_line(cfg, world, args, ms_step, value)
    R_all = int(counts_all.sum())
    out["config"] = _config(cfg, world, {
        "rows_R_per_gpu_mean": R_all / world, "mean_experts_per_token": R_all / (cfg.T * world),
        "max_over_mean_load": float(counts_all.sum(0).max() / max(1e-9, counts_all.sum(0).mean())),
        "parallelism": f"ep{world}: E/{world}={El} experts per GPU, T={cfg.T} tokens per GPU; " + (
            "NCCL grouped send/recv all-to-all-v (eager, host-planned)" if path == "nccl" else
            "fused NVLink peer-memory dispatch / combine (torch symmetric memory), " +
            ("one row per (token, owner) each way (moe_ep2d_*)" if path == "p2p-dedup" else "moe_ep2_*") +
            ("; exchange / GEMM overlap: no barrier between the x exchange and the expert GEMMs, each "
             "expert's GEMM1 tiles wait on its arrival counter" if path != "nccl" and getattr(r, "overlap", False)
             else "")),
        "ep_path": path + (f" ({note})" if note else ""),
        "row_capacity": None if path == "nccl" else {"R_cap": r.R_cap, "grows": r.grows},
        "launch": "cuda-graph replay (static capacity, no host sync)" if graph is not None else "eager",
        "wall_s_timed_region": wall})
    out["roofline"] = _roofline(cfg, flops_per_gpu, g_ms, wall, clk, world, None)
    out["nvlink_gbs"] = {"value": nvl / (ms_step / 1e3) / 1e9, "unit": "GB/s per GPU (algorithmic bytes / step time)",
                         "bytes_per_gpu_per_step": nvl, "frac_of_900": nvl / (ms_step / 1e3) / 1e9 / NVLINK_GBS}
    out["stages"] = {k: {"ms": max_over_ranks(sum(v) / len(v), world)} for k, v in stage_ms.items()} or None
    out["spawn"] = spawn
    out["gpu_launches"] = int(launches)
    out["clocks"] = clk
    if args.e2e:
        if path == "nccl":
            def eager_step(x_, u_, dy_):
                y_ = layer.forward(x_, u_, tau, c)
                return y_, layer.backward(dy_)["dx"]
            capture = None
        else:
            def eager_step(x_, u_, dy_):
                y_ = r.forward(x_, u_, tau, c, cfg.top1)
                return y_, r.backward(dy_)["dx"]

            def capture(X, U, DY):
                # DY is staged into the symmetric dy buffer inside the step (bwd_stage_dy)
                side = torch.cuda.Stream()
                side.wait_stream(torch.cuda.current_stream())
                with torch.cuda.stream(side):
                    eager_step(X, U, DY)
                torch.cuda.current_stream().wait_stream(side)
                torch.cuda.synchronize()
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g):
                    Y, DX = eager_step(X, U, DY)
                return g, Y, DX
        out["e2e"] = run_e2e(args, li, upool, cfg.T * world, world, eager_step,
                             capture if (path != "nccl" and args.graph) else None, check)
    if args.cpu_baseline and world == 1:
        # the oracle on the host (N = 1 only, as the single-GPU line)
        T_sub = args.cpu_tokens
        dt_cpu, _ = oracle_sample(cfg, T_sub)
        out["cpu_baseline"] = {"value": T_sub / dt_cpu, "unit": "tokens/s", "cores": cpu_cores(), "kind": "oracle",
                               "sample": f"first {T_sub} tokens of {cfg.name} (same d/d_ff/E/tau/c), fwd+bwd, "
                                         f"fp64 NumPy, {dt_cpu:.2f} s"}
    return out


# ------------------------------------------------------------------ reference arm (the oracle)
def run_reference(args, rank, world):
    if rank != 0:
        return None
    cfg = configs.get(args.config)
    T_sub = args.ref_tokens
    for _ in range(args.warmup):
        oracle_sample(cfg, T_sub)
    times = [oracle_sample(cfg, T_sub)[0] for _ in range(args.steps)]
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


def _json_stdout():
    """The contract is ONE JSON line on stdout.  Libraries print there too (NCCL's "NCCL version"
    banner at communicator init, for one): point fd 1 at stderr for the whole run and keep a
    private handle on the real stdout for the result line."""
    real = os.fdopen(os.dup(1), "w")
    sys.stdout.flush()
    os.dup2(2, 1)
    return real


def main():
    out_stream = _json_stdout()
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default=DEFAULT_CONFIG)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", dest="e2e", action="store_false")
    ap.add_argument("--no-cpu-baseline", dest="cpu_baseline", action="store_false")
    ap.add_argument("--cpu-tokens", type=int, default=4096)
    ap.add_argument("--ref-tokens", type=int, default=256)
    ap.add_argument("--no-graph", dest="graph", action="store_false",
                    help="launch the step eagerly instead of replaying a CUDA graph")
    ap.add_argument("--no-overlap", action="store_true",
                    help="peer-memory EP: put the barrier back between the x exchange and the expert GEMMs "
                         "(token-order copy pass, no arrival counters) -- the A/B of the overlap")
    ap.add_argument("--ep", default=None, choices=["p2p", "p2p-dedup", "nccl"],
                    help="expert-parallel exchange: the fused NVLink peer-memory path (moe_ep2_*, torch symmetric "
                         "memory; the default at N > 1), the same with one row per (token, owner) each way "
                         "(moe_ep2d_*), or NCCL grouped send/recv.  Given at N = 1 it runs that EP path on a "
                         "1-rank group instead of the single-GPU layer")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        print("warning: fewer than 3 warm-up steps", file=sys.stderr)
    if args.impl == "reference":
        rank = int(os.environ.get("RANK", "0"))
        world = int(os.environ.get("WORLD_SIZE", "1"))
        out = run_reference(args, rank, world)
        if out is not None:
            print(json.dumps(out), file=out_stream, flush=True)
        return 0
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return relaunch_under_torchrun(args, out_stream)
    world_env = int(os.environ.get("WORLD_SIZE", "1"))
    if world_env > 1:
        # NCCL's init lines (rank count, transport) on stderr; stdout carries only the JSON line
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
    if args.gpus != world_env:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world_env}; running {world_env} rank(s)",
              file=sys.stderr)
    rank, world, local = dist_setup(force_pg=args.ep is not None)
    if world > 1 and args.ep is None:
        args.ep = "p2p"
    out = run_ep(args, rank, world) if args.ep is not None else run_single(args)
    if rank == 0:
        print(json.dumps(out), file=out_stream, flush=True)
    import torch.distributed as dist
    if dist.is_initialized():
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
