"""Fused peer-memory expert parallelism ("ep2", include/moe_dts.h): the B200-native EP path.

The all-to-all exchanges of the DTS-Gate MoE layer are fused into the routing
kernels as NVLink peer loads / stores: the token side stores its x rows straight into the
owners' expert-side layouts, the combine / gate backward / dispatch backward gather e_out,
dG and dx_perm rows from the owners, and the expert side's combine backward reads dy rows
from the token owners.  Every rank's row buffers are symmetric (mapped into every rank):
`SymmetricBuffers` allocates them with torch symmetric memory (one process per GPU) or, for
tests, emulates `world` ranks inside ONE process on one device.

Marshalling only: every step is a libmoe_dts.so kernel (moe_ep2_* + the expert FFN calls).

    ranks = [EP2Rank(T, d, f, E, dtype, dev, r, W, syms) for r in range(W)]   # emulation
    EP2Rank.forward / backward / step run the phases of ONE rank (real multi-GPU: each
    process calls them; barriers are NCCL all-reduces).  The tests drive emulated ranks phase
    by phase in one process (tests/_ep_lockstep.py).

Row capacity ("adaptive capacity of experts"; nothing is dropped, R12).  The expert-side
row buffers are symmetric, so every rank sizes them identically, from the all-gathered counts
(identical on every rank): R_cap = the largest rank's 128-aligned recv layout times a headroom
factor.  The first step reads the counts once on the host to size them; later steps run at that
static capacity with no host synchronisation (the step can be captured as a CUDA graph).  A step
whose routing needs more rows raises MOE_ECAPACITY on EVERY rank (each rank's plan kernel checks
all ranks' layouts); `step()` then grows the buffers from that step's counts -- a collective
re-allocation every rank performs together -- and re-runs the step.  An explicit `capacity`
fixes R_cap instead (e.g. the worst case W*T*E_local + 127*E_local for tests).
"""
from __future__ import annotations

import math
from typing import Dict, Optional

import numpy as np
import torch

from . import _lib as L

_DT = {torch.float32: L.MOE_F32, torch.bfloat16: L.MOE_BF16}


class SymmetricBuffers:
    """Named symmetric buffers: buf(name, rank, shape, dtype) -> (local tensor, [peer tensors]).

    mode "emulated": all ranks live in this process on one device (tests).
    mode "symm_mem": one rank per process; torch.distributed._symmetric_memory maps every
    rank's allocation into every rank (NVLink P2P)."""

    def __init__(self, world: int, device: torch.device, mode: str = "emulated", group=None):
        self.world, self.device, self.mode, self.group = world, device, mode, group
        self._bufs: Dict[str, list] = {}

    def buf(self, name: str, rank: int, shape, dtype):
        shape = tuple(int(s) for s in shape)
        key = name
        have = self._bufs.get(key)
        if have is None or tuple(have[0].shape) != shape or have[0].dtype != dtype:
            if self.mode == "emulated":
                have = [torch.zeros(shape, dtype=dtype, device=self.device) for _ in range(self.world)]
            else:
                import torch.distributed._symmetric_memory as symm_mem
                t = symm_mem.empty(*shape, dtype=dtype, device=self.device)
                t.zero_()
                hdl = symm_mem.rendezvous(t, self.group)
                have = [t if q == rank else hdl.get_buffer(q, shape, dtype) for q in range(self.world)]
            self._bufs[key] = have
        return have[rank], have


class EP2Rank:
    """One rank of the fused peer-memory EP layer."""

    def __init__(self, T: int, d_model: int, d_ff: int, E: int, dtype: torch.dtype, device: torch.device, rank: int,
                 world: int, syms: SymmetricBuffers, comm: Optional[int] = None, dedup: bool = False,
                 capacity: Optional[int] = None, headroom: float = 1.25, overlap: Optional[bool] = None):
        self.T, self.d, self.f, self.E, self.El = T, d_model, d_ff, E, E // world
        # exchange / GEMM overlap (non-dedup path; moe_ep2_dispatch_ordered + moe_ep2_expert_ffn):
        # no barrier between the x exchange and the expert GEMMs -- each expert's GEMM1 tiles wait
        # on that expert's arrival counter instead.  Counters (symmetric) and targets (local) are
        # zero at construction and cumulative over steps (never reset, never re-allocated).
        self.overlap = (not dedup) if overlap is None else bool(overlap and not dedup)
        if self.overlap:
            self.arr_target = torch.zeros(E // world, dtype=torch.int32, device=device)
            self.sprefix = torch.zeros(E + 1, dtype=torch.int32, device=device)
            self.send = torch.empty(max(1, T * E), dtype=torch.int32, device=device)
        # dedup (moe_ep2d_*): one row per (token, owner) each way; U = world * T unique slots
        self.dedup, self.U = dedup, world * T
        self.dtype, self.device, self.rank, self.world, self.syms = dtype, device, rank, world, syms
        self.ctx = L.moe_create(T, d_model, d_ff, E, _DT[dtype], comm if comm else L.MOE_COMM_EMULATED, rank, world)
        self.ws = torch.empty(max(256, L.moe_workspace_bytes(self.ctx)), dtype=torch.uint8, device=device)
        L.moe_set_workspace(self.ctx, self.ws)
        # row capacity: fixed when given, else sized from the first step's all-gathered counts
        self.headroom = headroom
        self.R_cap: Optional[int] = None if capacity is None else self.round_rows(capacity)
        self.grows = 0                  # capacity re-allocations after an overflow (step())
        self.Wg = self.W1 = self.b1 = self.W2 = self.b2 = None
        self.st: Dict[str, torch.Tensor] = {}
        # optional {"experts_fwd": (ev0, ev1), "experts_bwd": (ev0, ev1)}: CUDA events recorded
        # around the expert FFN calls on the current stream (bench.py's GEMM time)
        self.events: Optional[Dict[str, tuple]] = None
        # optional dict receiving a (start, end) event pair per phase (per-stage breakdown; the
        # fused exchanges are inside the phases: dispatch stores rows to the owners, combine and
        # dispatch_bwd gather from them, combine_bwd reads dy from the token owners)
        self.stage_events: Optional[Dict[str, tuple]] = None

    def _mark(self, name: str, i: int):
        if self.events and name in self.events:
            self.events[name][i].record(torch.cuda.current_stream())

    def _stage(self, name: str, i: int):
        d = self.stage_events
        if d is None:
            return
        if name not in d:
            d[name] = (torch.cuda.Event(enable_timing=True, external=True),
                       torch.cuda.Event(enable_timing=True, external=True))
        d[name][i].record(torch.cuda.current_stream())

    def __del__(self):
        try:
            if getattr(self, "ctx", None):
                L.moe_destroy(self.ctx)
                self.ctx = None
        except Exception:
            pass

    # ------------------------------------------------------------ parameters
    def spawn(self, W1s, b1s, W2s, b2s, M1bits, M2bits):
        El, d, f, kw = self.El, self.d, self.f, dict(dtype=self.dtype, device=self.device)
        self.W1, self.b1 = torch.empty(El, f, d, **kw), torch.empty(El, f, **kw)
        self.W2, self.b2 = torch.empty(El, d, f, **kw), torch.empty(El, d, **kw)
        L.moe_dts_spawn(self.ctx, W1s, b1s, W2s, b2s, M1bits, M2bits, self.W1, self.b1, self.W2, self.b2)

    def set_gate(self, Wg):
        self.Wg = Wg

    def _sym(self, name, shape, dtype):
        return self.syms.buf(name, self.rank, shape, dtype)

    # ------------------------------------------------------------ row capacity
    @staticmethod
    def round_rows(n: int) -> int:
        return max(128, (int(n) + 127) // 128 * 128)

    def rows_needed(self, counts_all: np.ndarray) -> int:
        """Largest 128-aligned expert-side (recv) layout over the ranks for routing counts_all [W, E]."""
        tot = np.asarray(counts_all, np.int64).sum(0)
        pad = (tot + 127) // 128 * 128
        return int(pad.reshape(self.world, self.El).sum(1).max()) if tot.size else 0

    def capacity_for(self, counts_all: np.ndarray) -> int:
        need = self.rows_needed(counts_all)
        return self.round_rows(math.ceil(need * self.headroom))

    def counts_all_host(self) -> np.ndarray:
        """This rank's copy of the all-gathered counts (host read: synchronises the stream)."""
        ca, _ = self._sym("counts_all", (self.world, self.E), torch.int32)
        return ca.cpu().numpy()

    def worst_case_capacity(self) -> int:
        return self.round_rows(self.world * self.T * self.El + 127 * self.El)

    def prepare(self):
        """Create every symmetric buffer of the current capacity (a collective; do it before a
        CUDA-graph capture so the captured step performs no rendezvous)."""
        R, d = self.R_cap, self.d
        self._sym("counts_all", (self.world, self.E), torch.int32)
        for name, shape, dt in (("x_recv", (R, d), self.dtype), ("rtok", (R,), torch.int32),
                                ("rsrc", (R,), torch.int32), ("rgate", (R,), torch.float32),
                                ("e_out", (R, d), self.dtype), ("dG", (R,), torch.float32),
                                ("dx_perm", (R, d), self.dtype), ("dy", (self.T, d), self.dtype)):
            self._sym(name, shape, dt)
        if self.overlap:
            self._sym("arrive", (self.El,), torch.int32)
        if self.dedup:
            for name, shape, dt in (("ruid", (R,), torch.int32), ("tokbuf", (self.U, d), self.dtype),
                                    ("urows", (self.U, self.El), torch.int32), ("ysum", (self.U, d), self.dtype),
                                    ("dxu", (self.U, d), self.dtype)):
                self._sym(name, shape, dt)

    def dy_buffer(self) -> torch.Tensor:
        """The symmetric dy buffer the backward reads from (write dy here to skip the staging copy)."""
        return self._sym("dy", (self.T, self.d), self.dtype)[0]

    def barrier(self):
        L.moe_ep2_barrier(self.ctx)

    # ------------------------------------------------------------ forward phases
    def fwd_gate(self, x, u, tau: float, threshold: float, top1: bool = False):
        T, E, dev = self.T, self.E, self.device
        s = self.st
        s["x"], s["tau"] = x, tau
        s["probs"] = torch.empty(T, E, dtype=torch.float32, device=dev)
        s["slot"] = torch.empty(T, E, dtype=torch.int32, device=dev)
        s["counts"] = torch.empty(E, dtype=torch.int32, device=dev)
        s["near"] = torch.empty(1, dtype=torch.int32, device=dev)
        L.moe_dts_gate(self.ctx, x, self.Wg, u, tau, threshold, top1, s["probs"], s["slot"], s["counts"], s["near"])
        _, peers = self._sym("counts_all", (self.world, E), torch.int32)
        L.moe_ep2_counts(self.ctx, s["counts"], peers)

    def fwd_plan(self):
        if self.R_cap is None:           # first step: size the capacity from the gathered counts
            self.R_cap = self.capacity_for(self.counts_all_host())
        R, d = self.R_cap, self.d
        s = self.st
        ca, _ = self._sym("counts_all", (self.world, self.E), torch.int32)
        s["off"] = torch.empty(self.El + 1, dtype=torch.int32, device=self.device)
        L.moe_ep2_plan(self.ctx, ca, R, s["off"])
        if self.overlap:
            L.moe_ep2_arrival_plan(self.ctx, ca, self.sprefix, self.arr_target)
        xr, _ = self._sym("x_recv", (R, d), self.dtype)
        rt, _ = self._sym("rtok", (R,), torch.int32)
        rs, _ = self._sym("rsrc", (R,), torch.int32)
        rg, _ = self._sym("rgate", (R,), torch.float32)
        L.moe_ep2_prepare_recv(self.ctx, xr, rt, rs, rg, R)
        if self.dedup:
            self._sym("ruid", (R,), torch.int32)
            self._sym("tokbuf", (self.U, d), self.dtype)
            self._sym("urows", (self.U, self.El), torch.int32)
            s["uslot"] = torch.empty(self.T, self.world, dtype=torch.int32, device=self.device)

    def fwd_dispatch(self):
        R, d, s = self.R_cap, self.d, self.st
        if self.dedup:
            L.moe_ep2d_dispatch(self.ctx, s["x"], s["probs"], s["slot"], s["uslot"],
                                self._sym("tokbuf", (self.U, d), self.dtype)[1],
                                self._sym("urows", (self.U, self.El), torch.int32)[1],
                                self._sym("rtok", (R,), torch.int32)[1], self._sym("rsrc", (R,), torch.int32)[1],
                                self._sym("rgate", (R,), torch.float32)[1], self._sym("ruid", (R,), torch.int32)[1], R)
            return
        if self.overlap:
            L.moe_ep2_dispatch_ordered(self.ctx, s["x"], s["probs"], s["slot"],
                                       self._sym("x_recv", (R, d), self.dtype)[1],
                                       self._sym("rtok", (R,), torch.int32)[1], self._sym("rsrc", (R,), torch.int32)[1],
                                       self._sym("rgate", (R,), torch.float32)[1], R, self.sprefix, self.send,
                                       self._sym("arrive", (self.El,), torch.int32)[1])
            return
        L.moe_ep2_dispatch(self.ctx, s["x"], s["probs"], s["slot"], self._sym("x_recv", (R, d), self.dtype)[1],
                           self._sym("rtok", (R,), torch.int32)[1], self._sym("rsrc", (R,), torch.int32)[1],
                           self._sym("rgate", (R,), torch.float32)[1], R)

    def fwd_permute(self):
        """dedup, expert side: x_recv rows from the once-received token rows (local copy)."""
        R, d = self.R_cap, self.d
        L.moe_ep2d_permute(self.ctx, self._sym("tokbuf", (self.U, d), self.dtype)[0],
                           self._sym("rtok", (R,), torch.int32)[0], self._sym("ruid", (R,), torch.int32)[0], R,
                           self._sym("x_recv", (R, d), self.dtype)[0])

    def fwd_presum(self):
        """dedup, expert side: ysum[u] = sum over my experts of G e_out (one row per token and owner)."""
        R, d = self.R_cap, self.d
        L.moe_ep2d_presum(self.ctx, self._sym("e_out", (R, d), self.dtype)[0], self._sym("rgate", (R,), torch.float32)[0],
                          self._sym("urows", (self.U, self.El), torch.int32)[0],
                          self._sym("ysum", (self.U, d), self.dtype)[0])

    def fwd_experts(self):
        R, d, f, s = self.R_cap, self.d, self.f, self.st
        gph = torch.empty(2, R, f, dtype=self.dtype, device=self.device)   # one buffer: GEMM1 stores both per TMA op
        s["gp"], s["h"] = gph[0], gph[1]
        xr, eo = self._sym("x_recv", (R, d), self.dtype)[0], self._sym("e_out", (R, d), self.dtype)[0]
        self._mark("experts_fwd", 0)
        if self.overlap:
            L.moe_ep2_expert_ffn(self.ctx, xr, s["off"], R, self.W1, self.b1, self.W2, self.b2, s["gp"], s["h"], eo,
                                 self._sym("arrive", (self.El,), torch.int32)[0], self.arr_target)
        else:
            L.moe_expert_ffn(self.ctx, xr, s["off"], R, self.W1, self.b1, self.W2, self.b2, s["gp"], s["h"], eo)
        self._mark("experts_fwd", 1)

    def fwd_combine(self):
        R, d, s = self.R_cap, self.d, self.st
        s["y"] = torch.empty(self.T, d, dtype=self.dtype, device=self.device)
        if self.dedup:
            L.moe_ep2d_combine(self.ctx, self._sym("ysum", (self.U, d), self.dtype)[1], s["uslot"], s["y"])
        else:
            L.moe_ep2_combine(self.ctx, self._sym("e_out", (R, d), self.dtype)[1], s["probs"], s["slot"], s["y"])
        return s["y"]

    # ------------------------------------------------------------ backward phases
    def bwd_stage_dy(self, dy):
        buf, _ = self._sym("dy", (self.T, self.d), self.dtype)
        if dy.data_ptr() != buf.data_ptr():
            buf.copy_(dy)

    def bwd_gather_dy(self):
        """dedup, expert side: dyu[u] = the token's dy row, read once per (token, owner)."""
        s = self.st
        s["dyu"] = torch.empty(self.U, self.d, dtype=self.dtype, device=self.device)
        L.moe_ep2d_gather_dy(self.ctx, self._sym("dy", (self.T, self.d), self.dtype)[1],
                             self._sym("urows", (self.U, self.El), torch.int32)[0], s["dyu"])

    def bwd_combine(self):
        R, d, s = self.R_cap, self.d, self.st
        s["d_eout"] = torch.empty(R, d, dtype=self.dtype, device=self.device)
        s["db2"] = torch.empty(self.El, d, dtype=torch.float32, device=self.device)   # fused into the same pass
        dG, _ = self._sym("dG", (R,), torch.float32)
        if self.dedup:
            L.moe_ep2d_combine_bwd(self.ctx, s["dyu"], self._sym("e_out", (R, d), self.dtype)[0],
                                   self._sym("rgate", (R,), torch.float32)[0], self._sym("ruid", (R,), torch.int32)[0],
                                   s["off"], R, s["d_eout"], dG, s["db2"])
            return
        L.moe_ep2_combine_bwd(self.ctx, self._sym("dy", (self.T, d), self.dtype)[1],
                              self._sym("e_out", (R, d), self.dtype)[0], self._sym("rgate", (R,), torch.float32)[0],
                              self._sym("rtok", (R,), torch.int32)[0], self._sym("rsrc", (R,), torch.int32)[0],
                              s["off"], R, s["d_eout"], dG, s["db2"])

    def bwd_experts(self):
        R, d, f, El, s, dev = self.R_cap, self.d, self.f, self.El, self.st, self.device
        g = dict(dW1=torch.empty(El, f, d, dtype=torch.float32, device=dev),
                 db1=torch.empty(El, f, dtype=torch.float32, device=dev),
                 dW2=torch.empty(El, d, f, dtype=torch.float32, device=dev),
                 db2=s["db2"])
        dxp, _ = self._sym("dx_perm", (R, d), self.dtype)
        xr = self._sym("x_recv", (R, d), self.dtype)[0]
        self._mark("experts_bwd", 0)
        L.moe_expert_ffn_bwd(self.ctx, s["d_eout"], xr, s["gp"], s["h"], s["off"], R, self.W1, self.W2, s["gp"], dxp,
                             g["dW1"], g["db1"], g["dW2"], None)
        self._mark("experts_bwd", 1)
        s["grads"] = g

    def bwd_presum(self):
        """dedup, expert side: dxu[u] = sum over my experts of dx_perm (one row per token and owner)."""
        R, d = self.R_cap, self.d
        L.moe_ep2d_presum(self.ctx, self._sym("dx_perm", (R, d), self.dtype)[0], None,
                          self._sym("urows", (self.U, self.El), torch.int32)[0],
                          self._sym("dxu", (self.U, d), self.dtype)[0])

    def bwd_gate(self, balance_alpha: float = 0.0, B_total: Optional[int] = None):
        """dlogits, dW_g (this rank's tokens) and dx = dlogits W_g^T.  The balance term (Eq. 10)
        uses the GLOBAL counts: the kernel sums this rank's copy of the all-gathered counts_all."""
        s, dev = self.st, self.device
        g = s["grads"]
        g["dWg"] = torch.empty(self.d, self.E, dtype=torch.float32, device=dev)
        g["dlogits"] = torch.empty(self.T, self.E, dtype=torch.float32, device=dev)
        g["dx"] = torch.empty(self.T, self.d, dtype=self.dtype, device=dev)
        B = self.T * self.world if B_total is None else B_total
        ca, _ = self._sym("counts_all", (self.world, self.E), torch.int32)
        L.moe_ep2_gate_bwd(self.ctx, self._sym("dG", (self.R_cap,), torch.float32)[1], s["slot"], s["probs"], s["x"],
                           self.Wg, s["tau"], balance_alpha, ca if balance_alpha > 0 else None, B, g["dWg"],
                           g["dlogits"], g["dx"])

    def bwd_dispatch(self):
        """dx += the expert path's rows (gathered from the owners)."""
        s, g = self.st, self.st["grads"]
        if self.dedup:
            L.moe_ep2d_dispatch_bwd(self.ctx, self._sym("dxu", (self.U, self.d), self.dtype)[1], s["uslot"], True,
                                    g["dx"])
        else:
            L.moe_ep2_dispatch_bwd(self.ctx, self._sym("dx_perm", (self.R_cap, self.d), self.dtype)[1], s["slot"],
                                   True, g["dx"])
        return g

    def check(self):
        L.moe_check(self.ctx)

    # ------------------------------------------------------------ one rank, one process (multi-GPU)
    def forward(self, x, u, tau, threshold, top1=False):
        st = self._stage
        st("gate", 0)
        self.fwd_gate(x, u, tau, threshold, top1)
        st("gate", 1)
        self.barrier()
        st("dispatch", 0)
        self.fwd_plan()
        self.fwd_dispatch()
        st("dispatch", 1)
        if not self.overlap:          # overlap: the GEMMs wait per expert on the arrival counters
            self.barrier()
        st("expert_ffn", 0)
        if self.dedup:
            self.fwd_permute()
        self.fwd_experts()
        if self.dedup:
            self.fwd_presum()
        st("expert_ffn", 1)
        self.barrier()
        st("combine", 0)
        y = self.fwd_combine()
        st("combine", 1)
        return y

    def grow(self):
        """After MOE_ECAPACITY: size the buffers for the counts of the step that overflowed (every
        rank holds the same counts_all, so every rank picks the same capacity)."""
        need = self.capacity_for(self.counts_all_host())
        self.R_cap = max(need, self.R_cap or 0)
        self.grows += 1

    def step(self, x, u, dy, tau, threshold, top1=False, balance_alpha: float = 0.0, max_retries: int = 2):
        """forward + backward with the capacity policy: check the device flags after the step and,
        on MOE_ECAPACITY (raised on every rank together), grow and re-run the step."""
        for attempt in range(max_retries + 1):
            y = self.forward(x, u, tau, threshold, top1)
            g = self.backward(dy, balance_alpha)
            try:
                self.check()
                return y, g
            except L.MoEError as e:
                if e.code != 7 or attempt == max_retries:
                    raise
                self.grow()
        raise RuntimeError("unreachable")

    def backward(self, dy, balance_alpha: float = 0.0):
        st = self._stage
        self.bwd_stage_dy(dy)
        self.barrier()
        st("combine_bwd", 0)
        if self.dedup:
            self.bwd_gather_dy()
        self.bwd_combine()
        st("combine_bwd", 1)
        st("expert_ffn_bwd", 0)
        self.bwd_experts()
        if self.dedup:
            self.bwd_presum()
        st("expert_ffn_bwd", 1)
        self.barrier()
        st("gate_bwd", 0)
        self.bwd_gate(balance_alpha)
        L.moe_ep_allreduce(self.ctx, self.st["grads"]["dWg"], self.d * self.E)
        st("gate_bwd", 1)
        st("dispatch_bwd", 0)
        g = self.bwd_dispatch()
        st("dispatch_bwd", 1)
        return g
