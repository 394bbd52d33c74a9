"""DTSMoELayer: the public Python entry point -- runs the C-ABI call sequence of one
DTS-Gate MoE layer forward + backward.  Marshalling and buffer management only: every
step of the path runs in libmoe_dts.so kernels (see include/moe_dts.h).

Forward  : moe_dts_gate -> moe_dispatch -> moe_expert_ffn -> moe_combine
Backward : moe_combine_bwd (+ db2) -> moe_expert_ffn_bwd -> moe_dts_gate_bwd (dx = dL W_g^T) ->
           moe_dispatch_bwd (dx += the expert path's rows)

PyTorch provides device memory and streams only.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Optional

import torch

from . import _lib as L

DTYPES = {torch.float32: L.MOE_F32, torch.bfloat16: L.MOE_BF16}


def padded_rows(counts_host, align: int = L.ROW_ALIGN) -> int:
    return int(sum((int(c) + align - 1) // align * align for c in counts_host))


def make_nccl_comm(rank: int, world: int) -> int:
    """Create the library's own NCCL communicator over the ranks of the default
    torch.distributed process group (the 128-byte unique id is broadcast through it)."""
    import torch.distributed as dist
    uid = torch.zeros(128, dtype=torch.uint8)
    if rank == 0:
        uid = torch.frombuffer(bytearray(L.moe_nccl_unique_id()), dtype=torch.uint8).clone()
    if world > 1:
        if dist.get_backend() == "nccl":
            t = uid.cuda()
            dist.broadcast(t, 0)
            uid = t.cpu()
        else:
            dist.broadcast(uid, 0)
    return L.moe_nccl_comm_init(bytes(uid.numpy().tobytes()), world, rank)


class _Marker:
    """Records a (start, end) CUDA event pair per stage into `d` (no-op when d is None)."""

    def __init__(self, d):
        self.d = d

    def __call__(self, name, which):
        if self.d is None:
            return
        if name not in self.d:
            self.d[name] = (torch.cuda.Event(enable_timing=True, external=True),
                            torch.cuda.Event(enable_timing=True, external=True))
        self.d[name][which].record()


@dataclass
class ForwardState:
    tau: float
    threshold: float
    top1: bool
    x: torch.Tensor
    probs: torch.Tensor
    slot: torch.Tensor
    counts: torch.Tensor
    near_band: torch.Tensor
    offsets: torch.Tensor
    R_cap: int
    y: torch.Tensor


class DTSMoELayer:
    """One MoE FFN layer under the DTS gate on the current CUDA device (one rank)."""

    def __init__(self, T: int, d_model: int, d_ff: int, E: int, dtype: torch.dtype = torch.bfloat16,
                 device: Optional[torch.device] = None, rank: int = 0, world: int = 1, nccl_comm: int = 0,
                 recompute: bool = False, gpus_per_node: Optional[int] = None):
        if dtype not in DTYPES:
            raise ValueError(f"dtype must be one of {list(DTYPES)}")
        self.T, self.d, self.f, self.E = T, d_model, d_ff, E
        self.E_local = E // world
        self.dtype = dtype
        self.device = torch.device("cuda", torch.cuda.current_device()) if device is None else device
        self.rank, self.world = rank, world
        self.recompute = recompute        # NEXT #3: keep only x_perm between forward and backward
        self.ep = bool(nccl_comm)          # expert-parallel exchange (world > 1, or world == 1 self-exchange)
        if world > 1 and not self.ep:
            raise ValueError("world > 1 needs an NCCL communicator (see make_nccl_comm)")
        self.ctx = L.moe_create(T, d_model, d_ff, E, DTYPES[dtype], nccl_comm, rank, world)
        # NEXT #4: multi-node EP through the topology-aware hierarchical exchange
        self.hier = bool(self.ep and gpus_per_node and gpus_per_node < world)
        if self.hier:
            L.moe_ep_set_topology(self.ctx, gpus_per_node)
        nbytes = L.moe_workspace_bytes(self.ctx)
        self.ws = torch.empty(max(nbytes, 256), dtype=torch.uint8, device=self.device)
        L.moe_set_workspace(self.ctx, self.ws)
        self._rows = None      # row-layout buffers, grown on demand
        self._buf = {}
        self._counts_host = torch.empty(E, dtype=torch.int32, pin_memory=True)
        self.Wg = None
        self.W1 = self.b1 = self.W2 = self.b2 = None
        self.state: Optional[ForwardState] = None

    def __del__(self):
        try:
            if getattr(self, "ctx", None):
                L.moe_destroy(self.ctx)
                self.ctx = None
        except Exception:
            pass

    # ------------------------------------------------------------ parameters
    def spawn(self, W1s, b1s, W2s, b2s, M1bits, M2bits, stream=None):
        """Expert-diversify (Alg. 1 lines 4-5): local experts from the shared expert + masks."""
        El, d, f = self.E_local, self.d, self.f
        kw = dict(dtype=self.dtype, device=self.device)
        self.W1 = torch.empty(El, f, d, **kw)
        self.b1 = torch.empty(El, f, **kw)
        self.W2 = torch.empty(El, d, f, **kw)
        self.b2 = torch.empty(El, d, **kw)
        L.moe_dts_spawn(self.ctx, W1s, b1s, W2s, b2s, M1bits, M2bits, self.W1, self.b1, self.W2, self.b2, stream)

    def set_gate(self, Wg: torch.Tensor):
        self.Wg = Wg

    # ------------------------------------------------------------ buffers
    def _grow(self, name, rows, width, dtype):
        t = self._buf.get(name)
        if t is None or t.shape[0] < rows:
            t = torch.empty((max(rows, L.ROW_ALIGN),) + ((width,) if width else ()), dtype=dtype, device=self.device)
            self._buf[name] = t
        return t

    def _ensure_rows(self, R_send: int, R_recv: int):
        """Token-side ("send") and expert-side ("recv") row-layout buffers; without EP they
        are the same buffers."""
        d, f, D = self.d, self.f, self.dtype
        b = {}
        b["x_perm"] = self._grow("x_perm", R_send, d, D)
        b["row_token"] = self._grow("row_token", R_send, 0, torch.int32)
        b["row_gate"] = self._grow("row_gate", R_send, 0, torch.float32)
        b["e_out"] = self._grow("e_out", R_send, d, D)
        b["d_eout"] = self._grow("d_eout", R_send, d, D)
        b["dG_row"] = self._grow("dG_row", R_send, 0, torch.float32)
        b["dx_perm"] = self._grow("dx_perm", R_send, d, D)
        # gp and h as one [2, rows, d_ff] buffer: GEMM1's epilogue stores both with one TMA op
        gph = self._buf.get("gph")
        if gph is None or gph.shape[1] < R_recv:
            gph = torch.empty((2, max(R_recv, L.ROW_ALIGN), f), dtype=D, device=self.device)
            self._buf["gph"] = gph
        b["gp"], b["h"] = gph[0], gph[1]
        if self.ep:
            b["x_recv"] = self._grow("x_recv", R_recv, d, D)
            b["e_out_recv"] = self._grow("e_out_recv", R_recv, d, D)
            b["d_eout_recv"] = self._grow("d_eout_recv", R_recv, d, D)
            b["dx_perm_recv"] = self._grow("dx_perm_recv", R_recv, d, D)
        else:
            b["x_recv"], b["e_out_recv"] = b["x_perm"], b["e_out"]
            b["d_eout_recv"], b["dx_perm_recv"] = b["d_eout"], b["dx_perm"]
        b["R_send_cap"] = b["x_perm"].shape[0]
        b["R_recv_cap"] = min(b["gp"].shape[0], b["h"].shape[0], b["x_recv"].shape[0], b["e_out_recv"].shape[0],
                              b["d_eout_recv"].shape[0], b["dx_perm_recv"].shape[0])
        b["R_send_cap"] = min(b["R_send_cap"], b["row_token"].shape[0], b["row_gate"].shape[0], b["e_out"].shape[0],
                              b["d_eout"].shape[0], b["dG_row"].shape[0], b["dx_perm"].shape[0])
        if not self.ep:
            b["R_recv_cap"] = b["R_send_cap"] = min(b["R_send_cap"], b["R_recv_cap"])
        self._rows = b
        return b

    # ------------------------------------------------------------ forward
    def forward(self, x: torch.Tensor, u: Optional[torch.Tensor], tau: float, threshold: float,
                top1: bool = False, R_cap: Optional[int] = None, stream=None, events=None,
                stage_events: Optional[dict] = None) -> torch.Tensor:
        """events: optional (start, end) torch.cuda.Event pair recorded around moe_expert_ffn
        on the current stream (bench roofline timing).  stage_events: optional dict that
        receives a (start, end) event pair per C-ABI stage (per-stage breakdown)."""
        mark = _Marker(stage_events)
        T, E = self.T, self.E
        dev = self.device
        probs = torch.empty(T, E, dtype=torch.float32, device=dev)
        slot = torch.empty(T, E, dtype=torch.int32, device=dev)
        counts = torch.empty(E, dtype=torch.int32, device=dev)
        near = torch.empty(1, dtype=torch.int32, device=dev)
        mark("gate", 0)
        L.moe_dts_gate(self.ctx, x, self.Wg, u, tau, threshold, top1, probs, slot, counts, near, stream)
        mark("gate", 1)
        offsets = torch.empty(E + 1, dtype=torch.int32, device=dev)
        if self.ep:
            counts_all = L.moe_ep_exchange_counts(self.ctx, counts, self.world, E, stream)
            _, _, R_send, R_recv = L.moe_ep_plan(self.ctx, counts_all, E, self.E_local)
            rb = self._ensure_rows(R_send, R_recv)
            if self.hier:
                stage = self._grow("ep_stage", L.moe_ep_stage_rows(self.ctx), self.d, self.dtype)
                L.moe_ep_set_stage(self.ctx, stage, stage.shape[0])
            offsets_recv = torch.empty(self.E_local + 1, dtype=torch.int32, device=dev)
            L.moe_ep_upload(self.ctx, offsets_recv, stream)
        else:
            if R_cap is None:
                # size the row buffers from the routing result (one small D2H copy)
                self._counts_host.copy_(counts, non_blocking=True)
                torch.cuda.current_stream().synchronize() if stream is None else stream.synchronize()
                R_cap = padded_rows(self._counts_host.tolist())
            R_cap = max(L.ROW_ALIGN, (R_cap + L.ROW_ALIGN - 1) // L.ROW_ALIGN * L.ROW_ALIGN)
            rb = self._ensure_rows(R_cap, R_cap)
            offsets_recv = offsets
        R_send_cap, R_recv_cap = rb["R_send_cap"], rb["R_recv_cap"]
        R_out = torch.empty(1, dtype=torch.int32, device=dev)
        mark("dispatch", 0)
        L.moe_dispatch(self.ctx, x, probs, slot, rb["x_perm"], rb["row_token"], rb["row_gate"], offsets, R_send_cap,
                       R_out, stream)
        mark("dispatch", 1)
        if self.ep:
            L.moe_ep_dispatch(self.ctx, rb["x_perm"], rb["x_recv"], self.d, R_recv_cap, stream)
        if events:
            events[0].record()
        mark("expert_ffn", 0)
        L.moe_expert_ffn(self.ctx, rb["x_recv"], offsets_recv, R_recv_cap, self.W1, self.b1, self.W2, self.b2,
                         None if self.recompute else rb["gp"], rb["h"], rb["e_out_recv"], stream)
        mark("expert_ffn", 1)
        if events:
            events[1].record()
        if self.ep:
            L.moe_ep_combine(self.ctx, rb["e_out_recv"], rb["e_out"], self.d, stream)
        y = torch.empty(T, self.d, dtype=self.dtype, device=dev)
        mark("combine", 0)
        L.moe_combine(self.ctx, rb["e_out"], rb["row_gate"], slot, y, stream)
        mark("combine", 1)
        self.state = ForwardState(tau, threshold, top1, x, probs, slot, counts, near, offsets, R_send_cap, y)
        self.state.offsets_recv = offsets_recv
        self.state.R_recv_cap = R_recv_cap
        return y

    # ------------------------------------------------------------ backward
    def backward(self, dy: torch.Tensor, balance_alpha: float = 0.0, B_total: Optional[int] = None,
                 inplace_da: bool = True, stream=None, events=None, stage_events: Optional[dict] = None):
        st = self.state
        if st is None:
            raise RuntimeError("backward() before forward()")
        rb = self._rows
        El, d, f, dev = self.E_local, self.d, self.f, self.device
        mark = _Marker(stage_events)
        grads = dict(
            dW1=torch.empty(El, f, d, dtype=torch.float32, device=dev),
            db1=torch.empty(El, f, dtype=torch.float32, device=dev),
            dW2=torch.empty(El, d, f, dtype=torch.float32, device=dev),
            db2=torch.empty(El, d, dtype=torch.float32, device=dev),
            dWg=torch.empty(d, self.E, dtype=torch.float32, device=dev),
        )
        mark("combine_bwd", 0)
        # single rank: db2 is summed from the d_eout rows in the same pass; under the NCCL exchange it
        # is an expert-side sum over the received rows (moe_expert_ffn_bwd)
        L.moe_combine_bwd(self.ctx, dy, rb["e_out"], rb["row_gate"], rb["row_token"], st.offsets, st.R_cap,
                          rb["d_eout"], rb["dG_row"], None if self.ep else grads["db2"], stream)
        mark("combine_bwd", 1)
        if self.ep:
            L.moe_ep_dispatch(self.ctx, rb["d_eout"], rb["d_eout_recv"], d, st.R_recv_cap, stream)
        if self.recompute:
            L.moe_expert_ffn_recompute(self.ctx, rb["x_recv"], st.offsets_recv, st.R_recv_cap, self.W1, self.b1,
                                       rb["gp"], rb["h"], stream)
        da = rb["gp"] if inplace_da else torch.empty_like(rb["gp"])
        if events:
            events[0].record()
        mark("expert_ffn_bwd", 0)
        L.moe_expert_ffn_bwd(self.ctx, rb["d_eout_recv"], rb["x_recv"], rb["gp"], rb["h"], st.offsets_recv,
                             st.R_recv_cap, self.W1, self.W2, da, rb["dx_perm_recv"], grads["dW1"], grads["db1"],
                             grads["dW2"], grads["db2"] if self.ep else None, stream)
        mark("expert_ffn_bwd", 1)
        if events:
            events[1].record()
        if self.ep:
            L.moe_ep_combine(self.ctx, rb["dx_perm_recv"], rb["dx_perm"], d, stream)
        dlogits = torch.empty(self.T, self.E, dtype=torch.float32, device=dev)
        B = self.T * self.world if B_total is None else B_total
        counts = st.counts
        if balance_alpha > 0 and self.ep:
            counts = st.counts.clone()
            L.moe_ep_allreduce(self.ctx, counts, self.E, is_int32=True, stream=stream)
        dx = torch.empty(self.T, d, dtype=self.dtype, device=dev)
        mark("gate_bwd", 0)
        L.moe_dts_gate_bwd(self.ctx, rb["dG_row"], st.slot, st.probs, st.x, self.Wg, st.tau, balance_alpha,
                           counts if balance_alpha > 0 else None, B, grads["dWg"], dlogits, dx, stream)
        mark("gate_bwd", 1)
        if self.ep:
            L.moe_ep_allreduce(self.ctx, grads["dWg"], d * self.E, stream=stream)
        mark("dispatch_bwd", 0)
        L.moe_dispatch_bwd(self.ctx, rb["dx_perm"], st.slot, True, dx, stream)
        mark("dispatch_bwd", 1)
        grads["dx"] = dx
        grads["dlogits"] = dlogits
        grads["da"] = da
        self.last_grads = grads
        return grads

    def check(self, stream=None):
        L.moe_check(self.ctx, stream)

    @property
    def rows(self):
        return self._rows
