"""ctypes binding of libmoe_dts.so -- argument marshalling only.

Function names match include/moe_dts.h.  Tensors are passed as raw device pointers
(`tensor.data_ptr()`), streams as `torch.cuda.current_stream().cuda_stream`.  Every
non-zero status raises MoEError with moe_last_error().  There is NO fallback: if the
shared library is missing or fails to load, importing this module raises.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Optional

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("MOE_DTS_LIB", os.path.join(_PKG, "lib", "libmoe_dts.so"))

STATUS = {0: "MOE_OK", 1: "MOE_EINVAL", 2: "MOE_ESHAPE", 3: "MOE_EDTYPE", 4: "MOE_ECUDA", 5: "MOE_ENCCL",
          6: "MOE_ENONFINITE", 7: "MOE_ECAPACITY", 8: "MOE_EWORKSPACE", 9: "MOE_EARRIVAL"}
MOE_F32, MOE_BF16 = 0, 1
ROW_ALIGN = 128

# name -> (restype, argtypes)
_P, _I, _F, _L, _S = C.c_void_p, C.c_int, C.c_float, C.c_int64, C.c_size_t
SIGNATURES = {
    "moe_create": (_I, [C.POINTER(_P), _I, _I, _I, _I, _I, _P, _I, _I]),
    "moe_destroy": (_I, [_P]),
    "moe_last_error": (C.c_char_p, []),
    "moe_abi_version": (_I, []),
    "moe_kernel_launch_count": (C.c_uint64, []),
    "moe_workspace_bytes": (_S, [_P]),
    "moe_set_workspace": (_I, [_P, _P, _S]),
    "moe_check": (_I, [_P, _P]),
    "moe_dts_spawn": (_I, [_P] + [_P] * 10 + [_P]),
    "moe_dts_gate": (_I, [_P, _P, _P, _P, _F, _F, _I, _P, _P, _P, _P, _P]),
    "moe_dispatch": (_I, [_P, _P, _P, _P, _P, _P, _P, _P, _L, _P, _P]),
    "moe_expert_ffn": (_I, [_P, _P, _P, _L, _P, _P, _P, _P, _P, _P, _P, _P]),
    "moe_expert_ffn_recompute": (_I, [_P, _P, _P, _L, _P, _P, _P, _P, _P]),
    "moe_combine": (_I, [_P, _P, _P, _P, _P, _P]),
    "moe_combine_bwd": (_I, [_P, _P, _P, _P, _P, _P, _L, _P, _P, _P, _P]),
    "moe_expert_ffn_bwd": (_I, [_P, _P, _P, _P, _P, _P, _L, _P, _P, _P, _P, _P, _P, _P, _P, _P]),
    "moe_dts_gate_bwd": (_I, [_P, _P, _P, _P, _P, _P, _F, _F, _P, _L, _P, _P, _P, _P]),
    "moe_dispatch_bwd": (_I, [_P, _P, _P, _I, _P, _P]),
    "moe_balance_loss": (_I, [_P, _P, _P, _F, _L, _P, _P]),
    "moe_nccl_unique_id": (_I, [_P, _S]),
    "moe_nccl_comm_init": (_I, [C.POINTER(_P), _P, _I, _I]),
    "moe_nccl_comm_destroy": (_I, [_P]),
    "moe_ep_exchange_counts": (_I, [_P, _P, _P, _P]),
    "moe_ep_plan": (_I, [_P, _P, _P, _P, C.POINTER(_L), C.POINTER(_L)]),
    "moe_ep_plan_chunks": (_I, [_P, _I, _P, _P, _P, _I, C.POINTER(_I)]),
    "moe_ep_upload": (_I, [_P, _P, _P]),
    "moe_ep_dispatch": (_I, [_P, _P, _P, _I, _L, _P]),
    "moe_ep_combine": (_I, [_P, _P, _P, _I, _P]),
    "moe_ep_allreduce": (_I, [_P, _P, _L, _I, _P]),
    "moe_ep_set_topology": (_I, [_P, _I]),
    "moe_ep_stage_rows": (_I, [_P, C.POINTER(_L)]),
    "moe_ep_set_stage": (_I, [_P, _P, _L]),
    "moe_ep_hier_chunks": (_I, [_P, _I, _I, _P, _P, _P, _P, _I, C.POINTER(_I)]),
    "moe_ep_topology_stats": (_I, [_I, _I, _I, _P, _P]),
    "moe_ep2_barrier": (_I, [_P, _P]),
    "moe_ep2_counts": (_I, [_P, _P, _P, _P]),
    "moe_ep2_plan": (_I, [_P, _P, _L, _P, _P]),
    "moe_ep2_prepare_recv": (_I, [_P, _P, _P, _P, _P, _L, _P]),
    "moe_ep2_dispatch": (_I, [_P, _P, _P, _P, _P, _P, _P, _P, _L, _P]),
    "moe_ep2_arrival_plan": (_I, [_P, _P, _P, _P, _P]),
    "moe_ep2_dispatch_ordered": (_I, [_P, _P, _P, _P, _P, _P, _P, _P, _L, _P, _P, _P, _P]),
    "moe_ep2_expert_ffn": (_I, [_P, _P, _P, _L, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P]),
    "moe_ep2_combine": (_I, [_P, _P, _P, _P, _P, _P]),
    "moe_ep2_combine_bwd": (_I, [_P, _P, _P, _P, _P, _P, _P, _L, _P, _P, _P, _P]),
    "moe_ep2_gate_bwd": (_I, [_P, _P, _P, _P, _P, _P, _F, _F, _P, _L, _P, _P, _P, _P]),
    "moe_ep2_dispatch_bwd": (_I, [_P, _P, _P, _I, _P, _P]),
    "moe_ep2d_dispatch": (_I, [_P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _L, _P]),
    "moe_ep2d_permute": (_I, [_P, _P, _P, _P, _L, _P, _P]),
    "moe_ep2d_presum": (_I, [_P, _P, _P, _P, _P, _P]),
    "moe_ep2d_gather_dy": (_I, [_P, _P, _P, _P, _P]),
    "moe_ep2d_combine": (_I, [_P, _P, _P, _P, _P]),
    "moe_ep2d_combine_bwd": (_I, [_P, _P, _P, _P, _P, _P, _L, _P, _P, _P, _P]),
    "moe_ep2d_dispatch_bwd": (_I, [_P, _P, _P, _I, _P, _P]),
}
MOE_COMM_EMULATED = 1   # moe_create(nccl_comm=MOE_COMM_EMULATED): single-process emulation of `world` ranks


class MoEError(RuntimeError):
    def __init__(self, fn: str, code: int, msg: str):
        super().__init__(f"{fn} -> {STATUS.get(code, code)}: {msg}")
        self.code = code


def load(path: str = LIB_PATH) -> C.CDLL:
    if not os.path.exists(path):
        raise ImportError(f"libmoe_dts.so not built at {path}; run `python -m paper_2112_14397_b200.build` "
                          "(there is no CPU fallback)")
    lib = C.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


_lib: Optional[C.CDLL] = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        _lib = load()
    return _lib


def last_error() -> str:
    return (lib().moe_last_error() or b"").decode()


def _ptr(t) -> Optional[int]:
    if t is None:
        return None
    if isinstance(t, int):
        return t
    return t.data_ptr()


def _stream(stream) -> Optional[int]:
    if stream is None:
        import torch
        return torch.cuda.current_stream().cuda_stream
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


def _call(name: str, *args):
    rc = getattr(lib(), name)(*args)
    if rc != 0:
        raise MoEError(name, rc, last_error())
    return rc


# ---------------------------------------------------------------- same names as the C ABI
def moe_create(T: int, d_model: int, d_ff: int, E: int, dtype: int, nccl_comm: int = 0, rank: int = 0,
               world: int = 1) -> int:
    h = C.c_void_p()
    _call("moe_create", C.byref(h), T, d_model, d_ff, E, dtype, nccl_comm or None, rank, world)
    return h.value


def moe_destroy(ctx: int) -> None:
    _call("moe_destroy", ctx)


def moe_abi_version() -> int:
    return lib().moe_abi_version()


def moe_kernel_launch_count() -> int:
    return int(lib().moe_kernel_launch_count())


def moe_workspace_bytes(ctx: int) -> int:
    return lib().moe_workspace_bytes(ctx)


def moe_set_workspace(ctx: int, ws) -> None:
    _call("moe_set_workspace", ctx, _ptr(ws), ws.numel() * ws.element_size())


def moe_check(ctx: int, stream=None) -> None:
    _call("moe_check", ctx, _stream(stream))


def moe_dts_spawn(ctx, W1s, b1s, W2s, b2s, M1bits, M2bits, W1, b1, W2, b2, stream=None):
    _call("moe_dts_spawn", ctx, *[_ptr(t) for t in (W1s, b1s, W2s, b2s, M1bits, M2bits, W1, b1, W2, b2)],
          _stream(stream))


def moe_dts_gate(ctx, x, Wg, u, tau, threshold, top1, probs, slot, counts, near_band, stream=None):
    _call("moe_dts_gate", ctx, _ptr(x), _ptr(Wg), _ptr(u), float(tau), float(threshold), int(top1),
          _ptr(probs), _ptr(slot), _ptr(counts), _ptr(near_band), _stream(stream))


def moe_dispatch(ctx, x, probs, slot, x_perm, row_token, row_gate, offsets, R_cap, R_out, stream=None):
    _call("moe_dispatch", ctx, _ptr(x), _ptr(probs), _ptr(slot), _ptr(x_perm), _ptr(row_token),
          _ptr(row_gate), _ptr(offsets), int(R_cap), _ptr(R_out), _stream(stream))


def moe_expert_ffn(ctx, x_perm, offsets, R_cap, W1, b1, W2, b2, a_saved, h_saved, e_out, stream=None):
    _call("moe_expert_ffn", ctx, _ptr(x_perm), _ptr(offsets), int(R_cap), _ptr(W1), _ptr(b1), _ptr(W2),
          _ptr(b2), _ptr(a_saved), _ptr(h_saved), _ptr(e_out), _stream(stream))


def moe_expert_ffn_recompute(ctx, x_perm, offsets, R_cap, W1, b1, gp_saved, h_saved, stream=None):
    _call("moe_expert_ffn_recompute", ctx, _ptr(x_perm), _ptr(offsets), int(R_cap), _ptr(W1), _ptr(b1),
          _ptr(gp_saved), _ptr(h_saved), _stream(stream))


def moe_combine(ctx, e_out, row_gate, slot, y, stream=None):
    _call("moe_combine", ctx, _ptr(e_out), _ptr(row_gate), _ptr(slot), _ptr(y), _stream(stream))


def moe_combine_bwd(ctx, dy, e_out, row_gate, row_token, offsets, R_cap, d_eout, dG_row, db2=None, stream=None):
    _call("moe_combine_bwd", ctx, _ptr(dy), _ptr(e_out), _ptr(row_gate), _ptr(row_token), _ptr(offsets),
          int(R_cap), _ptr(d_eout), _ptr(dG_row), _ptr(db2), _stream(stream))


def moe_expert_ffn_bwd(ctx, d_eout, x_perm, a_saved, h_saved, offsets, R_cap, W1, W2, da, dx_perm,
                       dW1, db1, dW2, db2, stream=None):
    _call("moe_expert_ffn_bwd", ctx, _ptr(d_eout), _ptr(x_perm), _ptr(a_saved), _ptr(h_saved),
          _ptr(offsets), int(R_cap), _ptr(W1), _ptr(W2), _ptr(da), _ptr(dx_perm), _ptr(dW1), _ptr(db1),
          _ptr(dW2), _ptr(db2), _stream(stream))


def moe_dts_gate_bwd(ctx, dG_row, slot, probs, x, Wg, tau, balance_alpha, counts, B_total, dWg, dlogits, dx=None,
                     stream=None):
    _call("moe_dts_gate_bwd", ctx, _ptr(dG_row), _ptr(slot), _ptr(probs), _ptr(x), _ptr(Wg), float(tau),
          float(balance_alpha), _ptr(counts), int(B_total), _ptr(dWg), _ptr(dlogits), _ptr(dx), _stream(stream))


def moe_dispatch_bwd(ctx, dx_perm, slot, accumulate, dx, stream=None):
    _call("moe_dispatch_bwd", ctx, _ptr(dx_perm), _ptr(slot), int(bool(accumulate)), _ptr(dx), _stream(stream))


def moe_balance_loss(ctx, probs, counts, alpha, B_total, loss, stream=None):
    _call("moe_balance_loss", ctx, _ptr(probs), _ptr(counts), float(alpha), int(B_total), _ptr(loss),
          _stream(stream))


# ---------------------------------------------------------------- expert parallelism
def moe_nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    _call("moe_nccl_unique_id", C.cast(buf, C.c_void_p), 128)
    return buf.raw


def moe_nccl_comm_init(uid: bytes, world: int, rank: int) -> int:
    h = C.c_void_p()
    buf = C.create_string_buffer(uid, 128)
    _call("moe_nccl_comm_init", C.byref(h), C.cast(buf, C.c_void_p), world, rank)
    return h.value


def moe_nccl_comm_destroy(comm: int) -> None:
    _call("moe_nccl_comm_destroy", comm)


def _np_i32(a):
    import numpy as np
    a = np.ascontiguousarray(a, dtype=np.int32)
    return a, a.ctypes.data


def moe_ep_exchange_counts(ctx, counts, world: int, E: int, stream=None):
    import numpy as np
    out = np.zeros((world, E), dtype=np.int32)
    _call("moe_ep_exchange_counts", ctx, _ptr(counts), out.ctypes.data, _stream(stream))
    return out


def moe_ep_plan(ctx, counts_all, E: int, E_local: int):
    """Host-only.  Returns (offsets_send [E+1], offsets_recv [E_local+1], R_send, R_recv)."""
    import numpy as np
    ca, ca_p = _np_i32(counts_all)
    os_ = np.zeros(E + 1, dtype=np.int32)
    or_ = np.zeros(E_local + 1, dtype=np.int32)
    rs, rr = C.c_int64(), C.c_int64()
    _call("moe_ep_plan", ctx, ca_p, os_.ctypes.data, or_.ctypes.data, C.byref(rs), C.byref(rr))
    return os_, or_, rs.value, rr.value


def moe_ep_plan_chunks(ctx, which: int):
    """Host-only: list of (peer, row, nrows) in NCCL posting order (0 = sends, 1 = recvs)."""
    import numpy as np
    n = C.c_int()
    _call("moe_ep_plan_chunks", ctx, which, None, None, None, 0, C.byref(n))
    peer = np.zeros(max(1, n.value), np.int32)
    row = np.zeros(max(1, n.value), np.int64)
    nr = np.zeros(max(1, n.value), np.int32)
    _call("moe_ep_plan_chunks", ctx, which, peer.ctypes.data, row.ctypes.data, nr.ctypes.data, n.value, C.byref(n))
    return [(int(peer[i]), int(row[i]), int(nr[i])) for i in range(n.value)]


def moe_ep_upload(ctx, offsets_recv_dev, stream=None):
    _call("moe_ep_upload", ctx, _ptr(offsets_recv_dev), _stream(stream))


def moe_ep_dispatch(ctx, send_rows, recv_rows, width: int, R_recv_cap: int, stream=None):
    _call("moe_ep_dispatch", ctx, _ptr(send_rows), _ptr(recv_rows), int(width), int(R_recv_cap), _stream(stream))


def moe_ep_combine(ctx, recv_rows, send_rows, width: int, stream=None):
    _call("moe_ep_combine", ctx, _ptr(recv_rows), _ptr(send_rows), int(width), _stream(stream))


def moe_ep_allreduce(ctx, buf, n: int, is_int32: bool = False, stream=None):
    _call("moe_ep_allreduce", ctx, _ptr(buf), int(n), int(is_int32), _stream(stream))


# ---- NEXT #4: topology-aware hierarchical exchange
def moe_ep_set_topology(ctx, gpus_per_node: int):
    _call("moe_ep_set_topology", ctx, int(gpus_per_node))


def moe_ep_stage_rows(ctx) -> int:
    r = C.c_int64()
    _call("moe_ep_stage_rows", ctx, C.byref(r))
    return int(r.value)


def moe_ep_set_stage(ctx, stage, rows_cap: int):
    _call("moe_ep_set_stage", ctx, _ptr(stage) if stage is not None else None, int(rows_cap))


def moe_ep_hier_chunks(ctx, phase: int, is_recv: bool):
    """Host-only: list of (peer, buf, row, nrows) of hierarchical phase `phase` in NCCL posting
    order (buf: 0 send layout, 1 recv layout, 2 relay gather stage, 3 relay receive stage)."""
    import numpy as np
    n = C.c_int()
    _call("moe_ep_hier_chunks", ctx, int(phase), int(is_recv), None, None, None, None, 0, C.byref(n))
    k = max(1, n.value)
    peer, buf, nr = np.zeros(k, np.int32), np.zeros(k, np.int32), np.zeros(k, np.int32)
    row = np.zeros(k, np.int64)
    _call("moe_ep_hier_chunks", ctx, int(phase), int(is_recv), peer.ctypes.data, buf.ctypes.data, row.ctypes.data,
          nr.ctypes.data, n.value, C.byref(n))
    return [(int(peer[i]), int(buf[i]), int(row[i]), int(nr[i])) for i in range(n.value)]


def moe_ep_topology_stats(world: int, gpus_per_node: int, E: int, counts_all) -> dict:
    """Host-only cost-model identities of the flat and hierarchical plans (see moe_dts.h)."""
    import numpy as np
    ca = np.ascontiguousarray(counts_all, dtype=np.int32)
    st = np.zeros(8, np.int64)
    _call("moe_ep_topology_stats", int(world), int(gpus_per_node), int(E), ca.ctypes.data, st.ctypes.data)
    keys = ("flat_inter_pairs", "flat_inter_rows", "flat_intra_rows", "hier_inter_msgs", "hier_inter_rows",
            "hier_intra_rows", "node_pairs", "hier_max_msg_rows")
    return {k: int(v) for k, v in zip(keys, st)}


# ---- fused peer-memory EP ("ep2"): peers = list of `world` tensors (the same buffer on every rank)
def _peers(tensors):
    arr = (C.c_void_p * len(tensors))(*[t.data_ptr() for t in tensors])
    return C.cast(arr, C.c_void_p), arr           # keep `arr` alive for the call


def moe_ep2_barrier(ctx, stream=None):
    _call("moe_ep2_barrier", ctx, _stream(stream))


def moe_ep2_counts(ctx, counts, counts_all_peers, stream=None):
    p, keep = _peers(counts_all_peers)
    _call("moe_ep2_counts", ctx, _ptr(counts), p, _stream(stream))


def moe_ep2_plan(ctx, counts_all, R_recv_cap: int, offsets_recv=None, stream=None):
    _call("moe_ep2_plan", ctx, _ptr(counts_all), int(R_recv_cap), _ptr(offsets_recv), _stream(stream))


def moe_ep2_prepare_recv(ctx, x_recv, rtok, rsrc, rgate, R_recv_cap: int, stream=None):
    _call("moe_ep2_prepare_recv", ctx, _ptr(x_recv), _ptr(rtok), _ptr(rsrc), _ptr(rgate), int(R_recv_cap),
          _stream(stream))


def moe_ep2_dispatch(ctx, x, probs, slot, x_recv_peers, rtok_peers, rsrc_peers, rgate_peers, R_recv_cap: int,
                     stream=None):
    a, ka = _peers(x_recv_peers)
    b, kb = _peers(rtok_peers)
    c, kc = _peers(rsrc_peers)
    d, kd = _peers(rgate_peers)
    _call("moe_ep2_dispatch", ctx, _ptr(x), _ptr(probs), _ptr(slot), a, b, c, d, int(R_recv_cap), _stream(stream))


def moe_ep2_arrival_plan(ctx, counts_all, sprefix, arrive_target, stream=None):
    _call("moe_ep2_arrival_plan", ctx, _ptr(counts_all), _ptr(sprefix), _ptr(arrive_target), _stream(stream))


def moe_ep2_dispatch_ordered(ctx, x, probs, slot, x_recv_peers, rtok_peers, rsrc_peers, rgate_peers,
                             R_recv_cap: int, sprefix, send, arrive_peers, stream=None):
    a, ka = _peers(x_recv_peers)
    b, kb = _peers(rtok_peers)
    c, kc = _peers(rsrc_peers)
    d, kd = _peers(rgate_peers)
    e, ke = _peers(arrive_peers)
    _call("moe_ep2_dispatch_ordered", ctx, _ptr(x), _ptr(probs), _ptr(slot), a, b, c, d, int(R_recv_cap),
          _ptr(sprefix), _ptr(send), e, _stream(stream))


def moe_ep2_expert_ffn(ctx, x_recv, offsets_recv, R_recv_cap: int, W1, b1, W2, b2, gp_saved, h_saved, e_out,
                       arrive, arrive_target, stream=None):
    _call("moe_ep2_expert_ffn", ctx, _ptr(x_recv), _ptr(offsets_recv), int(R_recv_cap), _ptr(W1), _ptr(b1),
          _ptr(W2), _ptr(b2), _ptr(gp_saved), _ptr(h_saved), _ptr(e_out), _ptr(arrive), _ptr(arrive_target),
          _stream(stream))


def moe_ep2_combine(ctx, e_out_peers, probs, slot, y, stream=None):
    a, ka = _peers(e_out_peers)
    _call("moe_ep2_combine", ctx, a, _ptr(probs), _ptr(slot), _ptr(y), _stream(stream))


def moe_ep2_combine_bwd(ctx, dy_peers, e_out, rgate, rtok, rsrc, offsets_recv, R_recv_cap: int, d_eout, dG_row,
                        db2=None, stream=None):
    a, ka = _peers(dy_peers)
    _call("moe_ep2_combine_bwd", ctx, a, _ptr(e_out), _ptr(rgate), _ptr(rtok), _ptr(rsrc), _ptr(offsets_recv),
          int(R_recv_cap), _ptr(d_eout), _ptr(dG_row), _ptr(db2), _stream(stream))


def moe_ep2_gate_bwd(ctx, dG_peers, slot, probs, x, Wg, tau: float, balance_alpha: float, counts_all, B_total: int,
                     dWg, dlogits, dx=None, stream=None):
    """counts_all: this rank's [world, E] copy of the all-gathered counts (global counts = column sums)."""
    a, ka = _peers(dG_peers)
    _call("moe_ep2_gate_bwd", ctx, a, _ptr(slot), _ptr(probs), _ptr(x), _ptr(Wg), float(tau), float(balance_alpha),
          _ptr(counts_all), int(B_total), _ptr(dWg), _ptr(dlogits), _ptr(dx), _stream(stream))


def moe_ep2_dispatch_bwd(ctx, dx_perm_peers, slot, accumulate, dx, stream=None):
    a, ka = _peers(dx_perm_peers)
    _call("moe_ep2_dispatch_bwd", ctx, a, _ptr(slot), int(bool(accumulate)), _ptr(dx), _stream(stream))


# ---- ep2 with token dedup (include/moe_dts.h "ep2d")
def moe_ep2d_dispatch(ctx, x, probs, slot, uslot, tokbuf_peers, urows_peers, rtok_peers, rsrc_peers, rgate_peers,
                      ruid_peers, R_recv_cap: int, stream=None):
    ps = [_peers(t) for t in (tokbuf_peers, urows_peers, rtok_peers, rsrc_peers, rgate_peers, ruid_peers)]
    _call("moe_ep2d_dispatch", ctx, _ptr(x), _ptr(probs), _ptr(slot), _ptr(uslot), *[p for p, _ in ps],
          int(R_recv_cap), _stream(stream))


def moe_ep2d_permute(ctx, tokbuf, rtok, ruid, R_recv_cap: int, x_recv, stream=None):
    _call("moe_ep2d_permute", ctx, _ptr(tokbuf), _ptr(rtok), _ptr(ruid), int(R_recv_cap), _ptr(x_recv),
          _stream(stream))


def moe_ep2d_presum(ctx, rows, rgate, urows, out, stream=None):
    _call("moe_ep2d_presum", ctx, _ptr(rows), _ptr(rgate), _ptr(urows), _ptr(out), _stream(stream))


def moe_ep2d_gather_dy(ctx, dy_peers, urows, dyu, stream=None):
    a, ka = _peers(dy_peers)
    _call("moe_ep2d_gather_dy", ctx, a, _ptr(urows), _ptr(dyu), _stream(stream))


def moe_ep2d_combine(ctx, ysum_peers, uslot, y, stream=None):
    a, ka = _peers(ysum_peers)
    _call("moe_ep2d_combine", ctx, a, _ptr(uslot), _ptr(y), _stream(stream))


def moe_ep2d_combine_bwd(ctx, dyu, e_out, rgate, ruid, offsets_recv, R_recv_cap: int, d_eout, dG_row, db2=None,
                         stream=None):
    _call("moe_ep2d_combine_bwd", ctx, _ptr(dyu), _ptr(e_out), _ptr(rgate), _ptr(ruid), _ptr(offsets_recv),
          int(R_recv_cap), _ptr(d_eout), _ptr(dG_row), _ptr(db2), _stream(stream))


def moe_ep2d_dispatch_bwd(ctx, dxu_peers, uslot, accumulate, dx, stream=None):
    a, ka = _peers(dxu_peers)
    _call("moe_ep2d_dispatch_bwd", ctx, a, _ptr(uslot), int(bool(accumulate)), _ptr(dx), _stream(stream))
