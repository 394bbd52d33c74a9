"""Shared helpers for the GPU parity tests: run the CUDA path through the C ABI
(via DTSMoELayer) and the fp64 oracle on identical seeded inputs, then compare with
the band procedure of SURVEY.md §8c.  Test infrastructure only."""
from __future__ import annotations

import re
from dataclasses import dataclass
from typing import Dict, Optional

import numpy as np
import torch

from harness import inputs
from harness.configs import MoEConfig
from oracle import dts_moe as O

BAND = 1e-6


def rel_err(got: np.ndarray, ref: np.ndarray) -> float:
    """Norm-wise relative error ||got - ref|| / ||ref|| (reading R17)."""
    got = np.asarray(got, np.float64)
    ref = np.asarray(ref, np.float64)
    den = np.linalg.norm(ref)
    num = np.linalg.norm(got - ref)
    if den == 0.0:
        return float(num)
    return float(num / den)


def row_err(got: np.ndarray, ref: np.ndarray, allow: Optional[np.ndarray] = None) -> float:
    """Worst per-row error (VERDICT r1 "per-row bound"): max over rows i of
    max(0, ||got_i - ref_i|| - allow_i) / max(||ref_i||, median_j ||ref_j||).  A vector is treated
    as rows of one element.  Unlike the tensor norm, one wrong row (or one wrong 32-column chunk
    of a row) moves this by its own relative size, not by 1/sqrt(rows).  `allow` is an optional
    per-row absolute allowance for an error the tolerances themselves admit upstream (see
    gate_allowance)."""
    got = np.asarray(got, np.float64)
    ref = np.asarray(ref, np.float64)
    if ref.size == 0:
        return 0.0
    if ref.ndim == 1:
        got, ref = got[:, None], ref[:, None]
    got = got.reshape(-1, ref.shape[-1])
    ref = ref.reshape(-1, ref.shape[-1])
    rn = np.linalg.norm(ref, axis=1)
    floor = float(np.median(rn))
    if floor == 0.0:
        floor = float(rn.max()) if rn.max() > 0 else 1.0
    dn = np.linalg.norm(got - ref, axis=1)
    if allow is not None:
        dn = np.maximum(0.0, dn - np.asarray(allow, np.float64).reshape(-1))
    return float(np.max(dn / np.maximum(rn, floor)))


PROBS_TOL = 1e-5


def dG_scale(fw, dy: np.ndarray, dtype: str) -> np.ndarray:
    """[T, E] error scale of the GPU's combine-weight gradients dG_{t,e} = <dy_t, o_{t,e}>: a
    d-term dot product of bf16 values (dy, and e_out carrying ~2 bf16 roundings) has an absolute
    error of about 2^-8 ||dy_t|| ||o_{t,e}|| / sqrt(d) (random-sign rounding errors); 6 sigma of
    that.  A dot product that nearly cancels (|dG| << that scale) is known only to this absolute
    accuracy, whatever its size.  fp32 layers: 6 x 2^-20 instead of 6 x 2^-8."""
    T, d = dy.shape
    out = np.zeros(fw.p.shape)
    kappa = 6.0 * (2.0 ** -8 if dtype == "bf16" else 2.0 ** -20)
    dyn = np.linalg.norm(dy, axis=1)
    for e, toks in fw.toks.items():
        if len(toks):
            out[toks, e] = kappa * dyn[toks] * np.linalg.norm(fw.o[e], axis=1) / np.sqrt(d)
    return out


def gate_allowance(p: np.ndarray, m: np.ndarray, dG: np.ndarray, tau: float, tol: float,
                   dg_err: Optional[np.ndarray] = None) -> np.ndarray:
    """Per-token bound on how far dlogits may move when its inputs move within their error
    scales: the gate probabilities by PROBS_TOL absolute (BJ:5), the combine-weight gradients by
    dg_err (dG_scale: the absolute accuracy of a bf16 dot product; default tol |dG|).
    dlogits = p (.) (dp - s) / tau with dp = m dG, s = <p, dp>.
      probs: to first order a change delta of p moves it by (delta (.) (dp - s) - p <delta, dp>) / tau,
             so ||.|| <= 2 eps (||dp - s|| + ||p|| ||dp||_1) / tau (x2 margin);
      dG:    J = d dlogits / d dp = diag(p) (I - 1 p^T) / tau, so ||.|| <= sum_k g_k ||J[:, k]|| with
             ||J[:, k]||^2 = p_k^2 ((1 - p_k)^2 + ||p||^2 - p_k^2) / tau^2 (exact for one selected expert).
    Why a per-row bound needs it: at low tau with near-one-hot p a token's dlogits is set by
    1 - p_max (~1e-5), and a nearly cancelling dG (|<dy, o>| << ||dy|| ||o||) is known only to
    bf16 accuracy in ABSOLUTE terms; both are large RELATIVE errors of that token's small row,
    which the tensor norm hides.  dx inherits the allowance through ||W_g||_2."""
    dp = np.where(m, dG, 0.0)
    s = np.sum(p * dp, axis=1, keepdims=True)
    probs_term = 2.0 * PROBS_TOL * (np.linalg.norm(dp - s, axis=1) + np.linalg.norm(p, axis=1) * np.abs(dp).sum(1))
    g = np.where(m, np.abs(dG) * tol if dg_err is None else dg_err, 0.0)
    pn2 = np.sum(p * p, axis=1, keepdims=True)
    col = p * np.sqrt(np.maximum(0.0, (1.0 - p) ** 2 + pn2 - p * p))
    return probs_term / tau + np.sum(g * col, axis=1) / tau


def maxabs_rel(got: np.ndarray, ref: np.ndarray) -> float:
    """max |got - ref| / max |ref| (reported beside the norm-wise error)."""
    got = np.asarray(got, np.float64)
    ref = np.asarray(ref, np.float64)
    if ref.size == 0:
        return 0.0
    den = float(np.abs(ref).max())
    return float(np.abs(got - ref).max() / (den if den else 1.0))


def check_values(rep: Dict[str, float], name: str, got: np.ndarray, ref: np.ndarray, tol: float,
                 rows: bool = True, allow: Optional[np.ndarray] = None, explain=None) -> None:
    """Record the three errors of one value tensor and assert the norm-wise bound and (rows=True)
    the per-row bound, both at the BJ:5 tolerance; max-abs / max|ref| is reported, not bounded.
    rows=False for the reductions whose elements are sums with cancellation (db1, db2, dW_g,
    dG): their per-element error is set by the bf16 summands, not by the element's size, so
    they keep the norm-wise bound (their row error is still reported)."""
    rep[name] = rel_err(got, ref)
    rep[name + ".row"] = row_err(got, ref, allow)
    rep[name + ".maxabs"] = maxabs_rel(got, ref)
    assert rep[name] <= tol, f"{name}: norm-wise rel err {rep[name]:.3e} > {tol}"
    if rows and rep[name + ".row"] > tol:
        g2 = np.asarray(got, np.float64).reshape(-1, np.asarray(ref).shape[-1] if np.ndim(ref) > 1 else 1)
        r2 = np.asarray(ref, np.float64).reshape(g2.shape)
        rn, dn = np.linalg.norm(r2, axis=1), np.linalg.norm(g2 - r2, axis=1)
        a2 = np.zeros_like(dn) if allow is None else np.asarray(allow, np.float64).reshape(-1)
        i = int(np.argmax(np.maximum(0, dn - a2) / np.maximum(rn, np.median(rn))))
        raise AssertionError(f"{name}: worst row rel err {rep[name + '.row']:.3e} > {tol} (row {i}: |err| {dn[i]:.3e}, "
                             f"|ref| {rn[i]:.3e}, median |ref| {np.median(rn):.3e}, allowance {a2[i]:.3e}, "
                             f"norm-wise {rep[name]:.3e})" + (explain(i) if explain else ""))


def tol_for(cfg: MoEConfig) -> float:
    return 1e-4 if cfg.dtype == "f32" else 2e-2


def f32(v: float) -> float:
    return float(np.float32(v))


def band_tokens(p32: np.ndarray, m_gpu: np.ndarray, c: float, top1: bool) -> np.ndarray:
    """Tokens excluded from the bit-exact mask check (R18): any |p - c| < 1e-6 in the
    dense branch; top-2 gap < 1e-6 where the decision is argmax-based (guard / top-1)."""
    c32 = np.float32(c)
    dense_band = np.any(np.abs(p32 - c32) < np.float32(BAND), axis=1)
    srt = np.sort(p32, axis=1)
    gap = srt[:, -1] - srt[:, -2] if p32.shape[1] > 1 else np.full(p32.shape[0], np.inf, np.float32)
    argmax_decided = np.full(p32.shape[0], True) if top1 else ~np.any(p32 > c32, axis=1)
    return np.where(argmax_decided, gap < BAND, dense_band)


@dataclass
class GpuRun:
    layer: object
    y: np.ndarray
    probs: np.ndarray
    slot: np.ndarray
    counts: np.ndarray
    near_band: int
    offsets: np.ndarray
    rows: Dict[str, np.ndarray]
    W: Dict[str, np.ndarray]
    grads: Optional[Dict[str, np.ndarray]]


def _np(t: torch.Tensor) -> np.ndarray:
    if t.dtype == torch.bfloat16:
        t = t.float()
    return t.detach().cpu().numpy()


def run_gpu(cfg: MoEConfig, li: inputs.LayerInputs, backward: bool = True, recompute: bool = False) -> GpuRun:
    """recompute: NEXT #3 mode -- the forward keeps no [R, d_ff] activation; the gp rows checked
    are the ones moe_expert_ffn_recompute rebuilt before the expert backward."""
    from paper_2112_14397_b200.layer import DTSMoELayer
    dev = torch.device("cuda", 0)
    T = li.x.shape[0]
    layer = DTSMoELayer(T, cfg.d_model, cfg.d_ff, cfg.E, dtype=li.x.dtype, device=dev, recompute=recompute)
    layer.set_gate(li.Wg.to(dev))
    layer.spawn(*(t.to(dev) for t in (li.W1s, li.b1s, li.W2s, li.b2s, li.M1bits, li.M2bits)))
    u = li.u.to(dev) if li.u is not None else None
    y = layer.forward(li.x.to(dev), u, f32(cfg.tau), f32(cfg.threshold), top1=cfg.top1)
    torch.cuda.synchronize()
    layer.check()
    st = layer.state
    rb = layer.rows
    R = int(st.offsets[-1].item())
    rows = {k: _np(rb[k][:R]) for k in ("x_perm", "row_token", "row_gate", "h", "e_out")}
    if not recompute:
        rows["gp"] = _np(rb["gp"][:R])
    else:
        rb["gp"].fill_(float("nan"))            # the backward must rebuild it (and h) from x_perm
        rb["h"].fill_(float("nan"))
    W = {k: _np(getattr(layer, k)) for k in ("W1", "b1", "W2", "b2")}
    run = GpuRun(layer, _np(y), _np(st.probs), _np(st.slot), _np(st.counts), int(st.near_band.item()),
                 _np(st.offsets), rows, W, None)
    if backward:
        g = layer.backward(li.dy.to(dev), inplace_da=False)
        torch.cuda.synchronize()
        layer.check()
        run.grads = {k: _np(v) for k, v in g.items() if k not in ("da",)}
        run.grads["da"] = _np(g["da"][:R])
        for k in ("d_eout", "dG_row", "dx_perm"):
            run.rows[k] = _np(rb[k][:R])
        if recompute:
            run.rows["gp"] = _np(rb["gp"][:R])   # inplace_da=False: still the recomputed GELU'(a)
    return run


def run_oracle(cfg: MoEConfig, li: inputs.LayerInputs, mask_override=None, backward=True):
    ex = O.spawn(inputs.to_f64(li.W1s), inputs.to_f64(li.b1s), inputs.to_f64(li.W2s), inputs.to_f64(li.b2s),
                 inputs.bits_u32(li.M1bits), inputs.bits_u32(li.M2bits))
    fw = O.forward(inputs.to_f64(li.x), inputs.to_f64(li.Wg), inputs.to_f64(li.u), f32(cfg.tau),
                   f32(cfg.threshold), ex, top1=cfg.top1, mask_override=mask_override)
    bw = O.backward(fw, inputs.to_f64(li.dy)) if backward else None
    return ex, fw, bw


def compare(cfg: MoEConfig, li: inputs.LayerInputs, g: GpuRun, backward: bool = True) -> Dict[str, float]:
    """Full per-call comparison; asserts and returns the error report."""
    tol = tol_for(cfg)
    rep: Dict[str, float] = {}
    m_gpu = g.slot >= 0
    band = band_tokens(g.probs, m_gpu, cfg.threshold, cfg.top1)
    ex, fw, bw = run_oracle(cfg, li, backward=backward)
    flips = np.any(fw.m != m_gpu, axis=1)
    rep["band_tokens"] = int(band.sum())
    rep["mask_flips"] = int(flips.sum())
    assert not np.any(flips & ~band), f"routing mismatch outside the band on tokens {np.nonzero(flips & ~band)[0][:10]}"
    assert g.near_band == int(band.sum()), (g.near_band, int(band.sum()))
    if flips.any():
        ex, fw, bw = run_oracle(cfg, li, mask_override=m_gpu, backward=backward)
    # spawn: bit-exact
    for k in ("W1", "b1", "W2", "b2"):
        assert np.array_equal(g.W[k], ex[k]), f"spawn {k} not bit-exact"
    # gate probabilities (1e-5 abs, BJ:5)
    rep["probs_maxabs"] = float(np.max(np.abs(g.probs - fw.p)))
    assert rep["probs_maxabs"] <= 1e-5, rep
    # counts / dispatch layout: bit-exact vs the stable rule on the GPU's mask
    counts, offsets, slot, row_token = O.dispatch_layout(m_gpu)
    assert np.array_equal(g.counts, counts)
    assert np.array_equal(g.offsets, offsets)
    assert np.array_equal(g.slot, slot)
    assert np.array_equal(g.rows["row_token"], row_token)
    valid = row_token >= 0
    x64 = inputs.to_f64(li.x)
    assert np.array_equal(g.rows["x_perm"][valid], x64[row_token[valid]]), "x_perm not a bit-exact copy"
    assert not np.any(g.rows["x_perm"][~valid]), "pad rows not zero"
    toks, es = np.nonzero(m_gpu)
    assert np.array_equal(g.rows["row_gate"][slot[toks, es]], g.probs[toks, es]), "row_gate provenance"
    # expert FFN intermediates and output
    gp_ref = O.to_rows({e: O.gelu_prime(a) for e, a in fw.a.items()}, offsets, cfg.d_ff)
    h_ref = O.to_rows(fw.h, offsets, cfg.d_ff)
    e_ref = O.to_rows(fw.o, offsets, cfg.d_model)
    # every value tensor: norm-wise AND per-row (each token row of y / dx, each permuted row of
    # the row-layout tensors, each output row of the per-expert weight gradients)
    if "gp" in g.rows:
        check_values(rep, "gp", g.rows["gp"][valid], gp_ref[valid], tol)       # saved GELU'(a)
    check_values(rep, "h", g.rows["h"][valid], h_ref[valid], tol)
    check_values(rep, "e_out", g.rows["e_out"][valid], e_ref[valid], tol)
    check_values(rep, "y", g.y, fw.y, tol)
    if backward:
        do_ref = O.to_rows(bw.do, offsets, cfg.d_model)
        dxe_ref = O.to_rows(bw.dxe, offsets, cfg.d_model)
        check_values(rep, "d_eout", g.rows["d_eout"][valid], do_ref[valid], tol)
        assert not np.any(g.rows["d_eout"][~valid]), "d_eout pad rows not zero"
        check_values(rep, "dG_row", g.rows["dG_row"][slot[toks, es]], bw.dG[toks, es], tol, rows=False)
        check_values(rep, "dx_perm", g.rows["dx_perm"][valid], dxe_ref[valid], tol)
        allow = gate_allowance(fw.p, fw.m, bw.dG, fw.tau, tol, dG_scale(fw, inputs.to_f64(li.dy), cfg.dtype))
        check_values(rep, "dx", g.grads["dx"], bw.dx, tol, allow=allow * np.linalg.norm(fw.Wg, 2))
        check_values(rep, "dWg", g.grads["dWg"], bw.dWg, tol, rows=False)
        def why(t):
            o = np.argsort(-fw.p[t])[:4]
            sel = np.nonzero(m_gpu[t])[0]
            return (f"\n  token {t}: experts {o.tolist()} p_gpu {g.probs[t, o].tolist()} p_ref {fw.p[t, o].tolist()}"
                    f"\n  selected {sel.tolist()} dG_gpu {g.rows['dG_row'][slot[t, sel]].tolist()} dG_ref {bw.dG[t, sel].tolist()}"
                    f"\n  dlogits_gpu {g.grads['dlogits'][t, o].tolist()} dlogits_ref {bw.dlogits[t, o].tolist()}"
                    f" near_band {bool(band[t])}")
        check_values(rep, "dlogits", g.grads["dlogits"], bw.dlogits, tol, allow=allow, explain=why)
        for k, ref in (("dW1", bw.dW1), ("db1", bw.db1), ("dW2", bw.dW2), ("db2", bw.db2)):
            for e in range(cfg.E):
                if fw.counts[e] > 0:
                    check_values(rep, f"{k}[{e}]", g.grads[k][e], ref[e], tol, rows=k in ("dW1", "dW2"))
                else:
                    assert not np.any(g.grads[k][e]), f"{k}[{e}] must be zero for an empty expert"
    return rep


def summary(rep: Dict[str, float]) -> Dict[str, float]:
    """Compact report: the counts, and the worst norm-wise / per-row / max-abs error per tensor
    (per-expert entries folded into their tensor name)."""
    out: Dict[str, float] = {}
    for k, v in rep.items():
        base = re.sub(r"\[\d+\]", "", k)
        out[base] = max(out.get(base, 0.0), v)
    return out
