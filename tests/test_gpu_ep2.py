"""Fused peer-memory expert parallelism ("ep2") on ONE GPU: `world` ranks emulated in one
process (moe_create(nccl_comm=MOE_COMM_EMULATED)), each with its own buffers on the device;
the peer-pointer tables hand every rank the other ranks' buffers, exactly as NVLink
symmetric memory would on a multi-GPU node, and the ranks' launches are ordered phase by
phase on one stream (the barriers' role).  No kernel waits on another rank's kernel.

The result must equal the single-rank layer on the GLOBAL token set (all ranks' tokens
concatenated): bit for bit for routing, y, dx, dlogits and the expert weight gradients of
each rank's experts (same rows in the same order reach the same kernels); db1, db2 and dW_g
to fp32 rounding (different partial-sum partitions: the bias column sums split by the local
expert count, dW_g summed over ranks).
"""
import dataclasses

import numpy as np
import pytest
import torch

from harness import configs, inputs

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _built():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2112_14397_b200 import build
    build.build()


def _rel(a, b):
    a, b = a.double(), b.double()
    den = float(b.norm())
    return float((a - b).norm()) / (den if den else 1.0)


def _ep2(cfg, W, T):
    from paper_2112_14397_b200 import _lib as L
    dev = torch.device("cuda", 0)
    d, f, E = cfg.d_model, cfg.d_ff, cfg.E
    El = E // W
    dt = inputs.TORCH_DTYPE[cfg.dtype]
    mdt = L.MOE_BF16 if cfg.dtype == "bf16" else L.MOE_F32
    tau, c = float(np.float32(cfg.tau)), float(np.float32(cfg.threshold))
    ranks = [inputs.make_inputs(cfg, rank=q, T=T) for q in range(W)]
    li0 = ranks[0]
    Wg = li0.Wg.to(dev)
    R_cap = (W * T * El + 127 * El + 127) // 128 * 128
    ctx, wsp = [], []
    for q in range(W):
        h = L.moe_create(T, d, f, E, mdt, L.MOE_COMM_EMULATED, q, W)
        ws = torch.empty(max(256, L.moe_workspace_bytes(h)), dtype=torch.uint8, device=dev)
        L.moe_set_workspace(h, ws)
        ctx.append(h)
        wsp.append(ws)
    z = lambda *shape, dtype=dt: torch.zeros(*shape, dtype=dtype, device=dev)  # noqa: E731
    # per-rank weights (local experts spawned from the shared expert + global masks)
    Wt = []
    for q in range(W):
        w = dict(W1=z(El, f, d), b1=z(El, f), W2=z(El, d, f), b2=z(El, d))
        L.moe_dts_spawn(ctx[q], *(t.to(dev) for t in (li0.W1s, li0.b1s, li0.W2s, li0.b2s, li0.M1bits, li0.M2bits)),
                        w["W1"], w["b1"], w["W2"], w["b2"])
        Wt.append(w)
    # symmetric buffers
    sym = {k: [] for k in ("x_recv", "rtok", "rsrc", "rgate", "e_out", "d_eout", "dG", "dx_perm", "counts_all", "dy")}
    for q in range(W):
        sym["x_recv"].append(z(R_cap, d))
        sym["rtok"].append(z(R_cap, dtype=torch.int32))
        sym["rsrc"].append(z(R_cap, dtype=torch.int32))
        sym["rgate"].append(z(R_cap, dtype=torch.float32))
        sym["e_out"].append(z(R_cap, d))
        sym["d_eout"].append(z(R_cap, d))
        sym["dG"].append(z(R_cap, dtype=torch.float32))
        sym["dx_perm"].append(z(R_cap, d))
        sym["counts_all"].append(z(W, E, dtype=torch.int32))
        sym["dy"].append(ranks[q].dy.to(dev))
    loc = []
    for q in range(W):
        li = ranks[q]
        loc.append(dict(x=li.x.to(dev), u=li.u.to(dev), probs=z(T, E, dtype=torch.float32),
                        slot=z(T, E, dtype=torch.int32), counts=z(E, dtype=torch.int32),
                        near=z(1, dtype=torch.int32), off=z(El + 1, dtype=torch.int32), gp=z(R_cap, f), h=z(R_cap, f),
                        y=z(T, d), dx=z(T, d), dlogits=z(T, E, dtype=torch.float32),
                        dWg=z(d, E, dtype=torch.float32), dW1=z(El, f, d, dtype=torch.float32),
                        db1=z(El, f, dtype=torch.float32), dW2=z(El, d, f, dtype=torch.float32),
                        db2=z(El, d, dtype=torch.float32)))
    # ---- forward, phase by phase over the ranks
    for q in range(W):
        o = loc[q]
        L.moe_dts_gate(ctx[q], o["x"], Wg, o["u"], tau, c, cfg.top1, o["probs"], o["slot"], o["counts"], o["near"])
    for q in range(W):
        L.moe_ep2_counts(ctx[q], loc[q]["counts"], sym["counts_all"])
        L.moe_ep2_barrier(ctx[q])
    for q in range(W):
        L.moe_ep2_plan(ctx[q], sym["counts_all"][q], R_cap, loc[q]["off"])
        L.moe_ep2_prepare_recv(ctx[q], sym["x_recv"][q], sym["rtok"][q], sym["rsrc"][q], sym["rgate"][q], R_cap)
    for q in range(W):
        L.moe_ep2_dispatch(ctx[q], loc[q]["x"], loc[q]["probs"], loc[q]["slot"], sym["x_recv"], sym["rtok"],
                           sym["rsrc"], sym["rgate"], R_cap)
    for q in range(W):
        w, o = Wt[q], loc[q]
        L.moe_expert_ffn(ctx[q], sym["x_recv"][q], o["off"], R_cap, w["W1"], w["b1"], w["W2"], w["b2"], o["gp"], o["h"],
                         sym["e_out"][q])
    for q in range(W):
        L.moe_ep2_combine(ctx[q], sym["e_out"], loc[q]["probs"], loc[q]["slot"], loc[q]["y"])
    # ---- backward
    for q in range(W):
        L.moe_ep2_combine_bwd(ctx[q], sym["dy"], sym["e_out"][q], sym["rgate"][q], sym["rtok"][q], sym["rsrc"][q],
                              loc[q]["off"], R_cap, sym["d_eout"][q], sym["dG"][q], loc[q]["db2"])
    for q in range(W):
        w, o = Wt[q], loc[q]
        L.moe_expert_ffn_bwd(ctx[q], sym["d_eout"][q], sym["x_recv"][q], o["gp"], o["h"], o["off"], R_cap, w["W1"],
                             w["W2"], o["gp"], sym["dx_perm"][q], o["dW1"], o["db1"], o["dW2"], None)
    for q in range(W):
        o = loc[q]
        L.moe_ep2_gate_bwd(ctx[q], sym["dG"], o["slot"], o["probs"], o["x"], Wg, tau, 0.0, None, W * T, o["dWg"],
                           o["dlogits"], o["dx"])
    for q in range(W):
        o = loc[q]
        L.moe_ep2_dispatch_bwd(ctx[q], sym["dx_perm"], o["slot"], True, o["dx"])
    torch.cuda.synchronize()
    for q in range(W):
        L.moe_check(ctx[q])
    out = dict(loc=loc, dWg=sum(o["dWg"] for o in loc), counts_all=sym["counts_all"][0].cpu())
    for h in ctx:
        L.moe_destroy(h)
    return out, ranks


def _single(cfg, ranks):
    from paper_2112_14397_b200.layer import DTSMoELayer
    dev = torch.device("cuda", 0)
    x = torch.cat([r.x for r in ranks]).to(dev)
    u = torch.cat([r.u for r in ranks]).to(dev)
    dy = torch.cat([r.dy for r in ranks]).to(dev)
    li0 = ranks[0]
    layer = DTSMoELayer(x.shape[0], cfg.d_model, cfg.d_ff, cfg.E, dtype=x.dtype, device=dev)
    layer.set_gate(li0.Wg.to(dev))
    layer.spawn(*(t.to(dev) for t in (li0.W1s, li0.b1s, li0.W2s, li0.b2s, li0.M1bits, li0.M2bits)))
    y = layer.forward(x, u, float(np.float32(cfg.tau)), float(np.float32(cfg.threshold)), top1=cfg.top1)
    g = layer.backward(dy, inplace_da=False)
    torch.cuda.synchronize()
    layer.check()
    return layer, y, g


def _np(t):
    return (t.float() if t.dtype == torch.bfloat16 else t).detach().cpu().numpy()


def _vs_oracle(cfg, W, T, ranks_in, probs, slots, ys, dxs, dlogits, wgrads, dWg, y_tol=None, balance_alpha=0.0,
               dy_scale=1.0):
    """The W-rank result compared DIRECTLY with the fp64 oracle on the global token set (all
    ranks' tokens concatenated), with the band procedure of SURVEY §8(c): probs <= 1e-5, the
    mask bit-exact outside the band, every value tensor norm-wise and per row (y / dx /
    dlogits per token, dW1 / dW2 per output row of every expert on its owner rank, db1 / db2,
    dW_g summed over the ranks)."""
    from _parity import band_tokens, check_values, dG_scale, f32, gate_allowance, run_oracle, summary
    import types
    tol = 2e-2 if cfg.dtype == "bf16" else 1e-4
    cat = lambda k: torch.cat([getattr(r, k) for r in ranks_in])  # noqa: E731
    li = types.SimpleNamespace(**{k: getattr(ranks_in[0], k) for k in ("W1s", "b1s", "W2s", "b2s", "M1bits",
                                                                        "M2bits", "Wg")})
    li.x, li.u, li.dy = cat("x"), cat("u"), cat("dy") * dy_scale
    p32 = np.concatenate([_np(t) for t in probs])
    m_gpu = np.concatenate([_np(t) >= 0 for t in slots])
    _, fw, _ = run_oracle(cfg, li, backward=False)
    band = band_tokens(p32, m_gpu, f32(cfg.threshold), cfg.top1)
    flips = np.any(fw.m != m_gpu, axis=1)
    assert not np.any(flips & ~band), "routing mismatch outside the band"
    _, fw, _ = run_oracle(cfg, li, mask_override=m_gpu, backward=False)
    from oracle import dts_moe as O
    bw = O.backward(fw, inputs.to_f64(li.dy), balance_alpha=balance_alpha)   # global counts, |B| = W*T (R21)
    rep = {"band": int(band.sum()), "flips": int(flips.sum()),
           "probs_maxabs": float(np.abs(p32 - fw.p).max())}
    assert rep["probs_maxabs"] <= 1e-5, rep
    allow = gate_allowance(fw.p, fw.m, bw.dG, fw.tau, tol, dG_scale(fw, inputs.to_f64(li.dy), cfg.dtype))
    check_values(rep, "y", np.concatenate([_np(t) for t in ys]), fw.y, y_tol or tol)
    check_values(rep, "dx", np.concatenate([_np(t) for t in dxs]), bw.dx, y_tol or tol,
                 allow=allow * np.linalg.norm(fw.Wg, 2))
    check_values(rep, "dlogits", np.concatenate([_np(t) for t in dlogits]), bw.dlogits, tol, allow=allow)
    check_values(rep, "dWg", _np(dWg), bw.dWg, tol, rows=False)
    El = cfg.E // W
    for q in range(W):
        for j in range(El):
            e = q * El + j
            for k, ref in (("dW1", bw.dW1), ("db1", bw.db1), ("dW2", bw.dW2), ("db2", bw.db2)):
                got = _np(wgrads[q][k][j])
                if fw.counts[e]:
                    check_values(rep, f"{k}[{e}]", got, ref[e], tol, rows=k in ("dW1", "dW2"))
                else:
                    assert not np.any(got), f"{k}[{e}] of an empty expert must be zero"
    print(cfg.name, f"W={W} T={T} vs oracle", summary(rep))
    return rep


def _check(cfg, W, T):
    ep, ranks = _ep2(cfg, W, T)
    L_ = ep["loc"]
    _vs_oracle(cfg, W, T, ranks, [o["probs"] for o in L_], [o["slot"] for o in L_], [o["y"] for o in L_],
               [o["dx"] for o in L_], [o["dlogits"] for o in L_], L_, ep["dWg"])
    layer, y, g = _single(cfg, ranks)
    E, El = cfg.E, cfg.E // W
    st = layer.state
    for q in range(W):
        o = ep["loc"][q]
        sl = slice(q * T, (q + 1) * T)
        assert torch.equal(o["probs"], st.probs[sl]), f"rank {q} probs"
        assert torch.equal(o["slot"] >= 0, st.slot[sl] >= 0), f"rank {q} routing"
        assert torch.equal(o["counts"], (st.slot[sl] >= 0).sum(0).int()), f"rank {q} counts"
        assert torch.equal(o["y"], y[sl]), f"rank {q} y"
        assert torch.equal(o["dlogits"], g["dlogits"][sl]), f"rank {q} dlogits"
        assert torch.equal(o["dx"], g["dx"][sl]), f"rank {q} dx"
        es = slice(q * El, (q + 1) * El)
        for k in ("dW1", "dW2"):
            assert torch.equal(o[k], g[k][es]), f"rank {q} {k}"
        for k in ("db1", "db2"):      # column-sum split counts follow the local expert count
            assert _rel(o[k], g[k][es]) < 1e-5, f"rank {q} {k}"
    assert torch.equal(ep["counts_all"].sum(0), st.counts.cpu()), "all-gathered counts"
    assert _rel(ep["dWg"], g["dWg"]) < 1e-5, "dWg"


def test_ep2_c3_shape_two_ranks():
    _check(configs.C3, 2, 512)


def test_ep2_c3_shape_four_ranks_ragged():
    _check(configs.C3, 4, 300)


def test_ep2_c4_shape_eight_ranks_top1():
    cfg = dataclasses.replace(configs.C4, top1=True)
    _check(cfg, 8, 160)


def test_ep2_fp32_c1_two_ranks():
    _check(configs.C1, 2, 96)


def test_ep2_wide_rows_two_ranks():
    # d_model = 1280 > 1024: the expert-side combine backward takes the warp-per-row pass (dy
    # through the peer pointers) and a separate db2 pass instead of the fused register kernel
    _check(dataclasses.replace(configs.C3, name="C3w", d_model=1280, d_ff=512), 2, 192)


def test_ep2_bf16_dims_multiple_of_8_two_ranks():
    # d = 200, d_ff = 328 (multiples of 8, not 64): the CUDA-core GEMMs under the peer-memory EP path
    _check(dataclasses.replace(configs.C3, name="C3m8", d_model=200, d_ff=328), 2, 256)


def test_ep2_module_lockstep_c2_shape(poison_empty):
    # the same through paper_2112_14397_b200.ep2 (EP2Rank phases + SymmetricBuffers emulation)
    from paper_2112_14397_b200.ep2 import EP2Rank, SymmetricBuffers
    from _ep_lockstep import run_lockstep
    cfg, W, T = configs.C2, 2, 384
    dev = torch.device("cuda", 0)
    ranks_in = [inputs.make_inputs(cfg, rank=q, T=T) for q in range(W)]
    li0 = ranks_in[0]
    syms = SymmetricBuffers(W, dev)
    ranks = []
    for q in range(W):
        r = EP2Rank(T, cfg.d_model, cfg.d_ff, cfg.E, torch.bfloat16, dev, q, W, syms)
        r.set_gate(li0.Wg.to(dev))
        r.spawn(*(t.to(dev) for t in (li0.W1s, li0.b1s, li0.W2s, li0.b2s, li0.M1bits, li0.M2bits)))
        ranks.append(r)
    ys, grads, dWg = run_lockstep(ranks, [ri.x.to(dev) for ri in ranks_in], [ri.u.to(dev) for ri in ranks_in],
                                  [ri.dy.to(dev) for ri in ranks_in], float(np.float32(cfg.tau)),
                                  float(np.float32(cfg.threshold)))
    torch.cuda.synchronize()
    for r in ranks:
        r.check()
    layer, y, g = _single(cfg, ranks_in)
    El = cfg.E // W
    for q in range(W):
        sl, es = slice(q * T, (q + 1) * T), slice(q * El, (q + 1) * El)
        assert torch.equal(ys[q], y[sl])
        assert torch.equal(grads[q]["dx"], g["dx"][sl])
        assert torch.equal(grads[q]["dW1"], g["dW1"][es]) and torch.equal(grads[q]["dW2"], g["dW2"][es])
    assert _rel(dWg, g["dWg"]) < 1e-5


def _lockstep(cfg, W, T, dedup, balance_alpha=0.0, dy_scale=1.0):
    from paper_2112_14397_b200.ep2 import EP2Rank, SymmetricBuffers
    from _ep_lockstep import run_lockstep
    dev = torch.device("cuda", 0)
    dt = inputs.TORCH_DTYPE[cfg.dtype]
    ranks_in = [inputs.make_inputs(cfg, rank=q, T=T) for q in range(W)]
    li0 = ranks_in[0]
    syms = SymmetricBuffers(W, dev)
    ranks = []
    for q in range(W):
        r = EP2Rank(T, cfg.d_model, cfg.d_ff, cfg.E, dt, dev, q, W, syms, dedup=dedup)
        r.set_gate(li0.Wg.to(dev))
        r.spawn(*(t.to(dev) for t in (li0.W1s, li0.b1s, li0.W2s, li0.b2s, li0.M1bits, li0.M2bits)))
        ranks.append(r)
    ys, grads, dWg = run_lockstep(ranks, [ri.x.to(dev) for ri in ranks_in], [ri.u.to(dev) for ri in ranks_in],
                                  [ri.dy.to(dev) * dy_scale for ri in ranks_in], float(np.float32(cfg.tau)),
                                  float(np.float32(cfg.threshold)), top1=cfg.top1, balance_alpha=balance_alpha)
    torch.cuda.synchronize()
    for r in ranks:
        r.check()
    out = dict(y=[t.clone() for t in ys], g=[{k: v.clone() for k, v in g.items()} for g in grads], dWg=dWg.clone(),
               slot=[r.st["slot"].clone() for r in ranks], probs=[r.st["probs"].clone() for r in ranks])
    return out, ranks_in


@pytest.fixture
def poison_empty(monkeypatch):
    """Fill every new floating-point CUDA buffer from torch.empty with NaN, so a read of a row
    nobody wrote (instead of an exact zero or a finite leftover) fails the comparisons."""
    real = torch.empty

    def empty(*size, dtype=None, device=None, **kw):
        t = real(*size, dtype=dtype, device=device, **kw)
        if t.is_cuda and t.is_floating_point():
            t.fill_(float("nan"))
        return t
    monkeypatch.setattr(torch, "empty", empty)


@pytest.mark.parametrize("name,W,T", [("C1", 2, 96), ("C2", 2, 384), ("C3", 4, 300), ("C4", 8, 160)])
def test_ep2_dedup_matches_single_rank(poison_empty, name, W, T):
    # token dedup (moe_ep2d_*): one row per (token, owner) each way.  Routing, dlogits and the
    # expert weight gradients are bit-identical to the single-rank layer; y and dx differ only
    # by the rounding of the per-owner partial sums to bf16; the bias / gate weight gradients
    # to fp32 rounding (partial-sum partitions follow the local expert count).
    cfg = getattr(configs, name)
    ep, ranks_in = _lockstep(cfg, W, T, dedup=True)
    _vs_oracle(cfg, W, T, ranks_in, ep["probs"], ep["slot"], ep["y"], [gq["dx"] for gq in ep["g"]],
               [gq["dlogits"] for gq in ep["g"]], ep["g"], ep["dWg"])
    layer, y, g = _single(cfg, ranks_in)
    st = layer.state
    El = cfg.E // W
    for q in range(W):
        sl, es = slice(q * T, (q + 1) * T), slice(q * El, (q + 1) * El)
        assert torch.equal(ep["slot"][q] >= 0, st.slot[sl] >= 0), f"rank {q} routing"
        assert torch.equal(ep["g"][q]["dlogits"], g["dlogits"][sl]), f"rank {q} dlogits"
        for k in ("dW1", "dW2"):
            assert torch.equal(ep["g"][q][k], g[k][es]), f"rank {q} {k}"
        for k in ("db1", "db2"):
            assert _rel(ep["g"][q][k], g[k][es]) < 1e-5, f"rank {q} {k}"
        tol = 5e-3 if cfg.dtype == "bf16" else 1e-6      # fp32: the partial sums are not rounded further
        assert _rel(ep["y"][q], y[sl]) < tol, f"rank {q} y {_rel(ep['y'][q], y[sl])}"
        assert _rel(ep["g"][q]["dx"], g["dx"][sl]) < tol, f"rank {q} dx {_rel(ep['g'][q]['dx'], g['dx'][sl])}"
    assert _rel(ep["dWg"], g["dWg"]) < 1e-5


def test_ep2d_wide_rows_two_ranks(poison_empty):
    # the token-dedup path with d_model = 1280 > 1024 (warp-per-row combine backward + db2 pass)
    cfg = dataclasses.replace(configs.C3, name="C3w", d_model=1280, d_ff=512)
    ep, ranks_in = _lockstep(cfg, 2, 192, dedup=True)
    _vs_oracle(cfg, 2, 192, ranks_in, ep["probs"], ep["slot"], ep["y"], [gq["dx"] for gq in ep["g"]],
               [gq["dlogits"] for gq in ep["g"]], ep["g"], ep["dWg"])


def test_ep2_dedup_single_owner_rows_are_exact(poison_empty):
    # with one selected expert per (token, owner) -- top-1 routing -- the pre-sums are single
    # rows, so y and dx equal the non-dedup path bit for bit
    cfg = dataclasses.replace(configs.C3, top1=True)
    a, _ = _lockstep(cfg, 4, 256, dedup=True)
    b, _ = _lockstep(cfg, 4, 256, dedup=False)
    for q in range(4):
        assert torch.equal(a["y"][q], b["y"][q])
        assert torch.equal(a["g"][q]["dx"], b["g"][q]["dx"])


@pytest.mark.parametrize("name,W,T,dedup", [("C1", 2, 96, False), ("C3", 4, 300, True), ("C3", 2, 256, False)])
def test_ep2_balance_loss_uses_global_counts(poison_empty, name, W, T, dedup):
    # the peer-memory EP gate backward must take the GLOBAL per-expert counts for the
    # Eq. 10 term (|B| = the global batch, R21), not this rank's.  Compared with the
    # oracle's balance-loss gradient on the global token set.
    # With dy = 0 the balance term is the ONLY source of dlogits / dW_g / dx, so a rank-local count
    # (1/W of the global one) fails the comparison outright.
    cfg = getattr(configs, name)
    for dy_scale in (1.0, 0.0):
        ep, ranks_in = _lockstep(cfg, W, T, dedup=dedup, balance_alpha=0.1, dy_scale=dy_scale)
        _vs_oracle(cfg, W, T, ranks_in, ep["probs"], ep["slot"], ep["y"], [gq["dx"] for gq in ep["g"]],
                   [gq["dlogits"] for gq in ep["g"]], ep["g"], ep["dWg"], balance_alpha=0.1, dy_scale=dy_scale)


def _ranks(cfg, W, T, dedup=False, capacity=None):
    from paper_2112_14397_b200.ep2 import EP2Rank, SymmetricBuffers
    dev = torch.device("cuda", 0)
    dt = inputs.TORCH_DTYPE[cfg.dtype]
    ranks_in = [inputs.make_inputs(cfg, rank=q, T=T) for q in range(W)]
    li0 = ranks_in[0]
    syms = SymmetricBuffers(W, dev)
    ranks = []
    for q in range(W):
        r = EP2Rank(T, cfg.d_model, cfg.d_ff, cfg.E, dt, dev, q, W, syms, dedup=dedup, capacity=capacity)
        r.set_gate(li0.Wg.to(dev))
        r.spawn(*(t.to(dev) for t in (li0.W1s, li0.b1s, li0.W2s, li0.b2s, li0.M1bits, li0.M2bits)))
        ranks.append(r)
    return ranks, ranks_in


@pytest.mark.parametrize("dedup", [False, True], ids=["ep2", "ep2d"])
def test_ep2_capacity_overflow_recovers(poison_empty, dedup):
    """Adaptive row capacity ("adaptive capacity", nothing dropped, R12): the first step
    sizes the symmetric row buffers from its all-gathered counts (+25% headroom); a later step
    whose routing needs far more rows (c = 0: every token to every expert) overflows, which every
    rank reports (MOE_ECAPACITY), the ranks grow together and the re-run matches the oracle."""
    from _ep_lockstep import run_lockstep_with_recovery
    cfg, W, T = configs.C3, 2, 256
    ranks, ranks_in = _ranks(cfg, W, T, dedup=dedup)
    dev = torch.device("cuda", 0)
    xs, us, dys = ([getattr(ri, k).to(dev) for ri in ranks_in] for k in ("x", "u", "dy"))
    tau = float(np.float32(cfg.tau))
    *_, attempts = run_lockstep_with_recovery(ranks, xs, us, dys, tau, float(np.float32(cfg.threshold)))
    assert attempts == 0 and all(r.grows == 0 for r in ranks)
    cap0 = ranks[0].R_cap
    assert cap0 <= ranks[0].worst_case_capacity() // 3         # sized from the counts, not the worst case
    skew = dataclasses.replace(cfg, threshold=0.0)
    ys, grads, dWg, attempts = run_lockstep_with_recovery(ranks, xs, us, dys, tau, 0.0)
    assert attempts == 1 and all(r.grows == 1 for r in ranks) and ranks[0].R_cap > cap0
    _vs_oracle(skew, W, T, ranks_in, [r.st["probs"] for r in ranks], [r.st["slot"] for r in ranks], ys,
               [gq["dx"] for gq in grads], [gq["dlogits"] for gq in grads], grads, dWg)


@pytest.mark.parametrize("dedup", [False, True], ids=["ep2", "ep2d"])
def test_ep2_step_captures_as_cuda_graph(poison_empty, dedup):
    """With the capacity fixed after the first step, the EP step has no host synchronisation: the
    phases of all emulated ranks are captured as ONE CUDA graph, and every replay reproduces the
    eager step bit for bit (what bench.py times at N > 1)."""
    from _ep_lockstep import run_lockstep
    cfg, W, T = configs.C3, 4, 300
    ranks, ranks_in = _ranks(cfg, W, T, dedup=dedup)
    dev = torch.device("cuda", 0)
    xs, us, dys = ([getattr(ri, k).to(dev) for ri in ranks_in] for k in ("x", "u", "dy"))
    args = (xs, us, dys, float(np.float32(cfg.tau)), float(np.float32(cfg.threshold)))
    ys0, g0, dWg0 = run_lockstep(ranks, *args)
    torch.cuda.synchronize()
    ref = ([y.clone() for y in ys0], [{k: v.clone() for k, v in g.items()} for g in g0], dWg0.clone())
    for r in ranks:
        r.prepare()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        run_lockstep(ranks, *args)                       # warm-up on the side stream (allocator pools)
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        ys1, g1, dWg1 = run_lockstep(ranks, *args)
    for _ in range(2):
        graph.replay()
        torch.cuda.synchronize()
        for r in ranks:
            r.check()
        for q in range(W):
            assert torch.equal(ys1[q], ref[0][q])
            for k in ("dx", "dlogits", "dW1", "dW2", "db1", "db2", "dWg"):
                assert torch.equal(g1[q][k], ref[1][q][k]), (q, k)
        assert torch.equal(dWg1, ref[2])


@pytest.mark.gpu
@pytest.mark.parametrize("name,W,T", [("C2", 2, 384), ("C4", 4, 256), ("C1", 2, 256)])
def test_ep2_overlap_matches_barrier_path_and_counters(name, W, T):
    """Exchange / GEMM overlap (moe_ep2_arrival_plan + moe_ep2_dispatch_ordered + moe_ep2_expert_ffn,
    DESIGN §8): the ordered copy pass with arrival counters and the per-expert GEMM waits give the
    barrier path's results bit for bit, and after every step each rank's counters equal its
    cumulative targets (= the rows all sources sent to its experts, summed over the steps)."""
    from paper_2112_14397_b200.ep2 import EP2Rank, SymmetricBuffers
    from _ep_lockstep import run_lockstep
    cfg = getattr(configs, name)
    dev = torch.device("cuda", 0)
    dt = inputs.TORCH_DTYPE[cfg.dtype]
    ranks_in = [inputs.make_inputs(cfg, rank=q, T=T) for q in range(W)]
    li0 = ranks_in[0]
    args = ([ri.x.to(dev) for ri in ranks_in], [ri.u.to(dev) for ri in ranks_in], [ri.dy.to(dev) for ri in ranks_in],
            float(np.float32(cfg.tau)), float(np.float32(cfg.threshold)))
    res = {}
    for overlap in (False, True):
        syms = SymmetricBuffers(W, dev)
        ranks = []
        for q in range(W):
            r = EP2Rank(T, cfg.d_model, cfg.d_ff, cfg.E, dt, dev, q, W, syms, overlap=overlap)
            r.set_gate(li0.Wg.to(dev))
            r.spawn(*(t.to(dev) for t in (li0.W1s, li0.b1s, li0.W2s, li0.b2s, li0.M1bits, li0.M2bits)))
            ranks.append(r)
        assert all(r.overlap == overlap for r in ranks)
        for step in range(2):
            ys, grads, dWg = run_lockstep(ranks, *args, top1=cfg.top1)
            torch.cuda.synchronize()
            for r in ranks:
                r.check()
            if overlap:
                ca = ranks[0].counts_all_host()
                El = cfg.E // W
                for q, r in enumerate(ranks):
                    arrive = syms.buf("arrive", q, (El,), torch.int32)[0].cpu().numpy()
                    want = (step + 1) * ca[:, q * El:(q + 1) * El].sum(0)
                    assert np.array_equal(arrive, want), (q, arrive, want)
                    assert np.array_equal(r.arr_target.cpu().numpy(), want)
        res[overlap] = (ys, grads, dWg)
    (y0, g0, w0), (y1, g1, w1) = res[False], res[True]
    for q in range(W):
        assert torch.equal(y0[q], y1[q])
        for k in ("dx", "dW1", "dW2", "db1", "db2", "dWg"):
            assert torch.equal(g0[q][k], g1[q][k]), k
    assert torch.equal(w0, w1)
