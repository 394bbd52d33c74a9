"""Full-size parity at BASELINE.json's configurations, in the launch configuration
bench.py times (DTSMoELayer, whole T per GPU).

The oracle cannot redo a full fp64 fwd+bwd of C4 in test time, so the checks are:
  * routing for ALL tokens: the oracle gate (Eq. 8/9) on every token -> mask bit-exact
    outside the 1e-6 band, probs <= 1e-5, counts / offsets / slot / row_token bit-exact
    against the stable rule, band count equal to the GPU's near_band;
  * sampled tokens (random + the ragged tail): y, dx, dlogits against the oracle run on
    those tokens alone (every one of these is a per-token quantity);
  * sampled experts (first, last, largest): dW1, db1, dW2, db2 against the oracle run
    on exactly that expert's tokens with only that expert selected (an expert's
    gradient depends only on its own rows);
  * dW_g: the property dW_g = x^T dlogits, checked in fp64 against the GPU's own dlogits.
"""
import numpy as np
import pytest
import torch

from harness import configs, inputs
from oracle import dts_moe as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _built():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2112_14397_b200 import build
    build.build()


def _np(t):
    return (t.float() if t.dtype == torch.bfloat16 else t).detach().cpu().numpy()


def _rel(a, b):
    a = np.asarray(a, np.float64); b = np.asarray(b, np.float64)
    d = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / d) if d else float(np.linalg.norm(a))


def fullsize(cfg, step=0, n_random=160, tail=32):
    from _parity import band_tokens, check_values, dG_scale, f32, gate_allowance, summary
    from paper_2112_14397_b200.layer import DTSMoELayer
    li = inputs.make_inputs(cfg, step=step)
    T, E = li.x.shape[0], cfg.E
    dev = torch.device("cuda", 0)
    tau, c = f32(cfg.tau), f32(cfg.threshold)
    layer = DTSMoELayer(T, cfg.d_model, cfg.d_ff, E, dtype=li.x.dtype, device=dev)
    layer.set_gate(li.Wg.to(dev))
    layer.spawn(*(t.to(dev) for t in (li.W1s, li.b1s, li.W2s, li.b2s, li.M1bits, li.M2bits)))
    y = layer.forward(li.x.to(dev), li.u.to(dev), tau, c, top1=cfg.top1)
    g = layer.backward(li.dy.to(dev))
    torch.cuda.synchronize()
    layer.check()
    st = layer.state
    probs, slot = _np(st.probs), _np(st.slot)
    m_gpu = slot >= 0
    tol = 2e-2 if cfg.dtype == "bf16" else 1e-4
    rep = {}

    # ---- routing, all tokens
    x64, Wg64, u64, dy64 = (inputs.to_f64(t) for t in (li.x, li.Wg, li.u, li.dy))
    p = O.gumbel_softmax(x64, Wg64, u64, tau)
    m = O.threshold_select(p, c, cfg.top1)
    band = band_tokens(probs, m_gpu, c, cfg.top1)
    flips = np.any(m != m_gpu, axis=1)
    rep.update(band=int(band.sum()), flips=int(flips.sum()), probs_maxabs=float(np.abs(probs - p).max()))
    assert not np.any(flips & ~band), np.nonzero(flips & ~band)[0][:10]
    assert int(st.near_band.item()) == int(band.sum())
    assert rep["probs_maxabs"] <= 1e-5, rep
    counts, offsets, slot_ref, row_token = O.dispatch_layout(m_gpu)
    assert np.array_equal(_np(st.counts), counts)
    assert np.array_equal(_np(st.offsets), offsets)
    assert np.array_equal(slot, slot_ref)
    R = int(offsets[-1])
    assert np.array_equal(_np(layer.rows["row_token"][:R]), row_token)

    # ---- sampled tokens (random + ragged tail): per-token outputs
    rng = np.random.default_rng(7)
    S = np.unique(np.concatenate([rng.choice(T, size=min(n_random, T), replace=False),
                                  np.arange(max(0, T - tail), T)]))
    ex = O.spawn(inputs.to_f64(li.W1s), inputs.to_f64(li.b1s), inputs.to_f64(li.W2s), inputs.to_f64(li.b2s),
                 inputs.bits_u32(li.M1bits), inputs.bits_u32(li.M2bits))
    fw = O.forward(x64[S], Wg64, u64[S], tau, c, ex, mask_override=m_gpu[S])
    bw = O.backward(fw, dy64[S])
    # per-token rows: norm-wise and per-row bounds (tests/_parity.check_values)
    check_values(rep, "y", _np(y)[S], fw.y, tol)
    allow = gate_allowance(fw.p, fw.m, bw.dG, fw.tau, tol, dG_scale(fw, dy64[S], cfg.dtype))
    check_values(rep, "dx", _np(g["dx"])[S], bw.dx, tol, allow=allow * np.linalg.norm(Wg64, 2))
    check_values(rep, "dlogits", _np(g["dlogits"])[S], bw.dlogits, tol, allow=allow)
    # the permuted rows of the sampled tokens (row = slot[t, e]): e_out, d_eout, dx_perm
    rows = np.concatenate([slot[S[fw.toks[e]], e] for e in sorted(fw.o)])
    for name, per in (("e_out", fw.o), ("d_eout", bw.do), ("dx_perm", bw.dxe)):
        ref = np.concatenate([per[e] for e in sorted(fw.o)])
        check_values(rep, name, _np(layer.rows[name][torch.from_numpy(rows).to(dev).long()]), ref, tol)

    # ---- sampled experts: weight gradients over all of that expert's rows
    cnt = m_gpu.sum(0)
    for e in sorted({0, E - 1, int(np.argmax(cnt))}):
        toks = np.nonzero(m_gpu[:, e])[0]
        only = np.zeros((len(toks), E), bool)
        only[:, e] = True
        fe = O.forward(x64[toks], Wg64, u64[toks], tau, c, ex, mask_override=only)
        be = O.backward(fe, dy64[toks])
        for k, ref in (("dW1", be.dW1[e]), ("db1", be.db1[e]), ("dW2", be.dW2[e]), ("db2", be.db2[e])):
            if len(toks):   # every output row of dW1 / dW2; db1 / db2 norm-wise (sums with cancellation)
                check_values(rep, f"{k}[{e}]", _np(g[k][e]), ref, tol, rows=k in ("dW1", "dW2"))
            else:
                assert not np.any(_np(g[k][e])), f"{k}[{e}] of an empty expert must be zero"

    # ---- dW_g = x^T dlogits (property, fp64 product of the GPU's own dlogits)
    check_values(rep, "dWg_property", _np(g["dWg"]), x64.T @ _np(g["dlogits"]).astype(np.float64), 1e-3, rows=False)
    print(cfg.name, step, summary(rep))
    return rep


def test_c2_full_bench_config():
    fullsize(configs.C2)


def test_c3_full():
    fullsize(configs.C3)


def test_c4_full():
    fullsize(configs.C4)


@pytest.mark.parametrize("s", [0, 10, 19])
def test_c5_full_schedule(s):
    fullsize(configs.C5.at_step(s), step=s)


def test_c1_full_fp32():
    fullsize(configs.C1, n_random=200)


@pytest.mark.parametrize("name", ["C2", "C4"])
def test_graph_replay_matches_eager(name):
    # bench.py times the step as ONE CUDA-graph replay with the row capacity fixed to the
    # warm-up's (static capacity, no host sync).  That replay must give bit-identical outputs
    # and gradients to the eager path the checks above use, on every replay.
    from _parity import f32
    from paper_2112_14397_b200.layer import DTSMoELayer
    cfg = getattr(configs, name)
    li = inputs.make_inputs(cfg)
    dev = torch.device("cuda", 0)
    tau, c = f32(cfg.tau), f32(cfg.threshold)
    layer = DTSMoELayer(li.x.shape[0], cfg.d_model, cfg.d_ff, cfg.E, dtype=li.x.dtype, device=dev)
    layer.set_gate(li.Wg.to(dev))
    layer.spawn(*(t.to(dev) for t in (li.W1s, li.b1s, li.W2s, li.b2s, li.M1bits, li.M2bits)))
    x, u, dy = li.x.to(dev), li.u.to(dev), li.dy.to(dev)
    y0 = layer.forward(x, u, tau, c).clone()
    g0 = {k: v.clone() for k, v in layer.backward(dy).items()}
    torch.cuda.synchronize()
    layer.check()
    R_static = layer.state.R_cap
    layer.forward(x, u, tau, c, R_cap=R_static)       # as bench.py: one eager step at the static capacity
    layer.backward(dy)
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        y1 = layer.forward(x, u, tau, c, R_cap=R_static)
        g1 = layer.backward(dy)
    for _ in range(2):
        graph.replay()
        torch.cuda.synchronize()
        layer.check()
        assert torch.equal(y1, y0)
        for k in g0:
            if k == "da":
                continue
            assert torch.equal(g1[k], g0[k]), k
