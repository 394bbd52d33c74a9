"""The GPU parity checker itself (tests/_parity.compare) must catch localised corruption.

VERDICT r1 "What's weak" #1: with norm-wise errors only, one fully wrong e_out row among
16k rows, or one scribbled 32-column epilogue chunk of y, moved the tensor error by < 1%
and passed at 2e-2.  Here a fake "GPU run" is assembled from the oracle's own values rounded
to the GPU's storage dtypes (so it passes), then corrupted exactly that way: the per-row bound
must fail it while the tensor-norm error alone stays under the tolerance.  CPU only.
"""
import dataclasses

import numpy as np
import pytest
import torch

from harness import configs, inputs
from oracle import dts_moe as O

import _parity as P


def _bf16(a):
    return torch.from_numpy(np.asarray(a, np.float32)).bfloat16().float().numpy().astype(np.float64)


def _f32(a):
    return np.asarray(a, np.float32).astype(np.float64)


def _fake_run(cfg, li):
    ex, fw, bw = P.run_oracle(cfg, li)
    q = _bf16 if cfg.dtype == "bf16" else _f32
    counts, offsets, slot, row_token = O.dispatch_layout(fw.m)
    R = int(offsets[-1])
    valid = row_token >= 0
    x64 = inputs.to_f64(li.x)
    x_perm = np.zeros((R, cfg.d_model))
    x_perm[valid] = x64[row_token[valid]]
    p32 = _f32(fw.p)
    row_gate = np.zeros(R)
    toks, es = np.nonzero(fw.m)
    row_gate[slot[toks, es]] = p32[toks, es]
    dG_row = np.zeros(R)
    dG_row[slot[toks, es]] = bw.dG[toks, es]
    rows = dict(x_perm=x_perm, row_token=row_token, row_gate=row_gate,
                gp=q(O.to_rows({e: O.gelu_prime(a) for e, a in fw.a.items()}, offsets, cfg.d_ff)),
                h=q(O.to_rows(fw.h, offsets, cfg.d_ff)), e_out=q(O.to_rows(fw.o, offsets, cfg.d_model)),
                d_eout=q(O.to_rows(bw.do, offsets, cfg.d_model)), dG_row=_f32(dG_row),
                dx_perm=q(O.to_rows(bw.dxe, offsets, cfg.d_model)))
    for k in ("gp", "h", "e_out", "d_eout", "dx_perm"):
        rows[k][~valid] = 0.0            # the GPU's pad rows are zero
    grads = dict(dx=q(bw.dx), dWg=_f32(bw.dWg), dlogits=_f32(bw.dlogits), dW1=_f32(bw.dW1), db1=_f32(bw.db1),
                 dW2=_f32(bw.dW2), db2=_f32(bw.db2))
    band = P.band_tokens(p32, fw.m, cfg.threshold, cfg.top1)
    W = {k: ex[k] for k in ("W1", "b1", "W2", "b2")}
    return P.GpuRun(None, q(fw.y), p32, slot, counts, int(band.sum()), offsets, rows, W, grads)


@pytest.fixture(scope="module")
def c2_small():
    cfg = configs.C2
    li = inputs.make_inputs(cfg, T=256)
    g = _fake_run(cfg, li)
    # compare() reruns the oracle on every call; the inputs never change here, so memoise it
    real = P.run_oracle
    memo = real(cfg, li)
    P.run_oracle = lambda c, l, mask_override=None, backward=True: (
        memo if (c is cfg and l is li and mask_override is None and backward) else real(c, l, mask_override, backward))
    yield cfg, li, g
    P.run_oracle = real


def test_clean_fake_run_passes(c2_small):
    cfg, li, g = c2_small
    rep = P.compare(cfg, li, g)
    assert rep["y.row"] < 5e-3 and rep["e_out.row"] < 5e-3


def _mutated(g, where, fn):
    g2 = dataclasses.replace(g, rows=dict(g.rows), grads=dict(g.grads))
    if where == "y":
        g2.y = fn(g.y.copy())
    elif where in g.rows:
        g2.rows[where] = fn(g.rows[where].copy())
    else:
        g2.grads[where] = fn(g.grads[where].copy())
    return g2


def _zero_row(r):
    def f(a):
        a[r] = 0.0
        return a
    return f


def _scribble_chunk(r, c0):
    def f(a):
        a[r, c0:c0 + 32] = 0.0
        return a
    return f


@pytest.mark.parametrize("where,fn", [
    ("e_out", _zero_row(37)),                 # one fully wrong permuted expert-output row
    ("y", _scribble_chunk(11, 64)),           # one corrupted 32-column epilogue chunk of y
    ("dx_perm", _zero_row(5)),
    ("d_eout", _scribble_chunk(100, 0)),
    ("dx", _scribble_chunk(3, 32)),
    ("h", _scribble_chunk(50, 256)),
    ("dlogits", _zero_row(7)),                # still caught with the gate allowance (tests/_parity.gate_allowance)
])
def test_localised_corruption_fails(c2_small, where, fn):
    cfg, li, g = c2_small
    bad = _mutated(g, where, fn)
    # the hole: the whole-tensor norm error alone stays inside the 2e-2 tolerance ...
    ref = bad.y if where == "y" else (bad.rows.get(where) if where in bad.rows else bad.grads[where])
    good = g.y if where == "y" else (g.rows.get(where) if where in g.rows else g.grads[where])
    if where in ("e_out", "y", "dx_perm", "d_eout", "dx", "h"):
        assert P.rel_err(ref, good) < 2e-2
    # ... and the per-row bound catches it
    with pytest.raises(AssertionError, match=where):
        P.compare(cfg, li, bad)


def test_weight_gradient_row_corruption_fails(c2_small):
    cfg, li, g = c2_small

    def f(a):
        a[3, 17] = 0.0          # one output row of expert 3's dW1
        return a
    with pytest.raises(AssertionError, match=r"dW1\[3\]"):
        P.compare(cfg, li, _mutated(g, "dW1", f))


def test_row_err_floor_and_vectors():
    ref = np.ones((10, 4))
    got = ref.copy()
    got[2, 1] += 0.1                    # 0.1 / ||(1,1,1,1)|| = 0.05
    assert abs(P.row_err(got, ref) - 0.05) < 1e-12
    ref[7] = 1e-9                       # a near-zero row is judged against the median row norm
    got = ref.copy()
    got[7] = 1e-6
    assert P.row_err(got, ref) < 1e-5
    v = np.arange(1.0, 9.0)
    w = v.copy()
    w[0] += 0.9                          # vector: elementwise against max(|v_i|, median |v|)
    assert abs(P.row_err(w, v) - 0.9 / 4.5) < 1e-12
    assert abs(P.maxabs_rel(w, v) - 0.9 / 8.0) < 1e-12
