"""No hidden state across C-ABI calls.

ABI v2 carries every value that flows from one call to the next as an explicit argument:
  * db2 is either an output of moe_combine_bwd (summed in the same pass as d_eout) or summed by
    moe_expert_ffn_bwd from the d_eout it is given -- never a workspace leftover matched by
    pointer identity, so editing d_eout in place between the two calls gives the right db2;
  * the gate's input-gradient term dlogits W_g^T is written into dx by moe_dts_gate_bwd and
    moe_dispatch_bwd(accumulate=1) adds the expert rows onto it (no cached split of dlogits);
  * the one remaining carry, the per-block expert counts moe_dts_gate leaves for moe_dispatch,
    is checked: moe_dispatch refuses a (probs, slot) pair that is not the latest gate's.
"""
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


def _layer(cfg, T):
    from paper_2112_14397_b200.layer import DTSMoELayer
    li = inputs.make_inputs(cfg, T=T)
    dev = torch.device("cuda", 0)
    layer = DTSMoELayer(T, cfg.d_model, cfg.d_ff, cfg.E, dtype=li.x.dtype, device=dev)
    layer.set_gate(li.Wg.to(dev))
    layer.spawn(*(t.to(dev) for t in (li.W1s, li.b1s, li.W2s, li.b2s, li.M1bits, li.M2bits)))
    return layer, li, dev


def _colsum_per_expert(rows, offsets):
    rows = rows.double().cpu().numpy()
    off = offsets.cpu().numpy()
    return np.stack([rows[off[e]:off[e + 1]].sum(0) for e in range(len(off) - 1)])


@pytest.mark.parametrize("name,T", [("C3", 600), ("C1", None)])
def test_db2_follows_the_d_eout_it_is_given(name, T):
    from paper_2112_14397_b200 import _lib as L
    cfg = configs.get(name)
    T = T or cfg.T
    layer, li, dev = _layer(cfg, T)
    f32 = lambda v: float(np.float32(v))  # noqa: E731
    layer.forward(li.x.to(dev), li.u.to(dev), f32(cfg.tau), f32(cfg.threshold))
    st, rb = layer.state, layer.rows
    El, d = cfg.E, cfg.d_model
    db2_fused = torch.empty(El, d, dtype=torch.float32, device=dev)
    L.moe_combine_bwd(layer.ctx, li.dy.to(dev), rb["e_out"], rb["row_gate"], rb["row_token"], st.offsets, st.R_cap,
                      rb["d_eout"], rb["dG_row"], db2_fused)
    args = lambda db2: (layer.ctx, rb["d_eout"], rb["x_perm"], rb["gp"], rb["h"], st.offsets, st.R_cap,  # noqa: E731
                        layer.W1, layer.W2, torch.empty_like(rb["gp"]), torch.empty_like(rb["dx_perm"]),
                        torch.empty(El, cfg.d_ff, d, device=dev), torch.empty(El, cfg.d_ff, device=dev),
                        torch.empty(El, d, cfg.d_ff, device=dev), db2)
    db2_again = torch.empty_like(db2_fused)
    L.moe_expert_ffn_bwd(*args(db2_again))
    torch.cuda.synchronize()
    assert torch.equal(db2_fused, db2_again), "db2 of combine_bwd and of expert_ffn_bwd differ"
    ref = _colsum_per_expert(rb["d_eout"], st.offsets)
    assert np.allclose(db2_fused.cpu().numpy(), ref, rtol=1e-5, atol=1e-6)
    # edit d_eout IN PLACE (same pointer, offsets, R_cap) between the two calls
    rb["d_eout"].mul_(-2.0)
    db2_edit = torch.empty_like(db2_fused)
    L.moe_expert_ffn_bwd(*args(db2_edit))
    torch.cuda.synchronize()
    ref2 = _colsum_per_expert(rb["d_eout"], st.offsets)
    assert np.allclose(db2_edit.cpu().numpy(), ref2, rtol=1e-5, atol=1e-6), "stale db2 after an in-place edit"
    assert torch.equal(db2_edit, -2.0 * db2_fused)


def test_dispatch_bwd_accumulates_onto_the_gate_term():
    # dx = dlogits W_g^T from moe_dts_gate_bwd, then dispatch_bwd(accumulate) adds the rows; an
    # edit of dlogits after the gate backward cannot reach dx (nothing is cached from it)
    from paper_2112_14397_b200 import _lib as L
    cfg = configs.C3
    layer, li, dev = _layer(cfg, 500)
    f32 = lambda v: float(np.float32(v))  # noqa: E731
    layer.forward(li.x.to(dev), li.u.to(dev), f32(cfg.tau), f32(cfg.threshold))
    g = layer.backward(li.dy.to(dev))
    dx_ref = g["dx"].clone()
    st, rb = layer.state, layer.rows
    dx = torch.empty_like(dx_ref)
    dlogits = torch.empty(500, cfg.E, dtype=torch.float32, device=dev)
    dWg = torch.empty(cfg.d_model, cfg.E, dtype=torch.float32, device=dev)
    L.moe_dts_gate_bwd(layer.ctx, rb["dG_row"], st.slot, st.probs, st.x, layer.Wg, st.tau, 0.0, None, 500, dWg,
                       dlogits, dx)
    gate_only = dx.clone()
    dlogits.fill_(float("nan"))
    L.moe_dispatch_bwd(layer.ctx, rb["dx_perm"], st.slot, True, dx)
    torch.cuda.synchronize()
    assert torch.equal(dx, dx_ref)
    # without accumulate: the expert rows alone; gate term + rows (fp32 sum of the two bf16 rows)
    rows_only = torch.empty_like(dx)
    L.moe_dispatch_bwd(layer.ctx, rb["dx_perm"], st.slot, False, rows_only)
    torch.cuda.synchronize()
    assert torch.allclose(rows_only.float() + gate_only.float(), dx.float(), rtol=1e-2, atol=1e-2)


def test_dispatch_refuses_probs_slot_of_another_gate_call():
    from paper_2112_14397_b200 import _lib as L
    cfg = configs.C3
    T = 256
    layer, li, dev = _layer(cfg, T)
    E, d = cfg.E, cfg.d_model
    bufs = [dict(probs=torch.empty(T, E, device=dev), slot=torch.empty(T, E, dtype=torch.int32, device=dev),
                 counts=torch.empty(E, dtype=torch.int32, device=dev),
                 near=torch.empty(1, dtype=torch.int32, device=dev)) for _ in range(2)]
    x, u = li.x.to(dev), li.u.to(dev)
    R_cap = T * E + 128 * E
    out = dict(x_perm=torch.empty(R_cap, d, dtype=torch.bfloat16, device=dev),
               row_token=torch.empty(R_cap, dtype=torch.int32, device=dev),
               row_gate=torch.empty(R_cap, device=dev), offsets=torch.empty(E + 1, dtype=torch.int32, device=dev),
               R_out=torch.empty(1, dtype=torch.int32, device=dev))
    disp = lambda b: L.moe_dispatch(layer.ctx, x, b["probs"], b["slot"], out["x_perm"], out["row_token"],  # noqa: E731
                                    out["row_gate"], out["offsets"], R_cap, out["R_out"])
    for b in bufs:
        L.moe_dts_gate(layer.ctx, x, layer.Wg, u, 0.5, 0.05, 0, b["probs"], b["slot"], b["counts"], b["near"])
    with pytest.raises(L.MoEError) as e:
        disp(bufs[0])                                  # an older gate call's outputs
    assert e.value.code == 1 and "most recent moe_dts_gate" in str(e.value)
    disp(bufs[1])                                      # the latest: accepted
    torch.cuda.synchronize()
    layer.check()
    assert int(out["R_out"].item()) == int(out["offsets"][-1].item())
