"""GPU parity of the CUDA path (through the C ABI) against the fp64 oracle.

Sizes: C1 in full; C2-C5 at reduced T (same d, d_ff, E, tau, c -- several tiles and a
ragged tail), plus edge cases (ragged T, T=1, c=0, no noise, top-1, the guard).
Tolerances (BJ:5): probs 1e-5 abs; masks/counts/layout bit-exact outside the 1e-6
band; values 1e-4 (fp32) / 2e-2 (bf16) norm-wise relative.
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


def _run(cfg, T=None, step=0, with_noise=True, backward=True, recompute=False):
    from _parity import compare, run_gpu, summary
    li = inputs.make_inputs(cfg, step=step, with_noise=with_noise, T=T)
    g = run_gpu(cfg, li, backward=backward, recompute=recompute)
    rep = compare(cfg, li, g, backward=backward)
    print(cfg.name, T, "recompute" if recompute else "", summary(rep))
    return rep, g


def test_c1_full():
    _run(configs.C1)


def test_c1_ragged_tail():
    _run(configs.C1, T=200)


def test_c1_single_token():
    _run(configs.C1, T=1)


def test_c1_threshold_zero_all_selected():
    cfg = dataclasses.replace(configs.C1, threshold=0.0)
    rep, g = _run(cfg)
    assert np.all(g.slot >= 0)


def test_c1_guard_fires():
    # c >= 1/E makes empty selections possible; a low tau makes them common
    cfg = dataclasses.replace(configs.C1, threshold=0.6, tau=4.0)
    rep, g = _run(cfg)
    assert np.all((g.slot >= 0).sum(1) >= 1)


def test_c1_top1():
    cfg = dataclasses.replace(configs.C1, top1=True)
    rep, g = _run(cfg)
    assert np.all((g.slot >= 0).sum(1) == 1)


def test_c2_reduced_dense():
    _run(configs.C2, T=1024)


def test_c2_reduced_no_noise():
    _run(configs.C2, T=384, with_noise=False)


def test_c3_reduced():
    _run(configs.C3, T=1000)


def test_c3_reduced_top1():
    _run(dataclasses.replace(configs.C3, top1=True), T=512)


def test_c4_reduced():
    _run(configs.C4, T=640)


@pytest.mark.parametrize("s", [0, 2, 9, 19])
def test_c5_schedule_steps(s):
    _run(configs.C5.at_step(s), T=512, step=s)


def test_deterministic_rerun():
    from _parity import run_gpu
    cfg = configs.C3
    li = inputs.make_inputs(cfg, T=777)
    a = run_gpu(cfg, li)
    b = run_gpu(cfg, li)
    assert np.array_equal(a.y, b.y) and np.array_equal(a.slot, b.slot)
    for k in a.grads:
        assert np.array_equal(a.grads[k], b.grads[k]), k


def test_nonfinite_input_flagged():
    from paper_2112_14397_b200 import _lib as L
    from paper_2112_14397_b200.layer import DTSMoELayer
    cfg = configs.C1
    li = inputs.make_inputs(cfg)
    dev = torch.device("cuda", 0)
    layer = DTSMoELayer(cfg.T, cfg.d_model, cfg.d_ff, cfg.E, dtype=torch.float32, device=dev)
    x = li.x.clone()
    x[5, 3] = float("nan")
    layer.set_gate(li.Wg.to(dev))
    layer.spawn(*(t.to(dev) for t in (li.W1s, li.b1s, li.W2s, li.b2s, li.M1bits, li.M2bits)))
    layer.forward(x.to(dev), li.u.to(dev), 1.0, 0.1)
    with pytest.raises(L.MoEError) as e:
        layer.check()
    assert e.value.code == 6


def test_capacity_overflow_flagged():
    from paper_2112_14397_b200 import _lib as L
    from paper_2112_14397_b200.layer import DTSMoELayer
    cfg = configs.C1
    li = inputs.make_inputs(cfg)
    dev = torch.device("cuda", 0)
    layer = DTSMoELayer(cfg.T, cfg.d_model, cfg.d_ff, cfg.E, dtype=torch.float32, device=dev)
    layer.set_gate(li.Wg.to(dev))
    layer.spawn(*(t.to(dev) for t in (li.W1s, li.b1s, li.W2s, li.b2s, li.M1bits, li.M2bits)))
    layer.forward(li.x.to(dev), li.u.to(dev), 1.0, 0.1, R_cap=128)
    with pytest.raises(L.MoEError) as e:
        layer.check()
    assert e.value.code == 7


def test_invalid_scalars_rejected():
    from paper_2112_14397_b200 import _lib as L
    from paper_2112_14397_b200.layer import DTSMoELayer
    cfg = configs.C1
    layer = DTSMoELayer(cfg.T, cfg.d_model, cfg.d_ff, cfg.E, dtype=torch.float32)
    li = inputs.make_inputs(cfg)
    layer.set_gate(li.Wg.cuda())
    for tau, c in ((0.0, 0.1), (float("nan"), 0.1), (1.0, 1.0), (1.0, -0.1)):
        with pytest.raises(L.MoEError) as e:
            layer.forward(li.x.cuda(), li.u.cuda(), tau, c)
        assert e.value.code == 1


def test_ep_self_exchange_matches_single_rank():
    """The EP code path (NCCL counts all-gather, plan, grouped send/recv row exchange with
    pad zeroing, dW_g all-reduce) on a world-1 communicator must reproduce the non-EP
    layer bit for bit (C3 reduced, bf16)."""
    from paper_2112_14397_b200 import _lib as L
    from paper_2112_14397_b200.layer import DTSMoELayer
    cfg = configs.C3
    li = inputs.make_inputs(cfg, T=700)
    dev = torch.device("cuda", 0)
    comm = L.moe_nccl_comm_init(L.moe_nccl_unique_id(), 1, 0)
    outs = []
    for c in (0, comm):
        layer = DTSMoELayer(700, cfg.d_model, cfg.d_ff, cfg.E, dtype=torch.bfloat16, device=dev, nccl_comm=c)
        layer.set_gate(li.Wg.to(dev))
        layer.spawn(*(t.to(dev) for t in (li.W1s, li.b1s, li.W2s, li.b2s, li.M1bits, li.M2bits)))
        y = layer.forward(li.x.to(dev), li.u.to(dev), float(np.float32(cfg.tau)), float(np.float32(cfg.threshold)))
        g = layer.backward(li.dy.to(dev), inplace_da=False)
        torch.cuda.synchronize()
        layer.check()
        outs.append((y.float().cpu(), {k: v.float().cpu() for k, v in g.items() if k != "da"}))
        del layer
    assert torch.equal(outs[0][0], outs[1][0])
    for k in outs[0][1]:
        assert torch.equal(outs[0][1][k], outs[1][1][k]), k
    L.moe_nccl_comm_destroy(comm)


@pytest.mark.parametrize("cfg_name,T", [("C1", None), ("C3", 600)])
def test_balance_loss_and_gradient(cfg_name, T):
    """NEXT #1, Eq. 10: the loss value (moe_balance_loss) and its gradient folded
    into the gate backward (balance_alpha) against the oracle."""
    from _parity import f32, rel_err, run_oracle
    from oracle import dts_moe as O
    from paper_2112_14397_b200 import _lib as L
    from paper_2112_14397_b200.layer import DTSMoELayer
    cfg = configs.get(cfg_name)
    li = inputs.make_inputs(cfg, T=T)
    T_ = li.x.shape[0]
    dev = torch.device("cuda", 0)
    layer = DTSMoELayer(T_, cfg.d_model, cfg.d_ff, cfg.E, dtype=li.x.dtype, device=dev)
    layer.set_gate(li.Wg.to(dev))
    layer.spawn(*(t.to(dev) for t in (li.W1s, li.b1s, li.W2s, li.b2s, li.M1bits, li.M2bits)))
    layer.forward(li.x.to(dev), li.u.to(dev), f32(cfg.tau), f32(cfg.threshold))
    alpha = 0.1
    loss = torch.empty(1, dtype=torch.float32, device=dev)
    L.moe_balance_loss(layer.ctx, layer.state.probs, layer.state.counts, alpha, T_, loss)
    g = layer.backward(li.dy.to(dev), balance_alpha=alpha)
    torch.cuda.synchronize()
    layer.check()
    m_gpu = (layer.state.slot >= 0).cpu().numpy()
    ex, fw, _ = run_oracle(cfg, li, mask_override=m_gpu, backward=False)
    ref_loss = O.balance_loss(fw.p, fw.m, alpha)
    assert abs(loss.item() - ref_loss) <= 1e-5 * max(1.0, abs(ref_loss)), (loss.item(), ref_loss)
    bw = O.backward(fw, inputs.to_f64(li.dy), balance_alpha=alpha)
    tol = 1e-4 if cfg.dtype == "f32" else 2e-2
    assert rel_err(g["dWg"].cpu().numpy(), bw.dWg) <= tol
    assert rel_err(g["dx"].float().cpu().numpy(), bw.dx) <= tol


@pytest.mark.parametrize("cfg_name,T", [("C1", None), ("C4", 512)])
def test_recompute_mode_matches_saved_mode(cfg_name, T):
    """NEXT #3: with recompute=True nothing [R, d_ff]-sized is kept between the
    forward and the backward; GEMM1 + GELU are re-run from x_perm.  Results are bit-identical
    to the saved-activation mode (same kernels, same inputs, same order)."""
    from _parity import f32
    from paper_2112_14397_b200.layer import DTSMoELayer
    cfg = configs.get(cfg_name)
    li = inputs.make_inputs(cfg, T=T)
    T_ = li.x.shape[0]
    dev = torch.device("cuda", 0)
    outs = []
    for rc in (False, True):
        layer = DTSMoELayer(T_, cfg.d_model, cfg.d_ff, cfg.E, dtype=li.x.dtype, device=dev, recompute=rc)
        layer.set_gate(li.Wg.to(dev))
        layer.spawn(*(t.to(dev) for t in (li.W1s, li.b1s, li.W2s, li.b2s, li.M1bits, li.M2bits)))
        y = layer.forward(li.x.to(dev), li.u.to(dev), f32(cfg.tau), f32(cfg.threshold))
        if rc:
            layer.rows["h"].fill_(float("nan"))      # the forward's h must not be needed any more
            layer.rows["gp"].fill_(float("nan"))
        g = layer.backward(li.dy.to(dev))
        torch.cuda.synchronize()
        layer.check()
        outs.append((y.float().cpu(), {k: v.float().cpu() for k, v in g.items() if k not in ("da",)}))
    assert torch.equal(outs[0][0], outs[1][0])
    for k in outs[0][1]:
        assert torch.equal(outs[0][1][k], outs[1][1][k]), k


@pytest.mark.parametrize("cfg_name,T,step", [("C1", None, 0), ("C3", 700, 0), ("C4", 512, 0), ("C5", 384, 0),
                                              ("C5", 384, 19)])
def test_recompute_mode_against_oracle(cfg_name, T, step):
    """NEXT #3 against the fp64 oracle itself, not only against the saved mode: the
    forward keeps no [R, d_ff] activation (gp and h are NaN-filled after it), the backward's
    moe_expert_ffn_recompute rebuilds them from x_perm, and every output, intermediate and
    gradient passes the same element / row / tensor checks as the saved-activation path."""
    cfg = configs.get(cfg_name)
    if cfg_name == "C5":
        cfg = cfg.at_step(step)
    rep, g = _run(cfg, T=T, step=step, recompute=True)
    assert "gp" in rep and "h" in rep


@pytest.mark.parametrize("cfg_name,T", [("C1", None), ("C3", 600)])
def test_balance_gradient_alone(cfg_name, T):
    """With dy = 0 the Eq. 10 term is the only source of the gate gradient: dlogits,
    dW_g and dx (= dlogits W_g^T) against the oracle's balance-loss gradient, row by row."""
    from _parity import check_values, f32, run_oracle
    from oracle import dts_moe as O
    from paper_2112_14397_b200.layer import DTSMoELayer
    cfg = configs.get(cfg_name)
    li = inputs.make_inputs(cfg, T=T)
    T_ = li.x.shape[0]
    dev = torch.device("cuda", 0)
    layer = DTSMoELayer(T_, cfg.d_model, cfg.d_ff, cfg.E, dtype=li.x.dtype, device=dev)
    layer.set_gate(li.Wg.to(dev))
    layer.spawn(*(t.to(dev) for t in (li.W1s, li.b1s, li.W2s, li.b2s, li.M1bits, li.M2bits)))
    layer.forward(li.x.to(dev), li.u.to(dev), f32(cfg.tau), f32(cfg.threshold))
    g = layer.backward(torch.zeros_like(li.dy).to(dev), balance_alpha=0.1)
    torch.cuda.synchronize()
    layer.check()
    m_gpu = (layer.state.slot >= 0).cpu().numpy()
    _, fw, _ = run_oracle(cfg, li, mask_override=m_gpu, backward=False)
    bw = O.backward(fw, np.zeros_like(inputs.to_f64(li.dy)), balance_alpha=0.1)
    tol = 1e-4 if cfg.dtype == "f32" else 2e-2
    rep = {}
    check_values(rep, "dlogits", g["dlogits"].cpu().numpy(), bw.dlogits, tol)
    check_values(rep, "dWg", g["dWg"].cpu().numpy(), bw.dWg, tol, rows=False)
    check_values(rep, "dx", g["dx"].float().cpu().numpy(), bw.dx, tol)
    assert np.abs(bw.dlogits).max() > 0
    print(cfg_name, rep)


# ---- shapes off the benchmark grid: the other gate paths and partial GEMM tiles ----------
def _shape(name, T, d, f, E, tau, c, wg_var=None):
    import math
    return dataclasses.replace(configs.C3, name=name, T=T, d_model=d, d_ff=f, E=E, tau=tau, threshold=c,
                               wg_std=math.sqrt((wg_var if wg_var else 1.0) / d))


def test_bf16_simt_gemm_debug_path(monkeypatch):
    # MOE_GEMM=simt: the bf16 expert GEMMs on the CUDA-core grouped GEMM (the fp32 configs'
    # kernel) instead of tcgen05 -- a debug path, held to the same oracle checks
    monkeypatch.setenv("MOE_GEMM", "simt")
    _run(_shape("simt", 300, 256, 512, 16, 0.7, 0.05))


def test_bf16_E48_fused_gate_16_wide_boxes():
    # E % 32 != 0: fused gate with 12 experts per lane quarter; N=48 gate MMA
    _run(_shape("E48", 700, 256, 512, 48, 0.5, 0.03))


def test_bf16_E24_unfused_gate_path():
    # E % 16 != 0: tcgen05 logits (padded to 32) to HBM + thread-per-token softmax + fp64 refine queue
    _run(_shape("E24", 515, 192, 384, 24, 0.7, 0.05))


def test_bf16_unfused_gate_env_matches_oracle(monkeypatch):
    monkeypatch.setenv("MOE_GATE_UNFUSED", "1")
    _run(_shape("E16u", 400, 128, 256, 16, 1.0, 0.02))


def test_bf16_partial_tiles_simt_gate():
    # E > 64 (SIMT warp-per-token gate with inline fp64 refine); d = 192 and d_ff = 320 are
    # not multiples of the 256-wide GEMM tile: partial N tiles on every expert GEMM
    _run(_shape("odd", 300, 192, 320, 80, 0.8, 0.01))


def test_bf16_dims_multiple_of_8_not_64():
    # d = 200, d_ff = 328 (multiples of 8, not of 64): accepted by moe_create (SURVEY §8(b) asks for
    # multiples of 8); the CUDA-core GEMMs and the SIMT gate run them (the tensor-core GEMMs and
    # gate need 64-wide K boxes), every value checked against the oracle as usual
    _run(_shape("m8", 300, 200, 328, 16, 0.7, 0.05))
    _run(_shape("m8b", 257, 72, 136, 8, 1.0, 0.1))
    _run(_shape("m8r", 300, 200, 328, 16, 0.7, 0.05), recompute=True)


def test_bf16_single_expert_is_dense_ffn():
    # E = 1: every token to the one expert with weight 1 (P:311 special case), dW_g = 0
    rep, g = _run(_shape("E1", 256, 128, 256, 1, 1.0, 0.0))
    assert float(np.abs(g.grads["dWg"]).max()) == 0.0


# ---- the fp64 refine queue under load: tau = 200 squeezes every p towards 1/E and c = 1/E
# puts most tokens within the 5e-5 refine margin of the threshold, so most decisions (and
# the probs of those tokens) come from gate_refine_kernel (tau = 50 at E = 64).  Shapes cover one W_g chunk
# (E=16, d=768), four chunks (E=64, d=1024: 32 KB = 256 rows of W_g per chunk) and the
# scalar staging path (E=20: a W_g row is 40 bytes, not a multiple of 16) with a ragged
# second chunk (d=960, 819 rows per chunk); and short queues (fewer queued tokens than SMs:
# T = 40 at E = 64, T = 20 at E = 48 with d = 832 = 3 x 256 + 64 rows, T = 30 at E = 20).
@pytest.mark.parametrize("E,d,T,tau", [(16, 768, 1000, 200.0), (64, 1024, 700, 50.0), (20, 960, 515, 200.0),
                                       (64, 1024, 40, 50.0), (48, 832, 20, 200.0), (20, 960, 30, 200.0)])
def test_refine_queue_heavy(E, d, T, tau):
    cfg = _shape(f"RQ{E}", T, d, 256, E, tau, 1.0 / E)
    rep, g = _run(cfg, backward=False)
    from _parity import run_oracle
    li = inputs.make_inputs(cfg, T=T)
    _, fw, _ = run_oracle(cfg, li, backward=False)
    queued = np.any(np.abs(fw.p - np.float32(cfg.threshold)) < 5e-5, axis=1)
    assert queued.mean() > 0.5, queued.mean()


@pytest.mark.parametrize("dtype", ["bf16", "fp32"])
def test_empty_token_batch(dtype):
    # T = 0 (a rank with no tokens): every call succeeds, outputs are empty, the weight
    # gradients are exactly zero (sums over no rows), and a following non-empty layer is unaffected
    from paper_2112_14397_b200.layer import DTSMoELayer
    cfg = configs.C1 if dtype == "fp32" else dataclasses.replace(configs.C2, d_model=128, d_ff=256)
    dt = torch.float32 if dtype == "fp32" else torch.bfloat16
    dev = torch.device("cuda", 0)
    li = inputs.make_inputs(cfg, T=4)
    layer = DTSMoELayer(0, cfg.d_model, cfg.d_ff, cfg.E, dtype=dt, device=dev)
    layer.set_gate(li.Wg.to(dev))
    layer.spawn(*(t.to(dev) for t in (li.W1s, li.b1s, li.W2s, li.b2s, li.M1bits, li.M2bits)))
    x = torch.empty(0, cfg.d_model, dtype=dt, device=dev)
    u = torch.empty(0, cfg.E, dtype=torch.float32, device=dev)
    y = layer.forward(x, u, float(np.float32(cfg.tau)), float(np.float32(cfg.threshold)))
    g = layer.backward(torch.empty(0, cfg.d_model, dtype=dt, device=dev))
    torch.cuda.synchronize()
    layer.check()
    assert y.shape == (0, cfg.d_model)
    assert g["dx"].shape == (0, cfg.d_model)
    for k in ("dW1", "db1", "dW2", "db2", "dWg"):
        assert g[k].numel() > 0 and not torch.any(g[k] != 0), k
    _run(cfg, T=4)


def test_bf16_E128_maximum_experts():
    # E = 128, the largest expert count the gate supports (4 experts per lane in the
    # warp-per-token SIMT gate); 64-row experts on average, many partial GEMM tiles
    _run(_shape("E128", 640, 256, 512, 128, 1.0, 0.004))


def test_bf16_more_than_1024_gate_blocks():
    # T = 131149 tokens = 1025 gate blocks of 128 (+77): the dispatch scan walks each expert's
    # per-block counts in chunks of 1024 with a carry, so this is the first shape with two chunks
    # (C4's 131072 tokens fill exactly one); layout and routing bit-exact against the oracle
    _run(_shape("scan2", 1024 * 128 + 77, 64, 128, 8, 0.5, 0.05), backward=False)
