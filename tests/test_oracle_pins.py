"""Pins of the fp64 oracle against things other than itself (CPU only).

Each test names what fixes the expected value: a value printed in PAPER.md, a
textbook table, a closed form, an independent implementation (torch autograd on
a plain FFN), brute force on tiny inputs, or central finite differences.
"""
import json
import math
import os

import numpy as np
import pytest
import torch

from harness import configs, inputs
from oracle import dts_moe as O

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def _rand_layer(T=12, d=6, f=10, E=4, seed=0, wg_scale=1.0, keep=0.8):
    rng = np.random.default_rng(seed)
    x = rng.standard_normal((T, d))
    Wg = rng.standard_normal((d, E)) * wg_scale
    W1s = rng.standard_normal((f, d)) * 0.5
    b1s = rng.standard_normal(f) * 0.1
    W2s = rng.standard_normal((d, f)) * 0.5
    b2s = rng.standard_normal(d) * 0.1
    M1 = inputs.pack_bits(rng.random((E, f * d)) < keep)
    M2 = inputs.pack_bits(rng.random((E, d * f)) < keep)
    ex = O.spawn(W1s, b1s, W2s, b2s, M1, M2)
    u = rng.integers(1, 1 << 24, size=(T, E)) * 2.0 ** -24
    dy = rng.standard_normal((T, d))
    return x, Wg, ex, u, dy, (W1s, b1s, W2s, b2s)


# ---------------------------------------------------------------- paper values
def test_softmax_paper_worked_example():
    """softmax over the two kept logits [2.01, 2.64] prints [0.35, 0.65]."""
    g = _gold("paper_worked_example.json")
    logits = np.array(g["logits"])
    k = g["topk_k"]
    keep = np.argsort(-logits, kind="stable")[:k]
    assert list(np.argsort(-logits, kind="stable")) == g["preference_order"]
    # Run the oracle's gate with d=1, x=1, Wg = kept logits, tau=1, no noise.
    p = O.gumbel_softmax(np.ones((1, 1)), logits[keep][None, :], None, 1.0)[0]
    full = np.zeros(3)
    full[keep] = p
    np.testing.assert_allclose(np.round(full, g["printed_decimals"]), g["gate_weights"], atol=0)


def test_combine_paper_worked_example():
    """y_s = 0.35*e0 + 0.65*e1 given gate weights [0.35, 0.65, 0].
    Feed the oracle a layer whose softmax reproduces those weights on the two
    kept experts (logits log .35, log .65, -inf-ish) and check the combine."""
    g = _gold("paper_worked_example.json")
    w = np.array(g["gate_weights"])
    d, f, E = 3, 4, 3
    rng = np.random.default_rng(1)
    x = np.array([g["x_s"]])
    W1s = rng.standard_normal((f, d)); b1s = rng.standard_normal(f)
    W2s = rng.standard_normal((d, f)); b2s = rng.standard_normal(d)
    bits = [inputs.pack_bits(rng.random((E, f * d)) < 0.7), inputs.pack_bits(rng.random((E, d * f)) < 0.7)]
    ex = O.spawn(W1s, b1s, W2s, b2s, bits[0], bits[1])
    # logits whose softmax is (0.35, 0.65, ~0): e2 gets logit -200
    Lt = np.array([math.log(0.35), math.log(0.65), -200.0])
    # x @ Wg = Lt with x = [-0.2, 0.4, 1.5]: Wg = outer(x, Lt)/|x|^2
    Wg = np.outer(x[0], Lt) / np.dot(x[0], x[0])
    fw = O.forward(x, Wg, None, 1.0, 0.1, ex)
    assert list(np.nonzero(fw.m[0])[0]) == [0, 1]
    e = [O.gelu(x @ ex["W1"][i].T + ex["b1"][i]) @ ex["W2"][i].T + ex["b2"][i] for i in range(E)]
    np.testing.assert_allclose(fw.y[0], w[0] * e[0][0] + w[1] * e[1][0], rtol=1e-12, atol=1e-12)


# ---------------------------------------------------------------- primitives
def test_gelu_against_normal_table():
    g = _gold("normal_cdf_table.json")
    z = np.array(g["z"]); Phi = np.array(g["Phi"])
    np.testing.assert_allclose(O.gelu(z), z * Phi, atol=g["abs_tol"] * 4)


def test_gelu_prime_finite_difference():
    a = np.linspace(-5, 5, 41)
    h = 1e-6
    fd = (O.gelu(a + h) - O.gelu(a - h)) / (2 * h)
    np.testing.assert_allclose(O.gelu_prime(a), fd, atol=1e-8)
    assert O.gelu_prime(np.array([0.0]))[0] == 0.5


def test_gumbel_moments_and_mode():
    g = _gold("gumbel_moments.json")
    u = inputs.uniform_u(1000, 1000).numpy().astype(np.float64)
    z = O.gumbel_noise(u)
    assert abs(z.mean() - g["mean"]) < 0.01
    assert abs(z.var() - g["variance"]) < 0.02
    assert abs(O.gumbel_noise(np.array([math.exp(-1.0)]))[0]) < 1e-15
    # monotone increasing in u (a sign error would flip this)
    assert np.all(np.diff(O.gumbel_noise(np.linspace(0.01, 0.99, 50))) > 0)


def test_noise_added_before_tau_division():
    """Eq. 8: (x W_g + zeta)/tau, noise inside the tau division.
    zeta = 0 at u = 1/e and zeta = 1 at u = exp(-exp(-1)); logits 0, tau = 0.5:
    z = [0, 2] -> p = [1/(1+e^2), e^2/(1+e^2)]."""
    u = np.array([[math.exp(-1.0), math.exp(-math.exp(-1.0))]])
    p = O.gumbel_softmax(np.ones((1, 1)), np.zeros((1, 2)), u, 0.5)[0]
    e2 = math.exp(2.0)
    np.testing.assert_allclose(p, [1 / (1 + e2), e2 / (1 + e2)], rtol=1e-12)


def test_tau_limits():
    """tau up -> uniform; tau -> 0 -> one-hot on the argmax."""
    rng = np.random.default_rng(3)
    x = rng.standard_normal((50, 8)); Wg = rng.standard_normal((8, 5))
    p = O.gumbel_softmax(x, Wg, None, 1e9)
    np.testing.assert_allclose(p, 0.2, atol=1e-8)
    p0 = O.gumbel_softmax(x, Wg, None, 1e-4)
    np.testing.assert_array_equal(np.argmax(p0, 1), np.argmax(x @ Wg, 1))
    assert np.all(p0.max(1) > 1 - 1e-12)
    # equal logits: uniform at any tau
    np.testing.assert_allclose(O.gumbel_softmax(x, np.zeros((8, 5)), None, 0.37), 0.2, atol=1e-15)


# ---------------------------------------------------------------- selection
def test_threshold_examples_spec():
    """S:190, S:199-201 and strict '>' (R3), guard (R5), top-1."""
    m = O.threshold_select(np.array([[0.7, 0.2, 0.09, 0.01]]), 0.1)
    assert m.tolist() == [[True, True, False, False]]
    m = O.threshold_select(np.array([[0.4, 0.35, 0.25]]), 0.3)
    assert m.tolist() == [[True, True, False]]
    m = O.threshold_select(np.array([[0.5, 0.5]]), 0.999)           # guard, lowest index
    assert m.tolist() == [[True, False]]
    m = O.threshold_select(np.array([[0.25, 0.75]]), 0.25)          # strict: 0.25 not > 0.25
    assert m.tolist() == [[False, True]]
    m = O.threshold_select(np.array([[0.3, 0.6, 0.1]]), 0.05, top1=True)
    assert m.tolist() == [[False, True, False]]
    m = O.threshold_select(np.array([[0.3, 0.6, 0.1]]), 0.0)        # c = 0: all positive
    assert m.all()


def test_derived_dts_example_and_no_renormalisation():
    """Logits [2.01, 2.64, 1.8] through the DTS gate at tau=1, c=0.25:
    Id = {0, 1}, weights are the raw g' (not renormalised)."""
    fw = O.forward(np.ones((1, 1)), np.array([[2.01, 2.64, 1.8]]), None, 1.0, 0.25,
                   O.spawn(np.ones((2, 1)), np.zeros(2), np.ones((1, 2)), np.zeros(1),
                           inputs.pack_bits(np.ones((3, 2), bool)), inputs.pack_bits(np.ones((3, 2), bool))))
    assert fw.m.tolist() == [[True, True, False]]
    ez = np.exp([2.01, 2.64, 1.8])
    np.testing.assert_allclose(fw.G[0], [ez[0] / ez.sum(), ez[1] / ez.sum(), 0.0], rtol=1e-12)
    assert fw.G[0].sum() < 1.0
    assert np.all(fw.G[fw.m] == fw.p[fw.m])                          # provenance


def test_counts_conservation_and_guard():
    x, Wg, ex, u, dy, _ = _rand_layer(T=200, E=6, wg_scale=2.0)
    for c in (0.0, 0.1, 0.3, 0.9):
        fw = O.forward(x, Wg, u, 0.3, c, ex)
        assert fw.counts.sum() == fw.m.sum()
        assert np.all(fw.m.sum(1) >= 1)
        am = np.argmax(fw.p, 1)
        assert np.all(fw.m[np.arange(200), am])                     # argmax always kept


# ---------------------------------------------------------------- spawn
def test_spawn_special_cases():
    rng = np.random.default_rng(5)
    f, d, E = 6, 4, 3
    W1s = rng.standard_normal((f, d)); W2s = rng.standard_normal((d, f))
    b1s = rng.standard_normal(f); b2s = rng.standard_normal(d)
    ones = inputs.pack_bits(np.ones((E, f * d), bool))
    zeros = inputs.pack_bits(np.zeros((E, f * d), bool))
    ex = O.spawn(W1s, b1s, W2s, b2s, ones, ones)
    for e in range(E):
        assert np.array_equal(ex["W1"][e], W1s) and np.array_equal(ex["W2"][e], W2s)
    ex = O.spawn(W1s, b1s, W2s, b2s, zeros, zeros)
    assert not ex["W1"].any() and not ex["W2"].any()
    assert np.array_equal(ex["b1"][1], b1s) and np.array_equal(ex["b2"][2], b2s)
    # hand-made bit pattern: word 0 = 0b101 -> flat elements 0 and 2 kept
    words = np.zeros((1, 1), np.uint32); words[0, 0] = 0b101
    keep = O.unpack_bits(words, 24)[0]
    assert keep[0] and not keep[1] and keep[2] and not keep[3:].any()
    # round trip against the harness packer (independent code)
    k = rng.random((2, 77)) < 0.5
    assert np.array_equal(O.unpack_bits(inputs.pack_bits(k), 77), k)


# ---------------------------------------------------------------- dispatch layout
def test_dispatch_layout_hand_example():
    m = np.array([[1, 0], [1, 1], [0, 1], [1, 0]], bool)
    counts, offsets, slot, row_token = O.dispatch_layout(m, align=4)
    assert counts.tolist() == [3, 2]
    assert offsets.tolist() == [0, 4, 8]
    assert slot.tolist() == [[0, -1], [1, 4], [-1, 5], [2, -1]]
    assert row_token.tolist() == [0, 1, 3, -1, 1, 2, -1, -1]


def test_dispatch_roundtrip_identity():
    rng = np.random.default_rng(9)
    m = rng.random((300, 7)) < 0.3
    counts, offsets, slot, row_token = O.dispatch_layout(m)
    assert np.all(offsets % 128 == 0)
    for t, e in zip(*np.nonzero(m)):
        assert row_token[slot[t, e]] == t
    assert (row_token >= 0).sum() == m.sum()


# ---------------------------------------------------------------- layer special cases
def test_threshold_zero_is_dense_weighted_sum_bruteforce():
    """c = 0 -> y_s = sum_i g'_i e_i(x_s) over ALL experts (BJ:5), brute force per token."""
    x, Wg, ex, u, dy, _ = _rand_layer(T=9, E=5)
    fw = O.forward(x, Wg, u, 0.7, 0.0, ex)
    assert fw.m.all()
    for s in range(x.shape[0]):
        ys = np.zeros(x.shape[1])
        for i in range(5):
            a = [sum(ex["W1"][i][r, k] * x[s, k] for k in range(x.shape[1])) + ex["b1"][i][r]
                 for r in range(ex["W1"].shape[1])]
            h = [0.5 * v * (1 + math.erf(v / math.sqrt(2))) for v in a]
            o = [sum(ex["W2"][i][r, k] * h[k] for k in range(len(h))) + ex["b2"][i][r]
                 for r in range(x.shape[1])]
            ys += fw.p[s, i] * np.array(o)
        np.testing.assert_allclose(fw.y[s], ys, rtol=1e-11, atol=1e-12)


def _torch_ffn(x, W1, b1, W2, b2):
    return torch.nn.functional.linear(
        torch.nn.functional.gelu(torch.nn.functional.linear(x, W1, b1), approximate="none"), W2, b2)


def test_identical_experts_dense_equals_ffn():
    """keep = 1 (identical experts) and c = 0: y = sum_i p_i FFN(x) = FFN(x)."""
    x, Wg, _, u, dy, shared = _rand_layer(T=16, E=4)
    W1s, b1s, W2s, b2s = shared
    ones = inputs.pack_bits(np.ones((4, W1s.size), bool))
    ex = O.spawn(W1s, b1s, W2s, b2s, ones, ones)
    fw = O.forward(x, Wg, u, 1.3, 0.0, ex)
    ref = _torch_ffn(*[torch.from_numpy(a) for a in (x, W1s, b1s, W2s, b2s)]).numpy()
    np.testing.assert_allclose(fw.y, ref, rtol=1e-12, atol=1e-12)


def test_single_expert_is_plain_ffn_fwd_and_bwd():
    """E = 1: p == 1, y = FFN(x) and the gradients equal torch autograd of the plain FFN;
    dW_g == 0 exactly (BJ:5)."""
    x, Wg, ex, u, dy, _ = _rand_layer(T=10, E=1, keep=0.8)
    fw = O.forward(x, Wg, u, 0.5, 0.3, ex)
    assert np.all(fw.p == 1.0) and fw.m.all()
    tx = torch.from_numpy(x).requires_grad_()
    tw = [torch.from_numpy(ex[k][0]).clone().requires_grad_() for k in ("W1", "b1", "W2", "b2")]
    ty = _torch_ffn(tx, *tw)
    np.testing.assert_allclose(fw.y, ty.detach().numpy(), rtol=1e-12, atol=1e-12)
    ty.backward(torch.from_numpy(dy))
    bw = O.backward(fw, dy)
    np.testing.assert_allclose(bw.dx, tx.grad.numpy(), rtol=1e-10, atol=1e-12)
    for got, t in zip((bw.dW1[0], bw.db1[0], bw.dW2[0], bw.db2[0]), tw):
        np.testing.assert_allclose(got, t.grad.numpy(), rtol=1e-10, atol=1e-12)
    assert np.all(bw.dWg == 0.0)


@pytest.mark.parametrize("c,tau", [(0.0, 1.0), (0.15, 0.6), (0.3, 2.0)])
def test_gradients_finite_differences(c, tau):
    """Central differences in fp64, loss = sum(y * dy), mask frozen, and the
    |p - c| margin asserted so the frozen mask is the true local mask."""
    x, Wg, ex, u, dy, _ = _rand_layer(T=7, d=5, f=6, E=4, seed=11)
    fw = O.forward(x, Wg, u, tau, c, ex)
    if c > 0:
        assert np.min(np.abs(fw.p - c)) > 1e-3
    mask = fw.m.copy()
    bw = O.backward(fw, dy)

    def loss(x_, Wg_, ex_):
        return float(np.sum(O.forward(x_, Wg_, u, tau, c, ex_, mask_override=mask).y * dy))

    eps = 1e-6

    def fd(arr, fn):
        g = np.zeros_like(arr)
        it = np.nditer(arr, flags=["multi_index"])
        for _ in it:
            i = it.multi_index
            old = arr[i]
            arr[i] = old + eps; lp = fn()
            arr[i] = old - eps; lm = fn()
            arr[i] = old
            g[i] = (lp - lm) / (2 * eps)
        return g

    np.testing.assert_allclose(bw.dx, fd(x, lambda: loss(x, Wg, ex)), rtol=1e-6, atol=1e-8)
    np.testing.assert_allclose(bw.dWg, fd(Wg, lambda: loss(x, Wg, ex)), rtol=1e-6, atol=1e-8)
    for key, g in (("W1", bw.dW1), ("b1", bw.db1), ("W2", bw.dW2), ("b2", bw.db2)):
        np.testing.assert_allclose(g, fd(ex[key], lambda: loss(x, Wg, ex)), rtol=1e-6, atol=1e-8)


# ---------------------------------------------------------------- NEXT rows
def test_balance_loss_closed_forms():
    """balanced top-1 with uniform g' gives alpha; collapse gives alpha N."""
    N, B, a = 4, 8, 0.1
    p = np.full((B, N), 1.0 / N)
    m = np.zeros((B, N), bool); m[np.arange(B), np.arange(B) % N] = True
    assert abs(O.balance_loss(p, m, a) - a) < 1e-15
    p1 = np.zeros((B, N)); p1[:, 0] = 1.0
    m1 = np.zeros((B, N), bool); m1[:, 0] = True
    assert abs(O.balance_loss(p1, m1, a) - a * N) < 1e-15


def test_balance_loss_gradient_fd():
    x, Wg, ex, u, dy, _ = _rand_layer(T=6, d=4, f=5, E=3, seed=21)
    tau, c, alpha = 0.8, 0.2, 0.1
    fw = O.forward(x, Wg, u, tau, c, ex)
    mask = fw.m.copy()
    bw = O.backward(fw, np.zeros_like(dy), balance_alpha=alpha)

    def L():
        p = O.gumbel_softmax(x, Wg, u, tau)
        return O.balance_loss(p, mask, alpha)

    eps = 1e-6
    g = np.zeros_like(Wg)
    for i in np.ndindex(Wg.shape):
        old = Wg[i]
        Wg[i] = old + eps; lp = L()
        Wg[i] = old - eps; lm = L()
        Wg[i] = old
        g[i] = (lp - lm) / (2 * eps)
    np.testing.assert_allclose(bw.dWg, g, rtol=1e-6, atol=1e-10)


def test_temperature_schedule():
    """P:535 'annealing temperature from 2.0 to 0.3'; linear midpoint."""
    assert O.temperature_at(0) == 2.0
    assert O.temperature_at(15000) == 0.3 and O.temperature_at(10 ** 6) == 0.3
    assert abs(O.temperature_at(7500) - 1.15) < 1e-12
    assert abs(O.temperature_at(7500, shape="exp") - math.sqrt(2.0 * 0.3)) < 1e-12


def test_c5_schedule_endpoints():
    s = configs.c5_schedule()
    assert len(s) == 20 and s[0] == (2.0, 0.0)
    assert abs(s[-1][0] - 0.05) < 1e-15 and abs(s[-1][1] - 0.3) < 1e-15


def test_survey_appendix_b_values():
    """Printed closed-form values (tests/golden/survey_appendix_b.json): DTS probabilities on
    the paper's worked-example logits at tau = 2, 1, 0.5, 0.1 (no noise), the tau = 1,
    c = 0.25 selection, Gumbel noise at fixed u (incl. the harness extremes 2^-24 and
    1 - 2^-24) and GELU at fixed points, each to its printed precision."""
    g = _gold("survey_appendix_b.json")
    L = np.array([g["logits"]])
    for tau, ref in g["dts_no_noise"].items():
        p = O.gumbel_softmax(np.ones((1, 1)), L, None, float(tau))[0]
        np.testing.assert_allclose(p, ref, atol=0.6e-6, err_msg=f"tau={tau}")
    sel = g["threshold_tau1_c0.25"]
    p1 = O.gumbel_softmax(np.ones((1, 1)), L, None, 1.0)
    m = O.threshold_select(p1, 0.25)
    assert m[0].tolist() == sel["selected"]
    np.testing.assert_allclose(np.where(m, p1, 0.0)[0], sel["G"], atol=0.6e-6)
    for u, z in g["gumbel"]:
        assert abs(O.gumbel_noise(np.array([u]))[0] - z) < 0.6e-9, (u, z)
    for a, v in g["gelu"]:
        assert abs(O.gelu(np.array([a]))[0] - v) < 0.6e-9, (a, v)
