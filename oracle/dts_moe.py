"""Oracle: a plain, slow, obviously-correct fp64 CPU implementation of one
DTS-Gate MoE FFN layer (EvoMoE, arXiv 2112.14397) and its gradients.

TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs may import this module.  It shares no
code with the CUDA path (paper_2112_14397_b200/) and imports nothing from it.

Citations are PAPER.md line numbers (P:n) with the equation / algorithm they
fall in.  Where the paper is silent or garbled the reading taken is the one
listed in DESIGN.md §"Readings" (numbered R1..R21, mirroring SURVEY.md §8c).

Every function computes in float64 from inputs that are exact float64 copies
of the values the GPU receives (bf16/fp32 storage; tau and c as fp32 values).
Library primitives used as steps: numpy matmul, scipy.special.erf, np.exp/log.

Pins (tests/test_oracle_pins.py): softmax worked example, combine
worked example, Gumbel moments, tabulated normal CDF (GELU), E=1 ==
torch.nn.functional FFN + autograd, c=0 == dense weighted sum, tau->inf
uniform, tau->0 argmax, finite differences of every gradient, spawn special
cases, SPEC threshold examples, count conservation, balance-loss closed forms.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Dict, List, Optional

import numpy as np
from scipy.special import erf

SQRT2 = np.sqrt(2.0)
INV_SQRT_2PI = 1.0 / np.sqrt(2.0 * np.pi)


# --------------------------------------------------------------------------- #
# Primitives
# --------------------------------------------------------------------------- #
def gumbel_noise(u: np.ndarray) -> np.ndarray:
    """zeta ~ Gumbel(0,1) formed from uniform u as -log(-log u).
    P:326 ("sampled from Gumbel(0,1)"), Eq. 8; reading R2: i.i.d. per
    (token, expert), u supplied by the harness (BJ:5)."""
    return -np.log(-np.log(u))


def gelu(a: np.ndarray) -> np.ndarray:
    """GELU, erf form: a * Phi(a), Phi(a) = (1 + erf(a/sqrt 2))/2.
    Eq. 3 prints ReLU but §V.A uses GeLU for all models: reading R8."""
    return 0.5 * a * (1.0 + erf(a / SQRT2))


def gelu_prime(a: np.ndarray) -> np.ndarray:
    """d/da [a Phi(a)] = Phi(a) + a phi(a)."""
    return 0.5 * (1.0 + erf(a / SQRT2)) + a * INV_SQRT_2PI * np.exp(-0.5 * a * a)


def softmax_rows(z: np.ndarray) -> np.ndarray:
    """Row softmax with max subtraction (Eq. 5's softmax)."""
    z = z - z.max(axis=-1, keepdims=True)
    ez = np.exp(z)
    return ez / ez.sum(axis=-1, keepdims=True)


# --------------------------------------------------------------------------- #
# Gate: Eq. 6, Eq. 8, Eq. 9, Algorithm 2
# --------------------------------------------------------------------------- #
def gate_logits(x: np.ndarray, Wg: np.ndarray) -> np.ndarray:
    """L = x . W_g  (Eq. 6; W_g in R^{D x N}; no bias, R7)."""
    return x @ Wg


def gumbel_softmax(x: np.ndarray, Wg: np.ndarray, u: Optional[np.ndarray], tau: float) -> np.ndarray:
    """g'(x_s) = softmax over experts of (x_s W_g + zeta)/tau  (Eq. 8).
    Reading R1: the printed denominator's sum over s' is a softmax over the N
    experts.  Noise is added BEFORE dividing by tau, as printed (R2).  u=None
    means no noise."""
    L = gate_logits(x, Wg)
    zeta = 0.0 if u is None else gumbel_noise(u)
    return softmax_rows((L + zeta) / tau)


def argmax_lowest(p: np.ndarray) -> np.ndarray:
    """Row argmax, lowest index on ties (np.argmax returns the first maximum)."""
    return np.argmax(p, axis=1)


def threshold_select(p: np.ndarray, c: float, top1: bool = False) -> np.ndarray:
    """Expert selection mask m[T, E] (Alg. 2; Eq. 9).

    Dense branch (current_iteration < T_D): m_i = [g'_i > c]  -- strict '>' (R3),
    thresholding g' (R3), no renormalisation (R4).  If no expert passes,
    keep the argmax (Alg. 2 comment "N >= len(id_s) >= 1"; R5).
    Top-1 branch: m = onehot(argmax).

    Precision of the decision (task rule: float deciding an integer is taken in
    the kernel's precision): the comparison is made on g' rounded to fp32 against
    the fp32 value of c (R16/R18).  The argmax is taken on the fp64 g'.
    """
    T, E = p.shape
    am = argmax_lowest(p)
    if top1:
        m = np.zeros((T, E), dtype=bool)
        m[np.arange(T), am] = True
        return m
    m = p.astype(np.float32) > np.float32(c)
    empty = ~m.any(axis=1)
    m[np.where(empty)[0], am[empty]] = True
    return m


# --------------------------------------------------------------------------- #
# Expert diversify (Alg. 1 lines 4-5; Fig. P:241-247)
# --------------------------------------------------------------------------- #
def unpack_bits(words: np.ndarray, n: int) -> np.ndarray:
    """words: uint32 [..., nw]; bit (j % 32) of word j // 32 is element j."""
    words = np.asarray(words).view(np.uint32)
    j = np.arange(n)
    return ((words[..., j // 32] >> (j % 32).astype(np.uint32)) & 1).astype(bool)


def spawn(W1s, b1s, W2s, b2s, M1bits, M2bits, experts: Optional[List[int]] = None):
    """e_i <- diversify(e, i): W1_e = W1s (.) M1_e, W2_e = W2s (.) M2_e, biases copied
    unmasked (R10).  Returns dict of stacked fp64 arrays."""
    E = M1bits.shape[0]
    ids = list(range(E)) if experts is None else list(experts)
    f, d = W1s.shape
    W1 = np.stack([W1s * unpack_bits(M1bits[e], f * d).reshape(f, d) for e in ids])
    W2 = np.stack([W2s * unpack_bits(M2bits[e], d * f).reshape(d, f) for e in ids])
    b1 = np.stack([b1s.copy() for _ in ids])
    b2 = np.stack([b2s.copy() for _ in ids])
    return {"W1": W1, "b1": b1, "W2": W2, "b2": b2}


# --------------------------------------------------------------------------- #
# Dispatch layout (step 4): expert-major, stable, 128-row aligned
# --------------------------------------------------------------------------- #
def dispatch_layout(m: np.ndarray, align: int = 128):
    """Stable permute rule (R15): rows of expert e are offset_e + rank of s among
    tokens selecting e in ascending s; segments start on multiples of `align`.
    Returns (counts[E], offsets[E+1], slot[T,E] (-1 = not selected), row_token[R_pad])."""
    T, E = m.shape
    counts = m.sum(axis=0).astype(np.int64)
    padded = ((counts + align - 1) // align) * align
    offsets = np.concatenate([[0], np.cumsum(padded)]).astype(np.int64)
    slot = np.full((T, E), -1, dtype=np.int64)
    row_token = np.full(int(offsets[-1]), -1, dtype=np.int64)
    for e in range(E):
        toks = np.nonzero(m[:, e])[0]
        rows = offsets[e] + np.arange(len(toks))
        slot[toks, e] = rows
        row_token[rows] = toks
    return counts, offsets, slot, row_token


# --------------------------------------------------------------------------- #
# Layer forward / backward (Alg. 1 lines 7-12; Eq. 7)
# --------------------------------------------------------------------------- #
@dataclass
class Forward:
    x: np.ndarray
    Wg: np.ndarray
    tau: float
    p: np.ndarray               # g' [T, E]
    m: np.ndarray               # selection mask [T, E]
    G: np.ndarray               # combine weights [T, E] (p where selected, else 0)
    counts: np.ndarray          # [E]
    experts: Dict[str, np.ndarray]
    a: Dict[int, np.ndarray] = field(default_factory=dict)   # per expert, rows = tokens ascending
    h: Dict[int, np.ndarray] = field(default_factory=dict)
    o: Dict[int, np.ndarray] = field(default_factory=dict)
    toks: Dict[int, np.ndarray] = field(default_factory=dict)
    y: Optional[np.ndarray] = None


def forward(x, Wg, u, tau, c, experts, top1: bool = False,
            mask_override: Optional[np.ndarray] = None) -> Forward:
    """One DTS-Gate MoE layer forward.  x [T, d]; Wg [d, E]; u [T, E] or None;
    experts = spawn(...) output (E experts).  tau and c must already be the fp32
    values the GPU receives (as Python floats)."""
    p = gumbel_softmax(x, Wg, u, tau)                               # Alg. 2 line 2
    m = threshold_select(p, c, top1) if mask_override is None else mask_override.astype(bool)
    G = np.where(m, p, 0.0)                                          # Alg. 2 lines 9-12
    fw = Forward(x=x, Wg=Wg, tau=tau, p=p, m=m, G=G, counts=m.sum(axis=0), experts=experts)
    T, d = x.shape
    y = np.zeros((T, d))
    E = Wg.shape[1]
    for e in range(E):                                               # ascending e (R14)
        toks = np.nonzero(m[:, e])[0]
        xe = x[toks]
        a = xe @ experts["W1"][e].T + experts["b1"][e]               # Eq. 3, W1 x + b1
        h = gelu(a)
        o = h @ experts["W2"][e].T + experts["b2"][e]                # W2 h + b2
        fw.a[e], fw.h[e], fw.o[e], fw.toks[e] = a, h, o, toks
        y[toks] += G[toks, e][:, None] * o                           # Alg. 1 line 11 / Eq. 7
    fw.y = y
    return fw


@dataclass
class Backward:
    dx: np.ndarray
    dWg: np.ndarray
    dW1: np.ndarray
    db1: np.ndarray
    dW2: np.ndarray
    db2: np.ndarray
    dG: np.ndarray                       # [T, E], 0 where not selected
    dlogits: np.ndarray                  # [T, E]
    do: Dict[int, np.ndarray] = field(default_factory=dict)
    da: Dict[int, np.ndarray] = field(default_factory=dict)
    dxe: Dict[int, np.ndarray] = field(default_factory=dict)   # per-row dx contributions


def backward(fw: Forward, dy: np.ndarray, balance_alpha: float = 0.0) -> Backward:
    """Chain rule of Eq. 7 / Eq. 3 / Eq. 8 (the paper prints no backward).
    The mask m is a constant (no gradient through selection, u or tau).
    Non-selected experts still receive dz != 0 through the dense softmax.
    If balance_alpha > 0 the balance-loss gradient (Eq. 10) is added to dp."""
    x, p, m, G, ex = fw.x, fw.p, fw.m, fw.G, fw.experts
    T, d = x.shape
    E = p.shape[1]
    f = ex["W1"].shape[1]
    dx = np.zeros((T, d))
    dG = np.zeros((T, E))
    dW1 = np.zeros((E, f, d)); db1 = np.zeros((E, f))
    dW2 = np.zeros((E, d, f)); db2 = np.zeros((E, d))
    bw = Backward(dx, None, dW1, db1, dW2, db2, dG, None)
    for e in range(E):
        toks = fw.toks[e]
        o, h, a = fw.o[e], fw.h[e], fw.a[e]
        dye = dy[toks]
        dG[toks, e] = np.sum(dye * o, axis=1)                        # d y / d G = o
        do = G[toks, e][:, None] * dye                               # d y / d o = G
        dW2[e] = do.T @ h
        db2[e] = do.sum(axis=0)
        dh = do @ ex["W2"][e]
        da = dh * gelu_prime(a)
        dW1[e] = da.T @ x[toks]
        db1[e] = da.sum(axis=0)
        dxe = da @ ex["W1"][e]
        dx[toks] += dxe
        bw.do[e], bw.da[e], bw.dxe[e] = do, da, dxe
    dp = m * dG
    if balance_alpha > 0.0:
        dp = dp + balance_loss_grad_p(m, balance_alpha)[None, :]
    dz = p * (dp - np.sum(p * dp, axis=1, keepdims=True))           # softmax Jacobian
    dL = dz / fw.tau
    bw.dWg = x.T @ dL
    bw.dlogits = dL
    dx += dL @ fw.Wg.T
    bw.dx = dx
    return bw


# --------------------------------------------------------------------------- #
# Row-layout views (for comparing the GPU's permuted buffers)
# --------------------------------------------------------------------------- #
def to_rows(per_expert: Dict[int, np.ndarray], offsets: np.ndarray, width: int) -> np.ndarray:
    """Place per-expert row blocks into the expert-major padded layout; pad rows are NaN
    (they are excluded from comparisons)."""
    R = int(offsets[-1])
    out = np.full((R, width), np.nan)
    for e, blk in per_expert.items():
        out[offsets[e]:offsets[e] + blk.shape[0]] = blk
    return out


# --------------------------------------------------------------------------- #
# NEXT #1: balance loss, Eq. 10
# --------------------------------------------------------------------------- #
def balance_loss(p: np.ndarray, m: np.ndarray, alpha: float) -> float:
    """L = alpha N sum_i (count_i / |B|^2) sum_s g'_{s,i};  count_i = #{s : g(x_s)_i > 0}."""
    B, N = p.shape
    count = m.sum(axis=0).astype(np.float64)
    return float(alpha * N * np.sum(count / B ** 2 * p.sum(axis=0)))


def balance_loss_grad_p(m: np.ndarray, alpha: float) -> np.ndarray:
    """dL/dg'_{s,i} = alpha N count_i / |B|^2 (the count factor is an indicator: constant)."""
    B, N = m.shape
    return alpha * N * m.sum(axis=0).astype(np.float64) / B ** 2


# --------------------------------------------------------------------------- #
# NEXT #2: temperature scheduler
# --------------------------------------------------------------------------- #
def temperature_at(it: int, max_temp: float = 2.0, min_temp: float = 0.3,
                   decay_iters: int = 15000, shape: str = "linear") -> float:
    """tau decays from max_temp to min_temp over decay_iters, constant after (P:535,
    'annealing temperature from 2.0 to 0.3'; P:708 '15000 iterations')."""
    if decay_iters <= 0 or it >= decay_iters:
        return min_temp
    f = it / decay_iters
    if shape == "linear":
        return max_temp - (max_temp - min_temp) * f
    return max_temp * (min_temp / max_temp) ** f
