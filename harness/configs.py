"""Workload configurations C1-C5, verbatim from BASELINE.json `configs` (BJ:7-11).

This module is shared by the tests, bench.py and the oracle's callers.  It holds
*workload definitions only* (shapes, distributions, seeds, the C5 schedule as a
list of (tau, c) pairs) -- none of the method's arithmetic.

Every sigma is a standard deviation.  Readings:
  * BASELINE writes W_g ~ N(0, v); v is read as a VARIANCE, so sigma_g = sqrt(v).
  * "FFN weights ~ N(0, 0.02)" is read as sigma = 0.02 (GPT-2/FairSeq convention).
  * Biases are not specified; builder's choice sigma_b = 0.02 (nonzero so the bias
    paths are exercised).
  * C3/C4/C5 leave some distributions unstated; the C2 defaults are used and marked
    `builder_default`.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field, replace
from typing import Tuple

BASE_SEED = 2112


@dataclass(frozen=True)
class MoEConfig:
    name: str
    T: int                 # tokens per GPU
    d_model: int
    d_ff: int
    E: int                 # global number of experts
    dtype: str             # "f32" or "bf16" (activation / weight storage dtype)
    tau: float
    threshold: float
    x_std: float = 1.0
    wg_std: float = 0.0
    ffn_std: float = 0.02
    bias_std: float = 0.02
    keep_prob: float = 0.8
    top1: bool = False
    # C5: per-step (tau, c) pairs; empty for single-point configs
    schedule: Tuple[Tuple[float, float], ...] = field(default_factory=tuple)
    notes: str = ""

    def with_T(self, T: int) -> "MoEConfig":
        return replace(self, T=T, name=f"{self.name}[T={T}]")

    def at_step(self, s: int) -> "MoEConfig":
        if not self.schedule:
            return self
        tau, c = self.schedule[s]
        return replace(self, tau=tau, threshold=c, name=f"{self.name}[s={s}]")


def c5_schedule(steps: int = 20, tau0: float = 2.0, tau1: float = 0.05,
                c0: float = 0.0, c1: float = 0.3) -> Tuple[Tuple[float, float], ...]:
    """BJ:11: tau annealed geometrically 2.0 -> 0.05 and threshold linearly 0.0 -> 0.3
    over 20 steps; 'over 20 steps' read as inclusive endpoints."""
    out = []
    for s in range(steps):
        f = s / (steps - 1)
        out.append((tau0 * (tau1 / tau0) ** f, c0 + (c1 - c0) * f))
    return tuple(out)


C1 = MoEConfig("C1", T=256, d_model=64, d_ff=256, E=4, dtype="f32", tau=1.0, threshold=0.1,
               wg_std=math.sqrt(1.0 / 64), notes="BJ:7 tiny fp32 correctness config")
C2 = MoEConfig("C2", T=8 * 1024, d_model=768, d_ff=3072, E=16, dtype="bf16", tau=2.0,
               threshold=0.001, wg_std=math.sqrt(1.0 / 768),
               notes="BJ:8 GPT-small-shaped, near-dense routing")
C3 = MoEConfig("C3", T=32 * 512, d_model=768, d_ff=3072, E=32, dtype="bf16", tau=0.5,
               threshold=0.05, wg_std=math.sqrt(1.0 / 768),
               notes="BJ:9 RoBERTa-base-shaped; distributions builder_default (C2's)")
C4 = MoEConfig("C4", T=64 * 2048, d_model=1024, d_ff=4096, E=64, dtype="bf16", tau=0.1,
               threshold=0.2, wg_std=math.sqrt(4.0 / 1024),
               notes="BJ:10 large layer, sparse end; x/FFN distributions builder_default")
C5 = MoEConfig("C5", T=16384, d_model=512, d_ff=2048, E=32, dtype="bf16", tau=2.0,
               threshold=0.0, wg_std=math.sqrt(1.0 / 512), schedule=c5_schedule(),
               notes="BJ:11 dense-to-sparse sweep; distributions builder_default")

CONFIGS = {c.name: c for c in (C1, C2, C3, C4, C5)}


def get(name: str) -> MoEConfig:
    return CONFIGS[name]
