"""Host-side dense-to-sparse schedule (NEXT #2; Alg. 1 line 7 'temperature scheduler',
P:348-352; endpoints P:535 'annealing temperature from 2.0 to 0.3', duration and the switch
to Top-1 P:708 'in the first 15000 iterations and switch to Top1 then').

The schedule only produces the scalars the C ABI takes (tau, threshold, top1); it runs on
the host between steps.  `c5_sweep` is BASELINE.json's C5 workload schedule (geometric tau,
linear threshold, inclusive endpoints; reading R11).
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Iterator, Tuple


@dataclass(frozen=True)
class DTSSchedule:
    max_temp: float = 2.0
    min_temp: float = 0.3
    decay_iters: int = 15000
    dense_iters: int = 15000          # T_D of Alg. 2: iterations >= T_D use the Top-1 branch
    shape: str = "linear"             # "linear" | "exp" (geometric)
    threshold: float = 0.001          # c

    def tau(self, it: int) -> float:
        if self.decay_iters <= 0 or it >= self.decay_iters:
            return self.min_temp
        f = it / self.decay_iters
        if self.shape == "linear":
            return self.max_temp - (self.max_temp - self.min_temp) * f
        return self.max_temp * (self.min_temp / self.max_temp) ** f

    def top1(self, it: int) -> bool:
        return it >= self.dense_iters

    def at(self, it: int) -> Tuple[float, float, bool]:
        """(tau, threshold, top1) for training iteration `it` (Alg. 2 inputs)."""
        return self.tau(it), self.threshold, self.top1(it)


def c5_sweep(steps: int = 20, tau0: float = 2.0, tau1: float = 0.05, c0: float = 0.0,
             c1: float = 0.3) -> Iterator[Tuple[float, float]]:
    for s in range(steps):
        f = s / (steps - 1) if steps > 1 else 0.0
        yield tau0 * (tau1 / tau0) ** f, c0 + (c1 - c0) * f
