"""Test driver for the fused peer-memory EP ranks emulated in ONE process (test infrastructure,
not product: moved out of paper_2112_14397_b200/ep2.py).  Each phase runs
on every rank before the next phase starts -- the ordering the NCCL barriers give on a real
multi-GPU run -- and dW_g is summed over the ranks in torch, standing in for the NCCL
all-reduce (C6) of the real path."""
from typing import List

from paper_2112_14397_b200.ep2 import EP2Rank


def run_lockstep(ranks: List[EP2Rank], xs, us, dys, tau: float, threshold: float, top1: bool = False,
                 balance_alpha: float = 0.0):
    """Emulated ranks in one process: each phase runs on every rank before the next phase
    (the barriers' ordering); dW_g is summed over the ranks (the all-reduce)."""
    for r, x, u in zip(ranks, xs, us):
        r.fwd_gate(x, u, tau, threshold, top1)
    for r in ranks:
        r.fwd_plan()
    for r in ranks:
        r.fwd_dispatch()
    for r in ranks:
        if r.dedup:
            r.fwd_permute()
        r.fwd_experts()
        if r.dedup:
            r.fwd_presum()
    ys = [r.fwd_combine() for r in ranks]
    for r, dy in zip(ranks, dys):
        r.bwd_stage_dy(dy)
    for r in ranks:
        if r.dedup:
            r.bwd_gather_dy()
        r.bwd_combine()
    for r in ranks:
        r.bwd_experts()
        if r.dedup:
            r.bwd_presum()
    for r in ranks:
        r.bwd_gate(balance_alpha)
    dWg = sum(r.st["grads"]["dWg"] for r in ranks)
    grads = [r.bwd_dispatch() for r in ranks]
    return ys, grads, dWg


def check_all(ranks: List[EP2Rank]) -> List[int]:
    """moe_check on every rank; the status code of each (0 = ok)."""
    from paper_2112_14397_b200 import _lib as L
    codes = []
    for r in ranks:
        try:
            r.check()
            codes.append(0)
        except L.MoEError as e:
            codes.append(e.code)
    return codes


def run_lockstep_with_recovery(ranks: List[EP2Rank], *args, max_retries: int = 2, **kw):
    """EP2Rank.step()'s capacity policy for emulated ranks: run the step, check every rank; on
    MOE_ECAPACITY (which every rank must raise together) grow every rank and re-run.
    Returns (ys, grads, dWg, attempts)."""
    for attempt in range(max_retries + 1):
        out = run_lockstep(ranks, *args, **kw)
        codes = check_all(ranks)
        if all(c == 0 for c in codes):
            return out + (attempt,)
        assert all(c == 7 for c in codes), f"capacity overflow not raised on every rank: {codes}"
        for r in ranks:
            r.grow()
    raise AssertionError("capacity still exceeded after the retries")
