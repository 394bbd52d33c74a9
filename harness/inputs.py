"""Seeded synthetic inputs shared by the CUDA path and the oracle.

Holds NONE of the method's arithmetic: it only draws random numbers with
torch.Generator on the CPU, rounds them to the storage dtype and packs the
diversify masks into bit words.  Both sides receive identical bits; the oracle
converts them exactly to float64.

Seed offsets: x +1 (+1000*rank), W_g +2, shared expert +3,
masks +4, u +5 (+step), dy +6.

The uniform u fed to the Gumbel transform is k * 2^-24 with k ~ U{1, ..., 2^24-1},
which is exactly representable in fp32 and lies strictly inside (0, 1).
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Optional

import numpy as np
import torch

from .configs import BASE_SEED, MoEConfig

TORCH_DTYPE = {"f32": torch.float32, "bf16": torch.bfloat16}


def _gen(offset: int) -> torch.Generator:
    g = torch.Generator(device="cpu")
    g.manual_seed(BASE_SEED + offset)
    return g


def _randn(shape, std: float, offset: int, dtype: torch.dtype) -> torch.Tensor:
    t = torch.randn(*shape, generator=_gen(offset), dtype=torch.float32)
    if std != 1.0:
        t.mul_(std)
    return t.to(dtype)


def pack_bits(keep: np.ndarray) -> np.ndarray:
    """Pack a boolean array [E, n] into uint32 words [E, ceil(n/32)]:
    bit (j % 32) of word j // 32 is element j (1 = keep)."""
    E, n = keep.shape
    nw = (n + 31) // 32
    padded = np.zeros((E, nw * 32), dtype=np.uint8)
    padded[:, :n] = keep
    by = np.packbits(padded, axis=1, bitorder="little")          # [E, nw*4] bytes
    return np.ascontiguousarray(by).view("<u4").reshape(E, nw)


def mask_bits(cfg: MoEConfig, n_elems: int, which: int) -> torch.Tensor:
    """Bernoulli(keep_prob) masks for all E experts, packed; `which` = 1 (W1) or 2 (W2)."""
    g = _gen(4 + 100 * which)
    # generate in chunks to bound peak memory at the largest config
    E = cfg.E
    words = (n_elems + 31) // 32
    out = np.empty((E, words), dtype=np.uint32)
    for e in range(E):
        r = torch.rand(n_elems, generator=g) < cfg.keep_prob
        out[e] = pack_bits(r.numpy()[None, :])[0]
    return torch.from_numpy(out.view(np.int32))


def uniform_u(T: int, E: int, step: int = 0, rank: int = 0) -> torch.Tensor:
    g = _gen(5 + step + 1000 * rank)
    k = torch.randint(1, 1 << 24, (T, E), generator=g, dtype=torch.int64)
    return (k.to(torch.float64) * 2.0 ** -24).to(torch.float32)


@dataclass
class LayerInputs:
    cfg: MoEConfig
    x: torch.Tensor          # [T, d]          storage dtype
    Wg: torch.Tensor         # [d, E]          storage dtype
    W1s: torch.Tensor        # [d_ff, d]       shared expert (nn.Linear [out, in])
    b1s: torch.Tensor        # [d_ff]
    W2s: torch.Tensor        # [d, d_ff]
    b2s: torch.Tensor        # [d]
    M1bits: torch.Tensor     # [E, ceil(d_ff*d/32)] int32 bit words (uint32 semantics)
    M2bits: torch.Tensor     # [E, ceil(d*d_ff/32)]
    u: Optional[torch.Tensor]  # [T, E] fp32 in (0,1)
    dy: torch.Tensor         # [T, d]          storage dtype


def make_inputs(cfg: MoEConfig, step: int = 0, rank: int = 0, with_noise: bool = True,
                T: Optional[int] = None) -> LayerInputs:
    T = cfg.T if T is None else T
    d, f, E = cfg.d_model, cfg.d_ff, cfg.E
    dt = TORCH_DTYPE[cfg.dtype]
    x = _randn((T, d), cfg.x_std, 1 + 1000 * rank, dt)
    Wg = _randn((d, E), cfg.wg_std, 2, dt)
    g3 = _gen(3)
    W1s = (torch.randn(f, d, generator=g3) * cfg.ffn_std).to(dt)
    b1s = (torch.randn(f, generator=g3) * cfg.bias_std).to(dt)
    W2s = (torch.randn(d, f, generator=g3) * cfg.ffn_std).to(dt)
    b2s = (torch.randn(d, generator=g3) * cfg.bias_std).to(dt)
    M1 = mask_bits(cfg, f * d, 1)
    M2 = mask_bits(cfg, d * f, 2)
    u = uniform_u(T, E, step, rank) if with_noise else None
    dy = _randn((T, d), 1.0, 6 + 1000 * rank, dt)
    return LayerInputs(cfg, x, Wg, W1s, b1s, W2s, b2s, M1, M2, u, dy)


def to_f64(t: Optional[torch.Tensor]) -> Optional[np.ndarray]:
    """Exact conversion of a storage-dtype tensor to float64 NumPy."""
    if t is None:
        return None
    return t.to(torch.float64).numpy()


def bits_u32(t: torch.Tensor) -> np.ndarray:
    return t.numpy().view(np.uint32)
