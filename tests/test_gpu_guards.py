"""Out-of-bounds write guards for every device buffer the layer allocates.

compute-sanitizer is not available on the GPU pool, so every CUDA allocation made by
paper_2112_14397_b200.layer during a forward + backward is wrapped in 1 KiB guard zones on
both sides, pre-filled with a sentinel byte; after the step every guard must be intact.
Shapes: partial GEMM tiles and a ragged token count, every gate path (fused, unfused E % 16
!= 0, fp32 SIMT), top-1 at the C4 width, and the recomputation mode."""
import dataclasses
import math

import numpy as np
import pytest
import torch

from harness import configs, inputs

pytestmark = pytest.mark.gpu

GUARD = 1024
SENT = 0xA5


@pytest.fixture(scope="module", autouse=True)
def _built():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2112_14397_b200 import build
    build.build()


class _Guarded:
    def __init__(self):
        self.allocs = []
        self._empty, self._empty_like = torch.empty, torch.empty_like

    def empty(self, *size, dtype=None, device=None, **kw):
        if len(size) == 1 and isinstance(size[0], (tuple, list, torch.Size)):
            size = tuple(size[0])
        dev = torch.device(device) if device is not None else None
        if dev is None or dev.type != "cuda" or kw.get("pin_memory"):
            return self._empty(*size, dtype=dtype, device=device, **kw)
        dtype = dtype or torch.get_default_dtype()
        esz = torch.tensor([], dtype=dtype).element_size()
        nbytes = int(math.prod(size)) * esz
        base = self._empty(nbytes + 2 * GUARD, dtype=torch.uint8, device=dev)
        base.fill_(SENT)
        self.allocs.append((base, nbytes, tuple(size), dtype))
        return base[GUARD:GUARD + nbytes].view(dtype).view(size)

    def zeros(self, *size, dtype=None, device=None, **kw):
        t = self.empty(*size, dtype=dtype, device=device, **kw)
        return t.zero_()

    def empty_like(self, t, **kw):
        if t.is_cuda and not kw:
            return self.empty(tuple(t.shape), dtype=t.dtype, device=t.device)
        return self._empty_like(t, **kw)

    def check(self):
        torch.cuda.synchronize()
        bad = []
        for base, nbytes, size, dtype in self.allocs:
            lo, hi = base[:GUARD], base[GUARD + nbytes:]
            if bool((lo != SENT).any()) or bool((hi != SENT).any()):
                bad.append((size, dtype, int((lo != SENT).sum()), int((hi != SENT).sum())))
        assert not bad, f"guard zones overwritten (shape, dtype, bytes before, bytes after): {bad}"
        return len(self.allocs)


def _shape(name, T, d, f, E, tau, c, top1=False, dtype="bf16"):
    return dataclasses.replace(configs.C3, name=name, T=T, d_model=d, d_ff=f, E=E, tau=tau, threshold=c, top1=top1,
                               dtype=dtype, wg_std=math.sqrt(1.0 / d))


CASES = [
    ("partial_tiles_E20", _shape("g20", 777, 192, 320, 20, 0.7, 0.05), False),
    ("fused_E32", _shape("g32", 1000, 768, 3072, 32, 0.5, 0.05), False),
    ("fused_E32_recompute", _shape("g32r", 1000, 768, 3072, 32, 0.5, 0.05), True),
    ("c4_width_top1", _shape("g64", 640, 1024, 4096, 64, 0.1, 0.2, top1=True), False),
    ("simt_E80", _shape("g80", 300, 192, 320, 80, 0.8, 0.01), False),
    ("fp32_c1", configs.C1, False),
]


@pytest.mark.parametrize("name,cfg,recompute", CASES, ids=[c[0] for c in CASES])
def test_no_out_of_bounds_writes(monkeypatch, name, cfg, recompute):
    from paper_2112_14397_b200 import layer as LY
    g = _Guarded()
    monkeypatch.setattr(LY.torch, "empty", g.empty)
    monkeypatch.setattr(LY.torch, "empty_like", g.empty_like)
    li = inputs.make_inputs(cfg, T=cfg.T)
    dev = torch.device("cuda", 0)
    dt = inputs.TORCH_DTYPE[cfg.dtype]
    lay = LY.DTSMoELayer(cfg.T, cfg.d_model, cfg.d_ff, cfg.E, dtype=dt, device=dev, recompute=recompute)
    lay.set_gate(li.Wg.to(dev))
    lay.spawn(*(t.to(dev) for t in (li.W1s, li.b1s, li.W2s, li.b2s, li.M1bits, li.M2bits)))
    for _ in range(2):
        lay.forward(li.x.to(dev), li.u.to(dev), float(np.float32(cfg.tau)), float(np.float32(cfg.threshold)),
                    top1=cfg.top1)
        lay.backward(li.dy.to(dev))
    lay.check()
    n = g.check()
    assert n >= 20, n


@pytest.mark.parametrize("dedup", [False, True], ids=["ep2", "ep2_dedup"])
def test_ep2_no_out_of_bounds_writes(monkeypatch, dedup):
    # the fused peer-memory EP path, 4 emulated ranks: every rank's symmetric and local buffers
    # guarded (peer stores land in other ranks' buffers, so a bad row index shows up here)
    from paper_2112_14397_b200.ep2 import EP2Rank, SymmetricBuffers
    from _ep_lockstep import run_lockstep
    g = _Guarded()
    monkeypatch.setattr(torch, "empty", g.empty)
    monkeypatch.setattr(torch, "zeros", g.zeros)
    monkeypatch.setattr(torch, "empty_like", g.empty_like)
    cfg, W, T = _shape("gep", 300, 192, 320, 16, 0.7, 0.05), 4, 300
    dev = torch.device("cuda", 0)
    ranks_in = [inputs.make_inputs(cfg, rank=q, T=T) for q in range(W)]
    li0 = ranks_in[0]
    syms = SymmetricBuffers(W, dev)
    ranks = []
    for q in range(W):
        r = EP2Rank(T, cfg.d_model, cfg.d_ff, cfg.E, torch.bfloat16, dev, q, W, syms, dedup=dedup)
        r.set_gate(li0.Wg.to(dev))
        r.spawn(*(t.to(dev) for t in (li0.W1s, li0.b1s, li0.W2s, li0.b2s, li0.M1bits, li0.M2bits)))
        ranks.append(r)
    for _ in range(2):
        run_lockstep(ranks, [ri.x.to(dev) for ri in ranks_in], [ri.u.to(dev) for ri in ranks_in],
                     [ri.dy.to(dev) for ri in ranks_in], float(np.float32(cfg.tau)), float(np.float32(cfg.threshold)))
    for r in ranks:
        r.check()
    assert g.check() >= 40


@pytest.mark.parametrize("name,cfg,recompute", CASES, ids=[c[0] for c in CASES])
def test_no_reads_of_unwritten_memory(monkeypatch, name, cfg, recompute):
    # every new float CUDA buffer NaN-filled (ints -1): a step must give bit-identical results
    # to a step on zero-filled buffers, i.e. no kernel reads a value nobody wrote
    from paper_2112_14397_b200 import layer as LY
    real = torch.empty
    li = inputs.make_inputs(cfg, T=cfg.T)
    dev = torch.device("cuda", 0)
    dt = inputs.TORCH_DTYPE[cfg.dtype]
    outs = []
    for poison in (False, True):
        def empty(*size, dtype=None, device=None, **kw):
            t = real(*size, dtype=dtype, device=device, **kw)
            if t.is_cuda:
                t.fill_(float("nan") if poison and t.is_floating_point() else (-1 if poison else 0))
            return t
        monkeypatch.setattr(LY.torch, "empty", empty)
        lay = LY.DTSMoELayer(cfg.T, cfg.d_model, cfg.d_ff, cfg.E, dtype=dt, device=dev, recompute=recompute)
        lay.set_gate(li.Wg.to(dev))
        lay.spawn(*(t.to(dev) for t in (li.W1s, li.b1s, li.W2s, li.b2s, li.M1bits, li.M2bits)))
        y = lay.forward(li.x.to(dev), li.u.to(dev), float(np.float32(cfg.tau)), float(np.float32(cfg.threshold)),
                        top1=cfg.top1)
        g = lay.backward(li.dy.to(dev))
        torch.cuda.synchronize()
        lay.check()
        outs.append((y.clone(), {k: v.clone() for k, v in g.items() if k != "da"}))
        monkeypatch.setattr(LY.torch, "empty", real)
    assert torch.equal(outs[0][0], outs[1][0])
    for k in outs[0][1]:
        assert torch.equal(outs[0][1][k], outs[1][1][k]), k
