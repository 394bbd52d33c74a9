"""Expert-parallel (EP) exchange on the CPU: world_size 2 and 4 with the gloo backend.

Every rank computes its routing with the oracle, all-gathers the counts, asks the C ABI
(`moe_ep_plan`, host-only, no GPU) for the exchange plan, and moves the rows with gloo
point-to-point messages in exactly the chunk order the NCCL path posts
(`moe_ep_plan_chunks`).  The expert-side buffer must equal the single-rank layout of the
GLOBAL token set restricted to this rank's experts; running the expert FFN on it
(oracle arithmetic), exchanging back and combining must reproduce the single-process
oracle layer on the global token set -- forward and backward (dx, dW of local experts,
all-reduced dW_g).
"""
import dataclasses
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from harness import configs, inputs
from oracle import dts_moe as O

CFG = dataclasses.replace(configs.C1, name="ep-small", T=96, d_model=64, d_ff=128, E=8, tau=0.7, threshold=0.08)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _exchange(src, dst, sends, recvs):
    """Post every send/recv chunk (peer, row, nrows) like the NCCL group, then wait.
    Messages to oneself (NCCL handles them inside the group; gloo has no self pair) are
    matched in posting order and copied locally."""
    me = dist.get_rank()
    reqs, tmp = [], []
    self_src = [(row, n) for peer, row, n in sends if peer == me]
    self_dst = [(row, n) for peer, row, n in recvs if peer == me]
    assert [n for _, n in self_src] == [n for _, n in self_dst]
    for (rs, n), (rd, _) in zip(self_src, self_dst):
        dst[rd:rd + n] = src[rs:rs + n]
    for peer, row, n in sends:
        if peer != me:
            reqs.append(dist.isend(src[row:row + n].contiguous(), peer))
    for peer, row, n in recvs:
        if peer == me:
            continue
        buf = torch.empty((n,) + tuple(dst.shape[1:]), dtype=dst.dtype)
        tmp.append((row, n, buf))
        reqs.append(dist.irecv(buf, peer))
    for r in reqs:
        r.wait()
    for row, n, buf in tmp:
        dst[row:row + n] = buf


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2112_14397_b200 import _lib as L
        cfg = CFG
        T, d, f, E = cfg.T, cfg.d_model, cfg.d_ff, cfg.E
        El = E // world
        tau, c = float(np.float32(cfg.tau)), float(np.float32(cfg.threshold))
        per_rank = [inputs.make_inputs(cfg, rank=q) for q in range(world)]
        li = per_rank[rank]
        ex = O.spawn(inputs.to_f64(li.W1s), inputs.to_f64(li.b1s), inputs.to_f64(li.W2s), inputs.to_f64(li.b2s),
                     inputs.bits_u32(li.M1bits), inputs.bits_u32(li.M2bits))
        Wg = inputs.to_f64(li.Wg)
        x, u, dy = (inputs.to_f64(t) for t in (li.x, li.u, li.dy))
        # ---- local routing (oracle), counts all-gather
        p = O.gumbel_softmax(x, Wg, u, tau)
        m = O.threshold_select(p, c)
        G = np.where(m, p, 0.0)
        counts = torch.from_numpy(m.sum(0).astype(np.int32))
        gathered = [torch.zeros_like(counts) for _ in range(world)]
        dist.all_gather(gathered, counts)
        counts_all = torch.stack(gathered).numpy()
        # ---- plan from the C ABI (host-only)
        ctx = L.moe_create(T, d, f, E, L.MOE_F32, nccl_comm=1, rank=rank, world=world)
        off_send, off_recv, R_send, R_recv = L.moe_ep_plan(ctx, counts_all, E, El)
        sends, recvs = L.moe_ep_plan_chunks(ctx, 0), L.moe_ep_plan_chunks(ctx, 1)
        _, offs, slot, row_token = O.dispatch_layout(m)
        assert np.array_equal(offs, off_send) and offs[-1] == R_send
        valid = row_token >= 0
        # ---- dispatch: token side (send layout) -> expert side (recv layout)
        x_send = torch.zeros(R_send, d, dtype=torch.float64)
        x_send[torch.from_numpy(np.nonzero(valid)[0])] = torch.from_numpy(x[row_token[valid]])
        x_recv = torch.zeros(R_recv, d, dtype=torch.float64)
        _exchange(x_send, x_recv, sends, recvs)
        # expected: global token set, stable expert-major layout of my experts
        x_all = np.concatenate([inputs.to_f64(q.x) for q in per_rank])
        u_all = np.concatenate([inputs.to_f64(q.u) for q in per_rank])
        dy_all = np.concatenate([inputs.to_f64(q.dy) for q in per_rank])
        fw_all = O.forward(x_all, Wg, u_all, tau, c, ex)
        bw_all = O.backward(fw_all, dy_all)
        xr = x_recv.numpy()
        for j in range(El):
            e = rank * El + j
            toks = np.nonzero(fw_all.m[:, e])[0]
            seg = xr[off_recv[j]:off_recv[j + 1]]
            assert np.array_equal(seg[:len(toks)], x_all[toks]), f"rank {rank} expert {e} rows"
            assert not seg[len(toks):].any(), "recv pads must be zero"
        # ---- expert FFN on the recv layout (oracle arithmetic), combine exchange, combine
        e_out_recv = torch.zeros(R_recv, d, dtype=torch.float64)
        hs = {}
        for j in range(El):
            e = rank * El + j
            n = int(counts_all[:, e].sum())
            rows = xr[off_recv[j]:off_recv[j] + n]
            a = rows @ ex["W1"][e].T + ex["b1"][e]
            h = O.gelu(a)
            hs[j] = (rows, a, h)
            e_out_recv[off_recv[j]:off_recv[j] + n] = torch.from_numpy(h @ ex["W2"][e].T + ex["b2"][e])
        e_out_send = torch.zeros(R_send, d, dtype=torch.float64)
        _exchange(e_out_recv, e_out_send, recvs, sends)
        eo = e_out_send.numpy()
        y = np.zeros((T, d))
        for e in range(E):
            for t in np.nonzero(m[:, e])[0]:
                y[t] += G[t, e] * eo[slot[t, e]]
        np.testing.assert_allclose(y, fw_all.y[rank * T:(rank + 1) * T], rtol=1e-12, atol=1e-12)
        # ---- backward: d_eout to the experts, expert grads, dx_perm back, gate grads
        d_send = torch.zeros(R_send, d, dtype=torch.float64)
        dG = np.zeros((T, E))
        for e in range(E):
            for t in np.nonzero(m[:, e])[0]:
                r = slot[t, e]
                d_send[r] = torch.from_numpy(G[t, e] * dy[t])
                dG[t, e] = dy[t] @ eo[r]
        d_recv = torch.zeros(R_recv, d, dtype=torch.float64)
        _exchange(d_send, d_recv, sends, recvs)
        dxp_recv = torch.zeros(R_recv, d, dtype=torch.float64)
        dr = d_recv.numpy()
        for j in range(El):
            e = rank * El + j
            n = int(counts_all[:, e].sum())
            rows, a, h = hs[j]
            do = dr[off_recv[j]:off_recv[j] + n]
            np.testing.assert_allclose(do.T @ h, bw_all.dW2[e], rtol=1e-10, atol=1e-12)
            da = (do @ ex["W2"][e]) * O.gelu_prime(a)
            np.testing.assert_allclose(da.T @ rows, bw_all.dW1[e], rtol=1e-10, atol=1e-12)
            np.testing.assert_allclose(da.sum(0), bw_all.db1[e], rtol=1e-10, atol=1e-12)
            dxp_recv[off_recv[j]:off_recv[j] + n] = torch.from_numpy(da @ ex["W1"][e])
        dxp_send = torch.zeros(R_send, d, dtype=torch.float64)
        _exchange(dxp_recv, dxp_send, recvs, sends)
        dxs = dxp_send.numpy()
        dp = m * dG
        dL = p * (dp - np.sum(p * dp, axis=1, keepdims=True)) / tau
        dWg = torch.from_numpy(x.T @ dL)
        dist.all_reduce(dWg)
        dx = dL @ Wg.T
        for e in range(E):
            for t in np.nonzero(m[:, e])[0]:
                dx[t] += dxs[slot[t, e]]
        np.testing.assert_allclose(dx, bw_all.dx[rank * T:(rank + 1) * T], rtol=1e-10, atol=1e-12)
        np.testing.assert_allclose(dWg.numpy(), bw_all.dWg, rtol=1e-10, atol=1e-12)
        L.moe_destroy(ctx)
        out.put((rank, "ok", int(R_recv), len(sends)))
    except Exception as exc:  # pragma: no cover - reported to the parent
        import traceback
        out.put((rank, "fail", traceback.format_exc(), 0))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_ep_exchange_gloo(world):
    from paper_2112_14397_b200 import build
    build.build()
    ctx_mp = mp.get_context("spawn")
    q = ctx_mp.Queue()
    port = _free_port()
    procs = [ctx_mp.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=60)
    fails = [r for r in res if r[1] != "ok"]
    assert not fails, fails[0][2]


def test_ep_plan_single_rank_is_dispatch_layout():
    """world = 1: the plan is the identity exchange of the token-side layout."""
    from paper_2112_14397_b200 import build
    build.build()
    from paper_2112_14397_b200 import _lib as L
    rng = np.random.default_rng(0)
    m = rng.random((300, 6)) < 0.3
    counts = m.sum(0).astype(np.int32)[None, :]
    ctx = L.moe_create(300, 64, 128, 6, L.MOE_F32, nccl_comm=1, rank=0, world=1)
    os_, or_, rs, rr = L.moe_ep_plan(ctx, counts, 6, 6)
    _, offs, _, _ = O.dispatch_layout(m)
    assert np.array_equal(os_, offs) and np.array_equal(or_, offs) and rs == rr == offs[-1]
    sends, recvs = L.moe_ep_plan_chunks(ctx, 0), L.moe_ep_plan_chunks(ctx, 1)
    assert [(p, r, n) for p, r, n in sends] == [(p, r, n) for p, r, n in recvs]
    with pytest.raises(L.MoEError):
        L.moe_ep_plan(ctx, -counts, 6, 6)
    L.moe_destroy(ctx)
