"""NEXT #4: topology-aware hierarchical all-to-all on the CPU.

* Cost-model identities of the plan (host-only C ABI, virtual topologies, no GPU): for
  2 nodes x 8 GPUs with a uniform payload per GPU pair, the flat exchange has 64 inter-node
  (src, dst) GPU pairs per ordered node pair and the hierarchical one exactly 1 message of
  64x the size (the paper's "#GPU^2 times larger" message, SPEC ep-sim); inter-node and
  total rows are conserved.
* Data movement (gloo, world 4 = 2 nodes x 2 and world 8 = 4 nodes x 2, where every relay
  serves two remote nodes): the three phases, posted in exactly the NCCL order the library
  uses (`moe_ep_hier_chunks`), deliver the same expert-side layout as the flat exchange, and
  the reversed phases (combine) return the same token-side layout.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2112_14397_b200 import _lib as L


# ------------------------------------------------------------------ cost model (no comm)
def _uniform(world, E, b):
    return np.full((world, E), b, np.int32)


@pytest.mark.parametrize("E", [16, 32])
def test_two_nodes_of_eight_gpus_aggregate_64_to_1(E):
    b = 3                                   # rows per (source GPU, expert)
    counts = _uniform(16, E, b)
    st = L.moe_ep_topology_stats(16, 8, E, counts)
    El = E // 16
    pair_rows = b * El                      # payload of one (src GPU, dst GPU) pair
    assert st["node_pairs"] == 2
    assert st["flat_inter_pairs"] == 2 * 64                     # G^2 pairs per ordered node pair
    assert st["hier_inter_msgs"] == 2                           # one message per ordered node pair
    assert st["flat_inter_pairs"] // st["hier_inter_msgs"] == 64
    assert st["hier_max_msg_rows"] == 64 * pair_rows            # "#GPU^2 times larger"
    assert st["hier_inter_rows"] == st["flat_inter_rows"] == 2 * 64 * pair_rows
    total = int(counts.sum())
    assert st["flat_inter_rows"] + st["flat_intra_rows"] == total


def test_single_node_is_flat():
    counts = _uniform(8, 16, 5)
    st = L.moe_ep_topology_stats(8, 8, 16, counts)
    assert st["flat_inter_pairs"] == 0 and st["hier_inter_msgs"] == 0 and st["node_pairs"] == 0


@pytest.mark.parametrize("world,G", [(16, 8), (16, 4), (8, 2), (32, 8)])
def test_conservation_random_routing(world, G):
    rng = np.random.default_rng(world * 100 + G)
    E = world * 2
    counts = rng.integers(0, 40, size=(world, E)).astype(np.int32)
    counts[rng.random((world, E)) < 0.2] = 0               # some empty (source, expert) pairs
    st = L.moe_ep_topology_stats(world, G, E, counts)
    N = world // G
    assert st["hier_inter_rows"] == st["flat_inter_rows"]
    assert st["hier_inter_msgs"] == st["node_pairs"] <= N * (N - 1)
    assert st["flat_inter_pairs"] >= st["hier_inter_msgs"]
    # every inter-node row crosses the node boundary once, and moves intra-node at most twice
    # (gather to the relay, scatter from the relay); same-node rows move once
    assert st["hier_intra_rows"] <= st["flat_intra_rows"] + 2 * st["flat_inter_rows"]


# ------------------------------------------------------------------ data movement (gloo)
def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _post(bufs, sends, recvs):
    """One NCCL group: post every send/recv (peer, buf, row, n), self messages matched in
    posting order, then wait."""
    me = dist.get_rank()
    self_s = [(b, r, n) for p, b, r, n in sends if p == me]
    self_r = [(b, r, n) for p, b, r, n in recvs if p == me]
    assert [n for *_, n in self_s] == [n for *_, n in self_r]
    staged = [bufs[b][r:r + n].clone() for b, r, n in self_s]
    reqs, tmp = [], []
    for p, b, r, n in sends:
        if p != me:
            reqs.append(dist.isend(bufs[b][r:r + n].contiguous(), p))
    for p, b, r, n in recvs:
        if p == me:
            continue
        t = torch.empty((n,) + tuple(bufs[b].shape[1:]), dtype=bufs[b].dtype)
        tmp.append((b, r, n, t))
        reqs.append(dist.irecv(t, p))
    for q in reqs:
        q.wait()
    for (b, r, n), t in zip(self_r, staged):
        bufs[b][r:r + n] = t
    for b, r, n, t in tmp:
        bufs[b][r:r + n] = t


def _worker(rank, world, G, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        E, T, d = 2 * world, 64, 8
        El = E // world
        rng = np.random.default_rng(7)
        counts_all = rng.integers(0, 9, size=(world, E)).astype(np.int32)
        counts_all[rng.random((world, E)) < 0.25] = 0
        ctx = L.moe_create(T, 64, 64, E, L.MOE_F32, nccl_comm=1, rank=rank, world=world)
        L.moe_ep_set_topology(ctx, G)
        off_send, off_recv, R_send, R_recv = L.moe_ep_plan(ctx, counts_all, E, El)
        stage_rows = L.moe_ep_stage_rows(ctx)
        phases = [(L.moe_ep_hier_chunks(ctx, ph, False), L.moe_ep_hier_chunks(ctx, ph, True)) for ph in range(3)]
        flat_s, flat_r = L.moe_ep_plan_chunks(ctx, 0), L.moe_ep_plan_chunks(ctx, 1)
        # token-side rows: value encodes (source rank, expert, index) so every row is distinct
        send = torch.zeros(R_send, d, dtype=torch.float64)
        for e in range(E):
            for i in range(int(counts_all[rank, e])):
                send[off_send[e] + i] = torch.tensor([rank, e, i, 1.0, rank * 1000 + e, i * 7.0, -1.0, 2.0])
        stage = torch.zeros(max(stage_rows, 1), d, dtype=torch.float64)
        # stage buffer 3 starts after the gather stage: split the caller's buffer like the library
        out_rows = max([r + n for p, b, r, n in phases[0][1] + phases[1][0] if b == 2] + [0])
        bufs = {0: send, 1: torch.zeros(R_recv, d, dtype=torch.float64), 2: stage[:max(out_rows, 0)],
                3: stage[out_rows:]}
        in_rows = max([r + n for p, b, r, n in phases[1][1] + phases[2][0] if b == 3] + [0])
        assert out_rows + in_rows <= stage_rows
        for ph in range(3):                                  # dispatch
            _post(bufs, phases[ph][0], phases[ph][1])
        # reference: the flat exchange
        ref = {0: send, 1: torch.zeros(R_recv, d, dtype=torch.float64)}
        _post(ref, [(p, 0, r, n) for p, r, n in flat_s], [(p, 1, r, n) for p, r, n in flat_r])
        assert torch.equal(bufs[1], ref[1]), f"rank {rank}: hierarchical dispatch != flat"
        # combine: every message reversed, phases 2, 1, 0; the expert side sends back its rows + 1
        back = bufs[1] + 1.0
        cb = {0: torch.zeros(R_send, d, dtype=torch.float64), 1: back, 2: bufs[2], 3: bufs[3]}
        for ph in (2, 1, 0):
            _post(cb, phases[ph][1], phases[ph][0])
        rf = {0: torch.zeros(R_send, d, dtype=torch.float64), 1: back}
        _post(rf, [(p, 1, r, n) for p, r, n in flat_r], [(p, 0, r, n) for p, r, n in flat_s])
        assert torch.equal(cb[0], rf[0]), f"rank {rank}: hierarchical combine != flat"
        # inter-node phase: at most one message per (relay, partner) and only across nodes
        for p, b, r, n in phases[1][0]:
            assert p // G != rank // G and b == 2
        out[rank] = (len(phases[1][0]), stage_rows)
        L.moe_destroy(ctx)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,G", [(4, 2), (8, 2), (8, 4)])
def test_hierarchical_exchange_matches_flat(world, G):
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, G, _free_port(), out), nprocs=world, join=True)
    assert len(out) == world
    # one inter-node message per ordered node pair with payload, in total
    N = world // G
    assert sum(v[0] for v in out.values()) <= N * (N - 1)
