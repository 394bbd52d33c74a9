"""One rank of a real multi-process expert-parallel run (test infrastructure): launched by
tests/test_gpu_ep_multiproc.py through torch.distributed.run, one process per GPU, NCCL.

    python -m torch.distributed.run --nproc-per-node W tests/_ep_mp_worker.py MODE CONFIG T OUT_DIR

MODE: "nccl" (DTSMoELayer with the NCCL grouped send/recv exchange), "nccl-hier" (the same with
the hierarchical exchange over two virtual nodes of W/2 GPUs), "p2p" / "p2p-dedup" (EP2Rank
over torch symmetric memory: NVLink peer loads / stores; the step is also captured as a CUDA graph
and replayed, and the replay must equal the eager step bit for bit).  Each rank saves its tokens'
outputs and its experts' gradients to OUT_DIR/rank{r}.pt for the parent to compare with the oracle.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from harness import configs, inputs  # noqa: E402


def main():
    mode, cfg_name, T, out = sys.argv[1], sys.argv[2], int(sys.argv[3]), sys.argv[4]
    rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    from paper_2112_14397_b200.layer import DTSMoELayer, make_nccl_comm
    cfg = configs.get(cfg_name)
    li = inputs.make_inputs(cfg, rank=rank, T=T)
    tau, c = float(np.float32(cfg.tau)), float(np.float32(cfg.threshold))
    dt = inputs.TORCH_DTYPE[cfg.dtype]
    comm = make_nccl_comm(rank, world)
    x, u, dy = li.x.to(dev), li.u.to(dev), li.dy.to(dev)
    res = {}
    if mode in ("nccl", "nccl-hier"):
        # nccl-hier: NEXT #4, the topology-aware hierarchical exchange with the ranks split into
        # two virtual nodes of world/2 GPUs; results must equal the flat exchange's
        layer = DTSMoELayer(T, cfg.d_model, cfg.d_ff, cfg.E, dtype=dt, device=dev, rank=rank, world=world,
                            nccl_comm=comm, gpus_per_node=world // 2 if mode == "nccl-hier" else None)
        layer.set_gate(li.Wg.to(dev))
        layer.spawn(*(t.to(dev) for t in (li.W1s, li.b1s, li.W2s, li.b2s, li.M1bits, li.M2bits)))
        y = layer.forward(x, u, tau, c, top1=cfg.top1)
        g = layer.backward(dy)
        torch.cuda.synchronize()
        layer.check()
        st = layer.state
        res.update(probs=st.probs, slot=st.slot, y=y, **{k: g[k] for k in ("dx", "dlogits", "dW1", "db1", "dW2",
                                                                             "db2", "dWg")})
    else:
        from paper_2112_14397_b200.ep2 import EP2Rank, SymmetricBuffers
        syms = SymmetricBuffers(world, dev, mode="symm_mem", group=dist.group.WORLD)
        r = EP2Rank(T, cfg.d_model, cfg.d_ff, cfg.E, dt, dev, rank, world, syms, comm=comm, dedup=mode == "p2p-dedup")
        r.set_gate(li.Wg.to(dev))
        r.spawn(*(t.to(dev) for t in (li.W1s, li.b1s, li.W2s, li.b2s, li.M1bits, li.M2bits)))
        y, g = r.step(x, u, dy, tau, c, top1=cfg.top1)
        torch.cuda.synchronize()
        res.update(probs=r.st["probs"], slot=r.st["slot"], y=y, **{k: g[k] for k in ("dx", "dlogits", "dW1", "db1",
                                                                                       "dW2", "db2", "dWg")})
        res = {k: v.clone() for k, v in res.items()}
        # the same step captured as one CUDA graph (static capacity, no host sync) and replayed
        r.prepare()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            r.forward(x, u, tau, c, cfg.top1)
            r.backward(dy)
        torch.cuda.current_stream().wait_stream(s)
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            y1 = r.forward(x, u, tau, c, cfg.top1)
            g1 = r.backward(dy)
        same = True
        for _ in range(2):
            graph.replay()
            torch.cuda.synchronize()
            r.check()
            same &= bool(torch.equal(y1, res["y"]))
            for k in ("dx", "dlogits", "dW1", "dW2", "db1", "db2", "dWg"):
                same &= bool(torch.equal(g1[k], res[k]))
        res["graph_replay_identical"] = torch.tensor([int(same)])
        res["grows"] = torch.tensor([r.grows])
    torch.save({k: v.detach().cpu() for k, v in res.items()}, os.path.join(out, f"rank{rank}.pt"))
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
