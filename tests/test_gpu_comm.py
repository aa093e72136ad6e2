"""Multi-rank paths on ONE GPU: two processes share cuda:0 and talk through the
peer-memory communicator (CUDA IPC mapping of each other's mailbox, the same
mechanism NVLink peers use on an 8xB200 box).  Checks:
  * all-reduce: bit-identical sums in fixed rank order on both ranks;
  * pipeline hand-off: send/recv round trips;
  * if_run_stack by_tensor (TP=2) and by_layer (PP=2) == the oracle's stack.
Handles are exchanged with torch.distributed (gloo) all_gather_object.
"""
import os
import socket

import numpy as np
import pytest

from gpu_util import torch

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, mode, q):
    try:
        import sys
        sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
        import torch
        import torch.distributed as dist

        import oracle as O
        import paper_2401_08294_b200 as F
        import synth
        from paper_2401_08294_b200.model import Stack, deinterleave_rows

        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        dev = torch.device("cuda:0")
        torch.cuda.set_device(dev)
        cfg = dict(layers=2, hidden=512, heads=8, kv_heads=2, head_dim=64, ffn=1408)
        s = F.scheme(35, 64)
        shape = F.stack_shape(*[cfg[k] for k in ("layers", "hidden", "heads", "kv_heads", "head_dim", "ffn")], s)
        res = {}
        if mode == "collectives":
            plan = F.if_plan_partition(F.IF_BY_TENSOR, shape, world)
            comm = F.Comm(plan, rank, 64, cfg["hidden"])
            comm.exchange()
            for it in range(3):
                buf = torch.arange(1000, device=dev, dtype=torch.float32) * (rank + 1) + it
                comm.allreduce(buf)
                torch.cuda.synchronize()
                ref = torch.arange(1000, dtype=torch.float32) * sum(r + 1 for r in range(world)) + world * it
                res[f"ar{it}"] = bool(torch.equal(buf.cpu(), ref))
            comm.destroy()
            plan = F.if_plan_partition(F.IF_BY_LAYER, shape, world)
            comm = F.Comm(plan, rank, 64, cfg["hidden"])
            comm.exchange()
            for it in range(3):
                buf = torch.full((777,), float(it * 10 + 1), device=dev)
                if rank == 0:
                    comm.send_next(buf)
                else:
                    out = torch.zeros(777, device=dev)
                    comm.recv_prev(out)
                    torch.cuda.synchronize()
                    res[f"p2p{it}"] = bool(torch.all(out == it * 10 + 1).item())
            torch.cuda.synchronize()
            comm.destroy()
        else:
            if mode.startswith("hybrid"):
                # Table 4: 2 pipeline stages x 2 tensor-parallel ranks
                plan = F.if_plan_partition(F.IF_HYBRID, shape, world, 2, world // 2)
            else:
                strategy = F.IF_BY_TENSOR if mode == "tp" else F.IF_BY_LAYER
                plan = F.if_plan_partition(strategy, shape, world)
            stk = Stack(cfg, s, plan, rank, dev)
            comm = F.Comm(plan, rank, 8, cfg["hidden"])
            comm.exchange()
            T = 1 if mode in ("pp1", "hybrid1") else 2  # pp T = 1: each stage through the persistent engine
            h = synth.activations(T, cfg["hidden"], tid=5)
            hd = torch.from_numpy(h).to(dev)
            out = torch.zeros_like(hd)
            ws = torch.zeros(F.if_stack_workspace_bytes(shape, plan, rank, T, F.IF_DECODE), dtype=torch.uint8,
                             device=dev)
            F.if_run_stack(shape, plan, rank, comm, stk.arr, hd, T, F.IF_DECODE, out, None, ws)
            torch.cuda.synchronize()
            comm.destroy()
            last = plan.a[rank].stage == plan.stages - 1
            if last:
                # oracle: full stack from the host generator (independent of the GPU shards)
                d, H, G, hd_, Fd = cfg["hidden"], cfg["heads"], cfg["kv_heads"], cfg["head_dim"], cfg["ffn"]
                wq, wo, wgu, wdn = [], [], [], []
                for l in range(cfg["layers"]):
                    wq.append(O.quantize(35, 64, np.concatenate([synth.weight(l, "q", H * hd_, d, d),
                                                                 synth.weight(l, "k", G * hd_, d, d),
                                                                 synth.weight(l, "v", G * hd_, d, d)])))
                    wo.append(O.quantize(35, 64, synth.weight(l, "o", d, H * hd_, d)))
                    wgu.append(O.quantize(35, 64, np.concatenate([synth.weight(l, "gate", Fd, d, d),
                                                                  synth.weight(l, "up", Fd, d, d)])))
                    wdn.append(O.quantize(35, 64, synth.weight(l, "down", d, Fd, d)))
                ho, _ = O.stack_f64(dict(cfg, qtype=35, block=64), wq, wo, wgu, wdn, h)
                o = out.cpu().numpy().astype(np.float64)
                res["err"] = float(np.abs(o - ho).max() / np.abs(ho).max())
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, res))
    except Exception as e:  # pragma: no cover - reported to the parent
        import traceback
        q.put((rank, {"error": traceback.format_exc()}))


def _run(mode, world=2, timeout=240):
    import torch.multiprocessing as mp
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, mode, q)) for r in range(world)]
    for p in ps:
        p.start()
    out = {}
    try:
        for _ in range(world):
            r, res = q.get(timeout=timeout)
            out[r] = res
    finally:
        for p in ps:
            p.join(timeout=30)
            if p.is_alive():
                p.kill()
    for r, res in out.items():
        assert "error" not in res, res.get("error")
    return out


def test_comm_allreduce_and_p2p_two_ranks():
    out = _run("collectives")
    assert all(out[r][f"ar{i}"] for r in range(2) for i in range(3))
    assert all(out[1][f"p2p{i}"] for i in range(3))


def test_stack_tensor_parallel_two_ranks():
    out = _run("tp")
    for r in range(2):
        assert out[r]["err"] <= 1e-3, out


def test_stack_layer_parallel_two_ranks():
    out = _run("pp")
    assert out[1]["err"] <= 1e-3, out


def test_stack_layer_parallel_two_ranks_decode_engine():
    out = _run("pp1")
    assert out[1]["err"] <= 1e-3, out


def test_stack_hybrid_2x2_four_ranks():
    """Hybrid partition (Table 4): 2 stages x 2 TP ranks, 4 processes on one
    GPU; both last-stage ranks hold the full h_out and must equal the oracle."""
    out = _run("hybrid", world=4, timeout=360)
    for r in (2, 3):
        assert out[r]["err"] <= 1e-3, out


def test_stack_hybrid_2x2_four_ranks_batch1():
    out = _run("hybrid1", world=4, timeout=360)
    for r in (2, 3):
        assert out[r]["err"] <= 1e-3, out


def test_nccl_communicator_single_rank_in_graph():
    """if_comm_init (NCCL baseline): a 1-rank plan; all-reduce is the identity and is
    captured and replayed inside a CUDA graph; a 1-rank stack with the NCCL comm
    equals the comm-less run bit for bit."""
    import paper_2401_08294_b200 as F
    import synth
    from paper_2401_08294_b200.model import Stack
    dev = torch.device("cuda:0")
    torch.cuda.set_device(dev)
    cfg = dict(layers=2, hidden=512, heads=8, kv_heads=2, head_dim=64, ffn=1408)
    s = F.scheme(35, 64)
    shape = F.stack_shape(*[cfg[k] for k in ("layers", "hidden", "heads", "kv_heads", "head_dim", "ffn")], s)
    plan = F.if_plan_partition(F.IF_BY_TENSOR, shape, 1)
    comm = F.Comm(plan, 0, nccl_id=F.if_comm_nccl_unique_id())
    buf = torch.arange(4096, dtype=torch.float32, device=dev)
    st = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(st):
        comm.allreduce(buf, st)
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=st):
            comm.allreduce(buf, st)
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    assert torch.equal(buf.cpu(), torch.arange(4096, dtype=torch.float32))
    stk = Stack(cfg, s, plan, 0, dev)
    h = torch.from_numpy(synth.activations(3, cfg["hidden"])).to(dev)
    outs = []
    for c in (None, comm):
        out = torch.empty_like(h)
        ws = torch.zeros(F.if_stack_workspace_bytes(shape, plan, 0, 3, F.IF_DECODE), dtype=torch.uint8, device=dev)
        F.if_run_stack(shape, plan, 0, c, stk.arr, h, 3, F.IF_DECODE, out, None, ws)
        torch.cuda.synchronize()
        outs.append(out.cpu())
    assert torch.equal(outs[0], outs[1])
    comm.destroy()
