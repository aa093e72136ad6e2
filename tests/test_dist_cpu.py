"""Multi-process host logic on CPU (gloo, world_size 2): every rank plans its
share through the C ABI (if_plan_partition) and cuts its packed shards with
the product's slicing helpers; the ranks all-gather and rank 0 checks that the
assignments equal the oracle planner's, cover every (layer, head, FFN block)
once per group, and that the shards reassemble bit-exactly into the oracle's
unsharded packed tensors (block-aligned splits)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    try:
        import sys
        sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
        import oracle as O
        import paper_2401_08294_b200 as F
        import synth
        from paper_2401_08294_b200.model import col_slice, interleave_rows

        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        cfg = dict(layers=4, hidden=256, heads=4, kv_heads=2, head_dim=64, ffn=512)
        s = F.scheme(35, 64)
        shape = F.stack_shape(*[cfg[k] for k in ("layers", "hidden", "heads", "kv_heads", "head_dim", "ffn")], s)
        out = {}
        for strat in (F.IF_BY_LAYER, F.IF_BY_TENSOR):
            p = F.if_plan_partition(strat, shape, world)
            a = p.a[rank]
            mine = [a.stage, a.group_rank, a.layer_begin, a.layer_end, a.head_begin, a.head_end, a.kv_begin,
                    a.kv_end, a.ffn_blk_begin, a.ffn_blk_end]
            allv = [None] * world
            dist.all_gather_object(allv, mine)
            out[f"plan{strat}"] = allv
        # shards of layer 0 under by_tensor, cut on every rank from the oracle's packed tensors
        p = F.if_plan_partition(F.IF_BY_TENSOR, shape, world)
        a = p.a[rank]
        d, H, G, hd, Fd = cfg["hidden"], cfg["heads"], cfg["kv_heads"], cfg["head_dim"], cfg["ffn"]
        full_o = torch.from_numpy(O.quantize(35, 64, synth.weight(0, "o", d, H * hd, d)))
        full_g = torch.from_numpy(O.quantize(35, 64, synth.weight(0, "gate", Fd, d, d)))
        full_u = torch.from_numpy(O.quantize(35, 64, synth.weight(0, "up", Fd, d, d)))
        rb = (d // 64) * 32
        wo = col_slice(full_o, s, d, H * hd, a.head_begin * hd, a.head_end * hd)
        f0, f1 = a.ffn_blk_begin * 64, a.ffn_blk_end * 64
        wgu = interleave_rows(full_g[f0 * rb:f1 * rb], full_u[f0 * rb:f1 * rb], f1 - f0)
        shards = [None] * world
        dist.all_gather_object(shards, (wo.numpy(), wgu.numpy(), a.head_begin, a.head_end, f0, f1))
        if rank == 0:
            # reassemble W_o column shards -> the full packed tensor
            parts = sorted(shards, key=lambda t: t[2])
            nbh = [(t[3] - t[2]) * hd // 64 for t in parts]
            rows = [t[0].reshape(d, nb * 32) for t, nb in zip(parts, nbh)]
            out["wo_ok"] = bool(np.array_equal(np.concatenate(rows, axis=1).reshape(-1), full_o.numpy()))
            g_rows, u_rows = [], []
            for t in sorted(shards, key=lambda t: t[4]):
                v = t[1].reshape(-1, 2, rb)
                g_rows.append(v[:, 0])
                u_rows.append(v[:, 1])
            out["gu_ok"] = bool(np.array_equal(np.concatenate(g_rows).reshape(-1), full_g.numpy()) and
                                np.array_equal(np.concatenate(u_rows).reshape(-1), full_u.numpy()))
        dist.destroy_process_group()
        q.put((rank, out))
    except Exception:
        import traceback
        q.put((rank, {"error": traceback.format_exc()}))


def test_plan_and_shards_two_ranks_gloo():
    import oracle as O
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = {}
    for _ in range(2):
        r, o = q.get(timeout=180)
        res[r] = o
    for p in ps:
        p.join(timeout=30)
    for r in res:
        assert "error" not in res[r], res[r]["error"]
    out = res[0]
    keys = ["stage", "group_rank", "layer_begin", "layer_end", "head_begin", "head_end", "kv_begin", "kv_end",
            "ffn_blk_begin", "ffn_blk_end"]
    for strat in (0, 1):
        ref = O.plan(strat, 4, 4, 2, 512 // 64, 2)
        got = [dict(zip(keys, v)) for v in out[f"plan{strat}"]]
        assert got == ref
    assert out["wo_ok"] and out["gu_ok"]
