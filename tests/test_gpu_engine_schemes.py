"""The persistent decode engine for the k-bit schemes ("2, 3, 4, 5, 6, and 8"
bits, block sizes 32/64 P:176): batch-1 stacks and standalone GEMVs of
every k-bit scheme run through decode_mk (one launch per token), against the oracle's
fp64 stack / matmul at 1e-3 normwise.  Includes 7B-width rows (K = 4096 / 11008),
the 70B down projection (K = 28672: K-segmented staging for 32-weight blocks) and a
ragged GEMV (N not a multiple of the unit), and checks that a stack step is ONE launch.
"""
import numpy as np
import pytest

import oracle as O
import paper_2401_08294_b200 as F
import synth
from gpu_util import dev, normwise, oracle_rows_matmul, torch
from paper_2401_08294_b200.model import Stack, deinterleave_rows

pytestmark = pytest.mark.gpu

KBIT = [(2, 32), (2, 64), (3, 32), (3, 64), (4, 32), (4, 64), (5, 32), (5, 64), (6, 32), (6, 64), (8, 32), (8, 64)]
SMALL = dict(layers=2, hidden=1024, heads=8, kv_heads=4, head_dim=128, ffn=2048)


def _stack(cfg, qtype, bs, T=1):
    d = dev()
    s = F.scheme(qtype, bs)
    shape = F.stack_shape(*[cfg[k] for k in ("layers", "hidden", "heads", "kv_heads", "head_dim", "ffn")], s)
    plan = F.if_plan_partition(F.IF_BY_LAYER, shape, 1)
    stk = Stack(cfg, s, plan, 0, d)
    h = synth.activations(T, cfg["hidden"], tid=5)
    hd = torch.from_numpy(h).to(d)
    out = torch.empty_like(hd)
    nqkv = (cfg["heads"] + 2 * cfg["kv_heads"]) * cfg["head_dim"]
    qkv = torch.empty(T, nqkv, device=d)
    ws = torch.zeros(F.if_stack_workspace_bytes(shape, plan, 0, T, F.IF_DECODE), dtype=torch.uint8, device=d)
    F.if_launch_count(True)
    for _ in range(2):  # two launches on one workspace: the epoch / image versions advance
        F.if_run_stack(shape, plan, 0, None, stk.arr, hd, T, F.IF_DECODE, out, qkv, ws)
    launches = F.if_launch_count(True)
    torch.cuda.synchronize()
    host = [[t.cpu().numpy() for t in layer] for layer in stk.layers]
    ho, qo = O.stack_f64(dict(cfg, qtype=qtype, block=bs), [l[0] for l in host], [l[1] for l in host],
                         [deinterleave_rows(l[2], 2 * stk.local['lf']) for l in host], [l[3] for l in host], h)
    return out.cpu().numpy(), qkv.cpu().numpy(), ho, qo, launches


@pytest.mark.parametrize("qtype,bs", KBIT)
def test_engine_stack_every_kbit_scheme(qtype, bs):
    out, qkv, ho, qo, launches = _stack(SMALL, qtype, bs)
    assert normwise(out, ho) <= 1e-3
    assert normwise(qkv, qo) <= 1e-3
    assert launches == 2  # one engine kernel per call (the h_in copy is a memcpy node)


@pytest.mark.parametrize("qtype,bs", [(4, 32), (8, 64), (3, 32)])
def test_engine_stack_7b_width(qtype, bs):
    cfg = dict(synth.LLAMA["7b"], layers=2)
    out, qkv, ho, qo, _ = _stack(cfg, qtype, bs)
    assert normwise(out, ho) <= 1e-3
    assert normwise(qkv, qo) <= 1e-3


@pytest.mark.parametrize("qtype,bs,N,K", [(4, 32, 4096, 28672), (8, 64, 1000, 11008), (2, 32, 333, 4096),
                                           (5, 64, 8192, 28672), (6, 32, 4100, 8192)])
def test_engine_gemv_kbit(qtype, bs, N, K):
    """if_qgemv at B = 1 goes through the engine's single-phase mode (segmented staging
    for K = 28672); sampled rows vs the oracle's fp64 matmul of those rows."""
    d = dev()
    s = F.scheme(qtype, bs)
    W = torch.empty(N * K, dtype=torch.float32, device=d)
    F.if_synth_fill(synth.SEED_WEIGHTS, 900 + qtype, float(synth.scale(1 / np.sqrt(K))), W)
    p = torch.empty(F.if_packed_bytes(s, N, K), dtype=torch.uint8, device=d)
    F.if_quantize(s, W, N, K, p)
    x = synth.activations(1, K, tid=9)
    y = torch.empty(1, N, device=d)
    F.if_launch_count(True)
    F.if_qgemv(s, p, N, K, torch.from_numpy(x).to(d), 1, y)
    assert F.if_launch_count(True) == 1
    torch.cuda.synchronize()
    rows = sorted(set([0, 1, N // 3, N // 2, N - 2, N - 1] + list(range(0, N, max(1, N // 64)))))
    ref = oracle_rows_matmul(qtype, bs, p.cpu().numpy(), N, K, x, rows)
    assert normwise(y.cpu().numpy()[:, rows], ref) <= 1e-3
