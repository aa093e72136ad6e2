"""GPU parity of the KV-cache decode attention (if_run_stack_kv, attn.cu; NEXT-1,
DESIGN.md Q24) against the oracle's O.stack_kv_f64, element by element.

Decode gate 1e-3 normwise (fp32 path) on h_out and last_qkv at every step;
prefill (bf16 activations) is reported against a loose 5e-2 as the prefill stack.
Cases: multi-step decode of two slots (T = 2: per-layer path), batches through the
tensor-core qGEMV (T = 8, 16) with mixed positions, GQA with 8 heads per kv group
(Llama-2 70B's ratio), long positions through 16 position splits (caches filled
with the same synthetic values on both sides), a causal prefill chunk followed by
decode, and the out-of-range status.
"""
import numpy as np
import pytest

import oracle as O
import paper_2401_08294_b200 as F
import synth
from gpu_util import dev, normwise, torch
from paper_2401_08294_b200.model import Stack, deinterleave_rows

pytestmark = pytest.mark.gpu

SMALL = dict(layers=3, hidden=512, heads=8, kv_heads=2, head_dim=64, ffn=1408)
GQA8 = dict(layers=2, hidden=1024, heads=16, kv_heads=2, head_dim=128, ffn=1536)


class Rig:
    def __init__(self, cfg, slots, max_ctx, max_T=16, qtype=35, bs=64):
        self.d = dev()
        self.cfg = cfg
        s = F.scheme(qtype, bs)
        self.shape = F.stack_shape(*[cfg[k] for k in ("layers", "hidden", "heads", "kv_heads", "head_dim", "ffn")], s)
        self.plan = F.if_plan_partition(F.IF_BY_LAYER, self.shape, 1)
        self.stk = Stack(cfg, s, self.plan, 0, self.d)
        self.kv = F.KV(self.shape, self.plan, 0, slots, max_ctx, self.d)
        self.ws = torch.zeros(F.if_stack_workspace_bytes(self.shape, self.plan, 0, max_T, F.IF_DECODE),
                              dtype=torch.uint8, device=self.d)
        host = [[t.cpu().numpy() for t in layer] for layer in self.stk.layers]
        self.W = ([l[0] for l in host], [l[1] for l in host],
                  [deinterleave_rows(l[2], 2 * cfg["ffn"]) for l in host], [l[3] for l in host])
        self.oshape = dict(cfg, qtype=qtype, block=bs)
        self.K, self.V = O.kv_cache(self.oshape, slots, max_ctx)
        self.nqkv = (cfg["heads"] + 2 * cfg["kv_heads"]) * cfg["head_dim"]

    def step(self, h, slots, positions, mode=F.IF_DECODE):
        T = h.shape[0]
        hd = torch.from_numpy(h).to(self.d)
        out = torch.empty_like(hd)
        qkv = torch.empty(T, self.nqkv, device=self.d)
        sid = torch.tensor(slots, dtype=torch.int32, device=self.d)
        pos = torch.tensor(positions, dtype=torch.int32, device=self.d)
        F.if_run_stack_kv(self.shape, self.plan, 0, None, self.stk.arr, hd, T, mode, out, qkv, self.kv, sid, pos,
                          self.ws)
        torch.cuda.synchronize()
        ho, qo = O.stack_kv_f64(self.oshape, *self.W, h, slots, positions, self.K, self.V)
        return out.cpu().numpy(), qkv.cpu().numpy(), ho, qo


def test_decode_two_slots_eight_steps():
    r = Rig(SMALL, slots=2, max_ctx=16)
    for p in range(8):
        h = synth.activations(2, SMALL["hidden"], tid=100 + p)
        out, qkv, ho, qo = r.step(h, [0, 1], [p, p])
        assert normwise(out, ho) <= 1e-3, p
        assert normwise(qkv, qo) <= 1e-3, p
    assert int(r.kv.status.item()) == 0


@pytest.mark.parametrize("T", [1, 8, 16])
def test_decode_batches_mixed_positions(T):
    """T queries in distinct slots at different depths (slot t has t + 1 tokens
    cached before the batched step): per-layer B = 1 engine GEMV (T = 1) and the
    tensor-core batched qGEMV with the attention's fp16 split (T = 8, 16)."""
    r = Rig(SMALL, slots=T, max_ctx=T + 2, max_T=16)
    for p in range(T):  # fill: slot t receives tokens at positions 0..t (as a batch of the active slots)
        act = [t for t in range(T) if t >= p]
        h = synth.activations(len(act), SMALL["hidden"], tid=200 + p)
        out, _, ho, _ = r.step(h, act, [p] * len(act))
        assert normwise(out, ho) <= 1e-3
    h = synth.activations(T, SMALL["hidden"], tid=300)
    out, qkv, ho, qo = r.step(h, list(range(T)), [t + 1 for t in range(T)])
    assert normwise(out, ho) <= 1e-3
    assert normwise(qkv, qo) <= 1e-3


def test_gqa_eight_heads_per_group():
    r = Rig(GQA8, slots=1, max_ctx=8)
    for p in range(5):
        h = synth.activations(1, GQA8["hidden"], tid=400 + p)
        out, qkv, ho, qo = r.step(h, [0], [p])
        assert normwise(out, ho) <= 1e-3, p


@pytest.mark.parametrize("cfg", [SMALL, GQA8])
def test_long_position_sixteen_splits(cfg):
    """Position 700 of a 1024-position cache whose entries both sides hold as the same
    synthetic fp32 values: the attention runs 16 position splits + the merge."""
    P = 700
    r = Rig(cfg, slots=2, max_ctx=1024)
    rng = np.random.default_rng(7)
    k = (rng.standard_normal(r.K.shape) * 0.5).astype(np.float32)
    v = rng.standard_normal(r.V.shape).astype(np.float32)
    r.kv.k.copy_(torch.from_numpy(k.reshape(-1)))
    r.kv.v.copy_(torch.from_numpy(v.reshape(-1)))
    r.K[...] = k
    r.V[...] = v
    h = synth.activations(1, cfg["hidden"], tid=500)
    out, qkv, ho, qo = r.step(h, [1], [P])
    assert normwise(out, ho) <= 1e-3
    assert normwise(qkv, qo) <= 1e-3


def test_prefill_chunk_then_decode():
    """A 6-token causal prefill chunk (bf16 qGEMM) of one slot, then decode steps on top
    of the cache it wrote.  bf16 activations: held to 5e-2 like the prefill stack."""
    r = Rig(SMALL, slots=1, max_ctx=16)
    h = synth.activations(6, SMALL["hidden"], tid=600)
    out, _, ho, _ = r.step(h, [0] * 6, list(range(6)), mode=F.IF_PREFILL)
    err = normwise(out, ho)
    print(f"prefill chunk err {err:.2e}")
    assert err <= 5e-2
    for p in range(6, 9):
        out, _, ho, _ = r.step(synth.activations(1, SMALL["hidden"], tid=600 + p), [0], [p])
        assert normwise(out, ho) <= 5e-2


def test_out_of_range_position_reports_status():
    r = Rig(SMALL, slots=1, max_ctx=4)
    d = r.d
    h = torch.from_numpy(synth.activations(1, SMALL["hidden"])).to(d)
    out = torch.empty_like(h)
    sid = torch.tensor([0], dtype=torch.int32, device=d)
    pos = torch.tensor([4], dtype=torch.int32, device=d)
    F.if_run_stack_kv(r.shape, r.plan, 0, None, r.stk.arr, h, 1, F.IF_DECODE, out, None, r.kv, sid, pos, r.ws)
    torch.cuda.synchronize()
    assert int(r.kv.status.item()) == 1
    assert bool(torch.isfinite(out).all())


def test_graph_replay_with_device_positions():
    """Positions live in device memory: one captured graph decodes consecutive
    positions by updating them in place between replays."""
    r = Rig(SMALL, slots=1, max_ctx=8)
    d = r.d
    hd = torch.zeros(1, SMALL["hidden"], device=d)
    out = torch.empty_like(hd)
    sid = torch.zeros(1, dtype=torch.int32, device=d)
    pos = torch.zeros(1, dtype=torch.int32, device=d)
    st = torch.cuda.Stream(d)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(st):
        F.if_run_stack_kv(r.shape, r.plan, 0, None, r.stk.arr, hd, 1, F.IF_DECODE, out, None, r.kv, sid, pos, r.ws, st)
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=st):
            F.if_run_stack_kv(r.shape, r.plan, 0, None, r.stk.arr, hd, 1, F.IF_DECODE, out, None, r.kv, sid, pos,
                              r.ws, st)
    r.K[...] = 0
    r.V[...] = 0
    for p in range(5):
        h = synth.activations(1, SMALL["hidden"], tid=700 + p)
        hd.copy_(torch.from_numpy(h))
        pos.fill_(p)
        g.replay()
        torch.cuda.synchronize()
        ho, _ = O.stack_kv_f64(r.oshape, *r.W, h, [0], [p], r.K, r.V)
        assert normwise(out.cpu().numpy(), ho) <= 1e-3, p
