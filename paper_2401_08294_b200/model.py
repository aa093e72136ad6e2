"""Synthetic Llama-shaped stacks resident in HBM (Q18, Q19).

Weights are generated on the device by the library's counter-based generator
(if_synth_fill, same stream as synth/) and quantized by if_quantize, one
tensor at a time, so a 70B-shaped stack (34 GB packed) never needs its 274 GB
fp32 form.  Rank-local shards follow the plan (if_plan_partition):
  wqkv  rows q[h0*hd:h1*hd] | k[k0*hd:k1*hd] | v[k0*hd:k1*hd]    (column shard)
  wo    K-columns [h0*hd, h1*hd) of every row                      (row shard)
  wgu   rows gate[f0:f1] and up[f0:f1] interleaved (2f gate, 2f+1 up)  (column shard)
  wdown K-columns [f0, f1)                                          (row shard)
Shards are exact slices of the unsharded packed tensors (block-aligned splits).
"""
from __future__ import annotations

import math

import torch

import synth

from . import (IF_DECODE, Scheme, if_packed_bytes, if_quantize, if_synth_fill, layer_weights_array, stack_shape)


def _gen_rows(layer: int, name: str, N: int, K: int, hidden: int, r0: int, r1: int, scratch: torch.Tensor,
              stream=None) -> torch.Tensor:
    """fp32 rows [r0, r1) of the synthetic [N, K] tensor into scratch."""
    n = (r1 - r0) * K
    out = scratch[:n]
    if_synth_fill(synth.SEED_WEIGHTS, synth.tensor_id(layer, name), float(synth.scale(1.0 / math.sqrt(hidden))), out,
                  offset=r0 * K, stream=stream)
    return out


def quantize_rows(s: Scheme, layer: int, name: str, N: int, K: int, hidden: int, r0: int, r1: int,
                  scratch: torch.Tensor, dev_status: torch.Tensor) -> torch.Tensor:
    w = _gen_rows(layer, name, N, K, hidden, r0, r1, scratch)
    packed = torch.empty(if_packed_bytes(s, r1 - r0, K), dtype=torch.uint8, device=scratch.device)
    if_quantize(s, w, r1 - r0, K, packed, dev_status)
    return packed


def col_slice(packed: torch.Tensor, s: Scheme, N: int, K: int, c0: int, c1: int) -> torch.Tensor:
    """Block-aligned K-column window [c0, c1) of a packed [N, K] tensor."""
    from . import if_block_bytes
    bb = if_block_bytes(s)
    nb = K // s.block
    if c0 % s.block or c1 % s.block:
        raise ValueError(f"col_slice [{c0},{c1}) is not aligned to block {s.block}")
    v = packed.view(N, nb, bb)[:, c0 // s.block:c1 // s.block, :]
    return v.contiguous().view(-1)


def interleave_rows(a: torch.Tensor, b: torch.Tensor, rows: int) -> torch.Tensor:
    """Packed [rows, rb] tensors a, b -> [2*rows, rb] with rows a0, b0, a1, b1, ..."""
    rb = a.numel() // rows
    return torch.stack([a.view(rows, rb), b.view(rows, rb)], dim=1).reshape(-1).contiguous()


def deinterleave_rows(p, rows2: int):
    """Inverse of interleave_rows (numpy or torch): [2r, rb] -> concat(even rows, odd rows)."""
    rb = p.shape[0] // rows2
    v = p.reshape(rows2 // 2, 2, rb)
    if isinstance(p, torch.Tensor):
        return torch.cat([v[:, 0].reshape(-1), v[:, 1].reshape(-1)])
    import numpy as np
    return np.concatenate([v[:, 0].reshape(-1), v[:, 1].reshape(-1)])


class Stack:
    """Rank-local packed shards of a synthetic stack (all layers of the rank's stage)."""

    def __init__(self, cfg: dict, s: Scheme, plan, rank: int, device="cuda"):
        self.cfg = cfg
        self.s = s
        self.plan = plan
        self.rank = rank
        self.shape = stack_shape(cfg["layers"], cfg["hidden"], cfg["heads"], cfg["kv_heads"], cfg["head_dim"],
                                 cfg["ffn"], s)
        a = plan.a[rank]
        d, H, G, hd, F = cfg["hidden"], cfg["heads"], cfg["kv_heads"], cfg["head_dim"], cfg["ffn"]
        h0, h1, k0, k1 = a.head_begin, a.head_end, a.kv_begin, a.kv_end
        f0, f1 = a.ffn_blk_begin * 64, a.ffn_blk_end * 64
        self.local = dict(lh=h1 - h0, lkv=k1 - k0, lf=f1 - f0)
        biggest = max(H * hd * d, d * F, F * d, (H + 2 * G) * hd * d)
        scratch = torch.empty(biggest, dtype=torch.float32, device=device)
        self.dev_status = torch.zeros(1, dtype=torch.int32, device=device)
        self.layers = []
        for l in range(a.layer_begin, a.layer_end):
            q = quantize_rows(s, l, "q", H * hd, d, d, h0 * hd, h1 * hd, scratch, self.dev_status)
            k = quantize_rows(s, l, "k", G * hd, d, d, k0 * hd, k1 * hd, scratch, self.dev_status)
            v = quantize_rows(s, l, "v", G * hd, d, d, k0 * hd, k1 * hd, scratch, self.dev_status)
            wqkv = torch.cat([q, k, v])
            del q, k, v
            wo_full = quantize_rows(s, l, "o", d, H * hd, d, 0, d, scratch, self.dev_status)
            wo = col_slice(wo_full, s, d, H * hd, h0 * hd, h1 * hd) if (h1 - h0) != H else wo_full
            del wo_full
            g = quantize_rows(s, l, "gate", F, d, d, f0, f1, scratch, self.dev_status)
            u = quantize_rows(s, l, "up", F, d, d, f0, f1, scratch, self.dev_status)
            wgu = interleave_rows(g, u, f1 - f0)  # row 2f = gate f, row 2f+1 = up f (ABI layout)
            del g, u
            wd_full = quantize_rows(s, l, "down", d, F, d, 0, d, scratch, self.dev_status)
            wdown = col_slice(wd_full, s, d, F, f0, f1) if (f1 - f0) != F else wd_full
            del wd_full
            self.layers.append((wqkv, wo, wgu, wdown))
        del scratch
        torch.cuda.synchronize(device)
        st = int(self.dev_status.item())
        if st != 0:
            raise RuntimeError(f"quantization reported device status {st}")
        self.arr = layer_weights_array(self.layers)

    def weight_bytes(self) -> int:
        return sum(t.numel() for layer in self.layers for t in layer)
