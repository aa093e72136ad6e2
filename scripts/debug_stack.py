"""Localize a decode-engine mismatch: 1-2 layer SMALL stack vs the oracle."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import oracle as O
import paper_2401_08294_b200 as F
import synth
from paper_2401_08294_b200.model import Stack, deinterleave_rows

for layers in (1, 2):
    for cfg in (dict(layers=layers, hidden=512, heads=8, kv_heads=2, head_dim=64, ffn=1408),
                dict(layers=layers, hidden=4096, heads=32, kv_heads=32, head_dim=128, ffn=11008)):
        d = torch.device("cuda:0")
        s = F.scheme(35, 64)
        shape = F.stack_shape(*[cfg[k] for k in ("layers", "hidden", "heads", "kv_heads", "head_dim", "ffn")], s)
        plan = F.if_plan_partition(F.IF_BY_LAYER, shape, 1)
        stk = Stack(cfg, s, plan, 0, d)
        h = synth.activations(1, cfg["hidden"], tid=3)
        hd = torch.from_numpy(h).to(d)
        out = torch.empty_like(hd)
        nqkv = (cfg["heads"] + 2 * cfg["kv_heads"]) * cfg["head_dim"]
        qkv = torch.zeros(1, nqkv, device=d)
        ws = torch.zeros(F.if_stack_workspace_bytes(shape, plan, 0, 1, F.IF_DECODE), dtype=torch.uint8, device=d)
        F.if_run_stack(shape, plan, 0, None, stk.arr, hd, 1, F.IF_DECODE, out, qkv, ws)
        torch.cuda.synchronize()
        host = [[t.cpu().numpy() for t in layer] for layer in stk.layers]
        ho, qo = O.stack_f64(dict(cfg, qtype=35, block=64), [l[0] for l in host], [l[1] for l in host],
                             [deinterleave_rows(l[2], 2 * stk.local['lf']) for l in host], [l[3] for l in host], h)
        o, q = out.cpu().numpy(), qkv.cpu().numpy()
        eq = np.abs(q - qo).max() / np.abs(qo).max()
        eh = np.abs(o - ho).max() / np.abs(ho).max()
        nq = cfg["heads"] * cfg["head_dim"]
        nkv = cfg["kv_heads"] * cfg["head_dim"]
        eqq = np.abs(q[:, :nq] - qo[:, :nq]).max() / np.abs(qo[:, :nq]).max()
        evv = np.abs(q[:, nq + nkv:] - qo[:, nq + nkv:]).max() / np.abs(qo[:, nq + nkv:]).max()
        print(f"L={layers} d={cfg['hidden']}: qkv err {eq:.2e} (q {eqq:.2e}, v {evv:.2e})  h err {eh:.2e}", flush=True)
