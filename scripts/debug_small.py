"""Run the SMALL decode stack once (layers from argv) and compare with the oracle."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import torch
import oracle as O
import paper_2401_08294_b200 as F
import synth
from paper_2401_08294_b200.model import Stack, deinterleave_rows
layers = int(sys.argv[1]) if len(sys.argv) > 1 else 1
T = int(sys.argv[2]) if len(sys.argv) > 2 else 1
qt, bsz = (int(sys.argv[3]), int(sys.argv[4])) if len(sys.argv) > 4 else (35, 64)
cfg = dict(layers=layers, hidden=512, heads=8, kv_heads=2, head_dim=64, ffn=1408)
d = torch.device("cuda:0")
s = F.scheme(qt, bsz)
shape = F.stack_shape(*[cfg[k] for k in ("layers", "hidden", "heads", "kv_heads", "head_dim", "ffn")], s)
plan = F.if_plan_partition(F.IF_BY_LAYER, shape, 1)
stk = Stack(cfg, s, plan, 0, d)
h = synth.activations(T, cfg["hidden"], tid=3)
hd = torch.from_numpy(h).to(d)
out = torch.empty_like(hd)
ws = torch.zeros(F.if_stack_workspace_bytes(shape, plan, 0, T, F.IF_DECODE), dtype=torch.uint8, device=d)
F.if_run_stack(shape, plan, 0, None, stk.arr, hd, T, F.IF_DECODE, out, None, ws)
torch.cuda.synchronize()
host = [[t.cpu().numpy() for t in layer] for layer in stk.layers]
ho, qo = O.stack_f64(dict(cfg, qtype=qt, block=bsz), [l[0] for l in host], [l[1] for l in host],
                     [deinterleave_rows(l[2], 2 * stk.local['lf']) for l in host], [l[3] for l in host], h)
o = out.cpu().numpy()
print("layers", layers, "normwise", np.abs(o - ho).max() / np.abs(ho).max())
