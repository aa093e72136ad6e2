"""Dump the decode engine's transformed-input images after a 1-layer run and
check them against the oracle's intermediate vectors (debugging aid)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import oracle as O
import paper_2401_08294_b200 as F
import synth
from paper_2401_08294_b200.model import Stack, deinterleave_rows

POS = [0, 7, 14, 0, 7, 3, 10, 17, 0, 7, 6, 13, 0, 7, 2, 9, 16, 0, 7, 5, 12, 0, 7, 1, 8, 15, 0, 7, 4, 11, 0, 7]


def al(x):
    return (x + 255) & ~255


def untransform(img, K, xstride):
    """xs image [16][xstride] float4 -> x[K] (x_e, x_o per pair)."""
    x = np.zeros(K)
    for k in range(0, K, 2):
        b, j = k // 64, (k // 2) % 32
        jj, comp = j // 2, j % 2
        q = img[jj * xstride + b]
        xo = q[comp] * 2.0 ** (POS[j] - 85)
        xe = q[2 + comp] * 2.0 ** -85 + 11 * xo
        x[k], x[k + 1] = xe, xo
    return x


cfg = dict(layers=1, hidden=512, heads=8, kv_heads=2, head_dim=64, ffn=1408)
if len(sys.argv) > 1:
    cfg = dict(layers=1, hidden=4096, heads=32, kv_heads=32, head_dim=128, ffn=11008)
d = torch.device("cuda:0")
s = F.scheme(35, 64)
shape = F.stack_shape(*[cfg[k] for k in ("layers", "hidden", "heads", "kv_heads", "head_dim", "ffn")], s)
plan = F.if_plan_partition(F.IF_BY_LAYER, shape, 1)
stk = Stack(cfg, s, plan, 0, d)
h = synth.activations(1, cfg["hidden"], tid=3)
hd = torch.from_numpy(h).to(d)
out = torch.empty_like(hd)
ws = torch.zeros(F.if_stack_workspace_bytes(shape, plan, 0, 1, F.IF_DECODE), dtype=torch.uint8, device=d)
F.if_run_stack(shape, plan, 0, None, stk.arr, hd, 1, F.IF_DECODE, out, None, ws)
torch.cuda.synchronize()
D, H, G, hdim, Fd = cfg["hidden"], cfg["heads"], cfg["kv_heads"], cfg["head_dim"], cfg["ffn"]
nq, nkv = H * hdim, G * hdim
nqkv = nq + 2 * nkv
off = al(D * 4) + al(nqkv * 4) + al(nq * 4) + al(2 * Fd * 4) + al(Fd * 4) + al(D * 4) + al(5 * 4)
nbp_max = ((max(D, nq, Fd) // 64 + 31) // 32) * 32
img = 16 * (nbp_max + 16)
xstride = ((nbp_max + 1 + 7) // 8) * 8 + 1
raw = ws.cpu().numpy()[off:].view(np.float32)
xs_h = raw[:img * 4].reshape(-1, 4)
xs_ctx = raw[img * 4:2 * img * 4].reshape(-1, 4)
xs_act = raw[2 * img * 4:3 * img * 4].reshape(-1, 4)
ssq = raw[3 * img * 4:3 * img * 4 + 160]
# oracle intermediates (fp64)
host = [[t.cpu().numpy() for t in layer] for layer in stk.layers]
Wqkv = O.dequantize(35, 64, host[0][0], nqkv, D).astype(np.float64)
Wo = O.dequantize(35, 64, host[0][1], D, nq).astype(np.float64)
Wgu = O.dequantize(35, 64, deinterleave_rows(host[0][2], 2 * Fd), 2 * Fd, D).astype(np.float64)
hh = h[0].astype(np.float64)
a = hh / np.sqrt((hh ** 2).mean() + 1e-5)
qkv = Wqkv @ a
v = qkv[nq + nkv:].reshape(G, hdim)
ctx = np.repeat(v, H // G, axis=0).reshape(-1)
h2 = hh + Wo @ ctx
a2 = h2 / np.sqrt((h2 ** 2).mean() + 1e-5)
gu = Wgu @ a2
act = gu[:Fd] / (1 + np.exp(-gu[:Fd])) * gu[Fd:]
e = lambda x, r: np.abs(x - r).max() / np.abs(r).max()
print("ctx image err", e(untransform(xs_ctx, nq, xstride), ctx))
print("h (after o) image err", e(untransform(xs_h, D, xstride), h2), " (after down if overwritten)")
print("act image err", e(untransform(xs_act, Fd, xstride), act))
print("ssq", ssq[:4], "sum", ssq[:148].sum(), "expected (after down)", None, "h2^2 sum", (h2 ** 2).sum())
