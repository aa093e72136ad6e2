"""Engine (T=1) vs per-layer path (T=2, duplicated token) on a 2-layer stack; prints
per-segment normwise differences of h_out and last_qkv.  IFB_MODEL=70b|13b|7b."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2401_08294_b200 as F, synth
from paper_2401_08294_b200.model import Stack
m = os.environ.get("IFB_MODEL", "70b")
cfg = dict(synth.LLAMA[m], layers=int(os.environ.get("IFB_LAYERS", "2")))
dev = torch.device("cuda:0")
s = F.scheme(35, 64)
shape = F.stack_shape(*[cfg[k] for k in ("layers", "hidden", "heads", "kv_heads", "head_dim", "ffn")], s)
plan = F.if_plan_partition(F.IF_BY_LAYER, shape, 1)
stk = Stack(cfg, s, plan, 0, dev)
d = cfg["hidden"]; nqkv = (cfg["heads"] + 2 * cfg["kv_heads"]) * cfg["head_dim"]
h = torch.from_numpy(synth.activations(1, d)).to(dev)
res = {}
for T in (1, 8):
    hin = h.repeat(T, 1).contiguous()
    out = torch.empty_like(hin); qkv = torch.empty(T, nqkv, device=dev)
    ws = torch.zeros(F.if_stack_workspace_bytes(shape, plan, 0, T, F.IF_DECODE), dtype=torch.uint8, device=dev)
    F.if_run_stack(shape, plan, 0, None, stk.arr, hin, T, F.IF_DECODE, out, qkv, ws)
    torch.cuda.synchronize()
    res[T] = (out[0].cpu().numpy().astype(np.float64), qkv[0].cpu().numpy().astype(np.float64))
def nw(a, b): return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-30))
a, b = res[1], res[8]
nq, nk = cfg["heads"] * cfg["head_dim"], cfg["kv_heads"] * cfg["head_dim"]
print(m, "h_out", nw(a[0], b[0]), "q", nw(a[1][:nq], b[1][:nq]), "k", nw(a[1][nq:nq + nk], b[1][nq:nq + nk]),
      "v", nw(a[1][nq + nk:], b[1][nq + nk:]))
bad = np.where(np.abs(a[0] - b[0]) > 1e-2 * np.abs(b[0]).max())[0]
print("h_out bad rows:", len(bad), bad[:20], bad[-5:] if len(bad) else "")
