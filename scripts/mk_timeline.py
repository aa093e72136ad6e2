"""Per-phase timeline of the persistent decode kernel from %globaltimer stamps.

  python scripts/mk_timeline.py gemv N K
  python scripts/mk_timeline.py stack LAYERS
"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2401_08294_b200 as F
import synth
from paper_2401_08294_b200.model import Stack

L = F.lib()
L.ifx_set_mk_debug.argtypes = [ctypes.c_void_p]
dev = torch.device("cuda:0")
s = F.scheme(35, 64)
G = torch.cuda.get_device_properties(0).multi_processor_count
mode = sys.argv[1] if len(sys.argv) > 1 else "gemv"
if mode == "gemv":
    N, K = int(sys.argv[2]), int(sys.argv[3])
    p = torch.randint(0, 120, (F.if_packed_bytes(s, N, K),), dtype=torch.uint8, device=dev)
    v = p.view(-1, 32)
    v[:, 0] = 0x1F
    v[:, 1] = 0xA1
    v[:, 2] = 0x1F
    v[:, 3] = 0x21
    x = torch.randn(1, K, device=dev)
    y = torch.empty(1, N, device=dev)
    nph = 1
    dbg = torch.zeros(G * nph * 8, dtype=torch.int64, device=dev)
    for it in range(3):
        L.ifx_set_mk_debug(dbg.data_ptr() if it == 2 else None)
        F.if_qgemv(s, p, N, K, x, 1, y)
        torch.cuda.synchronize()
else:
    cfg = dict(synth.LLAMA["7b"], layers=int(sys.argv[2]) if len(sys.argv) > 2 else 4)
    shape = F.stack_shape(*[cfg[k] for k in ("layers", "hidden", "heads", "kv_heads", "head_dim", "ffn")], s)
    plan = F.if_plan_partition(F.IF_BY_LAYER, shape, 1)
    stk = Stack(cfg, s, plan, 0, dev)
    h = torch.randn(1, cfg["hidden"], device=dev)
    out = torch.empty_like(h)
    ws = torch.zeros(F.if_stack_workspace_bytes(shape, plan, 0, 1, F.IF_DECODE), dtype=torch.uint8, device=dev)
    nph = 4 * cfg["layers"]
    dbg = torch.zeros(G * nph * 8, dtype=torch.int64, device=dev)
    for it in range(3):
        L.ifx_set_mk_debug(dbg.data_ptr() if it == 2 else None)
        F.if_run_stack(shape, plan, 0, None, stk.arr, h, 1, F.IF_DECODE, out, None, ws)
        torch.cuda.synchronize()
L.ifx_set_mk_debug(None)
d = dbg.view(G, nph, 8).cpu().numpy().astype(np.float64)
t0 = d[:, 0, 0].min()
d = (d - t0) / 1e3  # us
names = ["start", "dep_ok", "x_ready", "staged", "units_done", "signalled", "st_bar", "st_loaded"]
print(f"== {' '.join(sys.argv[1:])}")
for p in range(min(nph, 12)):
    row = []
    for k in [0, 1, 2, 7, 6, 3, 4, 5]:
        col = d[:, p, k]
        row.append(f"{names[k]} {np.median(col):7.2f}")
    print(f"phase {p:3d}: " + " | ".join(row))
print("total span (us):", d[:, -1, 5].max())
