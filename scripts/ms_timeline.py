"""Per-CTA phase timeline of the fused batched chain (qgemv_ms.cu, globaltimer stamps).

  python scripts/ms_timeline.py B [LAYERS]
Launch order: prep, then (qkv, o, gu, down) per layer.  Per launch (us, medians over
CTAs): start->dep (pdl wait), dep->rec (records copy + rms), loop, reduce (cluster),
emit; plus the launch span (first start -> last end) and the gap to the previous.
"""
import ctypes, os, sys
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
B = int(sys.argv[1]) if len(sys.argv) > 1 else 8
layers = int(sys.argv[2]) if len(sys.argv) > 2 else 3
cfg = dict(synth.LLAMA["7b"], layers=layers)
shape = F.stack_shape(*[cfg[k] for k in ("layers", "hidden", "heads", "kv_heads", "head_dim", "ffn")], s)
plan = F.if_plan_partition(F.IF_BY_LAYER, shape, 1)
stk = Stack(cfg, s, plan, 0, dev)
h = torch.randn(B, cfg["hidden"], device=dev)
out = torch.empty_like(h)
ws = torch.zeros(F.if_stack_workspace_bytes(shape, plan, 0, B, F.IF_DECODE), dtype=torch.uint8, device=dev)
dbg = torch.zeros(16 * 1024 * 8, dtype=torch.int64, device=dev)
for it in range(4):
    L.ifx_set_mk_debug(dbg.data_ptr() if it == 3 else None)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    F.if_run_stack(shape, plan, 0, None, stk.arr, h, B, F.IF_DECODE, out, None, ws)
    e1.record()
    torch.cuda.synchronize()
    print("stack us", round(e0.elapsed_time(e1) * 1e3, 1))
L.ifx_set_mk_debug(None)
raw = dbg.view(16, 1024, 8).cpu().numpy().astype(np.float64)
t0 = raw[raw[:, :, 0] > 0, 0].min()
names = ["prep"] + [n for _ in range(layers) for n in ("qkv", "o", "gu", "down")]
prev_end = None
print("launch  nCTA   span  gap | dep   rec   loop  red   emit (median us) | loop max")
for q, n in enumerate(names[:16]):
    r = raw[q]
    ok = r[:, 0] > 0
    if not ok.any():
        continue
    r = (r[ok] - t0) / 1e3
    start, end = r[:, 0].min(), np.max(np.maximum(np.maximum(r[:, 5], r[:, 4]), r[:, 3]))
    def med(a, b):
        m = (r[:, b] > 0) & (r[:, a] > 0)
        return float(np.median(r[m, b] - r[m, a])) if n != "prep" and m.any() else 0.0
    gap = start - prev_end if prev_end is not None else 0.0
    print(f"{n:5s} {ok.sum():5d} {end - start:6.2f} {gap:5.2f} | {med(0,1):5.2f} {med(1,2):5.2f} {med(2,3):5.2f} "
          f"{med(3,4):5.2f} {np.median(r[r[:,5]>0,5]-r[r[:,5]>0,4]) if (r[:,5]>0).any() else 0:5.2f} | "
          f"{(r[:,3]-r[:,2]).max() if n != 'prep' else 0:5.2f}  starts {np.percentile(r[:,0]-start,[50,90,100]).round(2)}")
    prev_end = end
