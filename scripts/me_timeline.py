"""Per-phase timeline of the persistent batched engine (qgemv_ms.cu ms_engine_kernel).
  python scripts/me_timeline.py B LAYERS
Per phase: CTAs with units, median barrier wait, median loop (barrier-out -> last loop end),
median epilogue, phase span (first barrier-out -> last done) -- us."""
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
G = 2 * torch.cuda.get_device_properties(0).multi_processor_count
np_ = 1 + 4 * layers
dbg = torch.zeros(np_ * G * 4, dtype=torch.int64, device=dev)
for it in range(4):
    L.ifx_set_mk_debug(dbg.data_ptr() if it == 3 else None)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    F.if_run_stack(shape, plan, 0, None, stk.arr, h, B, F.IF_DECODE, out, None, ws)
    e1.record()
    torch.cuda.synchronize()
    print("stack us", round(e0.elapsed_time(e1) * 1e3, 1))
L.ifx_set_mk_debug(None)
r = dbg.view(np_, G, 4).cpu().numpy().astype(np.float64)
t0 = r[r > 0].min()
names = ["prep"] + [n for _ in range(layers) for n in ("qkv", "o", "gu", "down")]
print("phase  ctas  wait  loop  epi  span  (us)")
for p in range(1, np_):
    x = r[p]
    ok = x[:, 1] > 0
    if not ok.any(): continue
    x = (x[ok] - t0) / 1e3
    print(f"{names[p]:5s} {ok.sum():5d} {np.median(x[:,1]-x[:,0]):5.2f} {np.median(x[:,2]-x[:,1]):5.2f} "
          f"{np.median(x[:,3]-x[:,2]):5.2f} {x[:,3].max()-x[:,1].min():6.2f}  first-in {x[:,1].min():7.2f} last-done {x[:,3].max():7.2f}")
