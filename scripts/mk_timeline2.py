"""Per-phase-kind breakdown of the persistent decode kernel (globaltimer stamps).

  python scripts/mk_timeline2.py LAYERS
Columns (us, medians over CTAs and layers): wait = start->dep_ok, sync = dep_ok -
last CTA's signal of the previous phase, copy = dep_ok->x_ready, stage = x_ready->
staged, stream = staged->units_done, epi = units_done->signalled, skew = last -
median signal time of the phase.
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
G = torch.cuda.get_device_properties(0).multi_processor_count
layers = int(sys.argv[1]) if len(sys.argv) > 1 else 32
cfg = dict(synth.LLAMA[os.environ.get("IFB_MODEL", "7b")], layers=layers)
shape = F.stack_shape(*[cfg[k] for k in ("layers", "hidden", "heads", "kv_heads", "head_dim", "ffn")], s)
plan = F.if_plan_partition(F.IF_BY_LAYER, shape, 1)
stk = Stack(cfg, s, plan, 0, dev)
h = torch.randn(1, cfg["hidden"], device=dev)
out = torch.empty_like(h)
ws = torch.zeros(F.if_stack_workspace_bytes(shape, plan, 0, 1, F.IF_DECODE), dtype=torch.uint8, device=dev)
nph = 4 * layers
dbg = torch.zeros(G * nph * 16, dtype=torch.int64, device=dev)
for it in range(4):
    L.ifx_set_mk_debug(dbg.data_ptr() if it == 3 else None)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    F.if_run_stack(shape, plan, 0, None, stk.arr, h, 1, F.IF_DECODE, out, None, ws)
    e1.record()
    torch.cuda.synchronize()
    print("launch us", e0.elapsed_time(e1) * 1e3)
L.ifx_set_mk_debug(None)
raw = dbg.view(G, nph, 16).cpu().numpy()
dd = np.zeros(raw.shape)
dd[:, :, :8] = (raw[:, :, :8] - raw[:, 0, 0].min()).astype(np.float64)
dd[:, :, 8:] = (raw[:, :, 8:] - raw[:, 0, 8].min()).astype(np.float64)
d = dd[:, :, :8].copy()
ck = dd[:, :, 8:] / 1965.0  # us at max clock
d = d / 1e3
d[:, 0, 1] = d[:, 0, 0]  # phase 0 has no dependency stamp
print("total span", d[:, -1, 5].max() - d[:, 0, 0].min())
kinds = ["qkv", "o", "gu", "down"]
rows = {k: [] for k in range(4)}
for p in range(1, nph):
    k = p % 4
    last_prev = d[:, p - 1, 5].max()
    rows[k].append([np.median(d[:, p, 1] - d[:, p, 0]), np.median(d[:, p, 1]) - last_prev,
                    np.median(d[:, p, 2] - d[:, p, 1]), np.median(d[:, p, 3] - d[:, p, 2]),
                    np.median(d[:, p, 4] - d[:, p, 3]), np.median(d[:, p, 5] - d[:, p, 4]),
                    d[:, p, 5].max() - np.median(d[:, p, 5]), d[:, p, 5].max() - d[:, p - 1, 5].max()])
for k in range(4):
    ps = [p for p in range(1, nph) if p % 4 == k]
    first = np.median([np.median(d[:, p, 6] - d[:, p, 1]) for p in ps])
    repoll = dbg.view(G, nph, 16)[:, ps, 7].float().mean().item()
    print(f"{kinds[k]:5s} first-batch-return {first:6.2f} us after dep_ok; ct0 re-polls/phase {repoll:.2f}")
print("clock64-based intra-CTA durations (us @1965 MHz): start->dep, dep->copied, copied->staged, staged->units, units, epi-loop, bump")
for k in range(4):
    ps = [p for p in range(1, nph) if p % 4 == k]
    cols = []
    for a, b in [(0, 1), (1, 6), (6, 2), (2, 3), (3, 4), (4, 7), (7, 5)]:
        cols.append(np.median([np.median(ck[:, p, b] - ck[:, p, a]) for p in ps]))
    print(f"{kinds[k]:5s}" + "".join(f"{v:7.2f}" for v in cols))
print("kind   wait   sync   copy  stage stream    epi   skew  phase")
for k in range(4):
    a = np.median(np.array(rows[k]), axis=0)
    print(f"{kinds[k]:5s}" + "".join(f"{v:7.2f}" for v in a))
tot = np.sum([np.sum(np.array(rows[k]), axis=0) for k in range(4)], axis=0)
print("sum  " + "".join(f"{v:7.1f}" for v in tot))
w = dbg.view(G, nph, 16)[:, :, 15].cpu().numpy().astype(np.uint64)
if w.any():
    occ = (w & np.uint64(255)).astype(np.float64)
    wait = (w >> np.uint64(8)).astype(np.float64) / 1965.0
    print("IFB_MK_PROF: kind  ring-slots-landed-at-start  warp0-slot-wait-us (medians)")
    for k in range(4):
        ps = [p for p in range(1, nph) if p % 4 == k]
        print(f"  {kinds[k]:5s} {np.median(occ[:, ps]):5.1f} {np.median(wait[:, ps]):7.2f}")
