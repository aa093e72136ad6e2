"""Multi-rank plans run as concurrent streams on ONE GPU with in-process communicators
(if_comm_create_local): each rank's persistent decode engine gets SMs/devices CTAs,
the TP merges of o / down happen inside the engines (peer exchange regions), stage
hand-offs through the communicator's send/recv.  Several autoregressive steps (the
last stage's output is the next step's input) are compared with the oracle's
unpartitioned fp64 stack.  Prints one JSON line.  (Run in a subprocess by
tests/test_gpu_tp_engine.py: a protocol bug traps the GPU context after 2 s.)

    python scripts/tp_engine_check.py tensor|tensor4|hybrid|layer|single [steps]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import oracle as O
import paper_2401_08294_b200 as F
import synth
from paper_2401_08294_b200.model import Stack

mode = sys.argv[1] if len(sys.argv) > 1 else "tensor"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
CFG = dict(layers=4, hidden=1024, heads=8, kv_heads=4, head_dim=128, ffn=2048)
dev = torch.device("cuda:0")
torch.cuda.set_device(dev)
s = F.scheme(35, 64)
cfg = CFG
shape = F.stack_shape(*[cfg[k] for k in ("layers", "hidden", "heads", "kv_heads", "head_dim", "ffn")], s)
if mode == "tensor":
    plan = F.if_plan_partition(F.IF_BY_TENSOR, shape, 2)
elif mode == "tensor4":
    plan = F.if_plan_partition(F.IF_BY_TENSOR, shape, 4)
elif mode == "single":
    plan = F.if_plan_partition(F.IF_BY_LAYER, shape, 1)
elif mode == "hybrid":
    plan = F.if_plan_partition(F.IF_HYBRID, shape, 4, 2, 2)
else:
    plan = F.if_plan_partition(F.IF_BY_LAYER, shape, 2)
R = plan.devices
comms = F.Comm.local(plan, 8, cfg["hidden"]) if R > 1 else [None]
stacks = [Stack(cfg, s, plan, r, dev) for r in range(R)]
streams = [torch.cuda.Stream(dev) for _ in range(R)]
d = cfg["hidden"]
ws = [torch.zeros(F.if_stack_workspace_bytes(shape, plan, r, 1, F.IF_DECODE), dtype=torch.uint8, device=dev)
      for r in range(R)]
h_in = torch.from_numpy(synth.activations(1, d, tid=77)).to(dev)
outs = [torch.zeros(1, d, device=dev) for _ in range(R)]
last = [r for r in range(R) if plan.a[r].stage == plan.stages - 1]

# oracle: unpartitioned weights quantized by the oracle from the host generator
H, G, hd, Fd = cfg["heads"], cfg["kv_heads"], cfg["head_dim"], cfg["ffn"]
W = [[], [], [], []]
for l in range(cfg["layers"]):
    W[0].append(O.quantize(35, 64, np.concatenate([synth.weight(l, "q", H * hd, d, d), synth.weight(l, "k", G * hd, d, d),
                                                    synth.weight(l, "v", G * hd, d, d)])))
    W[1].append(O.quantize(35, 64, synth.weight(l, "o", d, H * hd, d)))
    W[2].append(O.quantize(35, 64, np.concatenate([synth.weight(l, "gate", Fd, d, d), synth.weight(l, "up", Fd, d, d)])))
    W[3].append(O.quantize(35, 64, synth.weight(l, "down", d, Fd, d)))
oshape = dict(cfg, qtype=35, block=64)

torch.cuda.synchronize()  # workspaces, inputs and weights are ready before the rank streams start
res = {"mode": mode, "ranks": R, "errs": [], "bitwise_equal_tp": True, "launches_per_step": []}
h_host = h_in.cpu().numpy()
for step in range(steps):
    F.if_launch_count(True)
    for r in range(R):
        with torch.cuda.stream(streams[r]):
            F.if_run_stack(shape, plan, r, comms[r], stacks[r].arr, h_in, 1, F.IF_DECODE, outs[r], None, ws[r],
                           streams[r])
    launches = F.if_launch_count(True)
    torch.cuda.synchronize()
    res["launches_per_step"].append(launches)
    got = [outs[r].cpu().numpy() for r in last]
    for g in got[1:]:
        res["bitwise_equal_tp"] &= bool(np.array_equal(g.view(np.uint32), got[0].view(np.uint32)))
    ref, _ = O.stack_f64(oshape, *W, h_host)
    err = float(np.abs(got[0] - ref).max() / np.abs(ref).max())
    res["errs"].append(err)
    # autoregressive feedback: the step output is the next input (exact fp32 values on both sides)
    h_host = got[0].astype(np.float32)
    h_in.copy_(torch.from_numpy(h_host))
# timing: 20 steps, device time
torch.cuda.synchronize()
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ev0.record()
for step in range(20):
    for r in range(R):
        with torch.cuda.stream(streams[r]):
            F.if_run_stack(shape, plan, r, comms[r], stacks[r].arr, h_in, 1, F.IF_DECODE, outs[r], None, ws[r],
                           streams[r])
torch.cuda.synchronize()
ev1.record()
torch.cuda.synchronize()
res["us_per_step_shared_gpu"] = ev0.elapsed_time(ev1) * 1e3 / 20
for c in comms:
    if c is not None:
        c.destroy()
print(json.dumps(res))
