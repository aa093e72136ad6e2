"""Dynamic-batching engine (if_engine AddQuery / Infer) at Llama-2-7B scale on
one B200: synthetic 7B stack (Q3H_B64), vocabulary 32000 (embedding fp32, LM head
Q3H_B64), KV cache for 16 slots x 512 positions.  Queries arrive over time (a new one
every few steps, as in Fig. 3) until 2 x slots have been served; each has a prompt of
16..64 tokens and 32 new tokens.  Reports generated tokens/s (wall clock around the
Infer() loop: the engine synchronises each step), the step-time distribution by active
batch size, and one speculative verification round (K = 4) of a running query.

    python scripts/engine_bench.py [--slots 16] [--new 32]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2401_08294_b200 as F
import synth
from paper_2401_08294_b200.model import Stack

ap = argparse.ArgumentParser()
ap.add_argument("--slots", type=int, default=16)
ap.add_argument("--new", type=int, default=32)
ap.add_argument("--vocab", type=int, default=32000)
ap.add_argument("--model", default="7b")
a = ap.parse_args()
dev = torch.device("cuda:0")
cfg = synth.LLAMA[a.model]
s = F.scheme(35, 64)
shape = F.stack_shape(*[cfg[k] for k in ("layers", "hidden", "heads", "kv_heads", "head_dim", "ffn")], s)
plan = F.if_plan_partition(F.IF_BY_LAYER, shape, 1)
stk = Stack(cfg, s, plan, 0, dev)
d, V = cfg["hidden"], a.vocab
E = torch.empty(V * d, device=dev)
F.if_synth_fill(synth.SEED_EMBED, 0, float(synth.scale(1.0)), E)
Wl = torch.empty(V * d, device=dev)
F.if_synth_fill(synth.SEED_WEIGHTS, synth.LM_TID, float(synth.scale(1.0 / np.sqrt(d))), Wl)
lm = torch.empty(F.if_packed_bytes(s, V, d), dtype=torch.uint8, device=dev)
F.if_quantize(s, Wl, V, d, lm)
del Wl
torch.cuda.synchronize()
eng = F.Engine(shape, stk.arr, E.view(V, d), lm, V, a.slots, 512, 64)
rng = np.random.default_rng(0)
total_q = 2 * a.slots
added, step, gen = 0, 0, 0
times, batch = [], []
t0 = time.perf_counter()
while True:
    while added < total_q and (step % 3 == 0 or added < a.slots // 2):  # staggered arrivals (Fig. 3)
        n = int(rng.integers(16, 65))
        eng.add_query(rng.integers(0, V, size=n).tolist(), a.new)
        added += 1
        if step % 3:
            break
    ts = time.perf_counter()
    out = eng.infer()
    times.append(time.perf_counter() - ts)
    batch.append(len(out))
    gen += len(out)
    step += 1
    if not out and added >= total_q:
        break
wall = time.perf_counter() - t0
b = np.array(batch)
tm = np.array(times) * 1e3
res = {"model": a.model, "vocab": V, "slots": a.slots, "queries": total_q, "new_tokens_each": a.new,
       "generated": gen, "steps": step, "wall_s": wall, "tokens_per_s": gen / wall,
       "step_ms_median_by_batch": {int(k): float(np.median(tm[b == k])) for k in sorted(set(b.tolist())) if k > 0}}
# one speculative verification round (Algorithm 1's target pass) on a fresh running query
q = eng.add_query(rng.integers(0, V, size=32).tolist(), 64)
while eng.query(q)[0] != 2:
    eng.infer()
K = 4
probs = torch.softmax(torch.randn(K, V, device=dev), dim=1)
draft = [int(x) for x in torch.multinomial(probs, 1).view(-1).tolist()]
torch.cuda.synchronize()
tv = time.perf_counter()
outv = eng.verify(q, draft, probs, [0.5] * K, 0.3)
res["verify_K4_ms"] = (time.perf_counter() - tv) * 1e3
res["verify_tokens"] = len(outv)
print(json.dumps(res))
