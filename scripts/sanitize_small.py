"""One small invocation of each hot kernel, for compute-sanitizer (memcheck / racecheck /
synccheck): the persistent decode engine on a 2-layer SMALL stack (B = 1), the fused
batched chain (B = 8 and 16; with the KV cache at B = 2), the batched tensor-core qGEMV (B = 8), the prefill qGEMM (M = 70), the KV-cache attention stack,
quantize / dequantize, the LM head and the speculative verification."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2401_08294_b200 as F, synth
from paper_2401_08294_b200.model import Stack
dev = torch.device("cuda:0")
s = F.scheme(35, 64)
cfg = dict(layers=2, hidden=512, heads=8, kv_heads=2, head_dim=64, ffn=1408)
shape = F.stack_shape(*[cfg[k] for k in ("layers", "hidden", "heads", "kv_heads", "head_dim", "ffn")], s)
plan = F.if_plan_partition(F.IF_BY_LAYER, shape, 1)
stk = Stack(cfg, s, plan, 0, dev)
for T in (1, 8, 16):
    h = torch.from_numpy(synth.activations(T, 512)).to(dev)
    out = torch.empty_like(h)
    ws = torch.zeros(F.if_stack_workspace_bytes(shape, plan, 0, T, F.IF_DECODE), dtype=torch.uint8, device=dev)
    for _ in range(2):
        F.if_run_stack(shape, plan, 0, None, stk.arr, h, T, F.IF_DECODE, out, None, ws)
kv = F.KV(shape, plan, 0, 2, 8, dev)
ws = torch.zeros(F.if_stack_workspace_bytes(shape, plan, 0, 2, F.IF_DECODE), dtype=torch.uint8, device=dev)
h = torch.from_numpy(synth.activations(2, 512)).to(dev)
out = torch.empty_like(h)
F.if_run_stack_kv(shape, plan, 0, None, stk.arr, h, 2, F.IF_DECODE, out, None, kv,
                  torch.tensor([0, 1], dtype=torch.int32, device=dev), torch.tensor([0, 3], dtype=torch.int32, device=dev), ws)
N, K = 512, 1024
W = torch.from_numpy(synth.weight(0, "q", N, K, K)).to(dev)
p = torch.empty(F.if_packed_bytes(s, N, K), dtype=torch.uint8, device=dev)
st = torch.zeros(1, dtype=torch.int32, device=dev)
F.if_quantize(s, W, N, K, p, st)
F.if_dequantize(s, p, N, K, torch.empty(N, K, device=dev), st)
x = torch.from_numpy(synth.activations(8, K)).to(dev)
F.if_qgemv(s, p, N, K, x, 8, torch.empty(8, N, device=dev))
F.if_qgemm(s, p, N, K, torch.randn(70, K, device=dev).to(torch.bfloat16), 70, torch.empty(70, N, device=dev))
lg = torch.randn(5, 1000, device=dev)
F.if_spec_verify(4, 1000, lg, torch.softmax(torch.randn(4, 1000, device=dev), 1), torch.tensor([1, 2, 3, 4], dtype=torch.int32, device=dev),
                 torch.rand(4, device=dev), 0.3, True, 5, 0.9, torch.empty(5, dtype=torch.int32, device=dev), torch.empty(1, dtype=torch.int32, device=dev))
torch.cuda.synchronize()
print("sanitize_small done")
