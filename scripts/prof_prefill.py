"""Prefill (a5) throughput: the 7B-shaped stack at M tokens per scheme, and the
bare qGEMM per stack shape.  Times CUDA-graph replays with CUDA events.

  python scripts/prof_prefill.py [--M 512] [--schemes Q3H:64,Q4:32,...] [--layers 32]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2401_08294_b200 as F
import synth
from paper_2401_08294_b200.model import Stack

SCHEMES = "Q2:32,Q2:64,Q3:32,Q3H:64,Q4:32,Q4:64,Q5:64,Q6:64,Q8:32,Q8:64"


def time_graph(fn, reps=5, warm=2):
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        fn(s)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            fn(s)
    for _ in range(warm):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        g.replay()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--M", type=int, default=512)
    ap.add_argument("--schemes", default=SCHEMES)
    ap.add_argument("--layers", type=int, default=32)
    ap.add_argument("--gemm-only", action="store_true")
    a = ap.parse_args()
    dev = torch.device("cuda:0")
    cfg = dict(synth.LLAMA["7b"], layers=a.layers)
    M, d = a.M, cfg["hidden"]
    flops_layer = 2 * M * d * ((cfg["heads"] + 2 * cfg["kv_heads"]) * cfg["head_dim"] + d + 2 * cfg["ffn"]) + \
        2 * M * cfg["ffn"] * d
    for spec in a.schemes.split(","):
        name, bs = spec.split(":")
        s = F.scheme(name, int(bs))
        # bare GEMM on the qkv shape
        N, K = 12288, 4096
        W = torch.empty(F.if_packed_bytes(s, N, K), dtype=torch.uint8, device=dev)
        scratch = torch.empty(N * K, device=dev)
        F.if_synth_fill(0x1F, 1, 1 / 64, scratch)
        F.if_quantize(s, scratch, N, K, W)
        del scratch
        X = torch.randn(M, K, device=dev).to(torch.bfloat16)
        Y = torch.empty(M, N, device=dev)
        ms = time_graph(lambda st: F.if_qgemm(s, W, N, K, X.view(torch.int16), M, Y, st))
        print(f"{spec:7s} qGEMM {M}x{N}x{K}: {ms * 1e3:8.1f} us  {2 * M * N * K / ms / 1e9:7.1f} TFLOP/s", flush=True)
        if a.gemm_only:
            continue
        shape = F.stack_shape(*[cfg[k] for k in ("layers", "hidden", "heads", "kv_heads", "head_dim", "ffn")], s)
        plan = F.if_plan_partition(F.IF_BY_LAYER, shape, 1)
        stk = Stack(cfg, s, plan, 0, dev)
        h = torch.randn(M, d, device=dev)
        out = torch.empty_like(h)
        ws = torch.zeros(F.if_stack_workspace_bytes(shape, plan, 0, M, F.IF_PREFILL), dtype=torch.uint8, device=dev)
        ms = time_graph(lambda st: F.if_run_stack(shape, plan, 0, None, stk.arr, h, M, F.IF_PREFILL, out, None, ws, st))
        print(f"{spec:7s} stack prefill M={M} L={cfg['layers']}: {ms:8.3f} ms  {M / ms * 1e3:9.0f} tokens/s  "
              f"{flops_layer * cfg['layers'] / ms / 1e9:7.1f} TFLOP/s  weights {stk.weight_bytes() / 1e9:.2f} GB", flush=True)
        del stk, ws


if __name__ == "__main__":
    main()
