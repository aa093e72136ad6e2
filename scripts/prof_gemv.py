"""Profile the qGEMV on the 7B stack shapes (for ncu / event timing).

  python scripts/prof_gemv.py [--reps 20] [--copies 8] [--B 1] [--shapes qkv,o,gu,down]

Each shape gets `copies` distinct packed matrices (rotated, > L2 in total) so
launches stream from HBM.  Prints per-shape average launch time and GB/s.
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch

import paper_2401_08294_b200 as F

SHAPES = {"qkv": (12288, 4096), "o": (4096, 4096), "gu": (22016, 4096), "down": (4096, 11008)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--copies", type=int, default=8)
    ap.add_argument("--B", type=int, default=1)
    ap.add_argument("--shapes", default="qkv,o,gu,down")
    ap.add_argument("--qtype", type=int, default=35)
    ap.add_argument("--block", type=int, default=64)
    a = ap.parse_args()
    dev = torch.device("cuda:0")
    s = F.scheme(a.qtype, a.block)
    for name in a.shapes.split(","):
        N, K = SHAPES[name]
        scratch = torch.empty(N * K, device=dev)
        mats = []
        for c in range(a.copies):
            F.if_synth_fill(0x1F, 1000 + c, 1.0 / 64, scratch)
            p = torch.empty(F.if_packed_bytes(s, N, K), dtype=torch.uint8, device=dev)
            F.if_quantize(s, scratch, N, K, p)
            mats.append(p)
        del scratch
        x = torch.randn(a.B, K, device=dev)
        y = torch.empty(a.B, N, device=dev)
        for p in mats:
            F.if_qgemv(s, p, N, K, x, a.B, y)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.reps):
            for p in mats:
                F.if_qgemv(s, p, N, K, x, a.B, y)
        e1.record()
        e1.synchronize()
        n = a.reps * len(mats)
        us = e0.elapsed_time(e1) * 1e3 / n
        gbs = F.if_packed_bytes(s, N, K) / (us * 1e-6) / 1e9
        print(f"{name:5s} N={N:6d} K={K:6d} B={a.B}: {us:8.2f} us/launch  {gbs:8.1f} GB/s")


if __name__ == "__main__":
    main()
