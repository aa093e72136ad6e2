"""Batched-decode qGEMV (tensor cores) time vs N at fixed K: intercept = fixed cost, slope = streaming rate.
  python scripts/prof_tc_sweep.py B [K]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2401_08294_b200 as F
B = int(sys.argv[1]) if len(sys.argv) > 1 else 8
K = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
s = F.scheme(35, 64)
dev = torch.device("cuda:0")
for N in [128, 1184, 4096, 16384, 65536]:
    p = torch.randint(0, 120, (F.if_packed_bytes(s, N, K),), dtype=torch.uint8, device=dev)
    v = p.view(-1, 32); v[:, 0] = 0x1F; v[:, 1] = 0xA1; v[:, 2] = 0x1F; v[:, 3] = 0x21
    x = torch.randn(B, K, device=dev)
    y = torch.empty(B, N, device=dev)
    for _ in range(3):
        F.if_qgemv(s, p, N, K, x, B, y)
    torch.cuda.synchronize()
    reps = 20
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        F.if_qgemv(s, p, N, K, x, B, y)
    e1.record(); e1.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / reps
    print(f"B={B} K={K} N={N:6d} {F.if_packed_bytes(s,N,K)/1e6:8.2f} MB {us:8.1f} us {F.if_packed_bytes(s,N,K)/us/1e3:8.1f} GB/s", flush=True)
