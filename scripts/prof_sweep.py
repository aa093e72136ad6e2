"""Time the B=1 Q3H qGEMV vs N at fixed K (intercept = fixed cost, slope = bandwidth)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2401_08294_b200 as F

K = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
s = F.scheme(35, 64)
dev = torch.device("cuda:0")
for N in [148, 1184, 4096, 16384, 65536, 131072]:
    copies = max(2, min(16, (1 << 30) // F.if_packed_bytes(s, N, K)))
    mats = [torch.randint(0, 255, (F.if_packed_bytes(s, N, K),), dtype=torch.uint8, device=dev) for _ in range(copies)]
    for m in mats:  # valid fp16 headers: lo=-0.01 hi=0.01 (0xA11F, 0x211F)
        v = m.view(-1, 32)
        v[:, 0] = 0x1F; v[:, 1] = 0xA1; v[:, 2] = 0x1F; v[:, 3] = 0x21
    x = torch.randn(1, K, device=dev)
    y = torch.empty(1, N, device=dev)
    for m in mats:
        F.if_qgemv(s, m, N, K, x, 1, y)
    torch.cuda.synchronize()
    reps = 10
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        for m in mats:
            F.if_qgemv(s, m, N, K, x, 1, y)
    e1.record(); e1.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / (reps * copies)
    print(f"K={K} N={N:7d} bytes={F.if_packed_bytes(s,N,K)/1e6:8.2f}MB  {us:8.2f} us  {F.if_packed_bytes(s,N,K)/us/1e3:8.1f} GB/s", flush=True)
