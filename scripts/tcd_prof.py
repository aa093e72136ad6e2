"""Where the batched-decode MMA thread's time goes (IFB_TCD_PROF build):
per CTA cycles waiting for the x tile, for the W' tile, issuing MMAs + commit."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2401_08294_b200 as F
B = int(sys.argv[1]) if len(sys.argv) > 1 else 8
N = int(sys.argv[2]) if len(sys.argv) > 2 else 16384
K = 4096
s = F.scheme(35, 64)
dev = torch.device("cuda:0")
p = torch.randint(0, 120, (F.if_packed_bytes(s, N, K),), dtype=torch.uint8, device=dev)
v = p.view(-1, 32); v[:, 0] = 0x1F; v[:, 1] = 0xA1; v[:, 2] = 0x1F; v[:, 3] = 0x21
x = torch.randn(B, K, device=dev); y = torch.empty(B, N, device=dev)
for _ in range(3):
    F.if_qgemv(s, p, N, K, x, B, y)
torch.cuda.synchronize()
from paper_2401_08294_b200 import _lib
buf = np.zeros((4096, 8), dtype=np.uint64)
_lib.load().ifx_tcd_prof(buf.ctypes.data_as(ctypes.c_void_p))
b = buf[buf[:, 3] > 0].astype(np.float64) / 1965.0
print(f"B={B} N={N} CTAs={len(b)}  median us  MMA thread: wait_x {np.median(b[:,0]):.2f}  wait_W' {np.median(b[:,1]):.2f}  "
      f"issue+commit {np.median(b[:,2]):.2f}  total {np.median(b[:,3]):.2f}")
print(f"  dequant (warp 2 lane 0): wait weight slot {np.median(b[:,4]):.2f}  wait free stage {np.median(b[:,5]):.2f}  "
      f"dequant+arrive {np.median(b[:,6]):.2f}  total {np.median(b[:,7]):.2f}")
