"""Per-CTA timeline of the prefill tensor-core qGEMM (IFB_TC_PROF build):
start, mainloop end (accumulator ready) and epilogue end per CTA, grouped by SM.

  IFB_NVCC_FLAGS=-DIFB_TC_PROF IFB_LIB_OUT=.../libif_P.so IFB_BUILD_DIR=.../_build_P python -c 'import ...build'
  IFB_LIB_PATH=.../libif_P.so python scripts/tc_timeline.py [--M 512] [--scheme Q3H:64]
"""
import argparse, ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2401_08294_b200 as F
from paper_2401_08294_b200 import _lib

ap = argparse.ArgumentParser()
ap.add_argument("--M", type=int, default=512)
ap.add_argument("--N", type=int, default=12288)
ap.add_argument("--K", type=int, default=4096)
ap.add_argument("--scheme", default="Q3H:64")
a = ap.parse_args()
dev = torch.device("cuda:0")
name, bs = a.scheme.split(":")
s = F.scheme(name, int(bs))
N, K, M = a.N, a.K, a.M
W = torch.empty(F.if_packed_bytes(s, N, K), dtype=torch.uint8, device=dev)
scratch = torch.empty(N * K, device=dev)
F.if_synth_fill(0x1F, 1, 1 / 64, scratch)
F.if_quantize(s, scratch, N, K, W)
X = torch.randn(M, K, device=dev).to(torch.bfloat16)
Y = torch.empty(M, N, device=dev)
for _ in range(3):
    F.if_qgemm(s, W, N, K, X.view(torch.int16), M, Y)
torch.cuda.synchronize()
lib = _lib.load()
buf = np.zeros((8192, 4), np.uint64)
lib.ifx_tc_tl(buf.ctypes.data_as(ctypes.c_void_p))
ctas = buf[buf[:, 1] > 0].astype(np.int64)
t0 = ctas[:, 1].min()
st, ml, ep = ctas[:, 1] - t0, ctas[:, 2] - t0, ctas[:, 3] - t0
print(f"{a.scheme} {M}x{N}x{K}: {len(ctas)} CTAs, span {ep.max() / 1e3:.1f} us")
print(f"  mainloop (start->acc ready) median {np.median(ml - st) / 1e3:.2f} us  max {np.max(ml - st) / 1e3:.2f}")
print(f"  epilogue (acc ready->end)   median {np.median(ep - ml) / 1e3:.2f} us  max {np.max(ep - ml) / 1e3:.2f}")
gaps = []
for sm in np.unique(ctas[:, 0]):
    idx = np.argsort(st[ctas[:, 0] == sm])
    s_sm, e_sm = st[ctas[:, 0] == sm][idx], ep[ctas[:, 0] == sm][idx]
    gaps += list(s_sm[1:] - e_sm[:-1])
if gaps:
    print(f"  gap end->next start on an SM: median {np.median(gaps) / 1e3:.2f} us  max {np.max(gaps) / 1e3:.2f}")
starts = np.sort(st)
for w in range(0, len(starts), 148):
    sel = (st >= starts[w]) & (st <= starts[min(w + 147, len(starts) - 1)])
    print(f"  wave {w // 148}: start {starts[w] / 1e3:7.2f} us .. last end {ep[sel].max() / 1e3:7.2f} us")
