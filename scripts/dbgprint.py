import runpy, sys, numpy as np
sys.argv = ["x", "4"]
g = runpy.run_path("scripts/mk_timeline2.py")
dd = g["dd"]
np.set_printoptions(linewidth=250)
for p in range(0, 6):
    print(p, (dd[0, p, :8] - dd[0, 0, 0]).astype(np.int64), (dd[0, p, 8:] - dd[0, 0, 8]).astype(np.int64))
