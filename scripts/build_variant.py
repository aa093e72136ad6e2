"""Build an experiment variant of libif_b200.so from a csrc directory (A/B only).
    python scripts/build_variant.py CSRC_DIR OUT_NAME [extra nvcc flags...]
-> paper_2401_08294_b200/OUT_NAME.so (travels to the GPU box with the snapshot)."""
import os, subprocess, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2401_08294_b200 import build as B
src, name, extra = sys.argv[1], sys.argv[2], sys.argv[3:]
B.CSRC = src
B.OUT = os.path.join(os.path.dirname(B.__file__), name + ".so")
B.BUILD = f"/tmp/build_{name}"
B.EXTRA = extra
print(B.build(force=True))
