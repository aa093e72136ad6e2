"""Build libif_b200.so in-tree: every csrc/*.cu compiled for sm_100a with nvcc.

    python -m paper_2401_08294_b200.build [--force] [-j N]

Flags: -gencode arch=compute_100a,code=sm_100a (tcgen05 needs the "a"
target), -O3 -lineinfo, C++20, no --use_fast_math (the codec kernels are
bit-exact with the oracle only under IEEE arithmetic).
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
ROOT = os.path.dirname(HERE)
OUT = os.environ.get("IFB_LIB_OUT", os.path.join(HERE, "libif_b200.so"))  # experiments: variant libraries
BUILD = os.environ.get("IFB_BUILD_DIR", os.path.join(HERE, "_build"))
EXTRA = os.environ.get("IFB_NVCC_FLAGS", "").split()

NVCC = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++20", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
                "-I", os.path.join(ROOT, "include"), "-Xptxas", "-warn-spills"]


def _sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def _headers():
    return sorted(glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(ROOT, "include", "*.h")))


def _newest(paths):
    return max((os.path.getmtime(p) for p in paths), default=0.0)


def _compile(src: str, force: bool) -> str:
    obj = os.path.join(BUILD, os.path.basename(src)[:-3] + ".o")
    if force or not os.path.exists(obj) or os.path.getmtime(obj) < max(os.path.getmtime(src), _newest(_headers())):
        flags = list(FLAGS)
        with open(src) as f:  # per-file override, e.g. "// ifb-build: -std=c++17" on line 1..5
            for line in [f.readline() for _ in range(5)]:
                if line.startswith("// ifb-build:"):
                    for opt in line.split(":", 1)[1].split():
                        if opt.startswith("-std="):
                            flags = [x for x in flags if not x.startswith("-std=")]
                        flags.append(opt)
        cmd = [NVCC, *flags, *EXTRA, "-c", src, "-o", obj + ".tmp"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
        os.replace(obj + ".tmp", obj)
    return obj


def build(force: bool = False, jobs: int | None = None) -> str:
    os.makedirs(BUILD, exist_ok=True)
    srcs = _sources()
    jobs = jobs or min(len(srcs), os.cpu_count() or 4)
    with cf.ThreadPoolExecutor(jobs) as ex:
        objs = list(ex.map(lambda s: _compile(s, force), srcs))
    if force or not os.path.exists(OUT) or os.path.getmtime(OUT) < _newest(objs):
        tmp = OUT + f".tmp{os.getpid()}"
        cmd = [NVCC, *ARCH, "-shared", "-o", tmp, *objs, "-lcudart", "-ldl"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
        os.replace(tmp, OUT)
    return OUT


if __name__ == "__main__":
    force = "--force" in sys.argv
    j = None
    if "-j" in sys.argv:
        j = int(sys.argv[sys.argv.index("-j") + 1])
    print(build(force, j))
