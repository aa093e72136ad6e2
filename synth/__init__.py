"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This module holds NO arithmetic of the method (no quantization, no products):
it is the counter-based input generator of DESIGN.md §Inputs, the one thing
both sides may share.  The CUDA library implements the *same* generator as a
device kernel (``if_synth_fill``) so that multi-GB weights can be generated in
HBM; ``tests/test_gpu_kernels.py::test_synth_generator_bitwise`` checks the two bit for bit.

Generator:
  h   = splitmix64(seed ^ tensor_id*0x9E3779B97F4A7C15 ^ idx*0xD1B54A32D192ED03)
  s   = sum_{i<4} ((h >> 16 i) & 0xFFFF) - 131070          (integer, exact in fp32)
  val = float32(s) * c,   c = float32(sigma * sqrt(3) / 65536)
Irwin-Hall(4): mean 0, std sigma, bounded by ±3.46 sigma.  Weights use
sigma = 1/sqrt(hidden), activations sigma = 1.
"""
from __future__ import annotations

import math

import numpy as np

SEED_WEIGHTS = 0x1F
SEED_ACTS = 0x2F
_M64 = (1 << 64) - 1
_G1 = np.uint64(0x9E3779B97F4A7C15)
_G2 = np.uint64(0xD1B54A32D192ED03)
_S1 = np.uint64(0xBF58476D1CE4E5B9)
_S2 = np.uint64(0x94D049BB133111EB)

# tensor ids inside layer l: 8*l + {q,k,v,o,gate,up,down}
TID = {"q": 0, "k": 1, "v": 2, "o": 3, "gate": 4, "up": 5, "down": 6}


def tensor_id(layer: int, name: str) -> int:
    return 8 * layer + TID[name]


def scale(sigma: float) -> np.float32:
    """The fp32 multiplier c passed verbatim to both generators."""
    return np.float32(sigma * math.sqrt(3.0) / 65536.0)


def _splitmix64(z: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        z = z + _G1
        z = (z ^ (z >> np.uint64(30))) * _S1
        z = (z ^ (z >> np.uint64(27))) * _S2
        return z ^ (z >> np.uint64(31))


def fill(seed: int, tid: int, c: np.float32, n: int, offset: int = 0) -> np.ndarray:
    """Elements idx = offset .. offset+n-1 of stream (seed, tid), as fp32."""
    idx = np.arange(offset, offset + n, dtype=np.uint64)
    with np.errstate(over="ignore"):
        base = np.uint64(seed & _M64) ^ (np.uint64(tid & _M64) * _G1)
        h = _splitmix64(base ^ (idx * _G2))
    m = np.uint64(0xFFFF)
    s = ((h & m) + ((h >> np.uint64(16)) & m) + ((h >> np.uint64(32)) & m) + ((h >> np.uint64(48)) & m))
    s = s.astype(np.int64) - 131070
    return s.astype(np.float32) * np.float32(c)


def matrix(seed: int, tid: int, sigma: float, N: int, K: int, row0: int = 0, row1: int | None = None) -> np.ndarray:
    """Rows [row0,row1) of the [N,K] tensor (seed, tid); element (n,k) has idx n*K+k."""
    row1 = N if row1 is None else row1
    return fill(seed, tid, scale(sigma), (row1 - row0) * K, row0 * K).reshape(row1 - row0, K)


def weight(layer: int, name: str, N: int, K: int, hidden: int, row0: int = 0, row1: int | None = None):
    return matrix(SEED_WEIGHTS, tensor_id(layer, name), 1.0 / math.sqrt(hidden), N, K, row0, row1)


def activations(T: int, d: int, tid: int = 0) -> np.ndarray:
    return matrix(SEED_ACTS, tid, 1.0, T, d)


SEED_EMBED = 0x3F
LM_TID = 7  # slot 7 of layer 0's tensor ids (8*l + 7 is unused by the layers)


def embedding(V: int, d: int) -> np.ndarray:
    """Token embedding table [V, d] fp32, sigma = 1 (the stack's input scale)."""
    return matrix(SEED_EMBED, 0, 1.0, V, d)


def lm_head(V: int, d: int) -> np.ndarray:
    """Output projection [V, d] fp32, sigma = 1/sqrt(d) like every weight matrix."""
    return matrix(SEED_WEIGHTS, LM_TID, 1.0 / math.sqrt(d), V, d)


# Llama-2 shapes (BASELINE.json configs)
LLAMA = {
    "7b": dict(layers=32, hidden=4096, heads=32, kv_heads=32, head_dim=128, ffn=11008),
    "13b": dict(layers=40, hidden=5120, heads=40, kv_heads=40, head_dim=128, ffn=13824),
    "70b": dict(layers=80, hidden=8192, heads=64, kv_heads=8, head_dim=128, ffn=28672),
}
