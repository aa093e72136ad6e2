"""Helpers for the -m gpu parity tests (tests only)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

SCHEMES = [(2, 32), (2, 64), (3, 32), (3, 64), (4, 32), (4, 64), (5, 32), (5, 64), (6, 32), (6, 64), (8, 32),
           (8, 64), (35, 32), (35, 64)]


def dev():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda:0")


def normwise(got, ref):
    """||got - ref||_inf / ||ref||_inf per output tensor (Q16)."""
    got = np.asarray(got, np.float64)
    ref = np.asarray(ref, np.float64)
    den = np.abs(ref).max()
    return float(np.abs(got - ref).max() / (den if den > 0 else 1.0))


def to_bf16_exact(a: np.ndarray):
    """fp32 -> bf16 (torch RN) and back: the exact bf16 values handed to the GPU."""
    t = torch.from_numpy(np.ascontiguousarray(a, np.float32)).to(torch.bfloat16)
    return t, t.to(torch.float32).numpy()
