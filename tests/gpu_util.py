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


def oracle_stack_per_token(shape: dict, wq, wo, wgu, wd, h: np.ndarray, threads: int = 0):
    """O.stack_f64 on every token row separately, rows run concurrently (the oracle's
    C call releases the GIL).  Tokens are independent in the stack (Q18: each
    token's attention sees only its own position), so the result equals one
    O.stack_f64 call on all rows; this only spreads the fp64 work over host cores."""
    import os
    from concurrent.futures import ThreadPoolExecutor

    import oracle as O
    T = h.shape[0]
    n = threads or min(T, os.cpu_count() or 1)
    with ThreadPoolExecutor(max(1, n)) as ex:
        outs = list(ex.map(lambda t: O.stack_f64(shape, wq, wo, wgu, wd, h[t:t + 1]), range(T)))
    return np.concatenate([o[0] for o in outs]), np.concatenate([o[1] for o in outs])


def oracle_rows_matmul(qtype: int, bs: int, packed: np.ndarray, N: int, K: int, X: np.ndarray, rows):
    """O.matmul_f64 of the sampled output rows `rows` only (packed rows are contiguous)."""
    import oracle as O
    rb = O.packed_bytes(qtype, bs, 1, K)
    sub = np.concatenate([packed[r * rb:(r + 1) * rb] for r in rows])
    return O.matmul_f64(qtype, bs, sub, len(rows), K, X)
