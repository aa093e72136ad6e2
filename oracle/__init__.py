"""CPU oracle for the Inferflow block-quantized GEMV/GEMM hot path (arxiv 2401.08294).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` leg may import this
package.  The product path (``paper_2401_08294_b200``) never imports it and
shares no code with it.

This module is argument marshalling (numpy <-> ctypes) over ``oracle.c``; all
of the method's arithmetic lives in ``oracle.c`` (C99, ``-ffp-contract=off``).

Parity status per function:
  quantize/dequantize/pack/unpack/bits_per_weight  pinned (Table 2, Table 3,
      exhaustive pair code, half-step bound, golden bytes)
  matmul_f64                                       pinned (brute force, one-hot,
      constant blocks, linearity)
  plan                                             pinned (Table 4)
  stack_f64                                        parity unpinned by the paper
      (no printed values); pinned only by special cases and by the
      virtual-partition replay.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_SRC = os.path.join(_HERE, "oracle.c")
_lock = threading.Lock()
_lib = None

CFLAGS = ["-O2", "-std=c99", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared", "-Wall"]


def build(force: bool = False) -> str:
    """Compile oracle.c -> liboracle.so with gcc (host only, no CUDA)."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < max(
        os.path.getmtime(_SRC), os.path.getmtime(os.path.join(_HERE, "oracle.h"))
    ):
        tmp = _SO + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *CFLAGS, "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _SO)
    return _SO


def lib():
    global _lib
    with _lock:
        if _lib is None:
            build()
            L = ctypes.CDLL(_SO)
            i32, i64, u16 = ctypes.c_int, ctypes.c_int64, ctypes.c_uint16
            vp = ctypes.c_void_p
            L.ref_scheme_valid.argtypes = [i32, i32]
            L.ref_levels.argtypes = [i32]
            L.ref_code_bytes.argtypes = [i32, i32]
            L.ref_code_bytes.restype = i64
            L.ref_block_bytes.argtypes = [i32, i32]
            L.ref_block_bytes.restype = i64
            L.ref_bits_per_weight.argtypes = [i32, i32, vp, vp]
            L.ref_f32_to_f16_rd.argtypes = [ctypes.c_float]
            L.ref_f32_to_f16_rd.restype = u16
            L.ref_f32_to_f16_ru.argtypes = [ctypes.c_float]
            L.ref_f32_to_f16_ru.restype = u16
            L.ref_f16_to_f32.argtypes = [u16]
            L.ref_f16_to_f32.restype = ctypes.c_float
            L.ref_pack_pair.argtypes = [i32, i32]
            L.ref_unpack_pair.argtypes = [i32, vp, vp]
            L.ref_quantize_block.argtypes = [i32, i32, vp, vp]
            L.ref_dequantize_block.argtypes = [i32, i32, vp, vp]
            L.ref_block_codes.argtypes = [i32, i32, vp, vp]
            L.ref_quantize.argtypes = [i32, i32, vp, i64, i64, vp]
            L.ref_dequantize.argtypes = [i32, i32, vp, i64, i64, vp]
            L.ref_matmul_f64.argtypes = [i32, i32, vp, i64, i64, vp, i64, vp]
            L.ref_stack_f64.argtypes = [vp, vp, vp, vp, vp, vp, i64, vp, vp]
            L.ref_stack_kv_f64.argtypes = [vp, vp, vp, vp, vp, vp, i64, vp, vp, i32, i32, vp, vp, vp, vp]
            L.ref_plan.argtypes = [i32] * 8 + [vp] * 10
            L.ref_spec_verify.argtypes = [i32, i32, vp, vp, vp, vp, ctypes.c_float, i32, i32, ctypes.c_float, vp, vp]
            L.ref_stack_partitioned_f64.argtypes = [vp, i32, i32, i32, i32, vp, vp, vp, vp, vp, i64, vp]
            L.ref_lm_logits_f64.argtypes = [i32, i32, vp, i64, i64, vp, i64, vp]
            L.ref_argmax_f64.argtypes = [vp, i64]
            L.ref_argmax_f64.restype = i64
            L.ref_cost_estimate.argtypes = [i32, i32, i32, ctypes.c_double, ctypes.c_double, ctypes.c_double, vp,
                                             ctypes.c_double, i32, vp, vp]
            _lib = L
    return _lib


class OracleError(RuntimeError):
    def __init__(self, status: int, what: str):
        super().__init__(f"oracle {what}: status {status}")
        self.status = status


def _ptr(a: np.ndarray) -> int:
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data


def _chk(st: int, what: str):
    if st != 0:
        raise OracleError(st, what)


# ---- scheme -----------------------------------------------------------------
QTYPES = {"Q2": 2, "Q3": 3, "Q3H": 35, "Q4": 4, "Q5": 5, "Q6": 6, "Q8": 8}


def scheme_valid(qtype: int, block: int) -> bool:
    return bool(lib().ref_scheme_valid(qtype, block))


def levels(qtype: int) -> int:
    return lib().ref_levels(qtype)


def code_bytes(qtype: int, n: int) -> int:
    return lib().ref_code_bytes(qtype, n)


def block_bytes(qtype: int, block: int) -> int:
    return lib().ref_block_bytes(qtype, block)


def bits_per_weight(qtype: int, block: int):
    num = np.zeros(1, np.int64)
    den = np.zeros(1, np.int64)
    lib().ref_bits_per_weight(qtype, block, _ptr(num), _ptr(den))
    return int(num[0]), int(den[0])


def packed_bytes(qtype: int, block: int, N: int, K: int) -> int:
    return N * (K // block) * block_bytes(qtype, block)


# ---- fp16 helpers -----------------------------------------------------------
def f32_to_f16_rd(f: float) -> int:
    return lib().ref_f32_to_f16_rd(float(np.float32(f)))


def f32_to_f16_ru(f: float) -> int:
    return lib().ref_f32_to_f16_ru(float(np.float32(f)))


def f16_to_f32(h: int) -> float:
    return lib().ref_f16_to_f32(h)


# ---- pair code --------------------------------------------------------------
def pack_pair(a: int, b: int) -> int:
    return lib().ref_pack_pair(a, b)


def unpack_pair(v: int):
    a = np.zeros(1, np.int32)
    b = np.zeros(1, np.int32)
    st = lib().ref_unpack_pair(v, _ptr(a), _ptr(b))
    _chk(st, "unpack_pair")
    return int(a[0]), int(b[0])


# ---- blocks -----------------------------------------------------------------
def quantize_block(qtype: int, w) -> bytes:
    w = np.ascontiguousarray(w, dtype=np.float32)
    out = np.zeros(4 + code_bytes(qtype, w.size), np.uint8)
    _chk(lib().ref_quantize_block(qtype, w.size, _ptr(w), _ptr(out)), "quantize_block")
    return out.tobytes()


def dequantize_block(qtype: int, n: int, blk: bytes) -> np.ndarray:
    b = np.frombuffer(blk, np.uint8).copy()
    out = np.zeros(n, np.float32)
    _chk(lib().ref_dequantize_block(qtype, n, _ptr(b), _ptr(out)), "dequantize_block")
    return out


def block_codes(qtype: int, n: int, blk: bytes) -> np.ndarray:
    b = np.frombuffer(blk, np.uint8).copy()
    out = np.zeros(n, np.int32)
    _chk(lib().ref_block_codes(qtype, n, _ptr(b), _ptr(out)), "block_codes")
    return out


# ---- tensors ----------------------------------------------------------------
def quantize(qtype: int, block: int, W: np.ndarray) -> np.ndarray:
    W = np.ascontiguousarray(W, dtype=np.float32)
    N, K = W.shape
    out = np.zeros(packed_bytes(qtype, block, N, K) if K % block == 0 else 1, np.uint8)
    _chk(lib().ref_quantize(qtype, block, _ptr(W), N, K, _ptr(out)), "quantize")
    return out


def dequantize(qtype: int, block: int, packed: np.ndarray, N: int, K: int) -> np.ndarray:
    packed = np.ascontiguousarray(packed, dtype=np.uint8)
    out = np.zeros((N, K), np.float32)
    _chk(lib().ref_dequantize(qtype, block, _ptr(packed), N, K, _ptr(out)), "dequantize")
    return out


def matmul_f64(qtype: int, block: int, packed: np.ndarray, N: int, K: int, X: np.ndarray) -> np.ndarray:
    """Y[M,N] = X[M,K] . W'^T in fp64; X given as fp32 (the exact values the GPU got)."""
    packed = np.ascontiguousarray(packed, dtype=np.uint8)
    X = np.ascontiguousarray(X, dtype=np.float32)
    if X.ndim == 1:
        X = X[None, :]
    M = X.shape[0]
    Y = np.zeros((M, N), np.float64)
    _chk(lib().ref_matmul_f64(qtype, block, _ptr(packed), N, K, _ptr(X), M, _ptr(Y)), "matmul_f64")
    return Y


# ---- stack ------------------------------------------------------------------
class StackShape(ctypes.Structure):
    _fields_ = [
        ("layers", ctypes.c_int32),
        ("hidden", ctypes.c_int32),
        ("heads", ctypes.c_int32),
        ("kv_heads", ctypes.c_int32),
        ("head_dim", ctypes.c_int32),
        ("ffn", ctypes.c_int32),
        ("qtype", ctypes.c_int32),
        ("block", ctypes.c_int32),
    ]


def _ptr_array(arrs):
    arrs = [np.ascontiguousarray(a, dtype=np.uint8) for a in arrs]
    P = (ctypes.c_void_p * len(arrs))(*[a.ctypes.data for a in arrs])
    return P, arrs


def stack_f64(shape: dict, wqkv, wo, wgu, wdown, h_in: np.ndarray, want_qkv: bool = True):
    s = StackShape(**shape)
    h_in = np.ascontiguousarray(h_in, dtype=np.float32)
    if h_in.ndim == 1:
        h_in = h_in[None, :]
    T = h_in.shape[0]
    nqkv = (shape["heads"] + 2 * shape["kv_heads"]) * shape["head_dim"]
    h_out = np.zeros((T, shape["hidden"]), np.float64)
    qkv = np.zeros((T, nqkv), np.float64)
    P1, k1 = _ptr_array(wqkv)
    P2, k2 = _ptr_array(wo)
    P3, k3 = _ptr_array(wgu)
    P4, k4 = _ptr_array(wdown)
    st = lib().ref_stack_f64(
        ctypes.addressof(s), P1, P2, P3, P4, _ptr(h_in), T, _ptr(h_out), _ptr(qkv) if want_qkv else None
    )
    _chk(st, "stack_f64")
    return h_out, qkv


def stack_kv_f64(shape: dict, wqkv, wo, wgu, wdown, h_in: np.ndarray, slot_ids, positions,
                 kcache: np.ndarray, vcache: np.ndarray):
    """ref_stack_kv_f64: the stack with GQA decode attention over a KV cache (Q24).
    kcache/vcache: fp64 [layers, slots, max_ctx, G, hd], updated in place (the
    caller's per-sequence state).  Returns (h_out fp64 [T, d], last_qkv fp64 with
    RoPE applied to q and k)."""
    s = StackShape(**shape)
    h_in = np.ascontiguousarray(h_in, dtype=np.float32)
    if h_in.ndim == 1:
        h_in = h_in[None, :]
    T = h_in.shape[0]
    slot_ids = np.ascontiguousarray(slot_ids, dtype=np.int32)
    positions = np.ascontiguousarray(positions, dtype=np.int32)
    assert kcache.dtype == np.float64 and kcache.flags.c_contiguous and vcache.shape == kcache.shape
    assert vcache.dtype == np.float64 and vcache.flags.c_contiguous
    L, slots, max_ctx = kcache.shape[:3]
    nqkv = (shape["heads"] + 2 * shape["kv_heads"]) * shape["head_dim"]
    h_out = np.zeros((T, shape["hidden"]), np.float64)
    qkv = np.zeros((T, nqkv), np.float64)
    P1, k1 = _ptr_array(wqkv)
    P2, k2 = _ptr_array(wo)
    P3, k3 = _ptr_array(wgu)
    P4, k4 = _ptr_array(wdown)
    st = lib().ref_stack_kv_f64(ctypes.addressof(s), P1, P2, P3, P4, _ptr(h_in), T, _ptr(slot_ids), _ptr(positions),
                                slots, max_ctx, _ptr(kcache), _ptr(vcache), _ptr(h_out), _ptr(qkv))
    _chk(st, "stack_kv_f64")
    return h_out, qkv


def spec_verify(tgt_logits: np.ndarray, draft_probs: np.ndarray, draft_tok, u_acc, u_smp: float,
                is_top: bool = False, top_k: int = 0, top_p: float = 1.0):
    """ref_spec_verify: one round of Algorithm 1 -> list of output tokens (accepted + 1)."""
    tgt_logits = np.ascontiguousarray(tgt_logits, np.float32)
    draft_probs = np.ascontiguousarray(draft_probs, np.float32)
    K1, V = tgt_logits.shape
    K = K1 - 1
    draft_tok = np.ascontiguousarray(draft_tok, np.int32)
    u_acc = np.ascontiguousarray(u_acc, np.float32)
    out = np.zeros(K + 1, np.int32)
    n = np.zeros(1, np.int32)
    _chk(lib().ref_spec_verify(K, V, _ptr(tgt_logits), _ptr(draft_probs), _ptr(draft_tok), _ptr(u_acc),
                               float(u_smp), int(is_top), int(top_k), float(top_p), _ptr(out), _ptr(n)),
         "spec_verify")
    return out[:n[0]].tolist()


def lm_logits_f64(qtype: int, block: int, lm_packed: np.ndarray, V: int, d: int, h: np.ndarray) -> np.ndarray:
    """ref_lm_logits_f64: final RMSNorm then the quantized output projection (Q27).
    h [T, d] (any float dtype, taken exactly as fp64) -> logits fp64 [T, V]."""
    h = np.ascontiguousarray(np.atleast_2d(h), np.float64)
    T = h.shape[0]
    out = np.zeros((T, V), np.float64)
    _chk(lib().ref_lm_logits_f64(qtype, block, _ptr(np.ascontiguousarray(lm_packed, np.uint8)), V, d, _ptr(h), T,
                                 _ptr(out)), "lm_logits_f64")
    return out


def argmax(x: np.ndarray) -> int:
    """ref_argmax_f64: greedy choice, first index of the maximum."""
    x = np.ascontiguousarray(x, np.float64)
    return int(lib().ref_argmax_f64(_ptr(x), x.size))


def lm_sequence_f64(shape: dict, wqkv, wo, wgu, wdown, embed: np.ndarray, lm_packed: np.ndarray, V: int,
                    prompt, continuation, max_ctx: int):
    """A sequential decode of one query with the plain pieces above (the "direct
    engine loop without batcher" of S:567): embedding rows of the prompt as one causal
    chunk at positions 0..n-1, then every continuation token one position at a time;
    after each call the logits of the last row.  Returns fp64 [1 + len(continuation), V]:
    row j is the target distribution's logits after prompt + continuation[:j]
    (teacher forcing with the tokens the caller emitted)."""
    K, Vc = kv_cache(shape, 1, max_ctx)
    d = shape["hidden"]
    qt, bs = shape["qtype"], shape["block"]
    prompt = list(prompt)
    rows = []
    h, _ = stack_kv_f64(shape, wqkv, wo, wgu, wdown, embed[prompt], [0] * len(prompt), list(range(len(prompt))),
                        K, Vc)
    rows.append(lm_logits_f64(qt, bs, lm_packed, V, d, h[-1:])[0])
    for j, tok in enumerate(continuation):
        h, _ = stack_kv_f64(shape, wqkv, wo, wgu, wdown, embed[[tok]], [0], [len(prompt) + j], K, Vc)
        rows.append(lm_logits_f64(qt, bs, lm_packed, V, d, h)[0])
    return np.stack(rows)


def cost_estimate(layers: int, stages: int, groups: int, t_fixed: float, layer_bytes: float, bw: float, t_merge,
                  t_hop: float, micro_batches: int = 1):
    """ref_cost_estimate (Q29) -> (decode tokens/s, throughput tokens/s).  t_merge:
    sequence indexed by group size (entry g = latency of one g-way merge)."""
    tm = np.zeros(9, np.float64)
    for g, v in enumerate(list(t_merge)[:9]):
        tm[g] = v
    dec, thr = ctypes.c_double(), ctypes.c_double()
    _chk(lib().ref_cost_estimate(layers, stages, groups, float(t_fixed), float(layer_bytes), float(bw), _ptr(tm),
                                 float(t_hop), micro_batches, ctypes.byref(dec), ctypes.byref(thr)), "cost_estimate")
    return dec.value, thr.value


def plan_auto(objective: str, layers: int, heads: int, kv_heads: int, ffn_blocks: int, devices: int, cost: dict,
              layer_bytes: float, micro_batches: int = 1):
    """The grid (stages, groups), stages x groups = devices, that a valid plan admits
    (ref_plan succeeds) and that maximises the objective ("decode" or "throughput");
    ties keep the grid found first, in order of increasing groups."""
    best = None
    for groups in range(1, devices + 1):
        if devices % groups:
            continue
        stages = devices // groups
        strategy = 0 if groups == 1 else (1 if stages == 1 else 2)
        try:
            plan(strategy, layers, heads, kv_heads, ffn_blocks, devices, stages, groups)
        except OracleError:
            continue
        dec, thr = cost_estimate(layers, stages, groups, cost["t_fixed"], layer_bytes, cost["bw"], cost["t_merge"],
                                 cost["t_hop"], micro_batches)
        val = dec if objective == "decode" else thr
        if best is None or val > best[0]:
            best = (val, stages, groups, dec, thr)
    return best


def kv_cache(shape: dict, slots: int, max_ctx: int):
    """A fresh (zeroed) oracle KV cache pair for stack_kv_f64."""
    dims = (shape["layers"], slots, max_ctx, shape["kv_heads"], shape["head_dim"])
    return np.zeros(dims, np.float64), np.zeros(dims, np.float64)


def stack_partitioned_f64(shape: dict, strategy: int, devices: int, stages: int, groups: int,
                          wqkv, wo, wgu, wdown, h_in: np.ndarray):
    s = StackShape(**shape)
    h_in = np.ascontiguousarray(h_in, dtype=np.float32)
    if h_in.ndim == 1:
        h_in = h_in[None, :]
    T = h_in.shape[0]
    h_out = np.zeros((T, shape["hidden"]), np.float64)
    P1, k1 = _ptr_array(wqkv)
    P2, k2 = _ptr_array(wo)
    P3, k3 = _ptr_array(wgu)
    P4, k4 = _ptr_array(wdown)
    st = lib().ref_stack_partitioned_f64(
        ctypes.addressof(s), strategy, devices, stages, groups, P1, P2, P3, P4, _ptr(h_in), T, _ptr(h_out)
    )
    _chk(st, "stack_partitioned_f64")
    return h_out


def plan(strategy: int, layers: int, heads: int, kv_heads: int, ffn_blocks: int, devices: int,
         stages: int = 0, groups: int = 0):
    """Returns a list of dicts (one per device) with 0-based half-open ranges."""
    arrs = [np.zeros(max(devices, 1), np.int32) for _ in range(10)]
    st = lib().ref_plan(strategy, layers, heads, kv_heads, ffn_blocks, devices, stages, groups,
                        *[_ptr(a) for a in arrs])
    _chk(st, "plan")
    keys = ["stage", "group_rank", "layer_begin", "layer_end", "head_begin", "head_end",
            "kv_begin", "kv_end", "ffn_blk_begin", "ffn_blk_end"]
    return [{k: int(a[d]) for k, a in zip(keys, arrs)} for d in range(devices)]
