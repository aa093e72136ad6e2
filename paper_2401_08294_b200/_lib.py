"""ctypes binding of libif_b200.so (include/if_b200.h).  Argument marshalling only.

Loading fails loudly when the library is missing: there is no CPU fallback.
"""
from __future__ import annotations

import ctypes
import os
import re

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
LIB_PATH = os.environ.get("IFB_LIB_PATH", os.path.join(HERE, "libif_b200.so"))  # override: experiments only
HEADER = os.path.join(ROOT, "include", "if_b200.h")

i32, i64, u64, f32, vp = ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64, ctypes.c_float, ctypes.c_void_p


class Scheme(ctypes.Structure):
    _fields_ = [("type", i32), ("block", i32)]


class StackShape(ctypes.Structure):
    _fields_ = [("layers", i32), ("hidden", i32), ("heads", i32), ("kv_heads", i32), ("head_dim", i32),
                ("ffn", i32), ("scheme", Scheme)]


class Assignment(ctypes.Structure):
    _fields_ = [(n, i32) for n in ("rank", "stage", "group_rank", "layer_begin", "layer_end", "head_begin",
                                   "head_end", "kv_begin", "kv_end", "ffn_blk_begin", "ffn_blk_end")]


class Plan(ctypes.Structure):
    _fields_ = [("strategy", i32), ("devices", i32), ("stages", i32), ("groups", i32), ("a", Assignment * 8)]


class KvCache(ctypes.Structure):
    _fields_ = [("k", vp), ("v", vp), ("slots", i32), ("max_ctx", i32), ("status", vp)]


class LayerWeights(ctypes.Structure):
    _fields_ = [("wqkv", vp), ("wo", vp), ("wgu", vp), ("wdown", vp)]


class CostModel(ctypes.Structure):
    _fields_ = [("t_fixed_s", ctypes.c_double), ("bw_bytes_s", ctypes.c_double), ("t_merge_s", ctypes.c_double * 9),
                ("t_hop_s", ctypes.c_double)]


class EngineConfig(ctypes.Structure):
    _fields_ = [("shape", StackShape), ("layers", vp), ("embed", vp), ("lm_head", vp), ("vocab", i32),
                ("slots", i32), ("max_ctx", i32), ("step_tokens", i32)]


_SIGS = {
    "if_block_bytes": (i64, [Scheme]),
    "if_packed_bytes": (i64, [Scheme, i64, i64]),
    "if_bits_per_weight": (i32, [Scheme, vp, vp]),
    "if_synth_fill": (i32, [u64, u64, f32, vp, i64, i64, vp]),
    "if_quantize": (i32, [Scheme, vp, i64, i64, vp, vp, vp]),
    "if_dequantize": (i32, [Scheme, vp, i64, i64, vp, vp, vp]),
    "if_qgemv": (i32, [Scheme, vp, i64, i64, vp, i64, vp, vp]),
    "if_qgemv_acc": (i32, [Scheme, vp, i64, i64, vp, i64, vp, vp]),
    "if_qgemm": (i32, [Scheme, vp, i64, i64, vp, i64, vp, vp]),
    "if_plan_partition": (i32, [i32, vp, i32, i32, i32, vp]),
    "if_comm_nccl_unique_id": (i32, [vp]),
    "if_comm_init": (i32, [vp, i32, vp, vp]),
    "if_comm_create": (i32, [vp, i32, i64, i32, vp]),
    "if_comm_ipc_handle": (i32, [vp, vp]),
    "if_comm_open_peers": (i32, [vp, vp]),
    "if_comm_destroy": (i32, [vp]),
    "if_comm_create_local": (i32, [vp, i64, i32, vp]),
    "if_comm_allreduce": (i32, [vp, vp, i64, vp]),
    "if_comm_send_next": (i32, [vp, vp, i64, vp]),
    "if_comm_recv_prev": (i32, [vp, vp, i64, vp]),
    "if_stack_workspace_bytes": (i32, [vp, vp, i32, i64, i32, vp]),
    "if_run_stack": (i32, [vp, vp, i32, vp, vp, vp, i64, i32, vp, vp, vp, vp]),
    "if_kv_cache_bytes": (i32, [vp, vp, i32, i32, i32, vp]),
    "if_run_stack_kv": (i32, [vp, vp, i32, vp, vp, vp, i64, i32, vp, vp, vp, vp, vp, vp, vp]),
    "if_embed": (i32, [vp, i32, i32, vp, i64, vp, vp, vp]),
    "if_lm_logits": (i32, [Scheme, vp, i64, i64, vp, i64, vp, vp, vp, vp]),
    "if_argmax": (i32, [vp, i64, i64, vp, vp]),
    "if_spec_verify": (i32, [i32, i64, vp, vp, vp, vp, f32, i32, i32, f32, vp, vp, vp]),
    "if_engine_create": (i32, [vp, vp]),
    "if_engine_add_query": (i32, [vp, vp, i32, i32, i32, vp]),
    "if_engine_infer": (i32, [vp, vp, vp, i32, vp, vp]),
    "if_engine_verify": (i32, [vp, i64, i32, vp, vp, vp, f32, i32, i32, f32, vp, vp, vp]),
    "if_engine_query": (i32, [vp, i64, vp, vp, vp]),
    "if_engine_last_logits": (i32, [vp, vp, vp, vp]),
    "if_engine_destroy": (i32, [vp]),
    "if_container_save": (i32, [ctypes.c_char_p, i32, vp, vp, vp, vp, vp, i32, vp]),
    "if_container_open": (i32, [ctypes.c_char_p, vp]),
    "if_container_count": (i32, [vp]),
    "if_container_info": (i32, [vp, i32, vp, i32, vp, vp, vp, vp]),
    "if_container_find": (i32, [vp, ctypes.c_char_p, vp]),
    "if_container_load": (i32, [vp, i32, vp, vp]),
    "if_container_read_host": (i32, [vp, i32, vp]),
    "if_container_close": (i32, [vp]),
    "if_cost_estimate": (i32, [vp, i32, i32, vp, i32, vp, vp]),
    "if_plan_auto": (i32, [i32, vp, i32, vp, i32, vp, vp, vp]),
    "if_last_error": (ctypes.c_char_p, []),
    "if_launch_count": (i64, [i32]),
}

_lib = None


def header_symbols() -> list[str]:
    """Every function declared in include/if_b200.h."""
    with open(HEADER) as f:
        txt = f.read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(if_[a-z0-9_]+)\s*\(", txt)))


def load():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `python -m paper_2401_08294_b200.build` "
                "(there is no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib
