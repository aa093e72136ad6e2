"""B200-native block-quantized GEMV/GEMM for Inferflow's hot path (arxiv 2401.08294).

Thin Python binding over the C ABI of include/if_b200.h (libif_b200.so): the
functions here carry the C names and only marshal arguments (torch CUDA
tensors -> device pointers, current CUDA stream).  Every step of the path runs
in the library's sm_100a kernels; there is no CPU or PyTorch fallback and a
missing library raises at import of the first call.
"""
from __future__ import annotations

import ctypes

from . import _lib
from ._lib import Assignment, CostModel, EngineConfig, KvCache, LayerWeights, Plan, Scheme, StackShape

QTYPES = {"Q2": 2, "Q3": 3, "Q3H": 35, "Q4": 4, "Q5": 5, "Q6": 6, "Q8": 8}
IF_BY_LAYER, IF_BY_TENSOR, IF_HYBRID = 0, 1, 2
IF_DECODE, IF_PREFILL = 0, 1
STATUS = {0: "OK", 1: "ARG", 2: "SHAPE", 3: "SCHEME", 4: "INPUT", 5: "DECODE", 6: "PLAN", 7: "GRID",
          8: "CUDA", 9: "COMM", 10: "UNSUPPORTED", 11: "IO"}


class IFError(RuntimeError):
    def __init__(self, status: int, fn: str):
        msg = _lib.load().if_last_error().decode(errors="replace")
        super().__init__(f"{fn}: IF_ERR_{STATUS.get(status, status)}: {msg}")
        self.status = status


def _check(st: int, fn: str):
    if st != 0:
        raise IFError(st, fn)


def lib():
    return _lib.load()


def scheme(qtype, block: int = 64) -> Scheme:
    if isinstance(qtype, str):
        qtype = QTYPES[qtype]
    return Scheme(int(qtype), int(block))


def _ptr(t) -> int:
    if t is None:
        return None
    return t.data_ptr()


def _stream(stream):
    if stream is None:
        import torch
        return torch.cuda.current_stream().cuda_stream
    if hasattr(stream, "cuda_stream"):
        return stream.cuda_stream
    return int(stream)


# ---- sizes ------------------------------------------------------------------
def if_block_bytes(s: Scheme) -> int:
    return lib().if_block_bytes(s)


def if_packed_bytes(s: Scheme, N: int, K: int) -> int:
    return lib().if_packed_bytes(s, N, K)


def if_bits_per_weight(s: Scheme):
    num, den = ctypes.c_int64(), ctypes.c_int64()
    _check(lib().if_bits_per_weight(s, ctypes.byref(num), ctypes.byref(den)), "if_bits_per_weight")
    return num.value, den.value


# ---- kernels ------------------------------------------------------------------
def if_synth_fill(seed: int, tensor_id: int, scale: float, out, offset: int = 0, stream=None):
    _check(lib().if_synth_fill(seed, tensor_id, float(scale), _ptr(out), out.numel(), offset, _stream(stream)),
           "if_synth_fill")


def if_quantize(s: Scheme, W, N: int, K: int, packed, dev_status=None, stream=None):
    _check(lib().if_quantize(s, _ptr(W), N, K, _ptr(packed), _ptr(dev_status), _stream(stream)), "if_quantize")


def if_dequantize(s: Scheme, packed, N: int, K: int, W_out, dev_status=None, stream=None):
    _check(lib().if_dequantize(s, _ptr(packed), N, K, _ptr(W_out), _ptr(dev_status), _stream(stream)),
           "if_dequantize")


def if_qgemv(s: Scheme, W, N: int, K: int, x, B: int, y, stream=None):
    _check(lib().if_qgemv(s, _ptr(W), N, K, _ptr(x), B, _ptr(y), _stream(stream)), "if_qgemv")


def if_qgemv_acc(s: Scheme, W, N: int, K: int, x, B: int, y, stream=None):
    _check(lib().if_qgemv_acc(s, _ptr(W), N, K, _ptr(x), B, _ptr(y), _stream(stream)), "if_qgemv_acc")


def if_qgemm(s: Scheme, W, N: int, K: int, X_bf16, M: int, Y, stream=None):
    _check(lib().if_qgemm(s, _ptr(W), N, K, _ptr(X_bf16), M, _ptr(Y), _stream(stream)), "if_qgemm")


# ---- partition ----------------------------------------------------------------
def stack_shape(layers, hidden, heads, kv_heads, head_dim, ffn, s: Scheme) -> StackShape:
    return StackShape(layers, hidden, heads, kv_heads, head_dim, ffn, s)


def if_plan_partition(strategy: int, shape: StackShape, devices: int, stages: int = 0, groups: int = 0) -> Plan:
    p = Plan()
    _check(lib().if_plan_partition(strategy, ctypes.byref(shape), devices, stages, groups, ctypes.byref(p)),
           "if_plan_partition")
    return p


# ---- communicator -------------------------------------------------------------
def if_comm_nccl_unique_id() -> bytes:
    buf = (ctypes.c_uint8 * 128)()
    _check(lib().if_comm_nccl_unique_id(buf), "if_comm_nccl_unique_id")
    return bytes(buf)


class Comm:
    """Peer-memory communicator (if_comm_*).  Handles are exchanged through
    torch.distributed.all_gather_object (plumbing only)."""

    def __init__(self, plan: Plan, rank: int, max_tokens: int = 0, hidden: int = 0, nccl_id: bytes | None = None):
        self.h = ctypes.c_void_p()
        self.plan = plan
        if nccl_id is not None:
            idb = (ctypes.c_uint8 * 128).from_buffer_copy(nccl_id)
            _check(lib().if_comm_init(ctypes.byref(plan), rank, idb, ctypes.byref(self.h)), "if_comm_init")
            self.kind = "nccl"
            return
        _check(lib().if_comm_create(ctypes.byref(plan), rank, max_tokens, hidden, ctypes.byref(self.h)),
               "if_comm_create")
        self.kind = "peer"

    @classmethod
    def nccl(cls, plan: Plan, rank: int, group=None):
        """NCCL communicator (if_comm_init); rank 0's unique id is broadcast with
        torch.distributed (plumbing only)."""
        import torch.distributed as dist
        obj = [if_comm_nccl_unique_id() if rank == 0 else None]
        if dist.is_initialized() and dist.get_world_size(group) > 1:
            dist.broadcast_object_list(obj, src=0, group=group)
        return cls(plan, rank, nccl_id=obj[0])

    def ipc_handle(self) -> bytes:
        buf = (ctypes.c_uint8 * 64)()
        _check(lib().if_comm_ipc_handle(self.h, buf), "if_comm_ipc_handle")
        return bytes(buf)

    def open_peers(self, handles: list[bytes]):
        blob = b"".join(handles)
        buf = (ctypes.c_uint8 * len(blob)).from_buffer_copy(blob)
        _check(lib().if_comm_open_peers(self.h, buf), "if_comm_open_peers")

    def exchange(self, group=None):
        if self.kind == "nccl":  # NCCL set itself up in if_comm_init
            return
        import torch.distributed as dist
        hs = [None] * dist.get_world_size(group)
        dist.all_gather_object(hs, self.ipc_handle(), group=group)
        self.open_peers(hs)

    def allreduce(self, buf, stream=None):
        _check(lib().if_comm_allreduce(self.h, _ptr(buf), buf.numel(), _stream(stream)), "if_comm_allreduce")

    def send_next(self, buf, stream=None):
        _check(lib().if_comm_send_next(self.h, _ptr(buf), buf.numel(), _stream(stream)), "if_comm_send_next")

    def recv_prev(self, buf, stream=None):
        _check(lib().if_comm_recv_prev(self.h, _ptr(buf), buf.numel(), _stream(stream)), "if_comm_recv_prev")

    @classmethod
    def local(cls, plan: Plan, max_tokens: int, hidden: int):
        """Every rank's peer-memory communicator in this process on the current device
        (if_comm_create_local): run a multi-rank plan on one GPU as concurrent streams."""
        hs = (ctypes.c_void_p * plan.devices)()
        _check(lib().if_comm_create_local(ctypes.byref(plan), max_tokens, hidden, hs), "if_comm_create_local")
        out = []
        for r in range(plan.devices):
            c = cls.__new__(cls)
            c.h = ctypes.c_void_p(hs[r])
            c.plan = plan
            c.kind = "peer"
            out.append(c)
        return out

    def destroy(self):
        if self.h:
            _check(lib().if_comm_destroy(self.h), "if_comm_destroy")
            self.h = ctypes.c_void_p()


# ---- stack --------------------------------------------------------------------
def if_stack_workspace_bytes(shape: StackShape, plan: Plan, rank: int, max_tokens: int, mode: int) -> int:
    n = ctypes.c_size_t()
    _check(lib().if_stack_workspace_bytes(ctypes.byref(shape), ctypes.byref(plan), rank, max_tokens, mode,
                                          ctypes.byref(n)), "if_stack_workspace_bytes")
    return n.value


def layer_weights_array(layers) -> ctypes.Array:
    """layers: list of (wqkv, wo, wgu, wdown) uint8 CUDA tensors."""
    arr = (LayerWeights * max(1, len(layers)))()
    for i, (a, b, c, d) in enumerate(layers):
        arr[i] = LayerWeights(a.data_ptr(), b.data_ptr(), c.data_ptr(), d.data_ptr())
    return arr


def if_run_stack(shape: StackShape, plan: Plan, rank: int, comm, layers_arr, h_in, T: int, mode: int, h_out,
                 last_qkv, workspace, stream=None):
    _check(lib().if_run_stack(ctypes.byref(shape), ctypes.byref(plan), rank, comm.h if comm else None, layers_arr,
                              _ptr(h_in), T, mode, _ptr(h_out), _ptr(last_qkv), _ptr(workspace), _stream(stream)),
           "if_run_stack")


def if_kv_cache_bytes(shape: StackShape, plan: Plan, rank: int, slots: int, max_ctx: int) -> int:
    n = ctypes.c_size_t()
    _check(lib().if_kv_cache_bytes(ctypes.byref(shape), ctypes.byref(plan), rank, slots, max_ctx, ctypes.byref(n)),
           "if_kv_cache_bytes")
    return n.value


class KV:
    """A device KV cache (if_kv_cache): two fp32 torch tensors + an optional status word."""

    def __init__(self, shape: StackShape, plan: Plan, rank: int, slots: int, max_ctx: int, device="cuda"):
        import torch
        n = if_kv_cache_bytes(shape, plan, rank, slots, max_ctx) // 4
        self.k = torch.zeros(n, dtype=torch.float32, device=device)
        self.v = torch.zeros(n, dtype=torch.float32, device=device)
        self.status = torch.zeros(1, dtype=torch.int32, device=device)
        self.c = KvCache(self.k.data_ptr(), self.v.data_ptr(), slots, max_ctx, self.status.data_ptr())


def if_run_stack_kv(shape: StackShape, plan: Plan, rank: int, comm, layers_arr, h_in, T: int, mode: int, h_out,
                    last_qkv, kv: "KV", slot_ids, positions, workspace, stream=None):
    _check(lib().if_run_stack_kv(ctypes.byref(shape), ctypes.byref(plan), rank, comm.h if comm else None, layers_arr,
                                 _ptr(h_in), T, mode, _ptr(h_out), _ptr(last_qkv), ctypes.byref(kv.c),
                                 _ptr(slot_ids), _ptr(positions), _ptr(workspace), _stream(stream)),
           "if_run_stack_kv")


# ---- language-model head, speculative verification --------------------------------
def if_embed(table, V: int, d: int, tokens, T: int, h, dev_status=None, stream=None):
    _check(lib().if_embed(_ptr(table), V, d, _ptr(tokens), T, _ptr(h), _ptr(dev_status), _stream(stream)), "if_embed")


def if_lm_logits(s: Scheme, lm, V: int, d: int, h, T: int, rows, logits, scratch, stream=None):
    _check(lib().if_lm_logits(s, _ptr(lm), V, d, _ptr(h), T, _ptr(rows), _ptr(logits), _ptr(scratch),
                              _stream(stream)), "if_lm_logits")


def if_argmax(logits, T: int, V: int, tokens, stream=None):
    _check(lib().if_argmax(_ptr(logits), T, V, _ptr(tokens), _stream(stream)), "if_argmax")


def if_spec_verify(K: int, V: int, tgt_logits, draft_probs, draft_tok, u_acc, u_smp: float, is_top: bool,
                   top_k: int, top_p: float, out_tok, n_out, stream=None):
    _check(lib().if_spec_verify(K, V, _ptr(tgt_logits), _ptr(draft_probs), _ptr(draft_tok), _ptr(u_acc),
                                float(u_smp), int(is_top), int(top_k), float(top_p), _ptr(out_tok), _ptr(n_out),
                                _stream(stream)), "if_spec_verify")


class Engine:
    """Dynamic-batching engine (if_engine_*): AddQuery / Infer and the
    speculative target pass (if_engine_verify).  Marshalling only."""

    def __init__(self, shape: StackShape, layers_arr, embed, lm_head, vocab: int, slots: int, max_ctx: int,
                 step_tokens: int = 64):
        self._keep = (layers_arr, embed, lm_head)
        self.vocab = vocab
        self.cfg = EngineConfig(shape, ctypes.cast(layers_arr, ctypes.c_void_p), embed.data_ptr(),
                                lm_head.data_ptr(), vocab, slots, max_ctx, step_tokens)
        self.h = ctypes.c_void_p()
        _check(lib().if_engine_create(ctypes.byref(self.cfg), ctypes.byref(self.h)), "if_engine_create")

    def add_query(self, prompt, max_new: int, eos: int = -1) -> int:
        arr = (ctypes.c_int32 * len(prompt))(*prompt)
        qid = ctypes.c_int64()
        _check(lib().if_engine_add_query(self.h, arr, len(prompt), max_new, eos, ctypes.byref(qid)),
               "if_engine_add_query")
        return qid.value

    def infer(self, stream=None):
        ids = (ctypes.c_int64 * 64)()
        toks = (ctypes.c_int32 * 64)()
        n = ctypes.c_int32()
        _check(lib().if_engine_infer(self.h, ids, toks, 64, ctypes.byref(n), _stream(stream)), "if_engine_infer")
        return [(ids[i], toks[i]) for i in range(n.value)]

    def verify(self, qid: int, draft_tok, draft_probs, u_acc, u_smp: float, is_top: bool = False, top_k: int = 0,
               top_p: float = 1.0, stream=None):
        K = len(draft_tok)
        dt = (ctypes.c_int32 * max(1, K))(*draft_tok)
        ua = (ctypes.c_float * max(1, K))(*u_acc)
        out = (ctypes.c_int32 * (K + 1))()
        n = ctypes.c_int32()
        _check(lib().if_engine_verify(self.h, qid, K, dt, _ptr(draft_probs), ua, float(u_smp), int(is_top),
                                      int(top_k), float(top_p), out, ctypes.byref(n), _stream(stream)),
               "if_engine_verify")
        return [out[i] for i in range(n.value)]

    def query(self, qid: int):
        ph, gen, pos = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()
        _check(lib().if_engine_query(self.h, qid, ctypes.byref(ph), ctypes.byref(gen), ctypes.byref(pos)),
               "if_engine_query")
        return ph.value, gen.value, pos.value

    def last_logits(self):
        """(device pointer, rows, query ids) of the last step's logits [rows, vocab]."""
        p, rows = ctypes.c_void_p(), ctypes.c_int32()
        ids = (ctypes.c_int64 * 64)()
        _check(lib().if_engine_last_logits(self.h, ctypes.byref(p), ctypes.byref(rows), ids), "if_engine_last_logits")
        return p.value, rows.value, [ids[i] for i in range(rows.value)]

    def destroy(self):
        if self.h:
            _check(lib().if_engine_destroy(self.h), "if_engine_destroy")
            self.h = ctypes.c_void_p()


# ---- packed-tensor container (NEXT-4) -------------------------------------------------
def if_container_save(path: str, tensors, on_device: bool, stream=None):
    """tensors: list of (name, Scheme, dims, packed uint8 tensor / numpy array)."""
    n = len(tensors)
    names = (ctypes.c_char_p * max(1, n))(*[t[0].encode() for t in tensors])
    schemes = (Scheme * max(1, n))(*[t[1] for t in tensors])
    ndims = (ctypes.c_int32 * max(1, n))(*[len(t[2]) for t in tensors])
    dims = (ctypes.c_int64 * (8 * max(1, n)))()
    for i, t in enumerate(tensors):
        for k, x in enumerate(t[2]):
            dims[8 * i + k] = int(x)
    data = (ctypes.c_void_p * max(1, n))(*[(t[3].data_ptr() if on_device else t[3].ctypes.data) for t in tensors])
    _check(lib().if_container_save(path.encode(), n, names, schemes, ndims, dims, data, int(on_device),
                                   _stream(stream) if on_device else None), "if_container_save")


class Container:
    def __init__(self, path: str):
        self.h = ctypes.c_void_p()
        _check(lib().if_container_open(path.encode(), ctypes.byref(self.h)), "if_container_open")

    def __len__(self):
        return lib().if_container_count(self.h)

    def info(self, i: int):
        name = ctypes.create_string_buffer(1024)
        s, nd, b = Scheme(), ctypes.c_int32(), ctypes.c_int64()
        dims = (ctypes.c_int64 * 8)()
        _check(lib().if_container_info(self.h, i, name, 1024, ctypes.byref(s), ctypes.byref(nd), dims, ctypes.byref(b)),
               "if_container_info")
        return name.value.decode(), (s.type, s.block), [dims[k] for k in range(nd.value)], b.value

    def find(self, name: str) -> int:
        i = ctypes.c_int32()
        _check(lib().if_container_find(self.h, name.encode(), ctypes.byref(i)), "if_container_find")
        return i.value

    def load(self, i: int, dst, stream=None):
        _check(lib().if_container_load(self.h, i, _ptr(dst), _stream(stream)), "if_container_load")

    def read_host(self, i: int, dst_numpy):
        _check(lib().if_container_read_host(self.h, i, dst_numpy.ctypes.data), "if_container_read_host")

    def close(self):
        if self.h:
            _check(lib().if_container_close(self.h), "if_container_close")
            self.h = ctypes.c_void_p()


# ---- cost model / auto-planner (NEXT-4) ---------------------------------------------------
def cost_model(t_fixed_s: float, bw_bytes_s: float, t_merge_s, t_hop_s: float) -> CostModel:
    tm = (ctypes.c_double * 9)(*([float(x) for x in list(t_merge_s)[:9]] + [0.0] * (9 - min(9, len(t_merge_s)))))
    return CostModel(float(t_fixed_s), float(bw_bytes_s), tm, float(t_hop_s))


def if_cost_estimate(shape: StackShape, stages: int, groups: int, cm: CostModel, micro_batches: int = 1):
    dec, thr = ctypes.c_double(), ctypes.c_double()
    _check(lib().if_cost_estimate(ctypes.byref(shape), stages, groups, ctypes.byref(cm), micro_batches,
                                  ctypes.byref(dec), ctypes.byref(thr)), "if_cost_estimate")
    return dec.value, thr.value


def if_plan_auto(objective: str, shape: StackShape, devices: int, cm: CostModel, micro_batches: int = 1):
    p = Plan()
    dec, thr = ctypes.c_double(), ctypes.c_double()
    _check(lib().if_plan_auto(0 if objective == "decode" else 1, ctypes.byref(shape), devices, ctypes.byref(cm),
                              micro_batches, ctypes.byref(p), ctypes.byref(dec), ctypes.byref(thr)), "if_plan_auto")
    return p, dec.value, thr.value


def if_launch_count(reset: bool = False) -> int:
    return lib().if_launch_count(1 if reset else 0)
