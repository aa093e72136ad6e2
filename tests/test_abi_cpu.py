"""CPU-side checks of the C ABI (no GPU): the library loads, exports every
symbol include/if_b200.h declares, and its host logic (sizes, planner,
argument validation) agrees with the oracle and the paper's tables."""
import ctypes
import json
import os

import pytest

import oracle as O
import paper_2401_08294_b200 as F
from paper_2401_08294_b200 import _lib


@pytest.fixture(scope="module", autouse=True)
def built():
    from paper_2401_08294_b200 import build
    build.build()


def test_exports_every_header_symbol():
    syms = _lib.header_symbols()
    assert len(syms) >= 20
    L = ctypes.CDLL(_lib.LIB_PATH)
    missing = [s for s in syms if not hasattr(L, s)]
    assert not missing, missing
    # and the binding wraps every one of them with the C name
    assert set(syms) <= set(_lib._SIGS), set(syms) - set(_lib._SIGS)


def test_sm100a_cubin():
    """The library carries sm_100a SASS (tcgen05-capable target)."""
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


@pytest.mark.parametrize("qtype,block", [(2, 32), (2, 64), (3, 32), (3, 64), (4, 32), (4, 64), (5, 32), (5, 64),
                                         (6, 32), (6, 64), (8, 32), (8, 64), (35, 32), (35, 64)])
def test_sizes_match_oracle(qtype, block):
    s = F.scheme(qtype, block)
    assert F.if_block_bytes(s) == O.block_bytes(qtype, block)
    assert F.if_bits_per_weight(s) == O.bits_per_weight(qtype, block)
    assert F.if_packed_bytes(s, 7, 4 * block) == 7 * 4 * O.block_bytes(qtype, block)
    assert F.if_packed_bytes(s, 7, 4 * block + 1) == -1


def test_table3_through_abi(golden_dir):
    with open(os.path.join(golden_dir, "table3.json")) as f:
        rows = json.load(f)["rows"]
    for r in rows:
        num, den = F.if_bits_per_weight(F.scheme(r["qtype"], r["block"]))
        assert num / den == r["bpw"]


def test_invalid_scheme_rejected_on_host():
    for q, b in [(7, 64), (4, 48), (35, 16), (1, 32)]:
        assert F.if_block_bytes(F.scheme(q, b)) == -1
        with pytest.raises(F.IFError) as e:
            F.if_qgemv(F.scheme(q, b), None, 4, 64, None, 1, None, stream=0)
        assert e.value.status == 3


def test_shape_and_arg_errors_on_host():
    s = F.scheme("Q3H", 64)
    L = F.lib()
    assert L.if_qgemv(s, None, 4, 100, None, 1, None, None) == 2   # K % block
    assert L.if_qgemv(s, None, 4, 128, None, 0, None, None) == 1   # B outside 1..64
    assert L.if_qgemv(s, None, 4, 128, None, 65, None, None) == 1
    assert L.if_qgemv(s, None, 4, 128, None, 1, None, None) == 1   # null pointers
    assert b"B=" in L.if_last_error() or b"null" in L.if_last_error()
    assert L.if_quantize(s, None, 4, 96, None, None, None) == 2
    assert L.if_qgemm(s, None, 4, 128, None, -1, None, None) == 2
    assert L.if_qgemv(s, None, 0, 128, None, 1, None, None) == 0   # empty output: no-op


LLAMA = {
    "7b": dict(layers=32, hidden=4096, heads=32, kv_heads=32, head_dim=128, ffn=11008),
    "13b": dict(layers=40, hidden=5120, heads=40, kv_heads=40, head_dim=128, ffn=13824),
    "70b": dict(layers=80, hidden=8192, heads=64, kv_heads=8, head_dim=128, ffn=28672),
}


def _shape(cfg, s=None):
    return F.stack_shape(cfg["layers"], cfg["hidden"], cfg["heads"], cfg["kv_heads"], cfg["head_dim"], cfg["ffn"],
                         s or F.scheme("Q3H", 64))


@pytest.mark.parametrize("model", ["7b", "13b", "70b"])
@pytest.mark.parametrize("strategy,devices,stages,groups", [
    (0, 1, 0, 0), (0, 2, 0, 0), (0, 4, 0, 0), (0, 8, 0, 0), (1, 2, 0, 0), (1, 4, 0, 0), (1, 8, 0, 0),
    (2, 4, 2, 2), (2, 8, 2, 4), (2, 8, 4, 2)])
def test_planner_matches_oracle(model, strategy, devices, stages, groups):
    cfg = LLAMA[model]
    try:
        ref = O.plan(strategy, cfg["layers"], cfg["heads"], cfg["kv_heads"], cfg["ffn"] // 64, devices, stages, groups)
    except O.OracleError as e:
        with pytest.raises(F.IFError) as e2:
            F.if_plan_partition(strategy, _shape(cfg), devices, stages, groups)
        assert e2.value.status == e.status
        return
    p = F.if_plan_partition(strategy, _shape(cfg), devices, stages, groups)
    assert p.devices == devices
    for d, r in enumerate(ref):
        a = p.a[d]
        got = dict(stage=a.stage, group_rank=a.group_rank, layer_begin=a.layer_begin, layer_end=a.layer_end,
                   head_begin=a.head_begin, head_end=a.head_end, kv_begin=a.kv_begin, kv_end=a.kv_end,
                   ffn_blk_begin=a.ffn_blk_begin, ffn_blk_end=a.ffn_blk_end)
        assert got == r


def test_table4_through_abi(golden_dir):
    with open(os.path.join(golden_dir, "table4.json")) as f:
        t = json.load(f)
    cfg = dict(layers=40, hidden=4096, heads=32, kv_heads=32, head_dim=128, ffn=4096)
    p = F.if_plan_partition(F.IF_HYBRID, _shape(cfg), 4, 2, 2)
    for row in t["devices_table"]:
        a = p.a[row["device"]]
        assert [a.layer_begin + 1, a.layer_end] == row["layers"]
        assert [a.head_begin + 1, a.head_end] == row["heads"]


def test_plan_errors_through_abi():
    cfg = LLAMA["70b"]
    with pytest.raises(F.IFError) as e:
        F.if_plan_partition(F.IF_HYBRID, _shape(cfg), 8, 3, 2)
    assert e.value.status == 7
    with pytest.raises(F.IFError) as e:
        F.if_plan_partition(F.IF_BY_TENSOR, _shape(dict(cfg, kv_heads=8)), 16)
    assert e.value.status == 1  # devices outside 1..8
    with pytest.raises(F.IFError) as e:
        F.if_plan_partition(F.IF_BY_TENSOR, _shape(LLAMA["13b"]), 6)
    assert e.value.status == 6  # 40 heads over 6 groups


def test_plan_rejects_head_ranges_off_block_boundaries():
    """W_o is split along K by heads, so each rank's column range
    h * head_dim must fall on a quantization-block boundary (else its shard is not
    a whole-block slice): heads = 12, head_dim = 80, 2 groups -> 480 % 64 != 0."""
    s = F.scheme(35, 64)
    shape = F.stack_shape(2, 960, 12, 12, 80, 1024, s)
    with pytest.raises(F.IFError) as e:
        F.if_plan_partition(F.IF_BY_TENSOR, shape, 2)
    assert e.value.status == 6
    F.if_plan_partition(F.IF_BY_TENSOR, shape, 3)  # 4 heads x 80 = 320 = 5 blocks: accepted


def test_nccl_unique_id_through_abi():
    """if_comm_nccl_unique_id (NCCL dlopen'ed by the library): 128 bytes, fresh each call."""
    a, b = F.if_comm_nccl_unique_id(), F.if_comm_nccl_unique_id()
    assert len(a) == 128 and len(b) == 128 and a != b
