"""Pins for the oracle's products, stack and planner (a4-a8).

  * brute-force matmul on exactly representable data (bitwise)
  * one-hot x -> a column of W' exactly; constant blocks -> lo*sum(x)
  * linearity in x
  * Table 4 plan + the balanced examples of S:618-619 + errors
  * virtual-partition replay == unpartitioned stack
  * stack special cases: zero weights -> identity; 1 layer composed by hand
    from independent numpy ops on the oracle's own dequantized matrices.
The stack composition itself is "parity unpinned" by the paper (Q18).
"""
import json
import math
import os

import numpy as np
import pytest

import oracle as O
import synth


def _pack_blocks_direct(qtype, bs, lo, hi, Q):
    """Build packed bytes for given fp16-exact lo/hi per block and integer codes,
    with an independent numpy packer (not oracle code)."""
    N, K = Q.shape
    nb = K // bs
    out = []
    for n in range(N):
        for b in range(nb):
            q = Q[n, b * bs:(b + 1) * bs]
            if qtype == 35:
                codes, width = [int(q[2 * j]) * 11 + int(q[2 * j + 1]) for j in range(bs // 2)], 7
            else:
                codes, width = [int(v) for v in q], qtype
            bits = []
            for c in codes:
                bits.extend([(c >> i) & 1 for i in range(width)])
            while len(bits) % 8:
                bits.append(0)
            out.append(np.array([lo[n, b], hi[n, b]], np.float16).tobytes())
            out.append(np.packbits(np.array(bits, np.uint8), bitorder="little").tobytes())
    return np.frombuffer(b"".join(out), np.uint8).copy()


@pytest.mark.parametrize("qtype,bs", [(4, 32), (35, 64), (3, 32), (8, 64), (2, 32), (5, 64), (6, 64)])
def test_bruteforce_integer_matmul(qtype, bs):
    """Integer lo, step exactly 1 (hi = lo + D): W' = q + lo are small integers,
    x small integers -> every fp64 sum is exact -> bitwise equality with an
    integer matmul."""
    rng = np.random.default_rng(qtype)
    D = O.levels(qtype)
    N, K, M = 5, 2 * bs, 3
    nb = K // bs
    lo = rng.integers(-8, 3, (N, nb)).astype(np.float64)
    hi = lo + D
    Q = rng.integers(0, D + 1, (N, K))
    packed = _pack_blocks_direct(qtype, bs, lo, hi, Q)
    X = rng.integers(-3, 4, (M, K)).astype(np.float32)
    Wint = Q + np.repeat(lo, bs, axis=1).astype(np.int64)
    expect = X.astype(np.int64) @ Wint.T
    Y = O.matmul_f64(qtype, bs, packed, N, K, X)
    assert np.array_equal(Y, expect.astype(np.float64))
    # the dequantized tensor itself is exactly q + lo
    assert np.array_equal(O.dequantize(qtype, bs, packed, N, K), Wint.astype(np.float32))


def test_one_hot_and_constant_blocks():
    rng = np.random.default_rng(5)
    N, K, bs = 7, 128, 64
    W = (rng.standard_normal((N, K)) * 0.05).astype(np.float32)
    p = O.quantize(35, bs, W)
    Wp = O.dequantize(35, bs, p, N, K)
    for k in [0, 63, 64, 127]:
        x = np.zeros(K, np.float32)
        x[k] = 1.0
        y = O.matmul_f64(35, bs, p, N, K, x)[0]
        assert np.array_equal(y, Wp[:, k].astype(np.float64))
    # constant fp16-exact blocks: y = lo * sum(x)
    Wc = np.full((3, K), 0.25, np.float32)
    pc = O.quantize(4, 32, Wc)
    x = rng.standard_normal(K).astype(np.float32)
    y = O.matmul_f64(4, 32, pc, 3, K, x)[0]
    assert np.allclose(y, 0.25 * x.astype(np.float64).sum(), rtol=1e-14, atol=1e-14)


def test_linearity():
    rng = np.random.default_rng(9)
    N, K = 9, 192
    W = (rng.standard_normal((N, K)) * 0.05).astype(np.float32)
    p = O.quantize(5, 64, W)
    a = rng.integers(-4, 5, K).astype(np.float32)
    b = rng.integers(-4, 5, K).astype(np.float32)
    ya = O.matmul_f64(5, 64, p, N, K, a)
    yb = O.matmul_f64(5, 64, p, N, K, b)
    yab = O.matmul_f64(5, 64, p, N, K, a + b)
    assert np.allclose(ya + yb, yab, rtol=1e-13, atol=1e-13)


# ---------------------------------------------------------------- planner
def test_table4_hybrid_plan(golden_dir):
    with open(os.path.join(golden_dir, "table4.json")) as f:
        t = json.load(f)
    plan = O.plan(2, t["layers"], t["heads"], t["heads"], 4, t["devices"], t["stages"], t["groups"])
    for row, a in zip(t["devices_table"], plan):
        # 1-based inclusive in the table, 0-based half-open in the API
        assert [a["layer_begin"] + 1, a["layer_end"]] == row["layers"]
        assert [a["head_begin"] + 1, a["head_end"]] == row["heads"]


def test_balanced_examples():
    p = O.plan(0, 40, 32, 32, 16, 4)
    assert [(a["layer_begin"] + 1, a["layer_end"]) for a in p] == [(1, 10), (11, 20), (21, 30), (31, 40)]
    assert all((a["head_begin"], a["head_end"]) == (0, 32) for a in p)
    p = O.plan(1, 40, 32, 32, 16, 4)
    assert [(a["head_begin"], a["head_end"]) for a in p] == [(0, 8), (8, 16), (16, 24), (24, 32)]
    assert all((a["layer_begin"], a["layer_end"]) == (0, 40) for a in p)
    # remainder to earlier stages; 7B FFN 172 blocks over 8 -> 22,22,22,22,21,21,21,21
    p = O.plan(0, 10, 8, 8, 4, 4)
    assert [a["layer_end"] - a["layer_begin"] for a in p] == [3, 3, 2, 2]
    p = O.plan(1, 32, 32, 32, 172, 8)
    assert [a["ffn_blk_end"] - a["ffn_blk_begin"] for a in p] == [22, 22, 22, 22, 21, 21, 21, 21]


def test_plan_errors():
    with pytest.raises(O.OracleError) as e:
        O.plan(2, 40, 32, 32, 16, 4, 3, 2)
    assert e.value.status == 7  # grid error
    with pytest.raises(O.OracleError) as e:
        O.plan(1, 40, 30, 30, 16, 4)
    assert e.value.status == 6  # indivisible heads
    with pytest.raises(O.OracleError) as e:
        O.plan(0, 3, 32, 32, 16, 4)
    assert e.value.status == 6  # layers < stages
    with pytest.raises(O.OracleError) as e:
        O.plan(1, 8, 64, 8, 16, 16)
    assert e.value.status == 6  # kv heads not divisible (70B G=8 at 16 groups)


def test_plan_completeness():
    """every (layer, head) pair covered exactly once per TP group."""
    for strat, dev, st, gr in [(0, 4, 0, 0), (1, 8, 0, 0), (2, 8, 2, 4), (2, 8, 4, 2), (2, 4, 2, 2)]:
        p = O.plan(strat, 80, 64, 8, 448, dev, st, gr)
        cover = np.zeros((80, 64), np.int32)
        for a in p:
            cover[a["layer_begin"]:a["layer_end"], a["head_begin"]:a["head_end"]] += 1
        assert np.all(cover == 1)


# ---------------------------------------------------------------- stack
SMALL = dict(layers=3, hidden=128, heads=4, kv_heads=2, head_dim=32, ffn=256)


def _make_stack(shape, qtype, bs):
    d, H, G, hd, F = shape["hidden"], shape["heads"], shape["kv_heads"], shape["head_dim"], shape["ffn"]
    wqkv, wo, wgu, wdown = [], [], [], []
    for l in range(shape["layers"]):
        q = synth.weight(l, "q", H * hd, d, d)
        k = synth.weight(l, "k", G * hd, d, d)
        v = synth.weight(l, "v", G * hd, d, d)
        wqkv.append(O.quantize(qtype, bs, np.concatenate([q, k, v])))
        wo.append(O.quantize(qtype, bs, synth.weight(l, "o", d, H * hd, d)))
        g = synth.weight(l, "gate", F, d, d)
        u = synth.weight(l, "up", F, d, d)
        wgu.append(O.quantize(qtype, bs, np.concatenate([g, u])))
        wdown.append(O.quantize(qtype, bs, synth.weight(l, "down", d, F, d)))
    return wqkv, wo, wgu, wdown


def test_stack_zero_weights_identity():
    shape = dict(SMALL, qtype=35, block=64)
    d, H, G, hd, F = 128, 4, 2, 32, 256
    z = lambda N, K: O.quantize(35, 64, np.zeros((N, K), np.float32))
    L = shape["layers"]
    wqkv = [z((H + 2 * G) * hd, d)] * L
    wo = [z(d, H * hd)] * L
    wgu = [z(2 * F, d)] * L
    wdown = [z(d, F)] * L
    h = synth.activations(2, d)
    h_out, qkv = O.stack_f64(shape, wqkv, wo, wgu, wdown, h)
    assert np.array_equal(h_out, h.astype(np.float64))
    assert np.all(qkv == 0)


def test_stack_one_layer_by_hand():
    """1 layer composed from independent numpy ops on the oracle's dequantized
    matrices (checks the glue: rms eps, v broadcast with GQA groups, silu, residuals)."""
    shape = dict(SMALL, layers=1, qtype=4, block=32)
    d, H, G, hd, F = 128, 4, 2, 32, 256
    wqkv, wo, wgu, wdown = _make_stack(shape, 4, 32)
    Wqkv = O.dequantize(4, 32, wqkv[0], (H + 2 * G) * hd, d).astype(np.float64)
    Wo = O.dequantize(4, 32, wo[0], d, H * hd).astype(np.float64)
    Wgu = O.dequantize(4, 32, wgu[0], 2 * F, d).astype(np.float64)
    Wd = O.dequantize(4, 32, wdown[0], d, F).astype(np.float64)
    h = synth.activations(3, d).astype(np.float64)
    a = h / np.sqrt((h ** 2).mean(1, keepdims=True) + 1e-5)
    qkv = a @ Wqkv.T
    v = qkv[:, (H + G) * hd:].reshape(3, G, hd)
    ctx = np.repeat(v, H // G, axis=1).reshape(3, H * hd)  # head i -> group i // (H/G)
    h2 = h + ctx @ Wo.T
    a2 = h2 / np.sqrt((h2 ** 2).mean(1, keepdims=True) + 1e-5)
    gu = a2 @ Wgu.T
    g, u = gu[:, :F], gu[:, F:]
    h3 = h2 + ((g * (1 / (1 + np.exp(-g)))) * u) @ Wd.T
    h_out, qkv_o = O.stack_f64(shape, wqkv, wo, wgu, wdown, h.astype(np.float32))
    assert np.allclose(h_out, h3, rtol=1e-12, atol=1e-12)
    assert np.allclose(qkv_o, qkv, rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("strategy,devices,stages,groups", [
    (0, 1, 0, 0), (0, 3, 0, 0), (1, 2, 0, 0), (2, 4, 2, 2)])
def test_virtual_partition_equivalence(strategy, devices, stages, groups):
    shape = dict(SMALL, qtype=35, block=64)
    ws = _make_stack(shape, 35, 64)
    h = synth.activations(2, 128)
    ref, _ = O.stack_f64(shape, *ws, h)
    got = O.stack_partitioned_f64(shape, strategy, devices, stages, groups, *ws, h)
    assert np.max(np.abs(got - ref)) <= 1e-12 * max(1.0, np.max(np.abs(ref)))
    if strategy == 0:  # layer-wise is just a reordering of nothing: bitwise
        assert np.array_equal(got, ref)
