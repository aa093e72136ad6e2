"""Pins for the oracle's codec (a1-a3): what the paper and mathematics fix.

Every test here checks oracle/ against something other than itself:
  * Table 2 codes, w' and averages             -> test_table2_*
  * Table 3 bits/weight                        -> test_table3_bits_per_weight
  * pair-code bijection + digit order          -> test_pair_code_*
  * bit layout vs an independent numpy packer (Q11/Q12)    -> test_golden_bytes_*
  * binary16 directed rounding vs numpy's float16          -> test_f16_*
  * half-step bound + containment              -> test_half_step_bound
  * monotone fidelity ordering                     -> test_monotone_fidelity
  * round-half-away tie (Q1)                               -> test_tie_rounds_away
"""
import json
import math
import os

import numpy as np
import pytest

import oracle as O

SCHEMES = [(8, 32), (8, 64), (6, 64), (5, 64), (4, 32), (4, 64), (35, 64), (35, 32),
           (3, 32), (3, 64), (2, 32), (2, 64), (6, 32), (5, 32)]


def table2(golden_dir):
    with open(os.path.join(golden_dir, "table2.json")) as f:
        return json.load(f)


# ---------------------------------------------------------------- Table 2
@pytest.mark.parametrize("col", ["4bit", "3bit", "3.5bit"])
def test_table2_codes(golden_dir, col):
    t = table2(golden_dir)
    c = t[col]
    blk = O.quantize_block(c["qtype"], t["w"])
    q = O.block_codes(c["qtype"], len(t["w"]), blk)
    assert q.tolist() == c["q"]


@pytest.mark.parametrize("col", ["4bit", "3bit", "3.5bit"])
def test_table2_dequantized(golden_dir, col):
    t = table2(golden_dir)
    c = t[col]
    blk = O.quantize_block(c["qtype"], t["w"])
    wp = O.dequantize_block(c["qtype"], len(t["w"]), blk)
    # printed to 3 decimals
    assert np.all(np.abs(wp.astype(np.float64) - np.array(c["w_prime"])) <= 0.0005 + 1e-9)
    delta = np.abs(np.array(t["w"], np.float32).astype(np.float64) - wp)
    bad = set(c.get("misprinted_delta_index", []))
    for i, (d, p) in enumerate(zip(delta, c["delta"])):
        if i in bad:
            continue
        assert abs(d - p) <= 0.0005 + 1e-6, (i, d, p)
    # printed average
    assert abs(delta.mean() - c["avg"]) <= 0.0005 + 1e-6


def test_table2_misprint_reading(golden_dir):
    """Q15: the two misprinted 3-bit cells; the printed average is the mean of the
    corrected cells, not of the printed ones."""
    t = table2(golden_dir)
    c = t["3bit"]
    printed_mean = np.mean(c["delta"])
    assert abs(printed_mean - 0.0715) < 0.001 and abs(printed_mean - c["avg"]) > 0.003
    blk = O.quantize_block(3, t["w"])
    wp = O.dequantize_block(3, 12, blk).astype(np.float64)
    d = np.abs(np.array(t["w"], np.float32) - wp)
    assert abs(d[3] - 0.114) < 0.0005 and abs(d[10] - 0.157) < 0.0005


def test_table2_header_is_min_max(golden_dir):
    """Q2: the two fp16 numbers are min(w) and max(w) (-1 and 1.5 are fp16-exact)."""
    t = table2(golden_dir)
    blk = O.quantize_block(35, t["w"])
    lo = np.frombuffer(blk[0:2], np.float16)[0]
    hi = np.frombuffer(blk[2:4], np.float16)[0]
    assert float(lo) == -1.0 and float(hi) == 1.5


# ---------------------------------------------------------------- Table 3
def test_table3_bits_per_weight(golden_dir):
    with open(os.path.join(golden_dir, "table3.json")) as f:
        rows = json.load(f)["rows"]
    for r in rows:
        num, den = O.bits_per_weight(r["qtype"], r["block"])
        assert num / den == r["bpw"], r
        # the serialized block: 2 fp16 + tight codes, exactly bpw*block/8 bytes
        assert O.block_bytes(r["qtype"], r["block"]) * 8 == r["bpw"] * r["block"]


def test_q3h_and_q3b32_same_cost():
    """Q3_B32 has the same actual bits/weight as Q3H (block 64)."""
    assert O.bits_per_weight(35, 64) == O.bits_per_weight(3, 32) == (4, 1)
    assert O.block_bytes(35, 64) == 32 and O.block_bytes(3, 32) == 16


# ---------------------------------------------------------------- pair code
def test_pair_code_bijection_exhaustive():
    seen = {}
    for a in range(11):
        for b in range(11):
            v = O.pack_pair(a, b)
            assert 0 <= v < 128  # fits the 7 bits of P:118
            assert v not in seen
            seen[v] = (a, b)
            assert O.unpack_pair(v) == (a, b)
    assert sorted(seen) == list(range(121))  # exactly the 121 valid codes
    for v in range(121, 128):
        with pytest.raises(O.OracleError) as e:
            O.unpack_pair(v)
        assert e.value.status == 5
    assert O.pack_pair(11, 0) == -1 and O.pack_pair(0, 11) == -1


def test_pair_code_digit_order():
    """Q10: the first (even) weight is the high digit: lexicographic order of
    (q_2i, q_2i+1) equals numeric order of the code."""
    codes = [O.pack_pair(a, b) for a in range(11) for b in range(11)]
    assert codes == sorted(codes)
    assert O.pack_pair(1, 0) > O.pack_pair(0, 10)


# ---------------------------------------------------------------- golden bytes
def _independent_pack(codes, width):
    """LSB-first tight packing written with numpy bit arrays (not oracle code)."""
    bits = []
    for c in codes:
        bits.extend([(c >> i) & 1 for i in range(width)])
    while len(bits) % 8:
        bits.append(0)
    return np.packbits(np.array(bits, np.uint8), bitorder="little").tobytes()


@pytest.mark.parametrize("col", ["4bit", "3bit", "3.5bit"])
def test_golden_bytes_table2(golden_dir, col):
    t = table2(golden_dir)
    c = t[col]
    q = c["q"]
    if c["qtype"] == 35:
        codes = [q[2 * j] * 11 + q[2 * j + 1] for j in range(len(q) // 2)]
        width = 7
    else:
        codes, width = q, c["qtype"]
    hdr = np.array([-1.0, 1.5], np.float16).tobytes()  # little-endian [lo16][hi16] (Q12)
    expect = hdr + _independent_pack(codes, width)
    assert O.quantize_block(c["qtype"], t["w"]) == expect


def test_golden_bytes_survey_hex():
    """The hex strings SURVEY §8c derived by hand for the Table 2 block."""
    w = [-1, -0.9, -0.6, -0.4, -0.2, 0, 0.1, 0.5, 0.7, 1, 1.3, 1.5]
    assert O.quantize_block(4, w).hex() == "00bc003e" + "10426597cafe"
    assert O.quantize_block(3, w).hex() == "00bc003e" + "40a48db50f"
    assert O.quantize_block(35, w).hex() == "00bc003e" + "004c49566d03"


def test_random_block_bytes_independent_repack():
    """Random blocks: re-derive the bytes from the oracle's own integer codes
    with the independent packer (bit order, density, header)."""
    rng = np.random.default_rng(1)
    for qtype, bs in SCHEMES:
        w = (rng.standard_normal(bs) * 0.02).astype(np.float32)
        blk = O.quantize_block(qtype, w)
        q = O.block_codes(qtype, bs, blk).tolist()
        if qtype == 35:
            codes, width = [q[2 * j] * 11 + q[2 * j + 1] for j in range(bs // 2)], 7
        else:
            codes, width = q, qtype
        assert blk[4:] == _independent_pack(codes, width)
        assert len(blk) == O.block_bytes(qtype, bs)


# ---------------------------------------------------------------- fp16
def test_f16_to_f32_exhaustive():
    h = np.arange(65536, dtype=np.uint16)
    ref = h.view(np.float16).astype(np.float32)
    lib = O.lib()
    got = np.array([lib.ref_f16_to_f32(int(v)) for v in h], np.float32)
    fin = np.isfinite(ref)
    assert np.array_equal(got[fin].view(np.uint32), ref[fin].view(np.uint32))
    assert np.all(np.isnan(got[np.isnan(ref)]))


def _numpy_directed(f32, down):
    """RD16/RU16 from numpy's round-to-nearest float16 + one nextafter step."""
    h = np.float16(f32)
    if np.isinf(h) and not np.isinf(f32):
        big = np.float16(65504.0)
        if down:
            return (big if f32 > 0 else np.float16(-np.inf))
        return (np.float16(np.inf) if f32 > 0 else -big)
    fh = np.float32(h)
    if down and fh > f32:
        h = np.nextafter(h, np.float16(-np.inf))
    if (not down) and fh < f32:
        h = np.nextafter(h, np.float16(np.inf))
    if h == 0:  # keep the sign of the input's zero side
        h = np.float16(-0.0) if (np.signbit(f32) or (down and f32 < 0)) else np.float16(0.0)
    return h


def test_f16_directed_rounding_sampled():
    rng = np.random.default_rng(7)
    vals = list(rng.standard_normal(4000).astype(np.float32) * np.float32(3.0))
    vals += list((rng.standard_normal(2000) * 1e-5).astype(np.float32))  # fp16 subnormal range
    vals += list((rng.standard_normal(1000) * 3e4).astype(np.float32))
    vals += [np.float32(x) for x in [65504, 65505, 65519, 65520, 70000, -65504, -65505, -70000,
                                     6.1e-5, 6.0e-8, 5.9e-8, 1e-9, -1e-9, 0.1, -0.1, 1.0, -1.0, 2049.0]]
    lib = O.lib()
    for f in vals:
        for down, fn in ((True, lib.ref_f32_to_f16_rd), (False, lib.ref_f32_to_f16_ru)):
            got = np.uint16(fn(float(f))).view(np.float16)
            exp = _numpy_directed(np.float32(f), down)
            assert np.float16(got).tobytes() == np.float16(exp).tobytes() or (got == exp and got != 0), (f, down, got, exp)
            if np.isfinite(got):
                if down:
                    assert np.float32(got) <= f
                else:
                    assert np.float32(got) >= f


# ---------------------------------------------------------------- invariants
def _gauss_blocks(rng, n_blocks, bs, sigma=1.0 / 64):
    return (rng.standard_normal((n_blocks, bs)) * sigma).astype(np.float32)


@pytest.mark.parametrize("qtype,bs", SCHEMES)
def test_half_step_bound(qtype, bs):
    """lo <= w' <= hi and |w - w'| <= step/2 (+ fp32 slack)."""
    rng = np.random.default_rng(qtype * 100 + bs)
    W = _gauss_blocks(rng, 3000, bs)
    W[0, :] = 0.5  # constant, fp16-exact
    W[1, :] = 0.1  # constant, not fp16-exact
    W[2, ::2] = -0.0
    packed = O.quantize(qtype, bs, W)
    Wp = O.dequantize(qtype, bs, packed, W.shape[0], bs)
    bb = O.block_bytes(qtype, bs)
    hdr = packed.reshape(W.shape[0], bb)[:, :4].copy().view(np.float16).astype(np.float64)
    lo, hi = hdr[:, 0:1], hdr[:, 1:2]
    D = O.levels(qtype)
    step = (hi - lo) / D
    assert np.all(lo <= W.min(1, keepdims=True)) and np.all(hi >= W.max(1, keepdims=True))
    # containment up to the single fp32 rounding of fma32(q, r/D, lo) (Q5)
    ulp = 2.0 ** -23 * np.maximum(np.maximum(np.abs(lo), np.abs(hi)), hi - lo)
    assert np.all(Wp >= lo - ulp) and np.all(Wp <= hi + ulp)
    err = np.abs(W.astype(np.float64) - Wp)
    slack = 4 * 2.0 ** -24 * np.maximum(np.abs(lo), np.abs(hi)) + 2.0 ** -22 * step
    assert np.all(err <= step / 2 + slack)
    # constant fp16-exact block: all codes 0, w' = lo exactly (Q6)
    assert np.all(Wp[0] == 0.5)
    q0 = O.block_codes(qtype, bs, packed[:bb].tobytes())
    assert np.all(q0 == 0)


def test_monotone_fidelity():
    """mean reconstruction error ordering Q8 <= Q6 <= Q5 <= Q4 <= Q3H <= Q3."""
    rng = np.random.default_rng(11)
    order = [(8, 64), (6, 64), (5, 64), (4, 64), (35, 64), (3, 64), (2, 64)]
    W = _gauss_blocks(rng, 1200, 64)
    errs = []
    for qtype, bs in order:
        p = O.quantize(qtype, bs, W)
        errs.append(np.abs(O.dequantize(qtype, bs, p, W.shape[0], bs) - W).mean())
    assert all(a < b for a, b in zip(errs, errs[1:])), errs
    # Q3H beats Q3_B32 at the same 4.0 bits/weight
    p3 = O.quantize(3, 32, W.reshape(-1, 32))
    e3 = np.abs(O.dequantize(3, 32, p3, W.size // 32, 32) - W.reshape(-1, 32)).mean()
    assert errs[4] < e3


def test_tie_rounds_away():
    """Q1: t = 0.5 exactly -> q = 1 (half away from zero), not 0 (half even)."""
    w = [-1.0, -0.875, 1.5, 1.5]
    blk = O.quantize_block(35, w)
    assert O.block_codes(35, 4, blk).tolist() == [0, 1, 10, 10]


def test_signed_zero_canonical():
    """Q7: -0 min/max is stored as +0."""
    blk = O.quantize_block(4, [-0.0] * 32)
    assert blk[:4] == b"\x00\x00\x00\x00"
    blk = O.quantize_block(4, [-0.0] * 31 + [1.0])
    assert blk[:2] == b"\x00\x00"


def test_errors():
    with pytest.raises(O.OracleError) as e:
        O.quantize_block(4, [float("nan")] + [0.0] * 31)
    assert e.value.status == 4
    with pytest.raises(O.OracleError) as e:
        O.quantize_block(4, [float("inf")] + [0.0] * 31)
    assert e.value.status == 4
    with pytest.raises(O.OracleError) as e:
        O.quantize_block(4, [70000.0] + [0.0] * 31)  # beyond fp16 (Q8)
    assert e.value.status == 4
    with pytest.raises(O.OracleError) as e:
        O.quantize_block(35, [0.0] * 3)  # odd Q3H length
    assert e.value.status == 3
    with pytest.raises(O.OracleError) as e:
        O.quantize(4, 32, np.zeros((2, 48), np.float32))
    assert e.value.status == 2
    # corrupted Q3H code > 120 -> decode error (Q14)
    blk = bytearray(O.quantize_block(35, [0.0] * 64))
    blk[4] = 0x7F
    with pytest.raises(O.OracleError) as e:
        O.dequantize_block(35, 64, bytes(blk))
    assert e.value.status == 5


def test_sharded_quantization_is_slice():
    """Quantization shards exactly: any block-aligned row/column
    window of W quantizes to the same bytes as the slice of the full tensor."""
    rng = np.random.default_rng(3)
    W = (rng.standard_normal((16, 256)) * 0.03).astype(np.float32)
    for qtype, bs in [(35, 64), (4, 32), (5, 64)]:
        full = O.quantize(qtype, bs, W).reshape(16, -1)
        bb = O.block_bytes(qtype, bs)
        part = O.quantize(qtype, bs, W[4:12, 64:192]).reshape(8, -1)
        assert np.array_equal(part, full[4:12, (64 // bs) * bb:(192 // bs) * bb])
