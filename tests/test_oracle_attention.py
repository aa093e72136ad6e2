"""Pins of the oracle's decode attention over a KV cache (O.stack_kv_f64, NEXT-1,
DESIGN.md Q24): scaled dot-product GQA with RoPE (Table 1
P:71).  Each pin is a property the paper/spec fixes, not a restatement:
  * position 0 == the single-position stack, bit for bit (softmax over one key,
    S:364; RoPE at position 0 is the identity);
  * RoPE is a rotation of consecutive pairs: norms preserved and the
    pair (2m, 2m+1) turned by exactly p * 10000^(-2m/hd), v untouched;
  * identical keys -> uniform scores -> context = mean of the cached values;
  * KV-cache consistency: one causal chunk == token-by-token decode;
  * batching transparency: slots in one batch == each slot alone;
  * out-of-range slot / position -> status 2.
"""
import math

import numpy as np
import pytest

import oracle as O
import synth

CFG = dict(layers=2, hidden=128, heads=4, kv_heads=2, head_dim=32, ffn=128)


def _weights(cfg, zero_k=False, zero_ffn=False, layers=None):
    d, H, G, hd, Fd = cfg["hidden"], cfg["heads"], cfg["kv_heads"], cfg["head_dim"], cfg["ffn"]
    ws = [[], [], [], []]
    for l in range(cfg["layers"] if layers is None else layers):
        k = np.zeros((G * hd, d), np.float32) if zero_k else synth.weight(l, "k", G * hd, d, d)
        ws[0].append(O.quantize(35, 64, np.concatenate([synth.weight(l, "q", H * hd, d, d), k,
                                                        synth.weight(l, "v", G * hd, d, d)])))
        ws[1].append(O.quantize(35, 64, synth.weight(l, "o", d, H * hd, d)))
        gu = np.concatenate([synth.weight(l, "gate", Fd, d, d), synth.weight(l, "up", Fd, d, d)])
        ws[2].append(O.quantize(35, 64, np.zeros_like(gu) if zero_ffn else gu))
        ws[3].append(O.quantize(35, 64, synth.weight(l, "down", d, Fd, d)))
    return ws


def _shape(cfg):
    return dict(cfg, qtype=35, block=64)


def test_position0_is_single_position_stack():
    ws = _weights(CFG)
    h = synth.activations(3, CFG["hidden"], tid=1)
    K, V = O.kv_cache(_shape(CFG), 3, 5)
    a, qa = O.stack_kv_f64(_shape(CFG), *ws, h, [2, 0, 1], [0, 0, 0], K, V)
    b, qb = O.stack_f64(_shape(CFG), *ws, h)
    assert np.array_equal(a, b) and np.array_equal(qa, qb)


@pytest.mark.parametrize("p", [1, 7, 1000])
def test_rope_is_a_rotation_by_p_theta(p):
    cfg = dict(CFG, layers=1)
    ws = _weights(cfg)
    h = synth.activations(1, cfg["hidden"], tid=2)
    H, G, hd = cfg["heads"], cfg["kv_heads"], cfg["head_dim"]
    K, V = O.kv_cache(_shape(cfg), 1, 1001)
    _, raw = O.stack_kv_f64(_shape(cfg), *ws, h, [0], [0], K, V)
    K, V = O.kv_cache(_shape(cfg), 1, 1001)
    _, rot = O.stack_kv_f64(_shape(cfg), *ws, h, [0], [p], K, V)
    nqk = (H + G) * hd
    r0 = raw[0, :nqk].reshape(-1, hd // 2, 2)  # [q and k heads, pairs, 2]
    r1 = rot[0, :nqk].reshape(-1, hd // 2, 2)
    # norms of consecutive pairs are preserved
    assert np.allclose(np.hypot(r1[..., 0], r1[..., 1]), np.hypot(r0[..., 0], r0[..., 1]), rtol=1e-12, atol=0)
    # each pair is turned by exactly p * 10000^(-2m/hd)
    turn = np.arctan2(r1[..., 1], r1[..., 0]) - np.arctan2(r0[..., 1], r0[..., 0])
    want = np.array([p * 10000.0 ** (-2.0 * m / hd) for m in range(hd // 2)])
    diff = np.angle(np.exp(1j * (turn - want[None, :])))
    assert np.abs(diff).max() < 1e-9
    # v is not rotated
    assert np.array_equal(rot[0, nqk:], raw[0, nqk:])


def test_identical_keys_give_mean_of_values():
    """W_k = 0: every cached key is 0, scores are uniform, ctx = mean of v_0..v_p;
    with zero FFN weights h_out - h = W_o' ctx exactly (up to fp64 rounding)."""
    cfg = dict(CFG, layers=1)
    ws = _weights(cfg, zero_k=True, zero_ffn=True)
    d, H, G, hd = cfg["hidden"], cfg["heads"], cfg["kv_heads"], cfg["head_dim"]
    nq, nkv = H * hd, G * hd
    P = 6
    hs = synth.activations(P, d, tid=3)
    K, V = O.kv_cache(_shape(cfg), 1, P)
    vs = []
    Wo = O.dequantize(35, 64, ws[1][0], d, nq).astype(np.float64)
    for p in range(P):
        out, qkv = O.stack_kv_f64(_shape(cfg), *ws, hs[p:p + 1], [0], [p], K, V)
        vs.append(qkv[0, nq + nkv:])
        vmean = np.mean(vs, axis=0)  # [G*hd]
        ctx = np.concatenate([vmean[(i // (H // G)) * hd:(i // (H // G) + 1) * hd] for i in range(H)])
        pred = hs[p].astype(np.float64) + Wo @ ctx
        assert np.abs(out[0] - pred).max() <= 1e-12 * np.abs(pred).max()


def test_chunk_equals_token_by_token():
    ws = _weights(CFG)
    T = 5
    h = synth.activations(T, CFG["hidden"], tid=4)
    K1, V1 = O.kv_cache(_shape(CFG), 2, 8)
    chunk, q1 = O.stack_kv_f64(_shape(CFG), *ws, h, [1] * T, list(range(T)), K1, V1)
    K2, V2 = O.kv_cache(_shape(CFG), 2, 8)
    steps = [O.stack_kv_f64(_shape(CFG), *ws, h[t:t + 1], [1], [t], K2, V2) for t in range(T)]
    tok = np.concatenate([s[0] for s in steps])
    assert np.abs(chunk - tok).max() <= 1e-12 * np.abs(tok).max()
    assert np.abs(K1 - K2).max() <= 1e-12 * np.abs(K2).max()


def test_batching_transparency():
    ws = _weights(CFG)
    h = synth.activations(6, CFG["hidden"], tid=5)
    # slot 0 gets tokens 0,1,2 and slot 1 tokens 3,4,5, decoded as 3 batched steps
    Kb, Vb = O.kv_cache(_shape(CFG), 2, 4)
    batched = [O.stack_kv_f64(_shape(CFG), *ws, h[[s, s + 3]], [0, 1], [s, s], Kb, Vb)[0] for s in range(3)]
    for slot in range(2):
        Ka, Va = O.kv_cache(_shape(CFG), 2, 4)
        for s in range(3):
            alone = O.stack_kv_f64(_shape(CFG), *ws, h[s + 3 * slot:s + 3 * slot + 1], [slot], [s], Ka, Va)[0]
            assert np.array_equal(alone[0], batched[s][slot])


def test_out_of_range_slot_or_position():
    ws = _weights(CFG)
    h = synth.activations(1, CFG["hidden"])
    K, V = O.kv_cache(_shape(CFG), 2, 4)
    for slot, pos in [(2, 0), (-1, 0), (0, 4), (0, -1)]:
        with pytest.raises(O.OracleError) as e:
            O.stack_kv_f64(_shape(CFG), *ws, h, [slot], [pos], K, V)
        assert e.value.status == 2
