"""Pins of the oracle's language-model head (O.lm_logits_f64, O.argmax, O.lm_sequence_f64;
DESIGN.md Q27: final RMSNorm + block-quantized output projection + greedy choice, the
step that makes Infer() return "a set of next tokens").  Not restatements:
  * one-hot hidden state: rms(s e_j) = e_j * s / sqrt(s^2/d + 1e-5) in closed form, so
    the logits are column j of the dequantized W' times that scalar (pins eps, the
    normalisation and which operand index is contracted: a transposed W' fails);
  * scale invariance of RMSNorm when eps is negligible (a dropped norm fails);
  * constant blocks (lo = hi): every logit is c_v * sum_i a_i;
  * argmax: numpy's first-maximum rule on random and tied vectors;
  * teacher-forced sequence: row j equals a fresh run of prompt + continuation[:j]
    as one prompt (the KV cache carries exactly the earlier positions).
"""
import numpy as np
import pytest

import oracle as O
import synth

QT, BS = 35, 64


def _lm(V, d):
    return O.quantize(QT, BS, synth.lm_head(V, d))


@pytest.mark.parametrize("j", [0, 37, 127])
def test_one_hot_hidden_state_selects_column(j):
    V, d = 96, 128
    lm = _lm(V, d)
    W = O.dequantize(QT, BS, lm, V, d).astype(np.float64)
    s = 0.01  # s^2/d = 7.8e-7 against eps 1e-5: the eps term dominates and is pinned
    h = np.zeros((1, d))
    h[0, j] = s
    got = O.lm_logits_f64(QT, BS, lm, V, d, h)[0]
    a_j = s / np.sqrt(s * s / d + 1e-5)
    assert np.allclose(got, W[:, j] * a_j, rtol=1e-14, atol=0)


def test_rmsnorm_scale_invariance():
    V, d = 64, 256
    lm = _lm(V, d)
    h = synth.activations(2, d, tid=9).astype(np.float64)
    a = O.lm_logits_f64(QT, BS, lm, V, d, h)
    b = O.lm_logits_f64(QT, BS, lm, V, d, 1000.0 * h)
    # eps/mean(h^2) ~ 1e-5 at sigma 1 -> relative change 5e-6 at scale 1, 5e-12 at 1000
    assert np.allclose(a, b, rtol=2e-5)
    assert not np.allclose(a, b, rtol=1e-9)


def test_constant_blocks_give_sum_of_normalised_state():
    V, d = 6, 128
    c = np.linspace(-0.5, 0.75, V).astype(np.float32)  # exact in fp16 -> lo = hi = c_v
    lm = O.quantize(QT, BS, np.repeat(c[:, None], d, axis=1))
    h = synth.activations(1, d, tid=3).astype(np.float64)
    a = h[0] / np.sqrt(np.mean(h[0] ** 2) + 1e-5)
    got = O.lm_logits_f64(QT, BS, lm, V, d, h)[0]
    assert np.allclose(got, c.astype(np.float64) * a.sum(), rtol=1e-12, atol=1e-12)


def test_argmax_first_maximum():
    rng = np.random.default_rng(0)
    for _ in range(50):
        x = rng.integers(-3, 4, size=17).astype(np.float64)  # many ties
        assert O.argmax(x) == int(np.argmax(x))
    assert O.argmax(np.array([2.0, 5.0, 5.0, 1.0])) == 1


def test_teacher_forced_sequence_equals_fresh_prompts():
    cfg = dict(layers=2, hidden=128, heads=4, kv_heads=2, head_dim=32, ffn=128, qtype=QT, block=BS)
    d, H, G, hd, Fd = 128, 4, 2, 32, 128
    ws = [[], [], [], []]
    for l in range(2):
        ws[0].append(O.quantize(QT, BS, np.concatenate([synth.weight(l, "q", H * hd, d, d),
                                                         synth.weight(l, "k", G * hd, d, d),
                                                         synth.weight(l, "v", G * hd, d, d)])))
        ws[1].append(O.quantize(QT, BS, synth.weight(l, "o", d, H * hd, d)))
        ws[2].append(O.quantize(QT, BS, np.concatenate([synth.weight(l, "gate", Fd, d, d),
                                                         synth.weight(l, "up", Fd, d, d)])))
        ws[3].append(O.quantize(QT, BS, synth.weight(l, "down", d, Fd, d)))
    V = 64
    E = synth.embedding(V, d)
    lm = _lm(V, d)
    prompt, cont = [5, 9, 1], [33, 2, 60]
    seq = O.lm_sequence_f64(cfg, *ws, E, lm, V, prompt, cont, max_ctx=8)
    for j in range(len(cont) + 1):
        fresh = O.lm_sequence_f64(cfg, *ws, E, lm, V, prompt + cont[:j], [], max_ctx=8)
        assert np.allclose(seq[j], fresh[0], rtol=1e-12, atol=1e-12), j
