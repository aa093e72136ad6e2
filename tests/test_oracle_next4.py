"""Pins of the NEXT-4 oracle pieces (Q28/Q29).

Container (oracle/container.py):
  * a hand-derived golden file (tests/golden/container_q4_const.hex: constant tensor,
    every byte worked out from the S:122 section layout and Eq. 1 with max = min);
  * quantize -> save -> load -> dequantize == quantize -> dequantize bit for bit;
  * truncated / trailing / inconsistent files are rejected with the byte offset.
Cost model (O.cost_estimate, Table 5):
  * Table 5: with the per-layer time and the 2- and 4-way merge latencies solved from
    the printed DECODE column (8 / 12 / 12 tokens/s, hop 0), the model predicts the
    printed THROUGHPUT column exactly (32 / 12 / 24): throughput = stages x decode;
  * groups = stages = 1 -> throughput == decode; a larger merge latency slows the
    tensor-wise decode and leaves the layer-wise one unchanged;
  * plan_auto picks tensor-wise for decode speed and layer-wise for throughput when
    merges are cheap and the pipeline is full.
"""
import os

import numpy as np
import pytest

import oracle as O
import synth
from oracle import container as C


def _golden_bytes(golden_dir):
    txt = open(os.path.join(golden_dir, "container_q4_const.hex")).read()
    hexs = "".join(l.split("#")[0] for l in txt.splitlines()).replace(" ", "")
    return bytes.fromhex(hexs)


def test_golden_container_bytes(tmp_path, golden_dir):
    W = np.full((2, 64), 0.5, np.float32)
    packed = O.quantize(4, 32, W)
    p = tmp_path / "w.ifq"
    C.write(str(p), [("w", 4, 32, [2, 64], packed)])
    assert p.read_bytes() == _golden_bytes(golden_dir)
    (name, qt, bs, dims, data), = C.read(str(p))
    assert (name, qt, bs, dims) == ("w", 4, 32, [2, 64]) and data == bytes(packed)


@pytest.mark.parametrize("qt,bs", [(35, 64), (4, 32), (3, 32), (8, 64), (5, 64), (35, 32)])
def test_quantize_save_load_dequantize_identity(tmp_path, qt, bs):
    tensors = []
    for tid, (name, (N, K)) in enumerate({"layers.0.wq": (96, 256), "layers.0.wdown": (64, 192),
                                           "lm_head": (50, 128)}.items()):
        W = synth.matrix(synth.SEED_WEIGHTS, 900 + tid, 1 / 16, N, K)
        tensors.append((name, qt, bs, [N, K], O.quantize(qt, bs, W), W))
    p = str(tmp_path / "m.ifq")
    C.write(p, [t[:5] for t in tensors])
    back = C.read(p)
    for (name, q, b, dims, packed, W), (n2, q2, b2, d2, data) in zip(tensors, back):
        assert (name, q, b, dims) == (n2, q2, b2, d2)
        got = O.dequantize(q, b, np.frombuffer(data, np.uint8), *dims)
        ref = O.dequantize(q, b, packed, *dims)
        assert np.array_equal(got.view(np.uint32), ref.view(np.uint32))


def test_malformed_containers_rejected(tmp_path, golden_dir):
    good = _golden_bytes(golden_dir)
    cases = {
        "truncated": good[:-1],
        "trailing": good + b"\0",
        "magic": b"XFQC" + good[4:],
        "blocks": good[:27] + b"\x05" + good[28:],  # block count 5 for dims [2, 64] / 32
        "scheme": good[:15] + b"\x07" + good[16:],  # qtype 7 is not a scheme
    }
    assert good[27] == 4 and good[15] == 4
    for what, blob in cases.items():
        p = tmp_path / f"{what}.ifq"
        p.write_bytes(blob)
        with pytest.raises(C.ContainerError, match="byte"):
            C.read(str(p))


def test_table5_throughput_column_predicted_from_decode_column():
    L = 60  # Falcon-40B's 60 layers (P:229 model); any L works, the parameters scale
    dec_layer, dec_tensor, dec_hybrid = 8.0, 12.0, 12.0  # Table 5 decoding speed
    # layer-wise (4 stages, hop 0): L * t = 1/8; tensor 1x4: L t/4 + 2 L m4 = 1/12;
    # hybrid 2x2: L t/2 + 2 L m2 = 1/12
    t = 1.0 / dec_layer / L
    m4 = (1.0 / dec_tensor - L * t / 4) / (2 * L)
    m2 = (1.0 / dec_hybrid - L * t / 2) / (2 * L)
    tm = [0, 0, m2, 0, m4]
    got = {}
    for name, (S, G) in {"layer": (4, 1), "tensor": (1, 4), "hybrid": (2, 2)}.items():
        got[name] = O.cost_estimate(L, S, G, 0.0, t, 1.0, tm, 0.0, micro_batches=4)
    assert np.allclose([got[k][0] for k in ("layer", "tensor", "hybrid")], [8, 12, 12], rtol=1e-12)
    # the printed throughput column, not used in the fit
    assert np.allclose([got[k][1] for k in ("layer", "tensor", "hybrid")], [32, 12, 24], rtol=1e-12)
    assert m4 > m2 > 0  # "especially when many GPU cards are involved"


def test_cost_model_identities_and_monotonicity():
    d, th = O.cost_estimate(32, 1, 1, 2e-6, 1e8, 5e12, [0] * 9, 1e-6, 8)
    assert d == th and np.isclose(1 / d, 32 * (2e-6 + 1e8 / 5e12))
    base = [0, 0, 2e-6, 0, 3e-6, 0, 0, 0, 4e-6]
    slow = [2 * x for x in base]
    assert O.cost_estimate(32, 1, 8, 0, 1e8, 5e12, slow, 0, 1)[0] < O.cost_estimate(32, 1, 8, 0, 1e8, 5e12, base, 0, 1)[0]
    assert O.cost_estimate(32, 8, 1, 0, 1e8, 5e12, slow, 1e-6, 1) == O.cost_estimate(32, 8, 1, 0, 1e8, 5e12, base, 1e-6, 1)


def test_plan_auto_objectives():
    cost = dict(t_fixed=1e-6, bw=5e12, t_merge=[0, 0, 2e-6, 0, 2.5e-6, 0, 0, 0, 3e-6], t_hop=1e-6)
    lb = 855638016 * 0.5  # a 70B layer at 0.5 B/weight
    dec = O.plan_auto("decode", 80, 64, 8, 448, 8, cost, lb, micro_batches=8)
    thr = O.plan_auto("throughput", 80, 64, 8, 448, 8, cost, lb, micro_batches=8)
    assert (dec[1], dec[2]) == (1, 8)  # tensor-wise: 8x the streaming bandwidth per token
    assert (thr[1], thr[2]) == (8, 1)  # layer-wise: every stage busy, no merges
