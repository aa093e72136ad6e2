"""The library's container I/O and cost model through the C ABI, on the host (no GPU
needed: host data and host reads), against the oracle (oracle/container.py,
O.cost_estimate, O.plan_auto) -- SURVEY NEXT-4, Q28/Q29.
"""
import numpy as np
import pytest

import oracle as O
import paper_2401_08294_b200 as F
import synth
from oracle import container as C


def _tensors():
    out = []
    for tid, (name, qt, bs, N, K) in enumerate([("layers.0.wqkv", 35, 64, 192, 512), ("layers.0.wo", 4, 32, 64, 256),
                                                ("lm_head", 8, 64, 70, 128), ("x", 35, 32, 3, 64)]):
        W = synth.matrix(synth.SEED_WEIGHTS, 700 + tid, 1 / 16, N, K)
        out.append((name, qt, bs, [N, K], O.quantize(qt, bs, W)))
    return out


def test_library_save_equals_oracle_file(tmp_path):
    ts = _tensors()
    a, b = str(tmp_path / "lib.ifq"), str(tmp_path / "ref.ifq")
    F.if_container_save(a, [(n, F.scheme(q, bs), dims, data) for n, q, bs, dims, data in ts], on_device=False)
    C.write(b, ts)
    assert open(a, "rb").read() == open(b, "rb").read()


def test_library_reads_oracle_file(tmp_path):
    ts = _tensors()
    p = str(tmp_path / "ref.ifq")
    C.write(p, ts)
    c = F.Container(p)
    assert len(c) == len(ts)
    for i, (name, q, bs, dims, data) in enumerate(ts):
        nm, sch, d, nbytes = c.info(i)
        assert (nm, sch, d, nbytes) == (name, (q, bs), dims, data.size)
        assert c.find(name) == i
        got = np.empty(nbytes, np.uint8)
        c.read_host(i, got)
        assert np.array_equal(got, data)
    c.close()


def test_library_rejects_malformed(tmp_path):
    ts = _tensors()[:1]
    p = tmp_path / "ref.ifq"
    C.write(str(p), ts)
    good = p.read_bytes()
    for what, blob in {"truncated": good[:-3], "trailing": good + b"x", "magic": b"IFQX" + good[4:],
                       "version": good[:4] + b"\x02" + good[5:]}.items():
        q = tmp_path / f"{what}.ifq"
        q.write_bytes(blob)
        with pytest.raises(F.IFError, match="IO.*byte"):
            F.Container(str(q))


def _layer_bytes(cfg, qt=35, bs=64):
    d, H, G, hd, Fd = cfg["hidden"], cfg["heads"], cfg["kv_heads"], cfg["head_dim"], cfg["ffn"]
    return sum(O.packed_bytes(qt, bs, N, K) for N, K in [((H + 2 * G) * hd, d), (d, H * hd), (2 * Fd, d), (d, Fd)])


@pytest.mark.parametrize("model", ["7b", "13b", "70b"])
def test_cost_estimate_and_plan_auto_equal_oracle(model):
    cfg = synth.LLAMA[model]
    shape = F.stack_shape(*[cfg[k] for k in ("layers", "hidden", "heads", "kv_heads", "head_dim", "ffn")],
                          F.scheme(35, 64))
    cost = dict(t_fixed=3.1e-6, bw=5.4e12, t_merge=[0, 0, 2.1e-6, 0, 2.6e-6, 0, 0, 0, 3.4e-6], t_hop=1.2e-6)
    cm = F.cost_model(cost["t_fixed"], cost["bw"], cost["t_merge"], cost["t_hop"])
    lb = _layer_bytes(cfg)
    for S, G in [(1, 1), (2, 1), (1, 2), (2, 2), (8, 1), (1, 8), (2, 4), (4, 2)]:
        for mb in (1, 4, 8):
            assert F.if_cost_estimate(shape, S, G, cm, mb) == O.cost_estimate(cfg["layers"], S, G, cost["t_fixed"], lb,
                                                                               cost["bw"], cost["t_merge"],
                                                                               cost["t_hop"], mb)
    for objective in ("decode", "throughput"):
        for devices in (1, 2, 4, 8):
            p, dec, thr = F.if_plan_auto(objective, shape, devices, cm, micro_batches=8)
            ref = O.plan_auto(objective, cfg["layers"], cfg["heads"], cfg["kv_heads"], cfg["ffn"] // 64, devices,
                              cost, lb, micro_batches=8)
            assert (p.stages, p.groups, dec, thr) == (ref[1], ref[2], ref[3], ref[4]), (objective, devices)
