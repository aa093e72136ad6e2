"""GPU parity of the CUDA path against the CPU oracle, through the C ABI.

Bar (BASELINE.json north_star): bit-exact packed codes and dequantized values;
qGEMV within 1e-3 normwise (fp32 accumulation); qGEMM within 2e-2 (bf16).
Shapes span several tiles/chunks with ragged tails; edge cases: empty
outputs, constant blocks, signed zeros, exact ties, subnormals, values at the
fp16 limit, non-finite inputs and invalid pair codes.
"""
import numpy as np
import pytest

import oracle as O
import paper_2401_08294_b200 as F
import synth
from gpu_util import SCHEMES, dev, normwise, to_bf16_exact, torch

pytestmark = pytest.mark.gpu


def _dq(qtype, bs, W):
    d = dev()
    N, K = W.shape
    s = F.scheme(qtype, bs)
    p = torch.empty(F.if_packed_bytes(s, N, K), dtype=torch.uint8, device=d)
    st = torch.zeros(1, dtype=torch.int32, device=d)
    F.if_quantize(s, torch.from_numpy(np.ascontiguousarray(W)).to(d), N, K, p, st)
    torch.cuda.synchronize()
    return p, int(st.item())


# ---------------------------------------------------------------- synth
def test_synth_generator_bitwise():
    d = dev()
    for tid, off, n, sig in [(0, 0, 10000, 1.0), (77, 12345, 4099, 1 / 64), (8 * 31 + 6, 11008 * 4095, 11008, 1 / 64)]:
        out = torch.empty(n, dtype=torch.float32, device=d)
        F.if_synth_fill(synth.SEED_WEIGHTS, tid, float(synth.scale(sig)), out, offset=off)
        ref = synth.fill(synth.SEED_WEIGHTS, tid, synth.scale(sig), n, off)
        assert np.array_equal(out.cpu().numpy().view(np.uint32), ref.view(np.uint32))


# ---------------------------------------------------------------- quantize
def _adversarial(K, bs, rng):
    rows = []
    rows.append(np.full(K, 0.5, np.float32))                         # constant, fp16-exact
    rows.append(np.full(K, 0.1, np.float32))                         # constant, not fp16-exact
    z = np.zeros(K, np.float32); z[::2] = -0.0; rows.append(z)       # signed zeros
    t = np.tile(np.array([-1.0, -0.875, 1.5, 1.5], np.float32), K // 4); rows.append(t)  # exact ties (Q1)
    rows.append((rng.standard_normal(K) * 1e-6).astype(np.float32))  # fp16 subnormal range
    rows.append((rng.standard_normal(K) * 1e-40).astype(np.float32))  # fp32 subnormals
    big = (rng.uniform(-65504, 65504, K)).astype(np.float32); big[::bs] = 65504.0; rows.append(big)
    rows.append((rng.standard_normal(K) * 300).astype(np.float32))
    return np.stack(rows)


@pytest.mark.parametrize("qtype,bs", SCHEMES)
def test_quantize_bitexact(qtype, bs):
    rng = np.random.default_rng(qtype * 7 + bs)
    K = bs * 17  # 17 blocks per row: ragged against 32-lane chunks
    W = np.concatenate([(rng.standard_normal((37, K)) * 0.02).astype(np.float32), _adversarial(K, bs, rng)])
    p, st = _dq(qtype, bs, W)
    assert st == 0
    ref = O.quantize(qtype, bs, W)
    assert np.array_equal(p.cpu().numpy(), ref)


@pytest.mark.parametrize("qtype,bs", [(35, 64), (4, 32), (8, 64), (35, 32)])
def test_quantize_errors(qtype, bs):
    K = bs * 4
    for bad in [np.nan, np.inf, -np.inf, 70000.0, -70000.0]:
        W = np.zeros((3, K), np.float32)
        W[1, 5] = bad
        _, st = _dq(qtype, bs, W)
        assert st == 4, bad


@pytest.mark.parametrize("qtype,bs", SCHEMES)
def test_dequantize_bitexact(qtype, bs):
    d = dev()
    rng = np.random.default_rng(100 + qtype * 7 + bs)
    N, K = 29, bs * 9
    W = np.concatenate([(rng.standard_normal((N, K)) * 0.05).astype(np.float32), _adversarial(K, bs, rng)])
    ref_p = O.quantize(qtype, bs, W)
    p = torch.from_numpy(ref_p).to(d)
    out = torch.empty(W.shape, dtype=torch.float32, device=d)
    st = torch.zeros(1, dtype=torch.int32, device=d)
    F.if_dequantize(F.scheme(qtype, bs), p, W.shape[0], K, out, st)
    torch.cuda.synchronize()
    assert int(st.item()) == 0
    ref = O.dequantize(qtype, bs, ref_p, W.shape[0], K)
    assert np.array_equal(out.cpu().numpy().view(np.uint32), ref.view(np.uint32))


@pytest.mark.parametrize("bs", [32, 64])
def test_dequantize_invalid_pair_code(bs):
    d = dev()
    W = np.zeros((2, bs * 2), np.float32)
    ref_p = O.quantize(35, bs, W)
    ref_p[4] = 0x7F  # first pair code of block 0 := 127 > 120
    out = torch.empty(W.shape, dtype=torch.float32, device=d)
    st = torch.zeros(1, dtype=torch.int32, device=d)
    F.if_dequantize(F.scheme(35, bs), torch.from_numpy(ref_p).to(d), 2, bs * 2, out, st)
    torch.cuda.synchronize()
    assert int(st.item()) == 5


# ---------------------------------------------------------------- qGEMV
def _gemv_case(qtype, bs, N, K, B, seed, acc=False):
    d = dev()
    rng = np.random.default_rng(seed)
    W = (rng.standard_normal((N, K)) / np.sqrt(K)).astype(np.float32)
    ref_p = O.quantize(qtype, bs, W)
    x = rng.standard_normal((B, K)).astype(np.float32)
    y0 = rng.standard_normal((B, N)).astype(np.float32)
    xd = torch.from_numpy(x).to(d)
    y = torch.from_numpy(y0.copy()).to(d)
    s = F.scheme(qtype, bs)
    pd = torch.from_numpy(ref_p).to(d)
    (F.if_qgemv_acc if acc else F.if_qgemv)(s, pd, N, K, xd, B, y)
    torch.cuda.synchronize()
    ref = O.matmul_f64(qtype, bs, ref_p, N, K, x)
    if acc:
        ref = ref + y0.astype(np.float64)
    return y.cpu().numpy(), ref, (s, pd, xd)


@pytest.mark.parametrize("qtype,bs", SCHEMES)
@pytest.mark.parametrize("B", [1, 3])
def test_qgemv_all_schemes(qtype, bs, B):
    got, ref, _ = _gemv_case(qtype, bs, 67, bs * 37, B, qtype * 100 + bs + B)
    assert normwise(got, ref) <= 1e-3


@pytest.mark.parametrize("N,K", [(1, 64), (5, 64 * 17), (131, 64 * 32), (70, 64 * 33), (300, 64 * 80),
                                 (64, 11008), (33, 64 * 448)])
@pytest.mark.parametrize("B", [1, 2, 4, 5, 8, 16, 64])
def test_qgemv_q3h64_shapes(N, K, B):
    got, ref, _ = _gemv_case(35, 64, N, K, B, N + K + B)
    assert normwise(got, ref) <= 1e-3


@pytest.mark.parametrize("qtype,bs,B", [(35, 64, 1), (35, 64, 4), (4, 32, 1), (5, 64, 8)])
def test_qgemv_accumulate(qtype, bs, B):
    got, ref, _ = _gemv_case(qtype, bs, 77, bs * 40, B, 5, acc=True)
    assert normwise(got, ref) <= 1e-3


def test_qgemv_config0_full_size():
    """BASELINE configs[0]: one 4096x4096 Q3H matrix, batch-1, synthetic weights."""
    d = dev()
    N = K = 4096
    W = synth.weight(0, "q", N, K, K)
    x = synth.activations(1, K)
    s = F.scheme(35, 64)
    Wd = torch.from_numpy(W).to(d)
    p = torch.empty(F.if_packed_bytes(s, N, K), dtype=torch.uint8, device=d)
    F.if_quantize(s, Wd, N, K, p)
    y = torch.empty(1, N, dtype=torch.float32, device=d)
    F.if_qgemv(s, p, N, K, torch.from_numpy(x).to(d), 1, y)
    y2 = torch.empty_like(y)
    F.if_qgemv(s, p, N, K, torch.from_numpy(x).to(d), 1, y2)
    torch.cuda.synchronize()
    ref_p = O.quantize(35, 64, W)
    assert np.array_equal(p.cpu().numpy(), ref_p)
    ref = O.matmul_f64(35, 64, ref_p, N, K, x)
    assert normwise(y.cpu().numpy(), ref) <= 1e-3
    assert torch.equal(y, y2)  # deterministic


def test_qgemv_one_hot_and_empty():
    d = dev()
    N, K = 40, 64 * 35
    rng = np.random.default_rng(1)
    W = (rng.standard_normal((N, K)) * 0.05).astype(np.float32)
    p = O.quantize(35, 64, W)
    Wp = O.dequantize(35, 64, p, N, K)
    s = F.scheme(35, 64)
    pd = torch.from_numpy(p).to(d)
    for k in [0, 1, 63, 64, 2047, K - 1]:
        x = torch.zeros(1, K, device=d)
        x[0, k] = 1.0
        y = torch.empty(1, N, device=d)
        F.if_qgemv(s, pd, N, K, x, 1, y)
        torch.cuda.synchronize()
        assert np.allclose(y.cpu().numpy()[0], Wp[:, k], rtol=2e-6, atol=1e-7)
    y = torch.full((1, 4), 7.0, device=d)
    F.if_qgemv(s, pd, 0, K, torch.zeros(1, K, device=d), 1, y)  # N = 0: no-op
    F.if_qgemv(s, pd, 4, 0, torch.zeros(1, 64, device=d), 1, y)  # K = 0: y = 0
    torch.cuda.synchronize()
    assert torch.all(y == 0)


# ---------------------------------------------------------------- qGEMM
@pytest.mark.parametrize("qtype,bs", SCHEMES)
@pytest.mark.parametrize("M", [70, 300])
def test_qgemm_all_schemes(qtype, bs, M):
    """M = 300 > 256: the wide-tile variant (512 tokens per tile, ragged)."""
    d = dev()
    rng = np.random.default_rng(qtype + bs + M)
    N, K = 136, 64 * 9
    W = (rng.standard_normal((N, K)) / np.sqrt(K)).astype(np.float32)
    p = O.quantize(qtype, bs, W)
    Xb, Xf = to_bf16_exact(rng.standard_normal((M, K)))
    Y = torch.empty(M, N, device=d)
    F.if_qgemm(F.scheme(qtype, bs), torch.from_numpy(p).to(d), N, K, Xb.to(d).view(torch.int16), M, Y)
    torch.cuda.synchronize()
    ref = O.matmul_f64(qtype, bs, p, N, K, Xf)
    assert normwise(Y.cpu().numpy(), ref) <= 2e-2


@pytest.mark.parametrize("M,N,K", [(1, 64, 64), (17, 200, 64 * 5), (128, 128, 4096), (512, 384, 64 * 20),
                                   (300, 1000, 64 * 3), (257, 130, 64 * 7), (700, 260, 64 * 11), (1024, 256, 4096)])
def test_qgemm_q3h_shapes(M, N, K):
    """M > 256: the wide-tile variant (512 tokens per weight tile, two TMEM accumulators)."""
    d = dev()
    rng = np.random.default_rng(M + N + K)
    W = (rng.standard_normal((N, K)) / np.sqrt(K)).astype(np.float32)
    p = O.quantize(35, 64, W)
    Xb, Xf = to_bf16_exact(rng.standard_normal((M, K)))
    Y = torch.empty(M, N, device=d)
    F.if_qgemm(F.scheme(35, 64), torch.from_numpy(p).to(d), N, K, Xb.to(d).view(torch.int16), M, Y)
    torch.cuda.synchronize()
    ref = O.matmul_f64(35, 64, p, N, K, Xf)
    assert normwise(Y.cpu().numpy(), ref) <= 2e-2


@pytest.mark.parametrize("B", [2, 4, 16])
@pytest.mark.parametrize("xscale", [1e-6, 1e5, "mixed"])
def test_qgemv_batched_scaled_x(B, xscale):
    """the tensor-core batched path splits x into fp16 hi + lo with a
    per-token power-of-two scale, so |x| > 65504 does not overflow and |x| ~ 1e-6
    does not fall into fp16 subnormals -- same 1e-3 gate as B = 1."""
    d = dev()
    rng = np.random.default_rng(B)
    N, K = 200, 64 * 40
    W = (rng.standard_normal((N, K)) / np.sqrt(K)).astype(np.float32)
    p = O.quantize(35, 64, W)
    x = rng.standard_normal((B, K))
    if xscale == "mixed":
        x *= np.array([10.0 ** (6 * (i % 3) - 6) for i in range(B)])[:, None]  # 1e-6, 1, 1e6 per token
    else:
        x *= xscale
    x = x.astype(np.float32)
    y = torch.empty(B, N, device=d)
    F.if_qgemv(F.scheme(35, 64), torch.from_numpy(p).to(d), N, K, torch.from_numpy(x).to(d), B, y)
    torch.cuda.synchronize()
    ref = O.matmul_f64(35, 64, p, N, K, x)
    got = y.cpu().numpy()
    for t in range(B):  # per token: each row has its own magnitude
        assert normwise(got[t], ref[t]) <= 1e-3, t
