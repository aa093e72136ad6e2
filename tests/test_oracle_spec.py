"""Pins of the oracle's speculative-sampling verification (O.spec_verify, Algorithm 1
P:351-384; Q25/Q26).  Not restatements -- properties the method fixes:
  * distribution preservation (the point of Algorithm 1's accept/resample rule):
    over uniform draws the first output token is distributed exactly as the target
    softmax, whatever the draft distribution (integrated on a grid of uniforms);
  * draft == target: every draft token is accepted and the extra token is a draw from the
    target at position K ("sample an extra token");
  * flexible accept: a draft token in the target's top-k / top-p pool is
    accepted even when a < q/p fails;
  * inverse-CDF sampling endpoints; invalid draft tokens -> status 2.
"""
import numpy as np
import pytest

import oracle as O


def _softmax(l):
    e = np.exp(l - l.max())
    return e / e.sum()


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_first_token_distribution_is_target(seed):
    rng = np.random.default_rng(seed)
    V = 5
    logits = rng.standard_normal((2, V)).astype(np.float32) * 1.5
    draft = rng.dirichlet(np.ones(V)).astype(np.float32)[None, :]
    target = _softmax(logits[0].astype(np.float64))
    N = 300
    grid = (np.arange(N) + 0.5) / N
    counts = np.zeros(V)
    for x in range(V):  # the draft token itself is drawn from the draft distribution
        for ua in grid:
            for us in grid[::3]:
                out = O.spec_verify(logits, draft, [x], [ua], us)
                counts[out[0]] += draft[0, x]
    emp = counts / counts.sum()
    assert np.abs(emp - target).max() < 1e-2, (emp, target)


def test_draft_equal_to_target_accepts_all_and_samples_extra():
    rng = np.random.default_rng(3)
    K, V = 3, 6
    logits = rng.standard_normal((K + 1, V)).astype(np.float32)
    draft = np.stack([_softmax(l.astype(np.float64)) for l in logits[:K]]).astype(np.float32)
    toks = [1, 4, 2]
    extra = np.zeros(V)
    grid = (np.arange(600) + 0.5) / 600
    for us in grid:
        out = O.spec_verify(logits, draft, toks, [0.999999] * K, us)
        assert out[:K] == toks and len(out) == K + 1
        extra[out[K]] += 1
    assert np.abs(extra / extra.sum() - _softmax(logits[K].astype(np.float64))).max() < 5e-3


def test_flexible_accept_top_k_and_top_p():
    V = 8
    q = np.array([0.40, 0.25, 0.15, 0.08, 0.05, 0.04, 0.02, 0.01])
    logits = np.log(q).astype(np.float32)[None, :].repeat(2, 0)
    draft = np.array([[0.02, 0.55, 0.35, 0.02, 0.02, 0.02, 0.01, 0.01]], np.float32)
    # q/p: token 1 -> 0.45, token 2 -> 0.43; a = 0.9 rejects both under the plain rule
    assert len(O.spec_verify(logits, draft, [1], [0.9], 0.5)) == 1
    assert len(O.spec_verify(logits, draft, [2], [0.9], 0.5)) == 1
    # token 1 (rank 2, mass strictly above it 0.40) is in the top-2 pool and the top-p 0.5 pool
    assert O.spec_verify(logits, draft, [1], [0.9], 0.5, is_top=True, top_k=2)[:1] == [1]
    assert O.spec_verify(logits, draft, [1], [0.9], 0.5, is_top=True, top_p=0.5)[:1] == [1]
    # token 2 (rank 3, mass above it 0.65) is outside top-2 and outside top-p 0.5 ...
    assert len(O.spec_verify(logits, draft, [2], [0.9], 0.5, is_top=True, top_k=2)) == 1
    assert len(O.spec_verify(logits, draft, [2], [0.9], 0.5, is_top=True, top_p=0.5)) == 1
    # ... and with both pools given it must lie in both
    assert len(O.spec_verify(logits, draft, [2], [0.9], 0.5, is_top=True, top_k=3, top_p=0.5)) == 1
    assert O.spec_verify(logits, draft, [2], [0.9], 0.5, is_top=True, top_k=3, top_p=0.7)[:1] == [2]
    # is_top off: the pools are ignored
    assert len(O.spec_verify(logits, draft, [1], [0.9], 0.5, is_top=False, top_k=2)) == 1


def test_resample_is_the_positive_residual():
    """Rejected token: the replacement is drawn from (q - p)_+ only -- tokens where the
    draft over-proposes (p >= q) are never drawn."""
    V = 4
    q = np.array([0.1, 0.2, 0.3, 0.4])
    p = np.array([0.4, 0.3, 0.2, 0.1], np.float32)[None, :]
    logits = np.log(q).astype(np.float32)[None, :].repeat(2, 0)
    seen = set()
    for us in (np.arange(200) + 0.5) / 200:
        out = O.spec_verify(logits, p, [0], [0.99], us)  # token 0: ratio 0.25 < 0.99 -> reject
        seen.add(out[0])
    assert seen == {2, 3}


def test_sampling_endpoints_and_errors():
    logits = np.log(np.array([[0.0, 0.5, 0.5], [0.2, 0.3, 0.5]]) + 1e-30).astype(np.float32)
    draft = np.array([[0.0, 0.5, 0.5]], np.float32)
    assert O.spec_verify(logits, draft, [1], [0.0], 0.0) == [1, 0]  # accepted; extra at u=0: first index
    assert O.spec_verify(logits, draft, [1], [0.0], 0.999999) == [1, 2]
    with pytest.raises(O.OracleError) as e:
        O.spec_verify(logits, draft, [3], [0.0], 0.0)
    assert e.value.status == 2
