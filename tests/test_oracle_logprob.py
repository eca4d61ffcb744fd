"""Pins for oracle.logprob (logp / H rows).

Each check ties the fp64 oracle to something other than itself: closed forms,
special cases, mpmath brute force and invariants of the softmax (§2,
P:94-108; BASELINE.json north_star: "exp(logp) summed over the vocabulary
equals 1", "brute-force softmax on tiny vocabularies").
"""
import math

import numpy as np
import pytest
import torch

from oracle import exact
from oracle.logprob import logprob_entropy


def _bf16(a):
    return torch.as_tensor(np.asarray(a, dtype=np.float32)).to(torch.bfloat16)


def _rand(shape, seed, scale=1.0):
    g = torch.Generator().manual_seed(seed)
    return (torch.randn(*shape, generator=g) * scale).to(torch.bfloat16)


def test_vocab_one_is_exactly_zero():
    H = _rand((5, 64), 1)
    W = _rand((1, 64), 2, 0.1)
    lp, ent = logprob_entropy(H, W, np.zeros(5, np.int64))
    assert np.all(lp == 0.0) and np.all(ent == 0.0)


@pytest.mark.parametrize("V", [2, 7, 1024, 151936])
def test_zero_weight_is_uniform(V):
    H = _rand((3, 64), 3)
    W = torch.zeros(V, 64, dtype=torch.bfloat16)
    ids = np.array([0, V // 2, V - 1])
    lp, ent = logprob_entropy(H, W, ids)
    assert np.allclose(lp, -math.log(V), atol=1e-12, rtol=0)
    assert np.allclose(ent, math.log(V), atol=1e-11, rtol=0)
    if V == 151936:
        assert abs(-math.log(V) - (-11.931215)) < 1e-6  # SURVEY C.5 closed form value


def test_vocab_two_is_minus_softplus():
    H = _rand((16, 32), 4)
    W = _rand((2, 32), 5, 0.7)
    ids = np.arange(16) % 2
    lp, _ = logprob_entropy(H, W, ids)
    z = H.double().numpy() @ W.double().numpy().T
    for t in range(16):
        xa, xb = z[t, ids[t]], z[t, 1 - ids[t]]
        d = xb - xa
        sp = d + math.log1p(math.exp(-d)) if d > 0 else math.log1p(math.exp(d))
        assert abs(lp[t] - (-sp)) < 1e-12


def test_probabilities_sum_to_one_over_full_vocab():
    V, d = 4096, 64
    H = _rand((3, d), 6)
    W = _rand((V, d), 7, 0.3)
    for t in range(3):
        lp_all, _ = logprob_entropy(H[t:t + 1].expand(V, d), W, np.arange(V))
        assert abs(math.fsum(np.exp(lp_all)) - 1.0) < 1e-12


@pytest.mark.parametrize("V,d,T", [(1, 16, 1.0), (2, 16, 1.0), (3, 24, 0.7), (8, 32, 1.0), (1024, 64, 1.3)])
def test_mpmath_brute_force(V, d, T):
    N = 3 if V < 1024 else 2
    H = _rand((N, d), 10 + V)
    W = _rand((V, d), 20 + V, 0.5)
    ids = np.array([(7 * t + 1) % V for t in range(N)])
    lp, ent = logprob_entropy(H, W, ids, temperature=T)
    lp_mp, ent_mp = exact.logprob_entropy_mp(H.float().numpy(), W.float().numpy(), ids, T)
    for t in range(N):
        assert abs(lp[t] - float(lp_mp[t])) < 1e-12
        assert abs(ent[t] - float(ent_mp[t])) < 1e-11


def test_temperature_two_equals_half_hidden_bitwise():
    V, d = 512, 64
    H = _rand((8, d), 30)
    W = _rand((V, d), 31, 0.5)
    ids = np.arange(8) * 37 % V
    lp2, e2 = logprob_entropy(H, W, ids, temperature=2.0)
    Hh = (H.float() * 0.5).to(torch.bfloat16)
    assert torch.equal(Hh.float() * 2, H.float())  # halving is exact in bf16 here
    lp1, e1 = logprob_entropy(Hh, W, ids, temperature=1.0)
    assert np.array_equal(lp1, lp2) and np.array_equal(e1, e2)


def test_per_token_temperature_matches_scalar_rows():
    V, d = 300, 32
    H = _rand((4, d), 40)
    W = _rand((V, d), 41, 0.5)
    ids = np.array([1, 50, 299, 7])
    temps = np.array([0.5, 1.0, 0.7, 2.0])
    lp, ent = logprob_entropy(H, W, ids, temperatures=temps)
    for t in range(4):
        l1, e1 = logprob_entropy(H[t:t + 1], W, ids[t:t + 1], temperature=temps[t])
        assert lp[t] == l1[0] and ent[t] == e1[0]


def test_shift_invariance_of_log_softmax():
    """Appending a constant feature c with a unit weight column shifts every logit by c."""
    V, d = 257, 32
    H = _rand((5, d), 50)
    W = _rand((V, d), 51, 0.4)
    ids = np.array([0, 1, 128, 255, 256])
    lp, ent = logprob_entropy(H, W, ids)
    H2 = torch.cat([H, torch.full((5, 1), 3.0, dtype=torch.bfloat16)], 1)
    W2 = torch.cat([W, torch.ones(V, 1, dtype=torch.bfloat16)], 1)
    lp2, ent2 = logprob_entropy(H2, W2, ids)
    assert np.allclose(lp, lp2, atol=1e-12, rtol=0) and np.allclose(ent, ent2, atol=1e-12, rtol=0)


def test_entropy_bounds_and_peaked_regime():
    import synth
    V, d = 2048, 256
    W = synth.head_weight(V, d, 60)
    ids = synth.token_ids(64, V, 61)
    H = synth.hidden_states(64, d, 62, weight=W, ids=ids, mode="peaked")
    lp, ent = logprob_entropy(H, W, ids)
    assert np.all(ent >= -1e-12) and np.all(ent <= math.log(V) + 1e-12)
    assert np.all(lp <= 1e-12)
    assert np.median(lp) > -3.0  # planted targets: most logp near 0 (Table 1 regime)


def test_permuting_vocab_rows_with_ids_is_invariant():
    V, d = 333, 48
    H = _rand((6, d), 70)
    W = _rand((V, d), 71, 0.5)
    ids = np.array([0, 5, 100, 200, 331, 332])
    perm = np.random.default_rng(0).permutation(V)
    inv = np.argsort(perm)
    lp, ent = logprob_entropy(H, W, ids)
    lp2, ent2 = logprob_entropy(H, W[torch.as_tensor(perm)], inv[ids])
    assert np.allclose(lp, lp2, atol=1e-12, rtol=0) and np.allclose(ent, ent2, atol=1e-12, rtol=0)


def test_logits_equal_mpmath_dot_products_at_temperature():
    """oracle.logprob.logits: x = H W^T / T against 40-digit dot products (§2 P:94 the
    head's logits; reading U7 for T).  A transposed operand, a dropped or inverted T fails."""
    import mpmath as mp
    from oracle.logprob import logits
    H = _rand((4, 48), 21)
    W = _rand((7, 48), 22, 0.3)
    for T in (0.7, 1.0, 2.5):
        x = logits(H, W, T)
        assert x.shape == (4, 7)
        with mp.workdps(40):
            for t in range(4):
                for v in range(7):
                    z = mp.fsum(mp.mpf(float(a)) * mp.mpf(float(b)) for a, b in zip(H[t].double(), W[v].double()))
                    ref = float(z / mp.mpf(T))
                    assert abs(x[t, v] - ref) <= 4 * math.ulp(abs(ref)) + 1e-300, (T, t, v)
