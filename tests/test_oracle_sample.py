"""Pins for oracle.sample (NEXT-1 rollout-side sampling twin).

Philox4x32-10 is pinned to the Random123 known-answer vectors (tests/golden/philox_kat.json);
Gumbel-max is pinned to the distribution it must realise, softmax(x) (§2 P:99 the
behavioural distribution of the rollout engine), by a chi-square test, and to the argmax
limit (one logit far above the rest is always chosen).
"""
import json
import math
import os

import numpy as np
import pytest
from scipy import stats

from oracle import sample as osm

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "philox_kat.json")


def test_philox_known_answer_vectors():
    with open(GOLDEN) as f:
        kat = json.load(f)
    for v in kat["vectors"]:
        c = [int(x, 16) for x in v["ctr"]]
        k = [int(x, 16) for x in v["key"]]
        out = osm.philox4x32_10(*c, *k)
        assert [int(o) for o in out] == [int(x, 16) for x in v["out"]]


def test_uniforms_open_interval_and_fp32_exact():
    u = osm.uniforms(123456789, (7 << 32) | 42, 10007)
    assert u.min() > 0 and u.max() < 1
    assert np.array_equal(u.astype(np.float32).astype(np.float64), u)
    assert abs(u.mean() - 0.5) < 0.01


@pytest.mark.parametrize("x", [[0.0, 1.0, -1.0, 2.0, 0.5, -3.0], [0.0] * 5])
def test_gumbel_max_realises_softmax(x):
    x = np.array(x)
    p = np.exp(x - x.max())
    p /= p.sum()
    n = 40000
    counts = np.zeros(x.size)
    for r in range(n):
        counts[osm.gumbel_argmax(x, 2026, r)[0]] += 1
    chi2 = ((counts - n * p) ** 2 / (n * p)).sum()
    assert stats.chi2.sf(chi2, x.size - 1) > 1e-4, (counts, n * p)


def test_dominant_logit_always_wins_and_seed_changes_draws():
    x = np.zeros(300)
    x[123] = 60.0
    assert all(osm.gumbel_argmax(x, s, r)[0] == 123 for s in (1, 2) for r in range(50))
    y = np.zeros(300)
    a = [osm.gumbel_argmax(y, 1, r)[0] for r in range(64)]
    b = [osm.gumbel_argmax(y, 2, r)[0] for r in range(64)]
    assert a != b and len(set(a)) > 30


# --------------------------------------------------------------------------- the T path of sample()
# sample() computes x = H W^T / T per row and draws argmax(x + g).  These pins tie the whole
# function (not only gumbel_argmax) to values fixed outside it: mpmath dot products, the softmax
# of the TEMPERED logits (§2, reading U7), the T -> 0 argmax limit, and the exact
# power-of-two metamorphic relation.  A dropped, doubled or inverted temperature fails them.

def _mp_tempered_softmax(h, W, T):
    import mpmath as mp
    with mp.workdps(40):
        xs = [mp.fsum(mp.mpf(float(a)) * mp.mpf(float(b)) for a, b in zip(h, w)) / mp.mpf(T) for w in W]
        m = max(xs)
        es = [mp.exp(x - m) for x in xs]
        s = mp.fsum(es)
        return np.array([float(e / s) for e in es]), [float(x) for x in xs]


def _small_head(seed, V=8, d=16, scale=0.9):
    import torch
    g = torch.Generator().manual_seed(seed)
    W = (torch.randn(V, d, generator=g) * scale).to(torch.bfloat16)
    h = torch.randn(1, d, generator=g).to(torch.bfloat16)
    return h, W


def test_sample_at_T07_realises_tempered_softmax_and_rejects_wrong_T():
    h, W = _small_head(11)
    n = 20000
    H = h.expand(n, -1)
    ids, _ = osm.sample(H, W, np.arange(n, dtype=np.uint64), seed=77, temperature=0.7)
    counts = np.bincount(ids, minlength=W.shape[0]).astype(np.float64)
    hv, Wv = h[0].double().numpy(), W.double().numpy()

    def chi2_sf(T):
        p, _ = _mp_tempered_softmax(hv, Wv, T)
        return stats.chi2.sf(((counts - n * p) ** 2 / (n * p)).sum(), W.shape[0] - 1)

    assert chi2_sf(0.7) > 1e-4
    # power: the same draws are incompatible with a dropped (T = 1), doubled (1.4) or squared-
    # away (0.35) temperature
    for wrong in (1.0, 1.4, 0.35):
        assert chi2_sf(wrong) < 1e-12, wrong


def test_sample_scores_equal_mpmath_tempered_logits_plus_gumbel():
    h, W = _small_head(12, V=40, d=24)
    keys = np.array([3, 99, 12345], dtype=np.uint64)
    H = h.expand(3, -1)
    T = 0.7
    ids, scores = osm.sample(H, W, keys, seed=5, temperature=T)
    _, xs = _mp_tempered_softmax(h[0].double().numpy(), W.double().numpy(), T)
    import mpmath as mp
    for r, k in enumerate(keys):
        u = osm.uniforms(5, int(k), W.shape[0])
        with mp.workdps(40):
            ref = [float(mp.mpf(x) - mp.log(-mp.log(mp.mpf(float(uu))))) for x, uu in zip(xs, u)]
        assert np.allclose(scores[r], ref, rtol=0, atol=1e-12)
        assert ids[r] == int(np.argmax(ref))


def test_sample_T_to_zero_is_argmax():
    import torch
    g = torch.Generator().manual_seed(13)
    V, d, n = 1000, 32, 64
    W = (torch.randn(V, d, generator=g) * 0.5).to(torch.bfloat16)
    H = torch.randn(n, d, generator=g).to(torch.bfloat16)
    z = H.double().numpy() @ W.double().numpy().T
    top2 = np.sort(z, axis=1)[:, -2:]
    clear = (top2[:, 1] - top2[:, 0]) > 0.05      # Gumbel noise spans < 20 nats; 0.05 / 1e-3 = 50
    assert clear.mean() > 0.5
    ids, _ = osm.sample(H, W, np.arange(n, dtype=np.uint64), seed=9, temperature=1e-3)
    assert np.array_equal(ids[clear], z.argmax(axis=1)[clear])


def test_sample_power_of_two_temperature_and_per_token_T():
    import torch
    g = torch.Generator().manual_seed(14)
    V, d, n = 300, 32, 16
    W = (torch.randn(V, d, generator=g) * 0.3).to(torch.bfloat16)
    H = torch.randn(n, d, generator=g).to(torch.bfloat16)
    keys = np.arange(n, dtype=np.uint64) * 7 + 1
    a = osm.sample(H, W, keys, seed=3, temperature=2.0)
    b = osm.sample((H.double() / 2).numpy(), W, keys, seed=3, temperature=1.0)   # H / 2 exact in fp64
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    Ts = np.where(np.arange(n) % 2 == 0, 0.7, 1.3)
    c = osm.sample(H, W, keys, seed=3, temperatures=Ts)
    for t in range(n):
        one = osm.sample(H[t:t + 1], W, keys[t:t + 1], seed=3, temperature=float(Ts[t]))
        assert c[0][t] == one[0][0] and np.array_equal(c[1][t], one[1][0])
