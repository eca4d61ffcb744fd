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
