"""Pins for oracle.correct (delta / TIS / K / RS rows).

Pinned against: the values Table 1 prints (fixture
tests/golden/table1.json), closed forms of K1/K3, 60-digit mpmath
evaluations of exp / K3, exact rational arithmetic for the fixed point and the
thresholds, the paper's zero-mismatch special case and the K1
cancellation property.
"""
import json
import math
import os
from fractions import Fraction

import numpy as np
import pytest

from oracle import correct as oc
from oracle import exact

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "table1.json")


@pytest.fixture(scope="module")
def table1():
    with open(GOLDEN) as f:
        return json.load(f)


def _cfg(**kw):
    return oc.Cfg(**kw)


# ---------------------------------------------------------------- Table 1 ----

def test_table1_delta_matches_printed(table1):
    d = oc.delta(table1["logp_train"], table1["logp_rollout"])
    assert np.allclose(d, table1["delta_printed"], atol=1e-6, rtol=0)
    assert abs(d[3] - (-0.133)) < 1e-6 and abs(d[5] - (-0.008)) < 1e-6 and abs(d[0] - 0.001) < 1e-6


def test_table1_tis_and_k_values(table1):
    d = oc.delta(table1["logp_train"], table1["logp_rollout"])
    r = oc.exp_contract(d)
    assert abs(r[3] - 0.875465) < 1e-6                      # r_corr("that") = e^-0.133
    k3 = oc.k3_contract(d)
    assert abs(k3[3] - 0.008465092) < 1e-8                   # K3("that")
    assert abs(math.fsum(k3) - 0.0084975) < 1e-7             # sum over the sentence
    assert abs(math.fsum(-d) - 0.14) < 1e-6                  # sum K1
    # TIS at tau_tok = 2: no token exceeds the cap, weight = r_corr
    res = oc.correct(table1["logp_train"], table1["logp_rollout"], [0, 8],
                     _cfg(tis=True, tis_cap=2.0, log_tis_cap=math.log(2.0)))
    assert np.allclose(res["tis_w"], r.astype(np.float32)) and res["stats"]["n_truncated"] == 0


@pytest.mark.parametrize("seq_rs,agg,kept", [(oc.SEQ_K3, oc.AGG_SUM, 0), (oc.SEQ_K3, oc.AGG_MEAN, 0),
                                             (oc.SEQ_K1, oc.AGG_SUM, 0)])
def test_table1_sentence_rejected(table1, seq_rs, agg, kept):
    res = oc.correct(table1["logp_train"], table1["logp_rollout"], [0, 8],
                     _cfg(seq_rs=seq_rs, seq_agg=agg, tau_seq=table1["tau_seq"]))
    assert res["seq_keep"][0] == kept
    assert np.all(res["coeff"] == 0)


@pytest.mark.parametrize("agg", [oc.AGG_SUM, oc.AGG_MEAN])
def test_table1_without_flip_token_kept(table1, agg):
    keep = [i for i in range(8) if i != 3]
    lt = [table1["logp_train"][i] for i in keep]
    lr = [table1["logp_rollout"][i] for i in keep]
    res = oc.correct(lt, lr, [0, 7], _cfg(seq_rs=oc.SEQ_K3, seq_agg=agg, tau_seq=table1["tau_seq"]))
    assert abs(res["seq_partials"][0, 0] * 2.0 ** -52 - 3.24e-5) < 1e-6
    assert res["seq_keep"][0] == 1


# ----------------------------------------------------- contract vs exact ----

def _sweep():
    mags = np.logspace(-300, math.log10(1024.0), 3000)
    extra = np.array([1e-12, 1e-8, 0.5, 0.999999, 1.0, 1.0000001, math.log(2), 6.9, 6.94, 7.0, 709.0, 700.0,
                      2.0 ** -6, np.nextafter(2.0 ** -6, 1.0), np.nextafter(2.0 ** -6, 0.0),
                      2.0 ** -2, np.nextafter(2.0 ** -2, 1.0), np.nextafter(2.0 ** -2, 0.0)])
    v = np.concatenate([mags, extra, np.linspace(1e-4, 2.0 ** -5, 700), np.linspace(2.0 ** -6, 0.3, 700)])
    return np.concatenate([v, -v, [0.0]])


def test_k3_contract_within_4_ulp_of_60_digit_reference():
    d = _sweep()
    k3 = oc.k3_contract(d)
    worst = 0.0
    for x, y in zip(d, k3):
        ref = float(exact.k3_mp(float(x)))
        if x == 0.0:
            assert y == 0.0
            continue
        if x > 709.0:              # exp_c rule: +inf (token saturates, C.3.8)
            assert y == math.inf
            continue
        err = abs(y - ref) / exact.ulp(ref)   # ulp(0) = 2^-1074 in the subnormal range
        worst = max(worst, err)
    assert worst <= 4.0, worst


def test_exp_contract_within_2_ulp():
    d = np.concatenate([np.linspace(-700, 709, 4001), np.linspace(-2, 2, 2001), np.linspace(-0.26, 0.26, 2001),
                        [2.0 ** -2, -(2.0 ** -2), np.nextafter(2.0 ** -2, 1.0), np.nextafter(-(2.0 ** -2), -1.0)]])
    e = oc.exp_contract(d)
    for x, y in zip(d, e):
        ref = float(exact.exp_mp(float(x)))
        assert abs(y - ref) <= 2 * exact.ulp(ref)
    assert oc.exp_contract(np.array([0.0]))[0] == 1.0
    assert oc.exp_contract(np.array([710.0]))[0] == math.inf
    assert oc.exp_contract(np.array([-701.0]))[0] == 0.0


def test_k_closed_forms():
    assert oc.k3_contract(np.array([0.0]))[0] == 0.0                              # K3(1) = 0
    assert abs(oc.k3_contract(np.array([math.log(2.0)]))[0] - (1 - math.log(2))) < 4e-16   # K3(2)
    assert -np.float64(1.0) == -1.0                                                # K1(e) = -ln e
    q = np.log(np.array([2.0, 2.0]))
    assert abs(math.fsum(oc.k3_contract(q)) - 0.6137056) < 1e-7                  # q = [2, 2]


def test_fixed_point_is_round_half_even_of_exact_product():
    rng = np.random.default_rng(1)
    K = np.concatenate([rng.normal(0, 1e-3, 2000), rng.normal(0, 10, 2000),
                        np.array([2.5 * 2.0 ** -52, 3.5 * 2.0 ** -52, -2.5 * 2.0 ** -52, 1024.0, -1024.0])])
    X, sat = oc.fixed_point(K)
    assert not sat.any()
    for k, x in zip(K, X):
        f = Fraction(float(k)) * 2 ** 52
        fl = math.floor(f)
        rem = f - fl
        want = fl + (1 if rem > Fraction(1, 2) or (rem == Fraction(1, 2) and fl % 2) else 0)
        assert int(x) == want
    X, sat = oc.fixed_point(np.array([1024.0000000001, -2000.0, math.inf]))
    assert sat.all() and list(X) == [2 ** 62, -(2 ** 62), 2 ** 62]


# ------------------------------------------------------ special cases ----

def test_zero_mismatch_collapses_everything():
    rng = np.random.default_rng(2)
    lp = -np.abs(rng.normal(0, 2, 5000)).astype(np.float32)
    cu = [0, 1000, 2500, 5000]
    cfg = _cfg(tis=True, tok_rs=True, seq_rs=oc.SEQ_K3, seq_agg=oc.AGG_SUM, tau_seq=1e-3)
    res = oc.correct(lp, lp.copy(), cu, cfg)
    assert np.all(res["delta"] == 0) and np.all(res["tis_w"] == 1.0)
    assert np.all(res["tok_keep"] == 1) and np.all(res["seq_keep"] == 1) and np.all(res["coeff"] == 1.0)
    st = res["stats"]
    assert st["sum_abs_delta"] == st["sum_k1"] == st["sum_k3"] == 0
    assert st["n_truncated"] == st["n_tok_rejected"] == st["n_seq_rejected"] == st["n_saturated"] == 0
    assert st["max_abs_delta"] == 0.0 and st["mean_k3"] == 0.0


def test_k1_cancels_exactly_k3_does_not():
    base = np.full(200, -1.0, np.float32)
    dd = np.float32(0.03125)
    num = base.copy()
    num[0::2] += dd
    num[1::2] -= dd
    res = oc.correct(num, base, [0, 200], _cfg(seq_rs=oc.SEQ_K1, seq_agg=oc.AGG_SUM, tau_seq=0.0))
    assert res["stats"]["sum_k1"] == 0 and res["stats"]["sum_k3"] > 0
    assert res["seq_partials"][0, 0] == 0 and res["seq_keep"][0] == 1   # S = 0 <= 0


def test_huge_thresholds_never_reject_or_truncate():
    rng = np.random.default_rng(3)
    den = -np.abs(rng.normal(0, 3, 3000)).astype(np.float32)
    num = (den + rng.normal(0, 0.3, 3000)).astype(np.float32)
    d = oc.delta(num, den)
    cap = float(np.exp(d.max())) * 2
    cfg = _cfg(tis=True, tis_cap=cap, log_tis_cap=math.log(cap), seq_rs=oc.SEQ_K3, tau_seq=1000.0)
    res = oc.correct(num, den, [0, 1000, 3000], cfg)
    assert res["stats"]["n_truncated"] == 0 and np.all(res["seq_keep"] == 1)


def test_less_equal_edge_sum_and_mean():
    # tau = 2^-10 -> threshold floor(2^-10 * 2^52) = 2^42; K1 = 2^-20 per token -> X = 2^32.
    den = np.full(1025, -1.0, np.float32)
    num = np.full(1025, np.float32(-1.0 - 2.0 ** -20), np.float32)
    assert float(num[0]) == -1.0 - 2.0 ** -20
    cfg = _cfg(seq_rs=oc.SEQ_K1, seq_agg=oc.AGG_SUM, tau_seq=2.0 ** -10)
    assert oc.correct(num[:1024], den[:1024], [0, 1024], cfg)["seq_keep"][0] == 1   # X_s == thr: keep
    assert oc.correct(num, den, [0, 1025], cfg)["seq_keep"][0] == 0                # one unit more: reject
    cfgm = _cfg(seq_rs=oc.SEQ_K1, seq_agg=oc.AGG_MEAN, tau_seq=2.0 ** -20)
    assert oc.correct(num, den, [0, 1025], cfgm)["seq_keep"][0] == 1               # mean == tau: keep
    num2 = num.copy()
    num2[7] = np.float32(-1.0 - 2.0 ** -19)
    assert oc.correct(num2, den, [0, 1025], cfgm)["seq_keep"][0] == 0


def test_mean_threshold_is_exact_rational_floor():
    rng = np.random.default_rng(4)
    for _ in range(3000):
        tau = float(10 ** rng.uniform(-8, 2)) * (1 if rng.random() < 0.9 else -1)
        T = int(rng.integers(0, 2 ** 31))
        thr = oc.seq_threshold(tau, T, oc.AGG_MEAN)
        # X <= tau 2^52 T  <=>  X <= thr, for X on both sides of thr
        for X in (thr, thr + 1):
            assert (Fraction(X) <= Fraction(tau) * 2 ** 52 * T) == (X <= thr)


def test_saturated_sequence_rejected_and_counted():
    den = np.array([-9.0, -1.0, -1.0, -1.0], np.float32)
    num = np.array([-1.0, -1.0, -1.0, -1.0], np.float32)   # delta = 8 -> K3 = e^8 - 9 > 2^10
    res = oc.correct(num, den, [0, 1, 4], _cfg(seq_rs=oc.SEQ_K3, seq_agg=oc.AGG_MEAN, tau_seq=1e3))
    assert list(res["seq_keep"]) == [0, 1] and res["stats"]["n_saturated"] == 1


def test_non_finite_is_a_data_error_with_first_index():
    num = np.zeros(10, np.float32)
    den = np.zeros(10, np.float32)
    num[6] = np.nan
    den[8] = -np.inf
    with pytest.raises(oc.DataError) as e:
        oc.correct(num, den, [0, 10], _cfg())
    assert e.value.index == 6


def test_prompt_only_sequence_is_kept_and_excluded():
    num = np.array([-1, -1, -5, -1], np.float32)
    den = np.array([-1, -3, -1, -1], np.float32)
    mask = np.array([1, 1, 0, 0], np.uint8)
    res = oc.correct(num, den, [0, 2, 4], _cfg(seq_rs=oc.SEQ_K3, seq_agg=oc.AGG_MEAN, tau_seq=1e-3), mask)
    assert list(res["seq_keep"]) == [0, 1]
    assert res["stats"]["n_resp_tok"] == 2 and res["coeff"][2] == 0 and res["coeff"][3] == 0


def test_token_rs_bounds_inclusive():
    lo, hi = math.log(0.5), math.log(2.0)
    den = np.zeros(4, np.float32) - 1.0
    d = np.array([hi, hi + 1e-3, lo, lo - 1e-3])
    num = (den + d).astype(np.float32)
    dd = oc.delta(num, den)
    cfg = _cfg(tok_rs=True, log_tok_lo=lo, log_tok_hi=hi)
    res = oc.correct(num, den, [0, 4], cfg)
    assert list(res["tok_keep"]) == [int(lo <= x <= hi) for x in dd]
    assert res["stats"]["n_tok_rejected"] == 4 - int(res["tok_keep"].sum())


def test_sharding_is_exact_and_order_free():
    rng = np.random.default_rng(5)
    N = 5000
    cu = np.array([0, 700, 701, 2600, 2600, 5000])   # includes an empty and a 1-token sequence
    den = -np.abs(rng.normal(0, 2, N)).astype(np.float32)
    num = (den + rng.laplace(0, 0.01, N)).astype(np.float32)
    mask = (rng.random(N) < 0.8).astype(np.uint8)
    cfg = _cfg(tis=True, tok_rs=True, seq_rs=oc.SEQ_K3, seq_agg=oc.AGG_MEAN, tau_seq=1e-3)
    full = oc.correct(num, den, cu, cfg, mask)
    for cuts in ([0, 1234, 5000], [0, 700, 2000, 2601, 5000], [0, 1, 2, 4999, 5000]):
        parts = []
        for a, b in zip(cuts[:-1], cuts[1:]):
            _, g, s = oc.local_partials(num[a:b], den[a:b], cu, cfg, mask[a:b], a)
            parts.append((g, s))
        for order in (parts, parts[::-1]):
            glob, seq = oc.combine(order)
            assert (seq == full["seq_partials"]).all()
            keep, score = oc.decide(seq, cfg)
            assert np.array_equal(keep, full["seq_keep"]) and np.array_equal(score, full["seq_score"])
            st = oc.finalize_stats(glob, keep, len(cu) - 1)
            assert st == full["stats"]


def test_contract_decisions_match_exact_real_decisions():
    """No seeded sequence lies in the tie band: the fixed-point decision equals the
    exact real-number decision sum_t K3(delta_t) <= tau (mpmath) everywhere."""
    import mpmath as mp
    rng = np.random.default_rng(6)
    S, L = 40, 64
    den = -np.abs(rng.normal(0, 2, S * L)).astype(np.float32)
    num = (den + rng.laplace(0, 2e-3, S * L)).astype(np.float32)
    cu = np.arange(0, S * L + 1, L)
    for tau in (1e-4, 1e-3, 3e-3):
        res = oc.correct(num, den, cu, _cfg(seq_rs=oc.SEQ_K3, tau_seq=tau))
        d = oc.delta(num, den)
        for s in range(S):
            with mp.workdps(40):
                Sx = mp.fsum(exact.k3_mp(float(x)) for x in d[cu[s]:cu[s + 1]])
            assert int(Sx <= mp.mpf(tau)) == res["seq_keep"][s]


def test_tokens_outside_the_sequences_are_a_data_error():
    """Reading U13b: a shard reaching past cu[S] (or starting before cu[0]) is a data error with
    the first offending global index, never a silent attribution to some sequence."""
    num = np.zeros(8, np.float32)
    den = np.zeros(8, np.float32)
    cfg = _cfg(seq_rs=oc.SEQ_K3)
    # local tokens 100..107 against sequences covering [0, 104)
    with pytest.raises(oc.DataError) as e:
        oc.local_partials(num, den, [0, 50, 104], cfg, None, 100)
    assert e.value.index == 104
    # a shard entirely past the end: its first token
    with pytest.raises(oc.DataError) as e:
        oc.local_partials(num, den, [0, 50, 104], cfg, None, 200)
    assert e.value.index == 200
    # an earlier non-finite token wins (min index)
    num[1] = np.nan
    with pytest.raises(oc.DataError) as e:
        oc.local_partials(num, den, [0, 50, 104], cfg, None, 100)
    assert e.value.index == 101
    # exactly covering shard: fine
    oc.local_partials(np.zeros(4, np.float32), np.zeros(4, np.float32), [0, 50, 104], cfg, None, 100)


# ------------------------------------------------ fused multiply-add (C.3 rev. 4) ----

def _fma_exact(a, b, c):
    """RN(a b + c) of the exact rational (CPython's int / int true division rounds correctly)."""
    return float(Fraction(float(a)) * Fraction(float(b)) + Fraction(float(c)))


def test_fma_is_the_correctly_rounded_exact_value():
    rng = np.random.default_rng(11)
    a, b, c = [], [], []
    # the contract's regime: Horner state Q in (0, 1], d in [-1, 1] at every scale, c = RN(1/n!)
    for n in range(2, 23):
        q = rng.uniform(0.0, 1.0, 300)
        d = rng.uniform(-1, 1, 300) * np.exp2(-rng.integers(0, 150, 300).astype(np.float64))
        a += list(q); b += list(d); c += [oc.INV_FACT[n]] * 300
    # general finite operands with every exponent gap between a b and c
    x = rng.normal(size=3000) * np.exp2(rng.integers(-60, 60, 3000).astype(np.float64))
    y = rng.normal(size=3000) * np.exp2(rng.integers(-60, 60, 3000).astype(np.float64))
    z = rng.normal(size=3000) * np.exp2(rng.integers(-180, 120, 3000).astype(np.float64))
    a += list(x); b += list(y); c += list(z)
    # exact ties and near-ties that only a single rounding resolves: A, B odd 53-bit integers,
    # C cancels the top bits of A B so that RN(A B + C) rounds a 54 / 55-bit remainder
    for k in (54, 55, 56):
        for _ in range(400):
            A = int(rng.integers(2 ** 52, 2 ** 53)) | 1
            B = int(rng.integers(2 ** 52, 2 ** 53)) | 1
            P = A * B
            C = -((P >> k) << k)
            a.append(math.ldexp(A, -53)); b.append(math.ldexp(B, -60)); c.append(math.ldexp(C, -113))
    a, b, c = np.array(a), np.array(b), np.array(c)
    got = oc.fma(a, b, c)
    want = np.array([_fma_exact(*t) for t in zip(a, b, c)])
    assert np.array_equal(got.view(np.int64), want.view(np.int64))
    # a plain a * b + c (two roundings) differs on some of these: the test can tell them apart
    assert not np.array_equal((a * b + c).view(np.int64), want.view(np.int64))
