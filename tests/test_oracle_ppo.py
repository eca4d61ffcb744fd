"""Pins for oracle.ppo (NEXT-2 fused PPO surrogate + diagnostics).

Tied to the paper's definitions by closed forms (eq:ppo_loss P:352-360 evaluated by hand),
an independent evaluation of -min(rA, clip(r) A) with mpmath, finite-difference gradients
(the score-function gradient, and "C has the same gradient as -r A"), exact
histogram edges, fsum for the sequence / batch averages and sharding exactness.
"""
import math

import mpmath as mp
import numpy as np
import pytest

from oracle import ppo as op

CFG = op.PPOCfg(clip_lo=0.8, clip_hi=1.2, hist_lo=-1.0, hist_inv_width=32.0, hist_bins=64)


def _lp(d):
    """lp_old = -1, lp_cur = -1 + d (fp32), so delta is the fp32-representable d."""
    old = np.full(len(d), -1.0, np.float32)
    cur = (old + np.asarray(d, np.float32)).astype(np.float32)
    return cur, old


def test_on_policy_closed_form():
    cur, old = _lp([0.0, 0.0, 0.0])
    adv = np.array([2.0, -1.5, 0.0], np.float32)
    res = op.ppo(cur, old, adv, [0, 3], CFG)
    assert list(res["loss"]) == [-2.0, 1.5, 0.0] and list(res["grad"]) == [-2.0, 1.5, 0.0]
    assert res["stats"]["n_clipped"] == 0 and res["stats"]["sum_k1"] == 0 and res["stats"]["sum_k3"] == 0
    assert res["hist"][0, 33] == 1 and res["hist"][1, 33] == 1 and res["stats"]["n_zero_adv"] == 1


def test_clip_branches_closed_form():
    cur, old = _lp([0.5, -0.5, -0.5, 0.5])
    adv = np.array([2.0, -1.0, 2.0, -1.0], np.float32)
    res = op.ppo(cur, old, adv, [0, 4], CFG)
    d = (cur.astype(np.float64) - old.astype(np.float64))
    r = np.exp(d)
    want = [-1.2 * 2.0, -0.8 * -1.0, -r[2] * 2.0, -r[3] * -1.0]
    assert np.allclose(res["loss"], want, rtol=1e-7, atol=0)
    assert list(res["clipped"]) == [1, 1, 0, 0] and res["grad"][0] == 0 and res["grad"][1] == 0
    assert res["grad"][2] == res["loss"][2] and res["grad"][3] == res["loss"][3]


def test_loss_is_minus_min_of_unclipped_and_clipped():
    rng = np.random.default_rng(0)
    d = rng.normal(0, 0.3, 2000)
    cur, old = _lp(d)
    adv = rng.normal(0, 1, 2000).astype(np.float32)
    w = rng.uniform(0, 2, 2000).astype(np.float32)
    res = op.ppo(cur, old, adv, [0, 2000], CFG, coeff=w)
    with mp.workdps(30):
        for t in range(0, 2000, 7):
            r = mp.exp(mp.mpf(float(cur[t])) - mp.mpf(float(old[t])))
            A = mp.mpf(float(adv[t]))
            want = -mp.mpf(float(w[t])) * min(r * A, min(max(r, mp.mpf(0.8)), mp.mpf(1.2)) * A)
            assert abs(float(want) - float(res["loss"][t])) <= 1e-6 * max(1.0, abs(float(want)))


def test_gradient_is_score_function_derivative():
    rng = np.random.default_rng(1)
    d = rng.normal(0, 0.3, 400)
    adv = rng.normal(0, 1, 400)
    h = 1e-6
    for t in range(400):
        A = adv[t]

        def L(x):
            r = math.exp(x)
            return -min(r * A, min(max(r, 0.8), 1.2) * A)

        if abs(math.exp(d[t]) - 1.2) < 1e-4 or abs(math.exp(d[t]) - 0.8) < 1e-4:
            continue   # kink of the clip
        fd = (L(d[t] + h) - L(d[t] - h)) / (2 * h)
        cur, old = _lp([d[t]])
        res = op.ppo(cur, old, np.array([A], np.float32), [0, 1], CFG)
        dd = float(cur[0]) - float(old[0])
        fd = (L(dd + h) - L(dd - h)) / (2 * h)
        assert abs(float(res["grad"][0]) - fd) < 1e-5 * max(1, abs(fd))


def test_zero_centred_contribution_and_its_gradient():
    rng = np.random.default_rng(2)
    d = rng.normal(0, 0.2, 300)
    cur, old = _lp(d)
    adv = rng.normal(0, 1, 300).astype(np.float32)
    res = op.ppo(cur, old, adv, [0, 300], CFG)
    r = np.exp(cur.astype(np.float64) - old.astype(np.float64))
    assert np.allclose(res["C"], -(r - 1) * adv, rtol=1e-12, atol=1e-15)
    # dC/dlp = -r A = d(-r A)/dlp: finite difference on the C definition
    h = 1e-6
    dd = cur.astype(np.float64) - old
    fd = (-(np.exp(dd + h) - 1) * adv - (-(np.exp(dd - h) - 1) * adv)) / (2 * h)
    assert np.allclose(fd, -r * adv, rtol=1e-5, atol=1e-8)


def test_histogram_edges_are_exact():
    # C = -(r - 1) A with r = 1 + k/32 exactly representable: pick A = -1 so C = r - 1
    ks = np.arange(-31, 50)
    r = 1.0 + ks / 32.0
    d = np.log(r)
    cur, old = _lp(d)
    res = op.local(cur, old, -np.ones(len(ks), np.float32), [0, len(ks)], CFG)
    C = res[0]["C"]
    raw = np.floor((C + 1.0) * 32.0)
    want = np.where(raw < 0, 0, np.where(raw >= 64, 65, raw + 1))
    assert res[1]["hist"][1].sum() == len(ks) and res[1]["hist"][0].sum() == 0
    assert np.array_equal(np.bincount(want.astype(int), minlength=66), res[1]["hist"][1])
    assert np.all((C >= -1.0 + (want - 1) / 32.0) | (want == 0))


def test_sequence_and_batch_averages():
    rng = np.random.default_rng(3)
    cu = np.array([0, 100, 100, 350, 351, 900])
    d = rng.normal(0, 0.05, 900)
    cur, old = _lp(d)
    adv = rng.normal(0, 1, 900).astype(np.float32)
    coeff = (rng.random(900) < 0.9).astype(np.float32) * rng.uniform(0.5, 2, 900).astype(np.float32)
    res = op.ppo(cur, old, adv, cu, CFG, coeff=coeff)
    r = np.exp(cur.astype(np.float64) - old.astype(np.float64))
    A = adv.astype(np.float64)
    L = -coeff.astype(np.float64) * np.minimum(r * A, np.clip(r, 0.8, 1.2) * A)   # eq:ppo_loss, fp64
    sums = [math.fsum(L[cu[s]:cu[s + 1]]) for s in range(5)]
    assert np.allclose(res["seq_loss"], sums, rtol=0, atol=1e-9)
    n_contrib_seq = sum(1 for s in range(5) if (coeff[cu[s]:cu[s + 1]] != 0).any())
    assert res["stats"]["n_seq_contrib"] == n_contrib_seq == 4
    assert abs(res["stats"]["batch_loss"] - math.fsum(sums) / 4) < 1e-9


def test_sharding_is_exact():
    rng = np.random.default_rng(4)
    cu = np.array([0, 700, 1300, 3000])
    d = rng.normal(0, 0.1, 3000)
    cur, old = _lp(d)
    adv = rng.normal(0, 1, 3000).astype(np.float32)
    mask = (rng.random(3000) < 0.7).astype(np.uint8)
    full = op.ppo(cur, old, adv, cu, CFG, resp_mask=mask)
    for cuts in ([0, 1000, 3000], [0, 699, 701, 2999, 3000]):
        parts = [op.local(cur[a:b], old[a:b], adv[a:b], cu, CFG, resp_mask=mask[a:b], tok_begin=a)[1:]
                 for a, b in zip(cuts[:-1], cuts[1:])]
        glob, seq = op.combine(parts)
        seq_loss, st = op.finish(glob, seq)
        assert np.array_equal(seq_loss, full["seq_loss"]) and st == full["stats"]
        assert np.array_equal(glob["hist"], full["hist"])


def test_non_finite_advantage_is_a_data_error():
    """Reading U13 for NEXT-2: a non-finite advantage (GRPO whitening of a zero-variance group
    gives NaN) or coefficient is a data error with the first index, not a histogrammed token."""
    cu = np.array([0, 6])
    cur = np.full(6, -1.0, np.float32)
    old = np.full(6, -1.0, np.float32)
    adv = np.ones(6, np.float32)
    adv[4] = np.nan
    with pytest.raises(op.DataError) as e:
        op.ppo(cur, old, adv, cu, CFG)
    assert e.value.index == 4
    adv[4] = 1.0
    coeff = np.ones(6, np.float32)
    coeff[2] = np.inf
    with pytest.raises(op.DataError) as e:
        op.ppo(cur, old, adv, cu, CFG, coeff=coeff)
    assert e.value.index == 2
    adv[3] = -np.inf
    with pytest.raises(op.DataError) as e:
        op.local(cur, old, adv, cu, CFG, tok_begin=0)
    assert e.value.index == 3
