"""GPU tests aimed at the correction kernel's chunk paths (csrc/correct.cu): the select-free fast
body with its warp-uniform sequence cursor, the in-lane redo of slow tokens (|delta| > 2^-6 or
non-finite) inside otherwise clean chunks, the masked body for chunks holding a sequence or
prompt/response boundary, and the non-interior configurations that route every chunk through the
masked body.  Every case is bit-exact against the oracle (oracle/correct.py), as in
test_gpu_correct.py; the inputs are shaped so that each path is taken many times."""
import math

import numpy as np
import pytest
import torch

from oracle import correct as oc

pytestmark = pytest.mark.gpu
DEV = "cuda"


def _ocfg(c):
    return oc.Cfg(tis=c.tis, tis_cap=c.tis_cap, log_tis_cap=math.log(c.tis_cap), tok_rs=c.tok_rs,
                  log_tok_lo=math.log(c.tok_lo), log_tok_hi=math.log(c.tok_hi), seq_rs=c.seq_rs,
                  seq_agg=c.seq_agg, tau_seq=c.tau_seq)


def _compare(res, ref):
    assert np.array_equal(res["tis_w"].cpu().numpy().view(np.uint32), ref["tis_w"].view(np.uint32))
    assert np.array_equal(res["tok_keep"].cpu().numpy(), ref["tok_keep"])
    assert np.array_equal(res["seq_keep"].cpu().numpy(), ref["seq_keep"])
    assert np.array_equal(res["coeff"].cpu().numpy().view(np.uint32), ref["coeff"].view(np.uint32))
    assert np.array_equal(res["seq_score"].cpu().numpy().view(np.uint64), ref["seq_score"].view(np.uint64))
    for k in ("n_tok", "n_resp_tok", "n_truncated", "n_tok_rejected", "n_seq_rejected", "n_saturated",
              "sum_abs_delta", "sum_k1", "sum_k3", "max_abs_delta"):
        assert res["stats"][k] == ref["stats"][k], (k, res["stats"][k], ref["stats"][k])


def _deltas(n, seed, p_slow):
    """den ~ -Exp(0.7); delta = 0 / Laplace(2e-3) / (w.p. p_slow) Laplace(0.3): the last are the
    slow tokens of an otherwise clean chunk."""
    g = np.random.default_rng(seed)
    den = -g.exponential(0.7, n).astype(np.float32)
    d = g.laplace(0, 2e-3, n)
    d[g.random(n) < 0.5] = 0.0
    big = g.random(n) < p_slow
    d[big] = g.laplace(0, 0.3, big.sum())
    num = np.minimum(den + d, 0.0).astype(np.float32)
    return num, den


def _run(tim, num, den, cu, mask, c):
    cu_t = torch.as_tensor(np.asarray(cu, np.int64))
    m_t = None if mask is None else torch.as_tensor(mask)
    res = tim.correct(torch.as_tensor(num).to(DEV), torch.as_tensor(den).to(DEV), cu_t.to(DEV), c,
                      None if m_t is None else m_t.to(DEV))
    ref = oc.correct(num, den, np.asarray(cu, np.int64), _ocfg(c), mask)
    _compare(res, ref)
    return res


CFGS = [
    dict(tis=True, tis_cap=2.0, seq_rs=oc.SEQ_K3, seq_agg=oc.AGG_SUM, tau_seq=1e-3),
    dict(tis=True, tis_cap=2.0, tok_rs=True, tok_lo=0.5, tok_hi=2.0, seq_rs=oc.SEQ_K1, seq_agg=oc.AGG_MEAN,
         tau_seq=3e-4),
    dict(tis=False, seq_rs=oc.SEQ_K3, seq_agg=oc.AGG_MEAN, tau_seq=1e-5),
    dict(tis=True, tis_cap=1.5, tok_rs=True, tok_lo=0.8, tok_hi=1.25),
]


@pytest.mark.parametrize("kw", CFGS)
@pytest.mark.parametrize("L", [4096, 128, 384])
def test_chunk_aligned_sequences(tim, kw, L):
    """Sequence and prompt boundaries on chunk boundaries: every chunk takes the fast body, the
    cursor advances at each sequence start; slow tokens sit inside clean chunks."""
    S = max(2, (1 << 18) // L)
    n = S * L
    num, den = _deltas(n, 1 + L, 2e-3)
    cu = np.arange(S + 1, dtype=np.int64) * L
    mask = (np.arange(n) % L >= L // 4).astype(np.uint8)
    _run(tim, num, den, cu, mask, tim.CorrectConfig(**kw))


@pytest.mark.parametrize("kw", CFGS)
def test_ragged_sequences_with_empty_ones(tim, kw):
    """Random lengths 0..700 (empty sequences included): boundaries inside chunks take the masked
    body, after which the lanes return to one cursor; prompts of random length."""
    g = np.random.default_rng(5)
    lens = g.integers(0, 700, 600)
    lens[g.random(600) < 0.05] = 0
    cu = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    n = int(cu[-1])
    num, den = _deltas(n, 6, 1e-3)
    mask = np.zeros(n, np.uint8)
    for s in range(600):
        a, b = int(cu[s]), int(cu[s + 1])
        mask[a + int(g.integers(0, max(1, b - a + 1))):b] = 1
    _run(tim, num, den, cu, mask, tim.CorrectConfig(**kw))


@pytest.mark.parametrize("kw", CFGS[:2])
def test_tiny_sequences(tim, kw):
    """1..5-token sequences: many boundaries per chunk (each lane walks several sequences)."""
    g = np.random.default_rng(7)
    lens = g.integers(1, 6, 40000)
    cu = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    n = int(cu[-1])
    num, den = _deltas(n, 8, 1e-2)
    _run(tim, num, den, cu, None, tim.CorrectConfig(**kw))


@pytest.mark.parametrize("kw", [dict(tis=True, tis_cap=1.01, seq_rs=oc.SEQ_K3, tau_seq=1e-3),
                                dict(tis=True, tis_cap=0.9, seq_rs=oc.SEQ_K1, seq_agg=oc.AGG_MEAN, tau_seq=1e-4),
                                dict(tok_rs=True, tok_lo=0.995, tok_hi=1.005, seq_rs=oc.SEQ_K3, tau_seq=1e-3),
                                dict(tis=True, tis_cap=2.0, tok_rs=True, tok_lo=1.001, tok_hi=3.0)])
def test_non_interior_configs(tim, kw):
    """Thresholds inside |delta| <= 2^-6 (truncation / rejection possible for small deltas): the
    launcher routes every chunk through the masked body."""
    L = 1024
    S = 64
    num, den = _deltas(S * L, 9, 2e-3)
    cu = np.arange(S + 1, dtype=np.int64) * L
    mask = (np.arange(S * L) % L >= 100).astype(np.uint8)
    _run(tim, num, den, cu, mask, tim.CorrectConfig(**kw))


def test_non_finite_inside_clean_chunks(tim):
    """NaN / inf in response and prompt tokens of chunks that are otherwise clean: status carries
    the first bad index, the token is excluded from every sum and count (oracle: drop the tokens)."""
    from paper_2605_14220_b200.tim import new_status, read_status
    L, S = 4096, 16
    n = L * S
    num, den = _deltas(n, 10, 1e-3)
    cu = np.arange(S + 1, dtype=np.int64) * L
    mask = (np.arange(n) % L >= 1024).astype(np.uint8)
    bad = [5000, 5001, 20000, 20480 + 3, 60000]   # response and prompt tokens
    num[bad[0]] = np.nan
    num[bad[1]] = np.inf
    den[bad[2]] = -np.inf
    num[bad[3]] = np.nan
    den[bad[4]] = np.nan
    c = tim.CorrectConfig(tis=True, seq_rs=oc.SEQ_K3, seq_agg=oc.AGG_MEAN, tau_seq=1e-4)
    st = new_status(DEV)
    res = tim.correct(torch.as_tensor(num).to(DEV), torch.as_tensor(den).to(DEV), torch.as_tensor(cu).to(DEV), c,
                      torch.as_tensor(mask).to(DEV), status=st)
    assert read_status(st) == (9, min(bad))
    w = res["tis_w"].cpu().numpy()
    assert np.isnan(w[bad]).all()
    assert (res["coeff"].cpu().numpy()[bad] == 0).all() and (res["tok_keep"].cpu().numpy()[bad] == 0).all()
    # the oracle's data error stops at the first bad token: compare the rest with the bad
    # tokens taken out of the response mask and given delta = 0 (they add nothing, count nothing)
    keep = np.ones(n, bool)
    keep[bad] = False
    num2, den2, mask2 = num.copy(), den.copy(), mask.copy()
    num2[bad] = den2[bad] = -1.0
    mask2[bad] = 0
    ref = oc.correct(num2, den2, cu, _ocfg(c), mask2)
    got = res["stats"]
    for k in ("n_resp_tok", "sum_abs_delta", "sum_k1", "sum_k3", "max_abs_delta", "n_seq_rejected"):
        assert got[k] == ref["stats"][k], k
    assert np.array_equal(res["seq_keep"].cpu().numpy(), ref["seq_keep"])
    assert np.array_equal(w[keep].view(np.uint32), ref["tis_w"][keep].view(np.uint32))


@pytest.mark.parametrize("P", [3, 7])
def test_split_form_with_unaligned_cuts(tim, P):
    """Shards cut at offsets that are not multiples of 128 (the warp's chunks straddle sequence
    starts at a different phase on every rank): the split form equals the single call."""
    L, S = 4096, 24
    n = L * S
    num, den = _deltas(n, 11, 2e-3)
    cu = torch.arange(S + 1, dtype=torch.int64) * L
    mask = torch.as_tensor((np.arange(n) % L >= 777).astype(np.uint8))
    c = tim.CorrectConfig(tis=True, tok_rs=True, tok_lo=0.6, tok_hi=1.7, seq_rs=oc.SEQ_K3, seq_agg=oc.AGG_SUM,
                          tau_seq=2e-2)
    numt, dent = torch.as_tensor(num).to(DEV), torch.as_tensor(den).to(DEV)
    full = tim.correct(numt, dent, cu.to(DEV), c, mask.to(DEV))
    ref = oc.correct(num, den, cu.numpy(), _ocfg(c), mask.numpy())
    _compare(full, ref)
    cuts = [0] + [r * n // P + 37 * r for r in range(1, P)] + [n]
    locs = []
    for r in range(P):
        a, b = cuts[r], cuts[r + 1]
        locs.append(tim.correct_local(numt[a:b], dent[a:b], cu.to(DEV), c, mask[a:b].to(DEV), tok_begin=a))
    gathered = torch.cat([loc["partial"] for loc in locs])
    for r in range(P):
        a, b = cuts[r], cuts[r + 1]
        out = tim.correct_finish(gathered, P, cu.to(DEV), c, locs[r]["coeff"], tok_begin=a)
        assert torch.equal(out["seq_keep"], full["seq_keep"])
        assert torch.equal(locs[r]["coeff"].view(torch.int32), full["coeff"][a:b].view(torch.int32))


@pytest.mark.parametrize("kw", CFGS)
def test_fused_single_launch_equals_split_launches(tim, kw):
    """P = 1: the cooperative one-launch form (pass 1 + decisions + zeroing behind grid barriers)
    and the split local / finish / zero launches give the same bits (both also == the oracle)."""
    from paper_2605_14220_b200.tim import debug_set_correct_split
    g = np.random.default_rng(12)
    lens = g.integers(1, 5000, 150)
    cu = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    n = int(cu[-1])
    num, den = _deltas(n, 13, 2e-3)
    mask = (g.random(n) < 0.9).astype(np.uint8)
    c = tim.CorrectConfig(**kw)
    split = _run(tim, num, den, cu, mask, c)
    try:
        debug_set_correct_split(False)
        fused = _run(tim, num, den, cu, mask, c)
    finally:
        debug_set_correct_split(True)
    for k in ("tis_w", "tok_keep", "seq_keep", "coeff", "seq_score", "stats_raw"):
        assert torch.equal(split[k], fused[k]), k
