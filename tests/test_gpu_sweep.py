"""C4 mismatch sweep: rollout log-probs from tim_logprob on a C1-shaped batch,
trainer log-probs from the three perturbation modes (P1 bf16 rounding of the log-probs, P2 one-ulp
flips of the hidden states re-scored by tim_logprob, P3 the Laplace mixture), and the correction
grid -- tau_tok x (tau_seq x {SUM, MEAN} x {K1, K3}) x masking signal {r_corr, r_ppo}.  Every
cell: masks, counts, weights, coefficients and statistics bit-exact vs the oracle, and the
split form over P = 2 / 8 fake ranks (sequences cut mid-way) identical to the single call."""
import math

import numpy as np
import pytest
import torch

import synth
from oracle import correct as oc

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
DEV = "cuda"
TAU_TOK = (1.25, 1.5, 2.0, 3.0, 5.0)
TAU_SEQ = (1e-4, 3e-4, 1e-3, 3e-3, 1e-2)


def _ocfg(c):
    return oc.Cfg(tis=c.tis, tis_cap=c.tis_cap, log_tis_cap=math.log(c.tis_cap), tok_rs=c.tok_rs,
                  log_tok_lo=math.log(c.tok_lo), log_tok_hi=math.log(c.tok_hi), seq_rs=c.seq_rs,
                  seq_agg=c.seq_agg, tau_seq=c.tau_seq)


@pytest.fixture(scope="module")
def batch(tim):
    cfg = synth.CONFIGS["c1"]
    n_seq, L = 16, cfg.seq_len                       # 65,536 tokens of the C1 shape
    N = n_seq * L
    W = synth.head_weight(cfg.vocab, cfg.hidden, cfg.seed, device=DEV)
    ids = synth.token_ids(N, cfg.vocab, cfg.seed, device=DEV)
    H = synth.hidden_states(N, cfg.hidden, cfg.seed, device=DEV, weight=W, ids=ids, mode="peaked")
    roll, _ = tim.logprob(H, W, ids)
    p2, _ = tim.logprob(synth.perturb_hidden_ulp(H, 1e-3, cfg.seed), W, ids)
    train = {"p1": synth.perturb_bf16(roll), "p2": p2, "p3": synth.perturb_laplace_mix(roll, cfg.seed)}
    cur = synth.policy_move(roll, cfg.seed, sd=0.01)
    cu = synth.cu_seqlens(n_seq, L)
    mask = synth.resp_mask(cu, cfg.prompt_len)
    del H, W
    torch.cuda.empty_cache()
    return roll, train, cur, cu, mask


def _cells():
    for tt in TAU_TOK:
        yield dict(tis=True, tis_cap=tt, seq_rs=oc.SEQ_K3, seq_agg=oc.AGG_SUM, tau_seq=1e-3)
    for ts in TAU_SEQ:
        for agg in (oc.AGG_SUM, oc.AGG_MEAN):
            for k in (oc.SEQ_K1, oc.SEQ_K3):
                yield dict(tis=True, tis_cap=2.0, tok_rs=True, tok_lo=0.5, tok_hi=2.0, seq_rs=k, seq_agg=agg,
                           tau_seq=ts)


@pytest.mark.parametrize("mode", ["p1", "p2", "p3"])
@pytest.mark.parametrize("signal", ["r_corr", "r_ppo"])
def test_c4_grid_bit_exact(tim, batch, mode, signal):
    roll, train, cur, cu, mask = batch
    num = train[mode] if signal == "r_corr" else cur   # r_corr: train_old / rollout; r_ppo: cur / rollout
    num_h, den_h, cu_h, m_h = num.cpu().numpy(), roll.cpu().numpy(), cu.numpy(), mask.numpy()
    cu_d, m_d = cu.to(DEV), mask.to(DEV)
    rejected = []
    for kw in _cells():
        c = tim.CorrectConfig(**kw)
        res = tim.correct(num, roll, cu_d, c, m_d)
        ref = oc.correct(num_h, den_h, cu_h, _ocfg(c), m_h)
        for k in ("tok_keep", "seq_keep"):
            assert np.array_equal(res[k].cpu().numpy(), ref[k]), (kw, k)
        for k in ("tis_w", "coeff"):
            assert np.array_equal(res[k].cpu().numpy().view(np.uint32), ref[k].view(np.uint32)), (kw, k)
        for k in ("n_resp_tok", "n_truncated", "n_tok_rejected", "n_seq_rejected", "n_saturated", "sum_abs_delta",
                  "sum_k1", "sum_k3", "max_abs_delta"):
            assert res["stats"][k] == ref["stats"][k], (kw, k)
        rejected.append(res["stats"]["n_seq_rejected"])
    assert len(rejected) == len(TAU_TOK) + 4 * len(TAU_SEQ)


@pytest.mark.parametrize("P", [2, 8])
def test_c4_split_form_across_ranks(tim, batch, P):
    roll, train, cur, cu, mask = batch
    num = train["p3"]
    N = num.numel()
    cu_d, m_d = cu.to(DEV), mask.to(DEV)
    for kw in (dict(tis=True, seq_rs=oc.SEQ_K3, seq_agg=oc.AGG_SUM, tau_seq=1e-3),
               dict(tis=True, tok_rs=True, seq_rs=oc.SEQ_K1, seq_agg=oc.AGG_MEAN, tau_seq=3e-4)):
        c = tim.CorrectConfig(**kw)
        full = tim.correct(num, roll, cu_d, c, m_d)
        cuts = [round(r * N / P) + (101 if 0 < r < P else 0) for r in range(P + 1)]   # mid-sequence cuts
        cuts[-1] = N
        locs = []
        for r in range(P):
            a, b = cuts[r], cuts[r + 1]
            locs.append(tim.correct_local(num[a:b], roll[a:b], cu_d, c, m_d[a:b], tok_begin=a))
        gathered = torch.cat([loc["partial"] for loc in locs])
        for r in range(P):
            a, b = cuts[r], cuts[r + 1]
            out = tim.correct_finish(gathered, P, cu_d, c, locs[r]["coeff"], tok_begin=a)
            assert torch.equal(out["seq_keep"], full["seq_keep"])
            assert torch.equal(locs[r]["coeff"].view(torch.int32), full["coeff"][a:b].view(torch.int32))
            assert torch.equal(locs[r]["tok_keep"], full["tok_keep"][a:b])
            st = tim.stats_from_bytes(out["stats_raw"])
            for k in ("n_seq_rejected", "sum_k1", "sum_k3", "sum_abs_delta", "n_tok_rejected", "max_abs_delta"):
                assert st[k] == full["stats"][k], (P, r, k)
