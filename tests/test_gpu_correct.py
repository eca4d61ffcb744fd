"""GPU tests of tim_correct / tim_mismatch_stats / the split local+finish form.

Bar (BASELINE.json north_star): masks, counts and sequence decisions bit-exact vs the oracle
on identical log-prob inputs; tis_w, coeff, seq_score and the exact integer statistics are
bit-exact too (same C.3 arithmetic contract on both sides).
"""
import itertools
import json
import math
import os

import numpy as np
import pytest
import torch

import synth
from oracle import correct as oc

pytestmark = pytest.mark.gpu
DEV = "cuda"


def _ocfg(c):
    return oc.Cfg(tis=c.tis, tis_cap=c.tis_cap, log_tis_cap=math.log(c.tis_cap), tok_rs=c.tok_rs,
                  log_tok_lo=math.log(c.tok_lo), log_tok_hi=math.log(c.tok_hi), seq_rs=c.seq_rs,
                  seq_agg=c.seq_agg, tau_seq=c.tau_seq)


def _inputs(n_seq, L, seed, variable=True, mode="p3", prompt=None):
    cu = synth.cu_seqlens(n_seq, L, seed, variable=variable)
    N = int(cu[-1])
    g = torch.Generator().manual_seed(seed)
    den = -torch.empty(N).exponential_(0.7, generator=g)
    if mode == "p3":
        num = synth.perturb_laplace_mix(den, seed)
    elif mode == "p1":
        num = synth.perturb_bf16(den)
    else:
        num = den.clone()
    mask = synth.resp_mask(cu, prompt if prompt is not None else max(1, L // 8))
    return num.float(), den.float(), cu, mask


def _compare(res, ref, cfg):
    assert np.array_equal(res["tis_w"].cpu().numpy().view(np.uint32), ref["tis_w"].view(np.uint32))
    assert np.array_equal(res["tok_keep"].cpu().numpy(), ref["tok_keep"])
    assert np.array_equal(res["seq_keep"].cpu().numpy(), ref["seq_keep"])
    assert np.array_equal(res["coeff"].cpu().numpy().view(np.uint32), ref["coeff"].view(np.uint32))
    assert np.array_equal(res["seq_score"].cpu().numpy().view(np.uint64), ref["seq_score"].view(np.uint64))
    s, r = res["stats"], ref["stats"]
    for k in ("n_tok", "n_resp_tok", "n_seq", "n_truncated", "n_tok_rejected", "n_seq_rejected", "n_saturated",
              "sum_abs_delta", "sum_k1", "sum_k3", "max_abs_delta", "mean_abs_delta", "mean_k1", "mean_k3"):
        assert s[k] == r[k], (k, s[k], r[k])


GRID = list(itertools.product([False, True], [False, True], [oc.SEQ_NONE, oc.SEQ_K1, oc.SEQ_K3],
                              [oc.AGG_SUM, oc.AGG_MEAN]))


@pytest.mark.parametrize("tis,tok_rs,seq_rs,agg", GRID)
def test_bit_exact_vs_oracle_grid(tim, tis, tok_rs, seq_rs, agg):
    num, den, cu, mask = _inputs(37, 700, 100 + seq_rs * 4 + agg * 2 + tis)
    for tau in (1e-4, 1e-3, 1e-2):
        c = tim.CorrectConfig(tis=tis, tis_cap=1.5 if tok_rs else 2.0, tok_rs=tok_rs, tok_lo=0.8, tok_hi=1.25,
                              seq_rs=seq_rs, seq_agg=agg, tau_seq=tau)
        res = tim.correct(num.to(DEV), den.to(DEV), cu.to(DEV), c, mask.to(DEV))
        ref = oc.correct(num.numpy(), den.numpy(), cu.numpy(), _ocfg(c), mask.numpy())
        _compare(res, ref, c)


@pytest.mark.parametrize("name", ["srs-k3-corr-ratio", "srs-k3-ppo-ratio", "tis-srs-k3-corr-ratio",
                                  "tis-srs-k1-corr-ratio"])
@pytest.mark.parametrize("mode", ["p1", "p3"])
def test_paper_presets(tim, name, mode):
    num, den, cu, mask = _inputs(64, 3072, 7, variable=False, mode=mode, prompt=1024)
    c = tim.PRESETS[name]
    res = tim.correct(num.to(DEV), den.to(DEV), cu.to(DEV), c, mask.to(DEV))
    ref = oc.correct(num.numpy(), den.numpy(), cu.numpy(), _ocfg(c), mask.numpy())
    _compare(res, ref, c)


def test_table1_on_gpu(tim):
    with open(os.path.join(os.path.dirname(__file__), "golden", "table1.json")) as f:
        t1 = json.load(f)
    num = torch.tensor(t1["logp_train"], dtype=torch.float32)
    den = torch.tensor(t1["logp_rollout"], dtype=torch.float32)
    cu = torch.tensor([0, 8])
    for seq_rs, agg in ((oc.SEQ_K3, oc.AGG_SUM), (oc.SEQ_K3, oc.AGG_MEAN), (oc.SEQ_K1, oc.AGG_SUM)):
        c = tim.CorrectConfig(tis=True, tis_cap=t1["tau_tok"], seq_rs=seq_rs, seq_agg=agg, tau_seq=t1["tau_seq"])
        res = tim.correct(num.to(DEV), den.to(DEV), cu.to(DEV), c)
        assert res["seq_keep"].item() == 0 and torch.all(res["coeff"] == 0)
        assert abs(res["tis_w"][3].item() - 0.875465) < 1e-6


def test_zero_mismatch_and_huge_thresholds(tim):
    num, den, cu, mask = _inputs(20, 500, 3, mode="zero")
    c = tim.CorrectConfig(tis=True, tok_rs=True, seq_rs=oc.SEQ_K3, tau_seq=1e-3)
    res = tim.correct(num.to(DEV), den.to(DEV), cu.to(DEV), c, mask.to(DEV))
    assert torch.all(res["tis_w"] == 1) and torch.all(res["tok_keep"] == 1) and torch.all(res["seq_keep"] == 1)
    st = res["stats"]
    assert st["sum_abs_delta"] == st["sum_k1"] == st["sum_k3"] == 0 and st["n_seq_rejected"] == 0
    assert st["max_abs_delta"] == 0.0


def test_less_equal_edge(tim):
    den = torch.full((1025,), -1.0)
    num = torch.full((1025,), -1.0 - 2.0 ** -20)
    c = tim.CorrectConfig(seq_rs=oc.SEQ_K1, seq_agg=oc.AGG_SUM, tau_seq=2.0 ** -10)
    keep = tim.correct(num[:1024].to(DEV), den[:1024].to(DEV), torch.tensor([0, 1024], device=DEV), c)["seq_keep"]
    rej = tim.correct(num.to(DEV), den.to(DEV), torch.tensor([0, 1025], device=DEV), c)["seq_keep"]
    assert keep.item() == 1 and rej.item() == 0


def test_mismatch_stats_matches_correct(tim):
    num, den, cu, mask = _inputs(16, 1000, 4)
    st = tim.mismatch_stats(num.to(DEV), den.to(DEV), cu.to(DEV), mask.to(DEV))
    ref = oc.correct(num.numpy(), den.numpy(), cu.numpy(), oc.Cfg(), mask.numpy())["stats"]
    for k in ("n_tok", "n_resp_tok", "sum_abs_delta", "sum_k1", "sum_k3", "max_abs_delta", "mean_abs_delta",
              "mean_k1", "mean_k3"):
        assert st[k] == ref[k], k


def test_nan_reported_in_status_word(tim):
    from paper_2605_14220_b200.tim import new_status, read_status
    num, den, cu, mask = _inputs(8, 300, 5)
    num[1234] = float("nan")
    den[1500] = float("-inf")
    st = new_status(DEV)
    tim.correct(num.to(DEV), den.to(DEV), cu.to(DEV), tim.CorrectConfig(seq_rs=oc.SEQ_K3), mask.to(DEV), status=st)
    assert read_status(st) == (9, 1234)


@pytest.mark.parametrize("P", [2, 3, 8])
def test_fake_ranks_split_form_equals_single_call(tim, P):
    """One process runs pass 1 on P token shards (sequences straddle shards), concatenates the
    partial blocks in rank order and finishes each shard: identical bits to the P = 1 call."""
    num, den, cu, mask = _inputs(23, 900, 9)
    N = num.numel()
    c = tim.CorrectConfig(tis=True, tok_rs=True, tok_lo=0.9, tok_hi=1.1, seq_rs=oc.SEQ_K3, seq_agg=oc.AGG_MEAN,
                          tau_seq=2e-3)
    full = tim.correct(num.to(DEV), den.to(DEV), cu.to(DEV), c, mask.to(DEV))
    cuts = [tim.shard_range(N, P, r, align=1) for r in range(P)]
    locs = [tim.correct_local(num[a:b].to(DEV), den[a:b].to(DEV), cu.to(DEV), c, mask[a:b].to(DEV), tok_begin=a)
            for a, b in cuts]
    gathered = torch.cat([l["partial"] for l in locs])
    coeff = []
    for (a, b), l in zip(cuts, locs):
        fin = tim.correct_finish(gathered, P, cu, c, l["coeff"], tok_begin=a)
        assert torch.equal(fin["seq_keep"], full["seq_keep"])
        assert torch.equal(fin["seq_score"], full["seq_score"])
        assert torch.equal(fin["stats_raw"], full["stats_raw"])
        coeff.append(l["coeff"])
    assert torch.equal(torch.cat(coeff).view(torch.int32), full["coeff"].view(torch.int32))


@pytest.mark.slow
def test_c3_scale_bit_exact(tim):
    """C3 (512 x 16384 tokens) sequence-RS K3 / MEAN and K1 / SUM at tau = 1e-3, bit-exact."""
    cfg = synth.CONFIGS["c3"]
    num, den, cu, mask = _inputs(cfg.n_seq, cfg.seq_len, cfg.seed, variable=False, prompt=cfg.prompt_len)
    for seq_rs, agg in ((oc.SEQ_K3, oc.AGG_MEAN), (oc.SEQ_K1, oc.AGG_SUM)):
        c = tim.CorrectConfig(tis=True, seq_rs=seq_rs, seq_agg=agg, tau_seq=1e-3)
        res = tim.correct(num.to(DEV), den.to(DEV), cu.to(DEV), c, mask.to(DEV))
        ref = oc.correct(num.numpy(), den.numpy(), cu.numpy(), _ocfg(c), mask.numpy())
        _compare(res, ref, c)


def test_nccl_comm_path_single_rank(tim):
    """tim_correct through a libtim-owned NCCL communicator (world size 1 on this one-GPU box):
    exercises tim_comm_unique_id / tim_comm_init / ncclAllGather / tim_comm_destroy and must give
    the same bits as the comm-less call."""
    import os
    import torch.distributed as dist
    own = not dist.is_initialized()
    if own:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29533")
        dist.init_process_group("gloo", rank=0, world_size=1)
    try:
        comm = tim.Comm()
        num, den, cu, mask = _inputs(9, 600, 21)
        c = tim.CorrectConfig(tis=True, seq_rs=oc.SEQ_K3, seq_agg=oc.AGG_MEAN, tau_seq=1e-3)
        a = tim.correct(num.to(DEV), den.to(DEV), cu.to(DEV), c, mask.to(DEV))
        b = tim.correct(num.to(DEV), den.to(DEV), cu.to(DEV), c, mask.to(DEV), comm=comm)
        for k in ("tis_w", "tok_keep", "seq_keep", "coeff", "seq_score", "stats_raw"):
            assert torch.equal(a[k], b[k]), k
        comm.close()
    finally:
        if own:
            dist.destroy_process_group()


def test_alignment_variants_match_the_oracle(tim):
    """The pass-1 load paths: 16-B aligned log-probs with a 16-B aligned mask (everything through
    the bulk-copy ring), with a mask that is only 4-B aligned (register prefetch of the mask), and
    4-B aligned log-probs (element-wise path) -- all bit-exact vs the oracle."""
    num, den, cu, mask = _inputs(24, 2000, 77)
    N = int(cu[-1])
    c = tim.CorrectConfig(tis=True, tok_rs=True, tok_lo=0.8, tok_hi=1.25, seq_rs=oc.SEQ_K3,
                          seq_agg=oc.AGG_MEAN, tau_seq=1e-3)
    pad = 8
    for off_lp, off_m in ((0, 0), (0, 4), (4, 4), (1, 3)):
        nb = torch.zeros(N + pad, dtype=torch.float32)
        db = torch.zeros(N + pad, dtype=torch.float32)
        mb = torch.zeros(N + pad, dtype=torch.uint8)
        nb[off_lp:off_lp + N] = num
        db[off_lp:off_lp + N] = den
        mb[off_m:off_m + N] = mask
        nd, dd, md = nb.to(DEV), db.to(DEV), mb.to(DEV)
        res = tim.correct(nd[off_lp:off_lp + N], dd[off_lp:off_lp + N], cu.to(DEV), c, md[off_m:off_m + N])
        ref = oc.correct(num.numpy(), den.numpy(), cu.numpy(), _ocfg(c), mask.numpy())
        _compare(res, ref, c)
