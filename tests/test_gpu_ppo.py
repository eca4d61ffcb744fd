"""GPU tests of tim_ppo_loss against the fp64 oracle (oracle/ppo.py).

Bit-exact: per-token loss / grad (fp32 bits), clip flags, sequence losses (f64 bits), the C(r)
histograms and every statistic (same decision-path contract on both sides, exact int sums).
"""
import math

import numpy as np
import pytest
import torch

import synth
from oracle import correct as oc
from oracle import ppo as op

pytestmark = pytest.mark.gpu
DEV = "cuda"


def _ocfg(c):
    return op.PPOCfg(clip_lo=1.0 - c.eps, clip_hi=1.0 + c.eps, hist_lo=c.hist_lo,
                     hist_inv_width=c.hist_bins / (c.hist_hi - c.hist_lo), hist_bins=c.hist_bins)


def _inputs(n_seq, L, seed, move=0.05):
    cu = synth.cu_seqlens(n_seq, L, seed, variable=True)
    N = int(cu[-1])
    g = torch.Generator().manual_seed(seed)
    old = -torch.empty(N).exponential_(0.7, generator=g)
    cur = synth.policy_move(old, seed, sd=move)
    adv = torch.randn(N, generator=g)
    adv[torch.rand(N, generator=g) < 0.05] = 0.0
    mask = synth.resp_mask(cu, max(1, L // 8))
    return cur.float(), old.float(), adv.float(), cu, mask


def _compare(res, ref):
    assert np.array_equal(res["loss"].cpu().numpy().view(np.uint32), ref["loss"].view(np.uint32))
    assert np.array_equal(res["grad"].cpu().numpy().view(np.uint32), ref["grad"].view(np.uint32))
    assert np.array_equal(res["clipped"].cpu().numpy(), ref["clipped"])
    assert np.array_equal(res["seq_loss"].cpu().numpy().view(np.uint64), ref["seq_loss"].view(np.uint64))
    assert np.array_equal(res["hist"].cpu().numpy(), ref["hist"])
    for k, v in ref["stats"].items():
        assert res["stats"][k] == v, (k, res["stats"][k], v)


@pytest.mark.parametrize("eps,move,bins", [(0.04, 0.05, 64), (0.1, 0.3, 200), (0.28, 0.01, 1)])
def test_ppo_bit_exact_vs_oracle_with_mask(tim, eps, move, bins):
    cur, old, adv, cu, mask = _inputs(29, 800, 40 + bins, move)
    cfg = tim.PPOConfig(eps=eps, hist_lo=-0.5, hist_hi=0.5, hist_bins=bins)
    res = tim.ppo_loss(cur.to(DEV), old.to(DEV), adv.to(DEV), cu.to(DEV), cfg, resp_mask=mask.to(DEV))
    ref = op.ppo(cur.numpy(), old.numpy(), adv.numpy(), cu.numpy(), _ocfg(cfg), resp_mask=mask.numpy())
    _compare(res, ref)
    assert 0 < res["stats"]["n_clipped"] < res["stats"]["n_contrib"] or bins == 1


def test_ppo_on_correction_coefficients(tim):
    """The App. A.4 chain: coeff = tim_correct(train_old vs rollout) weights the PPO tokens."""
    cur, old, adv, cu, mask = _inputs(17, 1200, 50)
    roll = synth.perturb_laplace_mix(old, 51)
    c = tim.PRESETS["tis-srs-k3-corr-ratio"]
    corr = tim.correct(old.to(DEV), roll.to(DEV), cu.to(DEV), tim.CorrectConfig(
        tis=True, tis_cap=2.0, seq_rs=oc.SEQ_K3, seq_agg=oc.AGG_MEAN, tau_seq=1e-3), mask.to(DEV))
    coeff = corr["coeff"]
    cfg = tim.PPOConfig(eps=0.2)
    res = tim.ppo_loss(cur.to(DEV), old.to(DEV), adv.to(DEV), cu.to(DEV), cfg, coeff=coeff)
    ref = op.ppo(cur.numpy(), old.numpy(), adv.numpy(), cu.numpy(), _ocfg(cfg), coeff=coeff.cpu().numpy())
    _compare(res, ref)
    assert res["stats"]["n_seq_contrib"] == int((corr["seq_keep"].cpu() != 0).sum())
    del c


def test_ppo_on_policy_is_minus_advantage(tim):
    cur, old, adv, cu, mask = _inputs(5, 300, 60)
    res = tim.ppo_loss(old.to(DEV), old.to(DEV), adv.to(DEV), cu.to(DEV), tim.PPOConfig(), resp_mask=mask.to(DEV))
    m = mask.bool()
    assert torch.equal(res["loss"].cpu()[m], -adv[m]) and res["stats"]["n_clipped"] == 0
    assert res["stats"]["sum_k1"] == 0 and res["stats"]["sum_k3"] == 0


@pytest.mark.parametrize("P", [2, 5])
def test_ppo_fake_ranks_split_form(tim, P):
    cur, old, adv, cu, mask = _inputs(13, 700, 70)
    N = cur.numel()
    cfg = tim.PPOConfig(eps=0.2, hist_bins=32)
    full = tim.ppo_loss(cur.to(DEV), old.to(DEV), adv.to(DEV), cu.to(DEV), cfg, resp_mask=mask.to(DEV))
    cuts = [tim.shard_range(N, P, r, align=1) for r in range(P)]
    locs = [tim.ppo_local(cur[a:b].to(DEV), old[a:b].to(DEV), adv[a:b].to(DEV), cu.to(DEV), cfg,
                          resp_mask=mask[a:b].to(DEV), tok_begin=a) for a, b in cuts]
    fin = tim.ppo_finish(torch.cat([l["partial"] for l in locs]), P, cu.numel() - 1, cfg)
    assert torch.equal(fin["seq_loss"], full["seq_loss"]) and torch.equal(fin["hist"], full["hist"])
    assert torch.equal(fin["stats_raw"], full["stats_raw"])
    assert torch.equal(torch.cat([l["loss"] for l in locs]).view(torch.int32), full["loss"].view(torch.int32))


def test_ppo_nan_status(tim):
    from paper_2605_14220_b200.tim import new_status, read_status
    cur, old, adv, cu, mask = _inputs(4, 400, 80)
    cur[777] = float("nan")
    st = new_status(DEV)
    res = tim.ppo_loss(cur.to(DEV), old.to(DEV), adv.to(DEV), cu.to(DEV), tim.PPOConfig(), status=st)
    assert read_status(st) == (9, 777) and math.isnan(res["loss"][777].item())


@pytest.mark.parametrize("wmode", ["coeff", "mask", "none"])
def test_ppo_lock_step_edges_bit_exact(tim, wmode):
    """The lock-step path's edges (csrc/ppo.cu): a single slow token inside an otherwise clean
    128-token chunk (|delta| just above / at 2^-2, |loss| just above 2^8, a non-finite advantage),
    A = 0 tokens (the per-lane sink slot of the C(r) histogram), C(r) below / above the histogram
    range and exactly on a bin edge, tokens clipped on both sides, sequence starts inside a lane's
    four tokens; every weight source (coefficient / response mask / none: three kernel
    instantiations).  Element-wise bit-exact against oracle/ppo.py."""
    from paper_2605_14220_b200.tim import new_status, read_status
    L = 128 * 6
    cu = torch.tensor([0, 130, 131, 640, 2 * L - 5, 2 * L, 3 * L], dtype=torch.int64)  # starts inside lanes
    N = int(cu[-1])
    g = torch.Generator().manual_seed(90 + len(wmode))
    old = -torch.empty(N).exponential_(0.7, generator=g)
    cur = synth.policy_move(old, 91, sd=0.03)
    adv = torch.randn(N, generator=g)
    d = torch.zeros(N)
    d[200], d[333], d[1000] = 0.25, 0.2500001, -0.75      # |delta| at / above the fast bound, large
    cur[200], cur[333], cur[1000] = old[200] + d[200], old[333] + d[333], old[1000] + d[1000]
    adv[444] = 300.0                                       # |loss| > 2^8 on a fast delta
    adv[445] = 0.0
    adv[512:640] = 0.0                                     # a whole chunk of A = 0
    cur[700], adv[700] = old[700] + 0.5, 1.0               # clipped high
    cur[701], adv[701] = old[701] - 0.5, -1.0              # clipped low
    cur[702], adv[702] = old[702], 0.25                    # r = 1 exactly: C = 0 on a bin edge
    cur[703], adv[703] = old[703] - 0.2, 100.0             # C far above the range
    cur[704], adv[704] = old[704] + 0.2, 100.0             # C far below the range
    cfg = tim.PPOConfig(eps=0.2, hist_lo=-0.5, hist_hi=0.5, hist_bins=40)
    mask = synth.resp_mask(cu, 7)
    coeff = (torch.rand(N, generator=g) * 2).float() * mask.float()
    kw, okw = {}, {}
    if wmode == "coeff":
        kw, okw = {"coeff": coeff.to(DEV)}, {"coeff": coeff.numpy()}
    elif wmode == "mask":
        kw, okw = {"resp_mask": mask.to(DEV)}, {"resp_mask": mask.numpy()}
    res = tim.ppo_loss(cur.float().to(DEV), old.float().to(DEV), adv.float().to(DEV), cu.to(DEV), cfg, **kw)
    ref = op.ppo(cur.float().numpy(), old.float().numpy(), adv.float().numpy(), cu.numpy(), _ocfg(cfg), **okw)
    _compare(res, ref)
    # a non-finite advantage inside a clean chunk: data error, token excluded, the rest unchanged
    adv2 = adv.clone()
    adv2[900] = float("inf")
    st = new_status(DEV)
    res2 = tim.ppo_loss(cur.float().to(DEV), old.float().to(DEV), adv2.float().to(DEV), cu.to(DEV), cfg,
                        status=st, **kw)
    assert read_status(st) == (9, 900)
    keep = torch.ones(N, dtype=torch.bool)
    keep[900] = False
    assert torch.equal(res2["loss"].cpu()[keep].view(torch.int32), res["loss"].cpu()[keep].view(torch.int32))
