"""GPU tests of the round-1 advisor / verdict robustness findings.

* a shard reaching past cu[n_seq] (or starting before cu[0]) is a data error with the first
  outside index, in correct and PPO, matching oracle.correct / oracle.ppo (reading U13b), and no
  access leaves the arrays (compute-sanitizer runs in scripts/sanitize.sh);
* a non-finite PPO advantage / coefficient is a data error: loss NaN, grad 0, clip flag 0, the
  token out of every count, sum and histogram (reading U13), matching the oracle on the same
  input with that token's weight zeroed;
* mixed host / device arguments never hand a host pointer to a kernel;
* calls on two CUDA streams at once do not share a workspace.
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
    return oc.Cfg(tis=c.tis, tis_cap=c.tis_cap, log_tis_cap=math.log(c.tis_cap), tok_rs=c.tok_rs,
                  log_tok_lo=math.log(c.tok_lo), log_tok_hi=math.log(c.tok_hi), seq_rs=c.seq_rs,
                  seq_agg=c.seq_agg, tau_seq=c.tau_seq)


@pytest.mark.parametrize("tok_begin,n", [(900, 300), (1500, 128), (1000, 200)])
def test_shard_past_the_sequences_is_a_data_error(tim, tok_begin, n):
    cu = torch.tensor([0, 400, 1000, 1100], dtype=torch.int64)
    g = torch.Generator().manual_seed(1)
    den = -torch.rand(n, generator=g)
    num = den + 0.01 * torch.randn(n, generator=g)
    cfg = tim.PRESETS["tis-srs-k3-corr-ratio"]
    st = tim.new_status(DEV)
    tim.correct(num.to(DEV), den.to(DEV), cu.to(DEV), cfg, tok_begin=tok_begin, status=st, return_stats=False)
    with pytest.raises(oc.DataError) as e:
        oc.local_partials(num.numpy(), den.numpy(), cu.numpy(), _ocfg(cfg), None, tok_begin)
    assert tim.read_status(st) == (9, e.value.index)
    # PPO: same range check
    st = tim.new_status(DEV)
    pc = tim.PPOConfig()
    tim.ppo_loss(num.to(DEV), den.to(DEV), torch.ones(n, device=DEV), cu.to(DEV), pc, tok_begin=tok_begin,
                 status=st, return_stats=False)
    assert tim.read_status(st) == (9, e.value.index)
    torch.cuda.synchronize()


def test_shard_inside_the_sequences_is_clean(tim):
    cu = torch.tensor([0, 400, 1000, 1100], dtype=torch.int64, device=DEV)
    den = -torch.rand(100, device=DEV)
    st = tim.new_status(DEV)
    tim.correct(den + 0.01, den, cu, tim.PRESETS["tis-srs-k3-corr-ratio"], tok_begin=1000, status=st)
    assert tim.read_status(st) == (0, 0)


@pytest.mark.parametrize("bad", ["nan_adv", "inf_adv", "nan_coeff"])
def test_ppo_non_finite_advantage_or_coeff(tim, bad):
    cu = synth.cu_seqlens(9, 700, 3, variable=True)
    N = int(cu[-1])
    g = torch.Generator().manual_seed(4)
    old = -torch.empty(N).exponential_(0.7, generator=g)
    cur = old + 0.05 * torch.randn(N, generator=g)
    adv = torch.randn(N, generator=g)
    coeff = torch.ones(N)
    k1, k2 = N // 3, 2 * N // 3
    if bad == "nan_adv":
        adv[k1] = float("nan")
        adv[k2] = float("nan")
    elif bad == "inf_adv":
        adv[k1] = float("-inf")
        adv[k2] = float("inf")
    else:
        coeff[k1] = float("nan")
        coeff[k2] = float("inf")
    cfg = tim.PPOConfig(eps=0.2, hist_lo=-0.5, hist_hi=0.5, hist_bins=32)
    st = tim.new_status(DEV)
    res = tim.ppo_loss(cur.to(DEV), old.to(DEV), adv.to(DEV), cu.to(DEV), cfg, coeff=coeff.to(DEV), status=st)
    ocfg = op.PPOCfg(clip_lo=0.8, clip_hi=1.2, hist_lo=-0.5, hist_inv_width=32.0, hist_bins=32)
    with pytest.raises(op.DataError) as e:
        op.ppo(cur.numpy(), old.numpy(), adv.numpy(), cu.numpy(), ocfg, coeff=coeff.numpy())
    assert tim.read_status(st) == (9, e.value.index) and e.value.index == k1
    loss, grad, clipped = res["loss"].cpu(), res["grad"].cpu(), res["clipped"].cpu()
    for k in (k1, k2):
        assert math.isnan(loss[k].item()) and grad[k].item() == 0.0 and clipped[k].item() == 0
    # every statistic equals the oracle's on the same input with the bad tokens' weight zeroed
    a2, c2 = adv.clone(), coeff.clone()
    a2[[k1, k2]] = 0.0
    c2[[k1, k2]] = 0.0
    ref = op.ppo(cur.numpy(), old.numpy(), a2.numpy(), cu.numpy(), ocfg, coeff=c2.numpy())
    assert np.array_equal(res["hist"].cpu().numpy(), ref["hist"])
    assert np.array_equal(res["seq_loss"].cpu().numpy().view(np.uint64), ref["seq_loss"].view(np.uint64))
    for k, v in ref["stats"].items():
        assert res["stats"][k] == v, (k, res["stats"][k], v)


def test_mixed_host_and_device_arguments(tim):
    cu = synth.cu_seqlens(5, 300, 6, variable=True)
    N = int(cu[-1])
    den = -torch.rand(N, generator=torch.Generator().manual_seed(6))
    num = den + 0.003
    mask = synth.resp_mask(cu, 30)
    cfg = tim.PRESETS["tis-srs-k3-corr-ratio"]
    ref = tim.correct(num.to(DEV), den.to(DEV), cu.to(DEV), cfg, mask.to(DEV))
    for a, b, c, m in [(num.to(DEV), den, cu, mask), (num.to(DEV), den.to(DEV), cu, mask), (num, den.to(DEV), cu.to(DEV), mask)]:
        got = tim.correct(a, b, c, cfg, m, device=DEV)
        assert torch.equal(got["coeff"].cpu(), ref["coeff"].cpu())
        assert torch.equal(got["seq_keep"].cpu(), ref["seq_keep"].cpu())


def test_two_streams_do_not_share_a_workspace(tim):
    V, d = 151936, 256
    W = synth.head_weight(V, d, 7, device=DEV)
    out = []
    for s in range(2):
        ids = synth.token_ids(3000, V, 7 + s, device=DEV)
        H = synth.hidden_states(3000, d, 7 + s, device=DEV, weight=W, ids=ids, mode="peaked")
        out.append((H, ids, tim.logprob(H, W, ids)))
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    torch.cuda.synchronize()
    with torch.cuda.stream(s1):
        a = tim.logprob(out[0][0], W, out[0][1])
    with torch.cuda.stream(s2):
        b = tim.logprob(out[1][0], W, out[1][1])
    torch.cuda.synchronize()
    for got, (_, _, ref) in zip((a, b), out):
        assert torch.equal(got[0].view(torch.int32), ref[0].view(torch.int32))
        assert torch.equal(got[1].view(torch.int32), ref[1].view(torch.int32))


def test_l2_persisting_set_aside(tim):
    """tim_l2_persisting (application-level L2 setup used by bench.py): the driver grants at least the
    request up to the device maximum (rounding up), 0 clears it, and a log-prob call after either
    setting gives the same bits (the set-aside is a cache policy, never a result)."""
    import synth
    W = synth.head_weight(3000, 256, 5, device="cuda")
    ids = synth.token_ids(700, 3000, 5, device="cuda")
    H = synth.hidden_states(700, 256, 5, device="cuda", weight=W, ids=ids, mode="peaked")
    g = tim.l2_persisting(48 << 20)
    assert g >= 48 << 20
    a = tim.logprob(H, W, ids)
    assert tim.l2_persisting(0) == 0
    b = tim.logprob(H, W, ids)
    assert torch.equal(a[0].view(torch.int32), b[0].view(torch.int32))
    assert tim.l2_persisting(1 << 40) == tim.l2_persisting(1 << 41)   # clamped to the device maximum
    tim.l2_persisting(0)
