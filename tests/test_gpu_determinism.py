"""Run-to-run determinism (SURVEY.md §5 "repeat 100x bitwise"): the same call repeated on the
same inputs returns the same bits every time -- the fixed reduction splits and orders (U20), the
exact integer sums of the corrections, and the block-ordered dW accumulation leave nothing to
scheduling or atomics order."""
import hashlib

import pytest
import torch

import synth

pytestmark = pytest.mark.gpu
DEV = "cuda"


def _digest(*ts):
    h = hashlib.sha256()
    for t in ts:
        h.update(t.contiguous().cpu().numpy().tobytes())
    return h.hexdigest()


def _head(N, d, V, seed):
    W = synth.head_weight(V, d, seed, device=DEV)
    ids = synth.token_ids(N, V, seed, device=DEV)
    H = synth.hidden_states(N, d, seed, device=DEV, weight=W, ids=ids, mode="peaked")
    return H, W, ids


def test_logprob_and_sample_repeat_100x_bitwise(tim):
    H, W, ids = _head(4096, 2048, 151936, 71)
    ref = _digest(*tim.logprob(H, W, ids))
    for _ in range(99):
        assert _digest(*tim.logprob(H, W, ids)) == ref
    keys = torch.arange(4096, device=DEV, dtype=torch.int64)
    sref = _digest(*tim.sample(H, W, keys, seed=5, temperature=0.7))
    for _ in range(19):
        assert _digest(*tim.sample(H, W, keys, seed=5, temperature=0.7)) == sref


def test_correct_and_ppo_repeat_100x_bitwise(tim):
    cu = synth.cu_seqlens(300, 4096, 72, variable=True)
    n = int(cu[-1])
    g = torch.Generator(device=DEV).manual_seed(72)
    den = -torch.empty(n, device=DEV).exponential_(0.7, generator=g)
    num = synth.perturb_laplace_mix(den, 72)
    mask = synth.resp_mask(cu, 512).to(DEV)
    cu = cu.to(DEV)
    cfg = tim.CorrectConfig(tis=True, tok_rs=True, seq_rs=tim.SEQ_K3, seq_agg=tim.AGG_MEAN, tau_seq=1e-6)
    pcfg = tim.PPOConfig(eps=0.2)
    adv = torch.randn(n, device=DEV, generator=g)

    def run():
        r = tim.correct(num, den, cu, cfg, mask, return_stats=False)
        p = tim.ppo_loss(num, den, adv, cu, pcfg, coeff=r["coeff"], return_stats=False)
        return _digest(r["tis_w"], r["tok_keep"], r["seq_keep"], r["coeff"], r["seq_score"], r["stats_raw"],
                       p["loss"], p["grad"], p["clipped"], p["seq_loss"], p["hist"], p["stats_raw"])

    ref = run()
    for _ in range(99):
        assert run() == ref


def test_head_backward_repeat_bitwise(tim):
    H, W, ids = _head(1500, 512, 151936, 73)
    g = torch.Generator(device=DEV).manual_seed(73)
    gl, ge = torch.randn(1500, device=DEV, generator=g), torch.randn(1500, device=DEV, generator=g)
    ref = _digest(*tim.head_backward(H, W, ids, gl, ge))
    for _ in range(9):
        assert _digest(*tim.head_backward(H, W, ids, gl, ge)) == ref
