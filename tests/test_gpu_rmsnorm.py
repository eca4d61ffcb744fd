"""GPU tests of the RMSNorm prologue (NEXT-4): tim_rmsnorm vs the oracle element by element
(bf16 results equal up to rare one-ulp rounding-boundary flips, since the GPU reduces in fp32
and the oracle in fp64), batch invariance, and tim_logprob_rmsnorm vs the oracle log-prob of
the oracle-normalized rows (2e-3)."""
import numpy as np
import pytest
import torch

import synth
from oracle.logprob import logprob_entropy
from oracle.rmsnorm import rmsnorm as o_rmsnorm

pytestmark = pytest.mark.gpu
DEV = "cuda"


def _pre(N, d, seed, scale=3.0):
    g = torch.Generator(device=DEV).manual_seed(seed)
    h = (torch.randn(N, d, generator=g, device=DEV) * scale).to(torch.bfloat16)
    gamma = (1.0 + 0.1 * torch.randn(d, generator=g, device=DEV)).to(torch.bfloat16)
    return h, gamma


@pytest.mark.parametrize("N,d", [(1, 64), (333, 256), (2048, 2048), (700, 4096)])
def test_rmsnorm_matches_oracle(tim, N, d):
    h, gamma = _pre(N, d, N + d)
    out = tim.rmsnorm(h, gamma, 1e-6).cpu().double().numpy()
    ref = o_rmsnorm(h.cpu(), gamma.cpu(), 1e-6)
    diff = out != ref
    assert diff.mean() < 1e-3, diff.mean()
    if diff.any():  # rounding-boundary flips of x1 (one bf16 ulp), at most two ulps after gamma * x1
        ulp = np.ldexp(1.0, np.floor(np.log2(np.abs(ref[diff]))).astype(int) - 7)
        assert np.all(np.abs(out[diff] - ref[diff]) <= 2 * ulp)


def test_rmsnorm_batch_invariance_and_strides(tim):
    N, d = 1000, 1024
    h, gamma = _pre(N, d, 5)
    ref = tim.rmsnorm(h, gamma).view(torch.int16)
    for a, b in ((0, 1), (7, 8), (100, 357), (0, 1000)):
        assert torch.equal(tim.rmsnorm(h[a:b], gamma).view(torch.int16), ref[a:b])
    big = torch.zeros(N, d + 64, dtype=torch.bfloat16, device=DEV)
    big[:, :d] = h
    assert torch.equal(tim.rmsnorm(big[:, :d], gamma).view(torch.int16), ref)


@pytest.mark.parametrize("d", [2048, 4096])
def test_logprob_rmsnorm_parity(tim, d):
    N, V = 512, 151936
    W = synth.head_weight(V, d, 77, device=DEV)
    ids = synth.token_ids(N, V, 77, device=DEV)
    h, gamma = _pre(N, d, 78)
    lp, ent = tim.logprob_rmsnorm(h, gamma, W, ids, eps=1e-6)
    x = o_rmsnorm(h.cpu(), gamma.cpu(), 1e-6)
    olp, oent = logprob_entropy(x, W.cpu(), ids.cpu(), row_chunk=32)
    assert np.abs(lp.cpu().double().numpy() - olp).max() <= 2e-3
    assert np.abs(ent.cpu().double().numpy() - oent).max() <= 2e-3
    # fused call == the two ABI calls in sequence, bitwise
    lp2, ent2 = tim.logprob(tim.rmsnorm(h, gamma, 1e-6), W, ids)
    assert torch.equal(lp.view(torch.int32), lp2.view(torch.int32))
