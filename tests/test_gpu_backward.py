"""GPU tests of the head backward (NEXT-3): tim_head_backward vs oracle.backward.

Tolerance (U24): the path rounds G = dL/dz to bf16 (relative error <= 2^-9 per
element, independent across elements) and the GEMMs accumulate in fp32, so the relative
Frobenius error of dhidden / dweight is ~2^-9 / sqrt(3) ~ 1.1e-3; the bound is 4e-3.
Exact properties: zero upstream gradients give exact zeros; repeated calls are bitwise equal;
token blocks accumulate dweight; a bad id reports its global index.
"""
import numpy as np
import pytest
import torch

import synth
from oracle.backward import grad_logits, head_backward as o_backward

pytestmark = pytest.mark.gpu
DEV = "cuda"
TOL = 4e-3


def _rel(a, ref):
    return float(np.linalg.norm(a - ref) / max(np.linalg.norm(ref), 1e-30))


def _problem(N, d, V, seed, mode="flat"):
    W = synth.head_weight(V, d, seed, device=DEV)
    ids = synth.token_ids(N, V, seed, device=DEV)
    H = synth.hidden_states(N, d, seed, device=DEV, weight=W, ids=ids, mode=mode)
    g = torch.Generator(device=DEV).manual_seed(seed)
    gl = torch.randn(N, generator=g, device=DEV)
    ge = torch.randn(N, generator=g, device=DEV)
    T = 0.6 + 0.8 * torch.rand(N, generator=g, device=DEV)
    return H, W, ids, gl, ge, T


@pytest.mark.parametrize("N,d,V,mode,ent,temps", [
    (300, 256, 5000, "flat", True, True),      # ragged M tile and vocab tail tile
    (1, 128, 257, "peaked", False, False),     # single token, 2 vocab tiles (tail of 1 column)
    (777, 512, 33000, "peaked", True, False),
])
def test_backward_matches_oracle(tim, N, d, V, mode, ent, temps):
    H, W, ids, gl, ge, T = _problem(N, d, V, N + V, mode)
    dh, dw = tim.head_backward(H, W, ids, gl, ge if ent else None, 1.0, T if temps else None)
    rh, rw = o_backward(H.cpu(), W.cpu(), ids.cpu(), gl.cpu(), ge.cpu() if ent else None, 1.0,
                        T.cpu() if temps else None)
    assert _rel(dh.cpu().double().numpy(), rh) <= TOL
    assert _rel(dw.cpu().double().numpy(), rw) <= TOL
    # row-wise too: no token's gradient is off
    eh = np.linalg.norm(dh.cpu().double().numpy() - rh, axis=1) / np.maximum(np.linalg.norm(rh, axis=1), 1e-30)
    assert eh.max() <= 4 * TOL


@pytest.mark.slow
@pytest.mark.parametrize("d", [2048, 4096])
def test_backward_full_vocab(tim, d):
    """BASELINE configs' head (V = 151936) at 512 tokens; dweight compared on sampled rows
    (the sampled ids plus random rows), dhidden in full."""
    N, V = 512, 151936
    H, W, ids, gl, ge, T = _problem(N, d, V, 40 + d, "peaked")
    dh, dw = tim.head_backward(H, W, ids, gl, ge)
    G = grad_logits(H.cpu(), W.cpu(), ids.cpu(), gl.cpu(), ge.cpu())
    rh = G @ W.cpu().double().numpy()
    assert _rel(dh.cpu().double().numpy(), rh) <= TOL
    rows = np.unique(np.concatenate([ids.cpu().numpy()[:64], np.random.default_rng(0).integers(0, V, 64),
                                     [0, V - 1]]))
    rw = G[:, rows].T @ H.cpu().double().numpy()
    assert _rel(dw[torch.as_tensor(rows, device=DEV)].cpu().double().numpy(), rw) <= TOL


def test_zero_gradient_and_determinism(tim):
    N, d, V = 600, 256, 3000
    H, W, ids, gl, ge, T = _problem(N, d, V, 9)
    z = torch.zeros(N, device=DEV)
    dh, dw = tim.head_backward(H, W, ids, z, z)
    assert torch.count_nonzero(dh) == 0 and torch.count_nonzero(dw) == 0
    a = tim.head_backward(H, W, ids, gl, ge, 1.0, T)
    b = tim.head_backward(H, W, ids, gl, ge, 1.0, T)
    assert torch.equal(a[0].view(torch.int32), b[0].view(torch.int32))
    assert torch.equal(a[1].view(torch.int32), b[1].view(torch.int32))
    # outputs may be skipped independently
    dh2, none = tim.head_backward(H, W, ids, gl, ge, 1.0, T, need_dweight=False)
    assert none is None and _rel(dh2.cpu().double().numpy(), a[0].cpu().double().numpy()) < 1e-6


def test_token_blocks_and_status(tim):
    """N above one token block (14080 rows at V = 151936): dweight is the sum of the blocks'
    contributions and dhidden rows match per-block calls (fp32 GEMM rounding only); a bad id
    in the second block is reported with its global index."""
    N, d, V = 14500, 128, 151936
    H, W, ids, gl, ge, T = _problem(N, d, V, 21)
    L = tim.lib()
    assert L.tim_head_backward_workspace_bytes(N, d, V) < L.tim_head_backward_workspace_bytes(2 * N, d, V) + 1
    dh, dw = tim.head_backward(H, W, ids, gl, ge)
    cut = 14080
    dh1, dw1 = tim.head_backward(H[:cut], W, ids[:cut], gl[:cut], ge[:cut])
    dh2, dw2 = tim.head_backward(H[cut:], W, ids[cut:], gl[cut:], ge[cut:])
    assert _rel(dw.cpu().double().numpy(), (dw1 + dw2).cpu().double().numpy()) < 1e-5
    assert _rel(dh.cpu().double().numpy(), torch.cat([dh1, dh2]).cpu().double().numpy()) < 1e-5
    bad = ids.clone()
    bad[14300] = V
    bad[14350] = -1
    st = tim.new_status(DEV)
    tim.head_backward(H, W, bad, gl, ge, status=st)
    code, idx = tim.read_status(st)
    assert code == 9 and idx == 14300, (code, idx)


def _lse2_oracle(H, W, T):
    """log2-sum-exp of y = z / T_t (in log2 units), fp64 from oracle.logprob.logits."""
    from oracle.logprob import logits
    x = logits(H.cpu(), W.cpu()) / T.cpu().double().numpy()[:, None]
    m = x.max(axis=1)
    return (m + np.log(np.exp(x - m[:, None]).sum(axis=1))) / np.log(2.0)


@pytest.mark.parametrize("N,d,V", [(300, 256, 5000), (14500, 128, 151936)])
def test_saved_forward_backward(tim, N, d, V):
    """tim_logprob_saved: logp / entropy bitwise those of tim_logprob, lse2 within the logp
    tolerance of the fp64 definition; tim_head_backward_saved: bitwise tim_head_backward (the
    forward is batch-invariant, so the saved per-token values are the ones it would recompute),
    also across the 14080-row token blocks."""
    H, W, ids, gl, ge, T = _problem(N, d, V, 5 + N)
    lp, ent, lse2 = tim.logprob_saved(H, W, ids, 1.0, T)
    lp0, ent0 = tim.logprob(H, W, ids, 1.0, T)
    assert torch.equal(lp.view(torch.int32), lp0.view(torch.int32))
    assert torch.equal(ent.view(torch.int32), ent0.view(torch.int32))
    rows = slice(0, 300)
    ref = _lse2_oracle(H[rows], W, T[rows])
    assert np.abs(lse2[rows].cpu().double().numpy() - ref).max() <= 2e-3
    a = tim.head_backward(H, W, ids, gl, ge, 1.0, T)
    b = tim.head_backward(H, W, ids, gl, ge, 1.0, T, saved=(ent, lse2))
    for x, y in zip(a, b):
        assert torch.equal(x.view(torch.int32), y.view(torch.int32))
