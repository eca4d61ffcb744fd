"""Pins for oracle.backward (NEXT-3).

* central finite differences of the forward oracle (oracle.logprob) -- a derivative taken
  numerically from the independent forward definition, so a dropped term, a wrong sign, a
  transposed operand or a missing 1/T fails;
* torch float64 autograd of the textbook forward (log_softmax / entropy) at a larger size;
* invariants: sum_v G[t, v] = 0 (both softmax derivatives are orthogonal to the ones vector),
  G = 0 for zero upstream gradients, and G = onehot - softmax for g = 1, e = 0, T = 1.
"""
import numpy as np
import pytest
import torch

from oracle.backward import grad_logits, head_backward
from oracle.logprob import logprob_entropy


def _problem(N, d, V, seed, temps=True):
    rng = np.random.default_rng(seed)
    H = rng.normal(0, 1, (N, d))
    W = rng.normal(0, 0.5, (V, d))
    ids = rng.integers(0, V, N)
    g = rng.normal(0, 1, N)
    e = rng.normal(0, 1, N)
    T = rng.uniform(0.5, 1.5, N) if temps else None
    return H, W, ids, g, e, T


def _loss(H, W, ids, g, e, T):
    lp, ent = logprob_entropy(H, W, ids, 1.0, T)
    return float((g * lp).sum() + (e * ent).sum())


@pytest.mark.parametrize("with_ent,temps", [(False, False), (True, False), (True, True)])
def test_finite_differences(with_ent, temps):
    N, d, V = 3, 6, 11
    H, W, ids, g, e, T = _problem(N, d, V, 7, temps)
    if not with_ent:
        e = np.zeros(N)
    dh, dw = head_backward(H, W, ids, g, e if with_ent else None, 1.0, T)
    eps = 1e-6
    fd_h = np.zeros_like(H)
    for i in range(N):
        for k in range(d):
            Hp, Hm = H.copy(), H.copy()
            Hp[i, k] += eps
            Hm[i, k] -= eps
            fd_h[i, k] = (_loss(Hp, W, ids, g, e, T) - _loss(Hm, W, ids, g, e, T)) / (2 * eps)
    fd_w = np.zeros_like(W)
    for v in range(V):
        for k in range(d):
            Wp, Wm = W.copy(), W.copy()
            Wp[v, k] += eps
            Wm[v, k] -= eps
            fd_w[v, k] = (_loss(H, Wp, ids, g, e, T) - _loss(H, Wm, ids, g, e, T)) / (2 * eps)
    assert np.abs(dh - fd_h).max() <= 1e-7 * max(1.0, np.abs(fd_h).max())
    assert np.abs(dw - fd_w).max() <= 1e-7 * max(1.0, np.abs(fd_w).max())


def test_torch_fp64_autograd():
    N, d, V = 40, 32, 300
    H, W, ids, g, e, T = _problem(N, d, V, 11)
    Ht = torch.tensor(H, requires_grad=True)
    Wt = torch.tensor(W, requires_grad=True)
    x = (Ht @ Wt.T) / torch.tensor(T)[:, None]
    ls = torch.log_softmax(x, dim=1)
    lp = ls[torch.arange(N), torch.tensor(ids)]
    ent = -(ls.exp() * ls).sum(dim=1)
    (torch.tensor(g) * lp + torch.tensor(e) * ent).sum().backward()
    dh, dw = head_backward(H, W, ids, g, e, 1.0, T, row_chunk=7)
    assert np.abs(dh - Ht.grad.numpy()).max() <= 1e-12 * max(1.0, np.abs(dh).max())
    assert np.abs(dw - Wt.grad.numpy()).max() <= 1e-12 * max(1.0, np.abs(dw).max())


def test_invariants():
    N, d, V = 16, 8, 50
    H, W, ids, g, e, T = _problem(N, d, V, 3)
    G = grad_logits(H, W, ids, g, e, 1.0, T)
    assert np.abs(G.sum(axis=1)).max() < 1e-14
    assert np.all(grad_logits(H, W, ids, np.zeros(N), np.zeros(N), 1.0, T) == 0)
    G1 = grad_logits(H, W, ids, np.ones(N), None, 1.0)
    z = H @ W.T
    p = np.exp(z - z.max(axis=1, keepdims=True))
    p /= p.sum(axis=1, keepdims=True)
    onehot = np.eye(V)[ids]
    assert np.abs(G1 - (onehot - p)).max() < 1e-15
    # row chunking changes only fp64 rounding (BLAS blocking, dweight's chunk sum)
    dh1, dw1 = head_backward(H, W, ids, g, e, 1.0, T, row_chunk=1)
    dh2, dw2 = head_backward(H, W, ids, g, e, 1.0, T, row_chunk=64)
    assert np.abs(dh1 - dh2).max() < 1e-13
    assert np.abs(dw1 - dw2).max() < 1e-13
