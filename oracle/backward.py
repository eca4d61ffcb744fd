"""fp64 oracle: backward of the head (TEST INFRASTRUCTURE ONLY).

What it computes, the gradient the trainer takes through the
recomputed log-probs -- PAPER.md §3 P:478 (the "score function gradient" of the policy-gradient
loss flows through log pi_theta(a_t | s_t)) -- of the scalar

  L = sum_t g_t logp_t + e_t H_t                (g, e: upstream gradients; e = 0 if absent)

with logp_t, H_t exactly as oracle.logprob (z = h W^T, x = z / T_t, p = softmax(x)):

  1. z = H W^T, x = z / T, lse = m + ln sum exp(x - m), p = exp(x - lse)   (as logprob steps 2-4)
  2. ent_t = lse_t - sum_v p_v x_v                                          (logprob step 6)
  3. dlogp_t / dx_v = 1[v = a_t] - p_v
     dH_t / dx_v    = -p_v (ln p_v + H_t)        (= -p_v (x_v - lse_t + H_t))
  4. G[t, v] = dL/dz[t, v] = (g_t (1[v = a_t] - p_v) + e_t dH_t/dx_v) / T_t
  5. dhidden = G W,  dweight = G^T H                                         (library dgemm)

Rows are independent except through step 5's token sum (dweight); rows are processed in
chunks with dweight accumulated chunk by chunk (fp64, so order is immaterial at test sizes).
Pinned in tests/test_oracle_backward.py by central finite differences of oracle.logprob, by
torch fp64 autograd, and by the invariants sum_v G[t, v] = 0 and G = 0 for g = e = 0.
"""
from __future__ import annotations

import numpy as np


def _as_f64(a) -> np.ndarray:
    if hasattr(a, "detach"):
        a = a.detach().cpu().double().numpy()
    return np.asarray(a, dtype=np.float64)


def _ints(a) -> np.ndarray:
    return np.asarray(a.cpu().numpy() if hasattr(a, "cpu") else a, dtype=np.int64)


def grad_logits(H, W, ids, grad_logp, grad_ent=None, temperature: float = 1.0, temperatures=None):
    """G = dL/dz [N, V] (float64), steps 1-4.

    Pinned by: test_oracle_backward.py::test_finite_differences, ::test_torch_fp64_autograd, ::test_invariants (sum_v G = 0, G = onehot - softmax at g = 1)."""
    H64, W64 = _as_f64(H), _as_f64(W)
    ids = _ints(ids)
    N = H64.shape[0]
    T = _as_f64(temperatures).reshape(N) if temperatures is not None else np.full(N, float(temperature))
    g = _as_f64(grad_logp).reshape(N)
    e = _as_f64(grad_ent).reshape(N) if grad_ent is not None else np.zeros(N)
    z = H64 @ W64.T                                             # step 1
    x = z / T[:, None]
    m = x.max(axis=1)
    lse = m + np.log(np.exp(x - m[:, None]).sum(axis=1))
    p = np.exp(x - lse[:, None])
    ent = lse - (p * x).sum(axis=1)                             # step 2
    onehot = np.zeros_like(p)
    onehot[np.arange(N), ids] = 1.0
    dlogp = onehot - p                                          # step 3
    dent = -p * ((x - lse[:, None]) + ent[:, None])
    return (g[:, None] * dlogp + e[:, None] * dent) / T[:, None]  # step 4


def head_backward(H, W, ids, grad_logp, grad_ent=None, temperature: float = 1.0, temperatures=None,
                  row_chunk: int = 64):
    """(dhidden [N, d], dweight [V, d]) in float64, step 5 over row chunks.

    Pinned by: test_oracle_backward.py::test_finite_differences (central differences of oracle.logprob), ::test_torch_fp64_autograd."""
    H64, W64 = _as_f64(H), _as_f64(W)
    ids = _ints(ids)
    N = H64.shape[0]
    g = _as_f64(grad_logp).reshape(N)
    e = _as_f64(grad_ent).reshape(N) if grad_ent is not None else None
    T = _as_f64(temperatures).reshape(N) if temperatures is not None else None
    dh = np.zeros_like(H64)
    dw = np.zeros_like(W64)
    for a in range(0, N, row_chunk):
        b = min(N, a + row_chunk)
        G = grad_logits(H64[a:b], W64, ids[a:b], g[a:b], None if e is None else e[a:b], temperature,
                        None if T is None else T[a:b])
        dh[a:b] = G @ W64                                       # step 5
        dw += G.T @ H64[a:b]
    return dh, dw
