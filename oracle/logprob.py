"""fp64 oracle: per-token log-prob and entropy (TEST INFRASTRUCTURE ONLY).

What it computes, §2 ("the
probability distribution on the vocabulary for the next token", P:99 the
token distributions pi(a_t | s_t)) and §4.1 ("the trainer re-evaluates
the sampled tokens"); temperature and entropy follow BASELINE.json north_star
(readings U7, U9 in DESIGN.md):

  1. H, W (bf16) -> float64 (exact).
  2. z = H W^T          (library dgemm; bf16*bf16 products are exact in fp64)
  3. x = z / T          (T scalar or per token)
  4. lse = m + ln sum_v exp(x_v - m),   m = max_v x_v
  5. logp_t = x_{t, a_t} - lse_t
  6. H_t = -sum_v p_v ln p_v = lse_t - sum_v p_v x_v,   p = exp(x - lse)

No blocking, fusion or reordering beyond splitting the token rows into
independent chunks (rows never interact).
"""
from __future__ import annotations

import numpy as np


def _as_f64(a) -> np.ndarray:
    if hasattr(a, "detach"):  # torch tensor (bf16 etc.): exact widening to float64
        a = a.detach().cpu().double().numpy()
    return np.asarray(a, dtype=np.float64)


def logprob_entropy(H, W, ids, temperature: float = 1.0, temperatures=None, row_chunk: int = 64):
    """Return (logp[N], entropy[N]) in float64.

    Pinned by: test_oracle_logprob.py (V = 1 exact zero, W = 0 closed form -ln V, V = 2 -softplus, sum exp(logp) = 1, 50-digit mpmath brute force, T = 2 == H / 2 bitwise, per-token T, shift / permutation invariance, entropy bounds).

    H: [N, d], W: [V, d] (bf16 values; torch or numpy), ids: [N] ints in [0, V).
    temperatures: optional per-token T [N] (overrides the scalar).
    """
    H64 = _as_f64(H)
    W64 = _as_f64(W)
    ids = np.asarray(ids.cpu().numpy() if hasattr(ids, "cpu") else ids, dtype=np.int64)
    N = H64.shape[0]
    if temperatures is not None:
        T = _as_f64(temperatures).reshape(N)
    else:
        T = np.full(N, float(temperature))
    logp = np.empty(N)
    ent = np.empty(N)
    WT = W64.T
    for a in range(0, N, row_chunk):
        b = min(N, a + row_chunk)
        z = H64[a:b] @ WT                      # step 2
        x = z / T[a:b, None]                   # step 3
        m = x.max(axis=1)                      # step 4
        lse = m + np.log(np.exp(x - m[:, None]).sum(axis=1))
        rows = np.arange(b - a)
        logp[a:b] = x[rows, ids[a:b]] - lse    # step 5
        p = np.exp(x - lse[:, None])           # step 6
        ent[a:b] = lse - (p * x).sum(axis=1)
    return logp, ent


def logits(H, W, temperature: float = 1.0):
    """fp64 scaled logits x = H W^T / T (used by GEMM bring-up tests).

    Pinned by: test_oracle_logprob.py::test_logits_equal_mpmath_dot_products_at_temperature (40-digit dot products at T = 0.7 / 1 / 2.5)."""
    return (_as_f64(H) @ _as_f64(W).T) / float(temperature)
