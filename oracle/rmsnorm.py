"""fp64 oracle of the RMSNorm prologue (NEXT-4; TEST INFRASTRUCTURE ONLY).

PAPER.md §3.1: vExact implements a batch-invariant RMSNorm -- the final norm in front
of the lm_head.  The paper's models use the Hugging Face Qwen3 definition
    x1 = to_bf16( h / sqrt(mean_k h_k^2 + eps) ),   out = to_bf16( gamma * x1 )
(SPEC.md S:72-80 rmsnorm_bi: y_i = gamma_i x_i / sqrt(mean(x^2) + eps)).  Here every product,
mean and square root is fp64; only the two roundings to bf16 the model itself performs are
kept (round to nearest even, 8 significant bits).
"""
from __future__ import annotations

import numpy as np

from .logprob import _as_f64


def to_bf16(x) -> np.ndarray:
    """Round float64 values to the nearest bf16 (ties to even); returned as float64.

    Pinned by: test_oracle_rmsnorm.py::test_bf16_rounding_matches_torch_for_fp32_values.
    """
    x = np.asarray(x, dtype=np.float64)
    m, e = np.frexp(x)                      # x = m 2^e, 0.5 <= |m| < 1
    r = np.ldexp(np.rint(np.ldexp(m, 8)), e - 8)
    return np.where(x == 0, x, r)


def rmsnorm(h, gamma, eps: float):
    """HF RMSNorm in fp64 with the model's two bf16 roundings.

    Pinned by: test_oracle_rmsnorm.py::test_spec_example_3_4 (SPEC.md S:77 worked example),
    ::test_zero_row_and_scale_invariance.
    """
    h64 = _as_f64(h)
    g64 = _as_f64(gamma)
    var = (h64 * h64).mean(axis=1)
    inv = 1.0 / np.sqrt(var + eps)
    x1 = to_bf16(h64 * inv[:, None])
    return to_bf16(g64[None, :] * x1)
