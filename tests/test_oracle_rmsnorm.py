"""Pins for oracle.rmsnorm (NEXT-4): SPEC.md S:77 worked example, the zero row, exact power-of-two
scale invariance, unit mean square, and the bf16 rounding helper against torch's own
float32 -> bfloat16 conversion (round to nearest even)."""
import math

import numpy as np
import torch

from oracle.rmsnorm import rmsnorm, to_bf16


def test_spec_example_3_4():
    out = rmsnorm(np.array([[3.0, 4.0]]), np.ones(2), 0.0)[0]
    exact = np.array([3.0, 4.0]) / math.sqrt(12.5)       # [0.8485..., 1.1314...]
    assert np.all(np.abs(out - exact) <= np.abs(exact) * 2.0 ** -8)
    assert abs(exact[0] - 0.848528) < 1e-6 and abs(exact[1] - 1.131371) < 1e-6


def test_zero_row_and_scale_invariance():
    rng = np.random.default_rng(0)
    h = rng.normal(0, 1, (16, 256))
    g = rng.normal(1, 0.1, 256)
    assert np.all(rmsnorm(np.zeros((1, 256)), g, 1e-6) == 0)
    a = rmsnorm(to_bf16(h), g, 0.0)
    b = rmsnorm(to_bf16(h) * 8.0, g, 0.0)
    assert np.array_equal(a, b)
    x1 = rmsnorm(to_bf16(h), np.ones(256), 0.0)
    assert np.allclose((x1 * x1).mean(axis=1), 1.0, atol=4e-3)


def test_bf16_rounding_matches_torch_for_fp32_values():
    rng = np.random.default_rng(1)
    x = np.concatenate([rng.normal(0, 3, 20000), rng.normal(0, 1e-3, 1000)]).astype(np.float32)
    ref = torch.from_numpy(x).to(torch.bfloat16).double().numpy()
    assert np.array_equal(to_bf16(x.astype(np.float64)), ref)
