"""fp64 oracle for the rollout-side sampling twin (TEST INFRASTRUCTURE ONLY).

SURVEY.md §8(f) NEXT-1: the rollout engine samples a_t ~ pi(.|s_t) (§2, "the
behavioral distribution realized by the rollout engine when the token is sampled") with the
same head arithmetic the trainer re-evaluates, so that log pi_rollout(a_t) and
log pi_train(a_t) coincide bit for bit (zero mismatch, §3.1).

Sampling rule (reading DESIGN.md U22): Gumbel-max, a_t = argmax_v (x_v + g_v), x = z / T,
g_v = -ln(-ln u_v), with u_v drawn from the counter-based Philox4x32-10 generator (Salmon et
al., "Parallel random numbers: as easy as 1, 2, 3", SC'11) keyed by the 64-bit seed and
counted by (vocab column / 4, 0, row_key lo, row_key hi): output word v % 4 of block v // 4 is
u_v = ((x >> 9) + 0.5) 2^-23 (exact in fp32).  argmax ties resolve to the lowest column.
"""
from __future__ import annotations

import numpy as np

from .logprob import _as_f64

PHILOX_M0 = np.uint64(0xD2511F53)
PHILOX_M1 = np.uint64(0xCD9E8D57)
PHILOX_W0 = np.uint32(0x9E3779B9)
PHILOX_W1 = np.uint32(0xBB67AE85)
MASK32 = np.uint64(0xFFFFFFFF)


def philox4x32_10(c0, c1, c2, c3, k0, k1):
    """Philox4x32 with 10 rounds on uint32 arrays (broadcasting); returns 4 uint32 arrays.

    Pinned by: test_oracle_sample.py::test_philox_known_answer_vectors (Random123 KATs)."""
    c0, c1, c2, c3 = (np.asarray(x, dtype=np.uint32) for x in (c0, c1, c2, c3))
    k0 = np.asarray(k0, dtype=np.uint32)
    k1 = np.asarray(k1, dtype=np.uint32)
    with np.errstate(over="ignore"):
        for r in range(10):
            p0 = PHILOX_M0 * c0.astype(np.uint64)
            p1 = PHILOX_M1 * c2.astype(np.uint64)
            hi0, lo0 = (p0 >> np.uint64(32)).astype(np.uint32), (p0 & MASK32).astype(np.uint32)
            hi1, lo1 = (p1 >> np.uint64(32)).astype(np.uint32), (p1 & MASK32).astype(np.uint32)
            c0, c1, c2, c3 = hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0
            if r < 9:
                k0 = k0 + PHILOX_W0
                k1 = k1 + PHILOX_W1
    return c0, c1, c2, c3


def uniforms(seed: int, row_key: int, vocab: int) -> np.ndarray:
    """u_v for v in [0, vocab) of one row (float64 holding the exact fp32 value).

    Pinned by: test_oracle_sample.py::test_uniforms_open_interval_and_fp32_exact, ::test_sample_scores_equal_mpmath_tempered_logits_plus_gumbel."""
    nblk = (vocab + 3) // 4
    blk = np.arange(nblk, dtype=np.uint32)
    k0, k1 = np.uint32(seed & 0xFFFFFFFF), np.uint32((seed >> 32) & 0xFFFFFFFF)
    lo, hi = np.uint32(row_key & 0xFFFFFFFF), np.uint32((row_key >> 32) & 0xFFFFFFFF)
    x = np.stack(philox4x32_10(blk, np.zeros_like(blk), np.full_like(blk, lo), np.full_like(blk, hi), k0, k1), 1)
    x = x.reshape(-1)[:vocab]
    return ((x >> np.uint32(9)).astype(np.float64) + 0.5) * 2.0 ** -23   # exact in fp32


def sample(H, W, row_keys, seed: int, temperature: float = 1.0, temperatures=None):
    """Gumbel-max samples in fp64: returns (ids, scores [N, V]) with scores = x + g (nats).

    Pinned by: test_oracle_sample.py::test_sample_at_T07_realises_tempered_softmax_and_rejects_wrong_T (chi-square vs the mpmath tempered softmax, with power against T = 1 / 1.4 / 0.35), ::test_sample_scores_equal_mpmath_tempered_logits_plus_gumbel, ::test_sample_T_to_zero_is_argmax, ::test_sample_power_of_two_temperature_and_per_token_T."""
    H64 = _as_f64(H)
    W64 = _as_f64(W)
    N = H64.shape[0]
    V = W64.shape[0]
    T = _as_f64(temperatures).reshape(N) if temperatures is not None else np.full(N, float(temperature))
    ids = np.empty(N, dtype=np.int64)
    scores = np.empty((N, V))
    for t in range(N):
        x = (H64[t] @ W64.T) / T[t]
        ids[t], scores[t] = gumbel_argmax(x, seed, int(row_keys[t]))
    return ids, scores


def gumbel_argmax(x, seed: int, row_key: int):
    """argmax_v (x_v - ln(-ln u_v)) for one row of tempered logits x (nats).

    Pinned by: test_oracle_sample.py::test_gumbel_max_realises_softmax (chi-square), ::test_dominant_logit_always_wins_and_seed_changes_draws."""
    u = uniforms(seed, row_key, x.shape[0])
    s = np.asarray(x, dtype=np.float64) - np.log(-np.log(u))
    return int(np.argmax(s)), s   # first maximum = lowest column
