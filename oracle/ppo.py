"""fp64 oracle: fused PPO / GRPO surrogate and the paper's loss diagnostics (TEST INFRASTRUCTURE ONLY).

SURVEY.md §8(f) NEXT-2.  From PAPER.md:
  L_ppo(r, A) = -min(r A, clip(r, 1 - eps, 1 + eps) A)                (eq:ppo_loss)
  r_ppo = pi_theta / pi_old, pi_old = pi_train_old (recompute) or pi_rollout_old (bypass)
                                                                       (eq:ppo_ratio)
  token-level terms summed over the response, averaged over the batch
  the patch objectives weight each token term by the correction coefficient
  (resp * tok_keep * seq_keep * min(r_corr, tau_tok), App. A.4) = `coeff`
  K1(r) = -log r, K3(r) = (r - 1) - log r on the PPO ratio             (§4.1)
  zero-centred contribution C(r) = -(r - 1) A, split by sign(A)

Decisions (clip flag, histogram bin, sums) follow the decision-path contract of
oracle/correct.py (one RN binary64 op per step, exact integer sums):
  delta = (double)lp_cur - (double)lp_old; r = exp_c(delta)
  clipped <=> (A > 0 and r > clip_hi) or (A < 0 and r < clip_lo)
  s = clipped ? (A > 0 ? clip_hi : clip_lo) * A : r * A;  loss = -(w s)   (w = coeff or 1)
  grad = d loss / d lp_cur = clipped ? 0 : loss                         (d r / d lp_cur = r)
  C = (-(r - 1)) * A;  bin = floor((C - hist_lo) * hist_inv_width): < 0 -> underflow slot 0,
        >= bins -> overflow slot bins + 1, else bin + 1;  histogram[A > 0 ? 0 : 1] (A == 0 counted apart)
  X = rint(loss 2^52) (saturated at |loss| > 2^10), per-sequence and batch sums exact;
  batch_loss = (sum over sequences of their loss sums) / (number of sequences with a contributing token)
Contributing tokens: coeff != 0 when coeff is given, else resp_mask (all tokens when absent).
Data errors (U13, U13b): a non-finite lp / advantage / coeff, or a token outside [cu[0], cu[S]).
"""
from __future__ import annotations

import dataclasses

import numpy as np

from .correct import DataError, _isum, delta, exp_contract, fixed_point, k3_contract, outside_sequences


@dataclasses.dataclass
class PPOCfg:
    clip_lo: float = 0.8
    clip_hi: float = 1.2
    hist_lo: float = -1.0
    hist_inv_width: float = 32.0   # bins / (hist_hi - hist_lo)
    hist_bins: int = 64


def local(lp_cur, lp_old, adv, cu_seqlens, cfg: PPOCfg, coeff=None, resp_mask=None, tok_begin: int = 0):
    """Pass 1 on one shard: per-token loss / grad / clip flag, C(r) histogram, exact partials.

    Pinned by: test_oracle_ppo.py::test_on_policy_closed_form, ::test_clip_branches_closed_form,
    ::test_loss_is_minus_min_of_unclipped_and_clipped (mpmath), ::test_gradient_is_score_function_derivative
    (finite differences), ::test_histogram_edges_are_exact, ::test_non_finite_advantage_is_a_data_error.
    """
    cu = np.asarray(cu_seqlens, dtype=np.int64)
    S = cu.size - 1
    d = delta(lp_cur, lp_old)
    n = d.size
    A = np.asarray(adv, dtype=np.float32).astype(np.float64)
    # data errors (reading U13): non-finite log-prob, advantage or weight; a token outside the
    # global sequences (U13b).  The first bad global index is reported.
    bad = ~np.isfinite(d) | ~np.isfinite(A) | outside_sequences(cu, tok_begin, n)
    if coeff is not None:
        bad |= ~np.isfinite(np.asarray(coeff, dtype=np.float32))
    if bad.any():
        raise DataError(tok_begin + int(np.argmax(bad)))
    r = exp_contract(d)
    if coeff is not None:
        c32 = np.asarray(coeff, dtype=np.float32)
        contrib = c32 != 0
        w = c32.astype(np.float64)
    else:
        contrib = np.ones(n, bool) if resp_mask is None else (np.asarray(resp_mask) != 0)
        w = contrib.astype(np.float64)
    clipped = ((A > 0) & (r > cfg.clip_hi)) | ((A < 0) & (r < cfg.clip_lo))
    rc = np.where(A > 0, cfg.clip_hi, cfg.clip_lo)
    s = np.where(clipped, rc * A, r * A)
    loss = -(w * s)
    grad = np.where(clipped, 0.0, loss)
    C = (-(r - 1.0)) * A
    raw = np.floor((C - cfg.hist_lo) * cfg.hist_inv_width)
    slot = np.where(raw < 0, 0, np.where(raw >= cfg.hist_bins, cfg.hist_bins + 1, raw + 1)).astype(np.int64)
    hist = np.zeros((2, cfg.hist_bins + 2), dtype=np.int64)
    np.add.at(hist[0], slot[contrib & (A > 0)], 1)
    np.add.at(hist[1], slot[contrib & (A < 0)], 1)
    X, sat = fixed_point(np.where(contrib, loss, 0.0))
    X1, _ = fixed_point(-d)
    X3, _ = fixed_point(k3_contract(d))
    glob = {
        "n_tok": n, "n_contrib": int(contrib.sum()), "n_clipped": int((contrib & clipped).sum()),
        "n_zero_adv": int((contrib & (A == 0)).sum()), "n_saturated": int((contrib & sat).sum()),
        "sum_loss": _isum(X[contrib]), "sum_k1": _isum(X1[contrib]), "sum_k3": _isum(X3[contrib]),
        "hist": hist,
    }
    seq = np.zeros((S, 3), dtype=object)
    seq[:] = 0
    g0, g1 = tok_begin, tok_begin + n
    for q in range(S):
        a, b = max(int(cu[q]), g0), min(int(cu[q + 1]), g1)
        if a >= b:
            continue
        sl = slice(a - g0, b - g0)
        c = contrib[sl]
        seq[q, 0] = _isum(X[sl][c])
        seq[q, 1] = int(c.sum())
        seq[q, 2] = int((sat[sl] & c).sum())
    tokens = {"loss": loss.astype(np.float32), "grad": grad.astype(np.float32), "clipped": clipped.astype(np.uint8),
              "C": C, "r": r}
    return tokens, glob, seq


def combine(parts):
    """Exact combination of the ranks' partials (integer sums).

    Pinned by: test_oracle_ppo.py::test_sharding_is_exact.
    """
    globs = [g for g, _ in parts]
    out = {k: sum(g[k] for g in globs) for k in globs[0] if k != "hist"}
    out["hist"] = sum(g["hist"] for g in globs)
    seq = parts[0][1].copy()
    for _, s in parts[1:]:
        seq = seq + s
    return out, seq


def finish(glob, seq):
    """Sequence losses and batch statistics from the combined exact partials.

    Pinned by: test_oracle_ppo.py::test_sequence_and_batch_averages (fsum).
    """
    S = seq.shape[0]
    seq_loss = np.array([float(int(seq[q, 0])) * 2.0 ** -52 for q in range(S)])
    n_seq_contrib = int(sum(1 for q in range(S) if int(seq[q, 1]) > 0))
    st = {k: v for k, v in glob.items() if k != "hist"}
    st["n_seq"] = S
    st["n_seq_contrib"] = n_seq_contrib
    st["batch_loss"] = (float(glob["sum_loss"]) * 2.0 ** -52) / n_seq_contrib if n_seq_contrib else 0.0
    nc = glob["n_contrib"]
    st["clip_frac"] = glob["n_clipped"] / nc if nc else 0.0
    st["mean_k1"] = (float(glob["sum_k1"]) * 2.0 ** -52) / nc if nc else 0.0
    st["mean_k3"] = (float(glob["sum_k3"]) * 2.0 ** -52) / nc if nc else 0.0
    return seq_loss, st


def ppo(lp_cur, lp_old, adv, cu_seqlens, cfg: PPOCfg, coeff=None, resp_mask=None):
    """Single-shard end-to-end oracle.

    Pinned by: every test in test_oracle_ppo.py.
    """
    tokens, glob, seq = local(lp_cur, lp_old, adv, cu_seqlens, cfg, coeff, resp_mask, 0)
    seq_loss, st = finish(glob, seq)
    return {**tokens, "seq_loss": seq_loss, "stats": st, "hist": glob["hist"], "seq_partials": seq}


def clip_bounds(eps: float) -> tuple[float, float]:
    """Paper's symmetric clip range (eq:ppo_loss): (1 - eps, 1 + eps) in binary64.

    Pinned by: test_oracle_ppo.py::test_clip_branches_closed_form.
    """
    return 1.0 - eps, 1.0 + eps

