"""fp64 oracle: mismatch statistics and TIS / RS corrections (TEST INFRASTRUCTURE ONLY).

Real-number semantics from PAPER.md:
  delta_t = log pi_train_old - log pi_rollout_old            (§2)
  r_corr  = pi_train_old / pi_rollout_old = e^delta          (§4.2)
  TIS weight  w_t = min(r_corr,t, tau_tok)                   (L_TIS)
  K1(r) = -log r,  K3(r) = (r - 1) - log r                   (§4.1)
  S_seq(q_1:T) = sum_t K(q_t), K in {K1, K3}                 (§4.2)
  sequence keep  1[S_seq <= tau_seq]                          (L_RS; App. A.4)
  tau_tok = 2, tau_seq = 0.001 in the paper's runs

Because integer outputs (masks, counts) must be bit-exact between this oracle
and the GPU, they are defined by the decision-path arithmetic contract of
SURVEY.md §8(c) C.3, which is written out here step by step.  Every floating
operation below is ONE IEEE binary64 round-to-nearest numpy ufunc (numpy never
fuses separate ufunc calls), except the K3 series' Horner steps, which are
single-rounding fused multiply-adds written out by `fma` (exact emulation).

  C.3.1  delta = (double)lp_num - (double)lp_den
  C.3.2  non-finite delta -> data error carrying the first bad (global) index
  C.3.3  threshold tests in the log domain on delta:
           truncated  <=> delta > ln tau_tok
           token keep <=> ln lo <= delta <= ln hi               (reading U4)
  C.3.5  K1 = -delta
  C.3.6  K3 = k3_c(delta): |delta| <= 1: delta^2 * P(delta), P the Horner
         series of (e^x - 1 - x)/x^2 with coefficients RN(1/n!), n = 2..9 for
         |delta| <= 2^-6, 2..15 for |delta| <= 2^-2, 2..23 for |delta| <= 1,
         each Horner step ONE fused multiply-add RN(P * delta + 1/n!) (`fma`,
         emulated exactly here, DFMA on the GPU; contract revision 4);
         otherwise (exp_c(delta) - 1) - delta.  exp_c = (1 + delta) + K3 for
         |delta| <= 2^-2 (same series), else Cody-Waite reduction
         k = rint(delta * log2 e), r = (delta - k*ln2_hi) - k*ln2_lo, degree-13
         Taylor Horner on r, then ldexp(., k); exp_c = +inf for delta > 709,
         0 for delta < -700.
  C.3.7  w = (float)(truncated ? tau_tok : min(exp_c(delta), tau_tok))
  C.3.8  fixed point X = rint(K * 2^52) (ties to even); |K| > 2^10 (or
         non-finite) saturates X = sign(K) * 2^62 and counts as saturated.
         Sums are exact Python integers.
  C.3.9  sequence keep: no saturated token and
           SUM : X_s <= floor(tau_seq * 2^52)
           MEAN: X_s <= floor(tau_seq * 2^52 * T_s)
         (T_s = contributing response tokens; T_s == 0 -> keep).  The floor is
         taken exactly with fractions.Fraction.
  C.3.10 statistics = exact integer totals; means = float(total) * 2^-52 / count.
"""
from __future__ import annotations

import dataclasses
import math
from fractions import Fraction

import numpy as np

# ---- constants of the contract (each the correctly rounded binary64 value) ----
LOG2E = float.fromhex("0x1.71547652b82fep+0")       # RN(1/ln 2)
LN2_HI = float.fromhex("0x1.62e42fee00000p-1")      # ln 2 split (fdlibm), hi has 32 zero low bits
LN2_LO = float.fromhex("0x1.a39ef35793c76p-33")
INV_FACT = [float(Fraction(1, math.factorial(n))) for n in range(0, 24)]  # RN(1/n!)
FX_SCALE = 2.0 ** 52
SAT_K = 2.0 ** 10
SAT_X = 2 ** 62

SEQ_NONE, SEQ_K1, SEQ_K3 = 0, 1, 3
AGG_SUM, AGG_MEAN = 0, 1


class DataError(ValueError):
    """Non-finite log-prob (TIM_ERR_DATA analogue); .index is the first bad global index."""

    def __init__(self, index: int):
        super().__init__(f"non-finite delta at token {index}")
        self.index = index


@dataclasses.dataclass
class Cfg:
    tis: bool = False
    tis_cap: float = 2.0
    log_tis_cap: float = math.log(2.0)
    tok_rs: bool = False
    log_tok_lo: float = -math.log(2.0)
    log_tok_hi: float = math.log(2.0)
    seq_rs: int = SEQ_NONE
    seq_agg: int = AGG_SUM
    tau_seq: float = 1e-3


def delta(lp_num, lp_den) -> np.ndarray:
    """C.3.1: one rounded subtraction of the widened fp32 inputs.

    Pinned by: test_oracle_correct.py::test_table1_delta_matches_printed (Table 1), ::test_zero_mismatch_collapses_everything.
    """
    return np.asarray(lp_num, dtype=np.float32).astype(np.float64) - \
        np.asarray(lp_den, dtype=np.float32).astype(np.float64)


SMALL = 2.0 ** -6  # |delta| <= SMALL: short Horner polynomial n = 2..9 (truncation < 1e-19 relative)
MID = 2.0 ** -2    # |delta| <= MID:   n = 2..15 (first dropped term < 4e-22 relative)


def _two_sum(a, b):
    """Knuth's TwoSum: s = RN(a + b) and the exact error e, a + b = s + e."""
    s = a + b
    bb = s - a
    return s, (a - (s - bb)) + (b - bb)


def _split(a):
    """Veltkamp split: a = hi + lo exactly, each half with at most 26 significant bits."""
    c = 134217729.0 * a  # 2^27 + 1
    hi = c - (c - a)
    return hi, a - hi


def _two_prod(a, b):
    """Dekker's product: p = RN(a b) and the exact error e, a b = p + e (no over- / underflow)."""
    p = a * b
    ah, al = _split(a)
    bh, bl = _split(b)
    return p, ((ah * bh - p) + ah * bl + al * bh) + al * bl


def fma(a, b, c) -> np.ndarray:
    """RN(a * b + c) with ONE rounding (IEEE 754 fusedMultiplyAdd; the GPU's DFMA), which numpy
    does not expose.  Boldo & Melquiond's emulation through rounding to odd: uh + ul = a b and
    th + tl = c + uh exactly, v = RO(tl + ul), result RN(th + v).  Valid for finite operands whose
    product neither overflows nor underflows (here |a|, |c| <= 1 and |b| >= 2^-150 or b == 0: the
    contract's Horner steps).  Round to odd of x + y: RN, and when inexact with an even last bit,
    the neighbour on the side of the exact sum (which has an odd last bit).

    Pinned by: test_oracle_correct.py::test_fma_is_the_correctly_rounded_exact_value (exact rationals,
    incl. constructed ties and near-ties).
    """
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    c = np.asarray(c, dtype=np.float64)
    uh, ul = _two_prod(a, b)
    th, tl = _two_sum(c, uh)
    v, e = _two_sum(tl, ul)
    even = (v.view(np.int64) & 1) == 0
    v = np.where((e != 0) & even, np.nextafter(v, np.where(e > 0, np.inf, -np.inf)), v)
    return th + v


def _k3_series(d, top: int) -> np.ndarray:
    """d^2 Q(d), Q = Horner of (e^x - 1 - x)/x^2 with coefficients RN(1/n!), n = top..2; every
    Horner step is one fused multiply-add Q <- RN(Q d + 1/n!) (contract revision 4)."""
    Q = np.full_like(d, INV_FACT[top])
    for n in range(top - 1, 1, -1):
        Q = fma(Q, d, INV_FACT[n])
    return (d * d) * Q


def exp_contract(d) -> np.ndarray:
    """C.3.6 exp_c.  |d| <= 2^-2: (1 + d) + K3_series(d) with the K3 branch's own series (n = 2..9
    for |d| <= 2^-6, n = 2..15 above), i.e. e^d = 1 + d + (e^d - 1 - d).  Otherwise Cody-Waite
    reduction + degree-13 Taylor Horner + ldexp; +inf above 709, 0 below -700.

    Pinned by: test_oracle_correct.py::test_exp_contract_within_2_ulp (60-digit mpmath).
    """
    d = np.asarray(d, dtype=np.float64)
    dd = np.where(np.isfinite(d), np.clip(d, -700.0, 709.0), 0.0)
    k = np.rint(dd * LOG2E)
    r = (dd - k * LN2_HI) - k * LN2_LO
    p = np.full_like(r, INV_FACT[13])
    for n in range(12, -1, -1):
        p = p * r + INV_FACT[n]
    out = np.ldexp(p, k.astype(np.int64))
    small = np.abs(dd) <= SMALL
    mid = ~small & (np.abs(dd) <= MID)
    ds = np.where(small, dd, 0.0)
    dm = np.where(mid, dd, 0.0)
    out = np.where(mid, (1.0 + dm) + _k3_series(dm, 15), out)
    out = np.where(small, (1.0 + ds) + _k3_series(ds, 9), out)
    out = np.where(d > 709.0, np.inf, out)
    out = np.where(d < -700.0, 0.0, out)
    return out


def k3_contract(d) -> np.ndarray:
    """C.3.6 K3 = e^d - 1 - d = d^2 P(d): P = Horner series of RN(1/n!) with n = 2..9 for
    |d| <= 2^-6, n = 2..15 for |d| <= 2^-2 and n = 2..23 for |d| <= 1; (exp_c(d) - 1) - d
    otherwise.

    Pinned by: test_oracle_correct.py::test_k3_contract_within_4_ulp_of_60_digit_reference, ::test_k_closed_forms.
    """
    d = np.asarray(d, dtype=np.float64)
    ad = np.abs(d)
    tiny = ad <= SMALL
    mid = ~tiny & (ad <= MID)
    med = ~tiny & ~mid & (ad <= 1.0)
    out = (exp_contract(d) - 1.0) - d
    out = np.where(med, _k3_series(np.where(med, d, 0.0), 23), out)
    out = np.where(mid, _k3_series(np.where(mid, d, 0.0), 15), out)
    out = np.where(tiny, _k3_series(np.where(tiny, d, 0.0), 9), out)
    return out


def fixed_point(K) -> tuple[np.ndarray, np.ndarray]:
    """C.3.8: X = rint(K * 2^52) as int64; |K| > 2^10 or non-finite -> +-2^62, saturated.

    Pinned by: test_oracle_correct.py::test_fixed_point_is_round_half_even_of_exact_product (exact rationals), ::test_saturated_sequence_rejected_and_counted.
    """
    K = np.asarray(K, dtype=np.float64)
    sat = ~(np.abs(K) <= SAT_K)
    Ks = np.where(sat, 0.0, K)
    X = np.rint(Ks * FX_SCALE).astype(np.int64)
    sgn = np.where(np.signbit(K), -1, 1).astype(np.int64)
    X = np.where(sat, sgn * np.int64(SAT_X), X)
    return X, sat


def _isum(x: np.ndarray) -> int:
    """Exact integer sum (Python ints)."""
    return int(sum(int(v) for v in x.tolist()))


def seq_threshold(tau: float, T: int, agg: int) -> int:
    """C.3.9 exact floor(tau * 2^52 * (T if MEAN else 1)).

    Pinned by: test_oracle_correct.py::test_mean_threshold_is_exact_rational_floor (fractions.Fraction), ::test_less_equal_edge_sum_and_mean.
    """
    f = Fraction(tau) * (2 ** 52) * (T if agg == AGG_MEAN else 1)
    return math.floor(f)


def outside_sequences(cu, tok_begin: int, n: int) -> np.ndarray:
    """Reading U13b: a local token whose global index lies outside [cu[0], cu[S]) belongs to no
    sequence -- a data error, like a non-finite log-prob.

    Pinned by: test_oracle_correct.py::test_tokens_outside_the_sequences_are_a_data_error.
    """
    g = np.arange(tok_begin, tok_begin + n, dtype=np.int64)
    return (g < int(cu[0])) | (g >= int(cu[-1]))


def local_partials(lp_num, lp_den, cu_seqlens, cfg: Cfg, resp_mask=None, tok_begin: int = 0):
    """Pass 1 on one shard [tok_begin, tok_begin + n): per-token outputs and the exact
    per-sequence / global integer partials that one rank contributes.

    Pinned by: test_oracle_correct.py::test_sharding_is_exact_and_order_free, ::test_table1_tis_and_k_values, ::test_token_rs_bounds_inclusive, ::test_non_finite_is_a_data_error_with_first_index, ::test_prompt_only_sequence_is_kept_and_excluded.
    """
    cu = np.asarray(cu_seqlens, dtype=np.int64)
    S = cu.size - 1
    d = delta(lp_num, lp_den)
    n = d.size
    bad = ~np.isfinite(d) | outside_sequences(cu, tok_begin, n)
    if bad.any():
        raise DataError(tok_begin + int(np.argmax(bad)))
    resp = np.ones(n, bool) if resp_mask is None else (np.asarray(resp_mask) != 0)
    trunc = (d > cfg.log_tis_cap) if cfg.tis else np.zeros(n, bool)
    if cfg.tis:
        w64 = np.where(trunc, cfg.tis_cap, np.minimum(exp_contract(d), cfg.tis_cap))
        w = w64.astype(np.float32)
    else:
        w = np.ones(n, np.float32)
    keep = ((cfg.log_tok_lo <= d) & (d <= cfg.log_tok_hi)) if cfg.tok_rs else np.ones(n, bool)
    coeff = np.where(resp & keep, w, np.float32(0.0)).astype(np.float32)

    k1 = -d
    k3 = k3_contract(d)
    X_abs, _ = fixed_point(np.abs(d))
    X_k1, _ = fixed_point(k1)
    X_k3, _ = fixed_point(k3)
    glob = {
        "n_tok": n,
        "n_resp_tok": int(resp.sum()),
        "n_truncated": int((resp & trunc).sum()),
        "n_tok_rejected": int((resp & ~keep).sum()),
        "n_saturated": 0,
        "max_abs_delta": float(np.abs(d[resp]).max()) if resp.any() else 0.0,
        "sum_abs_delta": _isum(X_abs[resp]),
        "sum_k1": _isum(X_k1[resp]),
        "sum_k3": _isum(X_k3[resp]),
    }
    seq = np.zeros((S, 3), dtype=object)  # (X_s, T_s, nsat_s) Python ints
    seq[:] = 0
    if cfg.seq_rs != SEQ_NONE:
        Xq, satq = fixed_point(k1 if cfg.seq_rs == SEQ_K1 else k3)
        contrib = resp & keep
        glob["n_saturated"] = int((contrib & satq).sum())
        g0, g1 = tok_begin, tok_begin + n
        for s in range(S):
            a, b = max(int(cu[s]), g0), min(int(cu[s + 1]), g1)
            if a >= b:
                continue
            sl = slice(a - g0, b - g0)
            c = contrib[sl]
            seq[s, 0] = _isum(Xq[sl][c])
            seq[s, 1] = int(c.sum())
            seq[s, 2] = int((satq[sl] & c).sum())
    tokens = {"delta": d, "tis_w": w, "tok_keep": keep.astype(np.uint8), "coeff_prov": coeff}
    return tokens, glob, seq


def combine(parts):
    """Exact combination of the (glob, seq) partials of all ranks (order-free: integers / max).

    Pinned by: test_oracle_correct.py::test_sharding_is_exact_and_order_free.
    """
    globs = [g for g, _ in parts]
    out = {k: sum(g[k] for g in globs) for k in globs[0] if k != "max_abs_delta"}
    out["max_abs_delta"] = max(g["max_abs_delta"] for g in globs)
    seq = parts[0][1].copy()
    for _, s in parts[1:]:
        seq = seq + s
    return out, seq


def decide(seq, cfg: Cfg):
    """C.3.9: per-sequence keep flags and scores from the combined exact partials.

    Pinned by: test_oracle_correct.py::test_table1_sentence_rejected, ::test_table1_without_flip_token_kept, ::test_less_equal_edge_sum_and_mean, ::test_contract_decisions_match_exact_real_decisions (mpmath), ::test_huge_thresholds_never_reject_or_truncate.
    """
    S = seq.shape[0]
    keep = np.ones(S, np.uint8)
    score = np.zeros(S, np.float64)
    if cfg.seq_rs == SEQ_NONE:
        return keep, score
    for s in range(S):
        X, T, nsat = int(seq[s, 0]), int(seq[s, 1]), int(seq[s, 2])
        sc = float(X) * (2.0 ** -52)
        if cfg.seq_agg == AGG_MEAN:
            sc = sc / T if T > 0 else 0.0
        score[s] = sc
        if T == 0:
            keep[s] = 1
        elif nsat > 0:
            keep[s] = 0
        else:
            keep[s] = 1 if X <= seq_threshold(cfg.tau_seq, T, cfg.seq_agg) else 0
    return keep, score


def finalize_stats(glob, seq_keep, n_seq: int):
    """C.3.10: host-side statistics from exact totals.

    Pinned by: test_oracle_correct.py::test_zero_mismatch_collapses_everything, ::test_k1_cancels_exactly_k3_does_not.
    """
    st = dict(glob)
    st["n_seq"] = n_seq
    st["n_seq_rejected"] = int((np.asarray(seq_keep) == 0).sum())
    n = glob["n_resp_tok"]
    for k in ("abs_delta", "k1", "k3"):
        st["mean_" + k] = (float(glob["sum_" + k]) * (2.0 ** -52)) / n if n else 0.0
    return st


def seq_index(cu_seqlens, tok_begin: int, n: int) -> np.ndarray:
    """Sequence id of every local token (searchsorted on the global offsets).

    Pinned by: test_oracle_correct.py::test_sharding_is_exact_and_order_free (cuts inside sequences).
    """
    cu = np.asarray(cu_seqlens, dtype=np.int64)
    g = np.arange(tok_begin, tok_begin + n, dtype=np.int64)
    return np.searchsorted(cu, g, side="right") - 1


def correct(lp_num, lp_den, cu_seqlens, cfg: Cfg, resp_mask=None):
    """Single-shard (P = 1) end-to-end oracle: returns a dict with every output.

    Pinned by: every test in test_oracle_correct.py (Table 1 values, closed forms, zero mismatch, K1 cancellation, thresholds).
    """
    tokens, glob, seq = local_partials(lp_num, lp_den, cu_seqlens, cfg, resp_mask, 0)
    glob, seq = combine([(glob, seq)])
    seq_keep, score = decide(seq, cfg)
    sid = seq_index(cu_seqlens, 0, tokens["delta"].size)
    coeff = np.where(seq_keep[sid] != 0, tokens["coeff_prov"], np.float32(0.0)).astype(np.float32)
    stats = finalize_stats(glob, seq_keep, seq.shape[0])
    return {
        "delta": tokens["delta"], "tis_w": tokens["tis_w"], "tok_keep": tokens["tok_keep"],
        "seq_keep": seq_keep, "seq_score": score, "coeff": coeff, "stats": stats,
        "seq_partials": seq,
    }
