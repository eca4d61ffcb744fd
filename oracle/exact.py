"""Arbitrary-precision references used ONLY to pin the oracle (TEST INFRASTRUCTURE ONLY).

These evaluate the real-number definitions (§2 P:94-108 softmax /
log-prob, §4.1 P:393 K1/K3, §4.2 P:496 r_corr) with mpmath at 50-60 digits,
independently of numpy, so that a dropped term, a wrong sign or a transposed
operand in ``oracle.logprob`` / ``oracle.correct`` fails a pin.
"""
from __future__ import annotations

import mpmath as mp


def logprob_entropy_mp(H, W, ids, temperature=1.0, dps: int = 50):
    """Brute force: every logit as an exact dot product, then log-softmax and entropy."""
    with mp.workdps(dps):
        out_lp, out_h = [], []
        T = mp.mpf(temperature)
        for t, row in enumerate(H):
            xs = []
            for w in W:
                z = mp.fsum(mp.mpf(float(a)) * mp.mpf(float(b)) for a, b in zip(row, w))
                xs.append(z / T)
            lse = mp.log(mp.fsum(mp.exp(x) for x in xs))
            ps = [mp.exp(x - lse) for x in xs]
            out_lp.append(xs[int(ids[t])] - lse)
            out_h.append(-mp.fsum(p * mp.log(p) for p in ps if p > 0))
        return out_lp, out_h


def k3_mp(d, dps: int = 60):
    """K3(r) = (r - 1) - log r at r = e^d, i.e. expm1(d) - d.

    expm1(d) - d cancels ~|log10 d| digits for small d, so the working precision
    grows with that cancellation."""
    import math
    if d != 0:
        dps += max(0, int(-math.log10(abs(d))) + 5)
    with mp.workdps(dps):
        x = mp.mpf(d)
        return mp.expm1(x) - x


def exp_mp(d, dps: int = 60):
    with mp.workdps(dps):
        return mp.exp(mp.mpf(d))


def ulp(x: float) -> float:
    import math
    return math.ulp(abs(x)) if x != 0 else math.ulp(0.0)
