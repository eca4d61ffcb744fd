// contract.cuh -- device side of the decision-path arithmetic contract (DESIGN.md §2 C.3) and the
// exact-integer reduction helpers shared by the correction (correct.cu) and PPO (ppo.cu) kernels.
// Every fp64 op is an explicit round-to-nearest intrinsic (__dadd_rn / __dmul_rn are never contracted;
// the K3 series' Horner steps are explicit single-rounding __fma_rn, contract revision 4); every sum of
// quantised values is an int128 integer sum, so results do not depend on reduction order,
// sharding or the number of GPUs.
#pragma once
#include <cuda_runtime.h>
#include <math_constants.h>

#include <climits>
#include <cstdint>

#include "tim_internal.h"

namespace tim {

// RN(1/n!), n = 0..23 (binary64), and the Cody-Waite split of ln 2 (fdlibm ln2_hi / ln2_lo).
static __constant__ double kInvFact[24] = {
    0x1.0000000000000p+0,  0x1.0000000000000p+0,  0x1.0000000000000p-1,  0x1.5555555555555p-3,
    0x1.5555555555555p-5,  0x1.1111111111111p-7,  0x1.6c16c16c16c17p-10, 0x1.a01a01a01a01ap-13,
    0x1.a01a01a01a01ap-16, 0x1.71de3a556c734p-19, 0x1.27e4fb7789f5cp-22, 0x1.ae64567f544e4p-26,
    0x1.1eed8eff8d898p-29, 0x1.6124613a86d09p-33, 0x1.93974a8c07c9dp-37, 0x1.ae7f3e733b81fp-41,
    0x1.ae7f3e733b81fp-45, 0x1.952c77030ad4ap-49, 0x1.6827863b97d97p-53, 0x1.2f49b46814157p-57,
    0x1.e542ba4020225p-62, 0x1.71b8ef6dcf572p-66, 0x1.0ce396db7f853p-70, 0x1.761b41316381ap-75};
constexpr double kLog2e = 0x1.71547652b82fep+0;
constexpr double kLn2Hi = 0x1.62e42fee00000p-1;
constexpr double kLn2Lo = 0x1.a39ef35793c76p-33;
constexpr double kTwo52 = 0x1p52;
constexpr long long kSatX = 1ll << 62;

constexpr double kSmall = 0x1p-6;  // |d| <= 2^-6: short Horner polynomial (n = 2..9)
constexpr double kMid = 0x1p-2;    // |d| <= 2^-2: n = 2..15

// K3 series d^2 Q(d), Q = Horner of RN(1/n!), n = kTop..2, each step one fused multiply-add.
template <int kTop>
__device__ __forceinline__ double k3_series(double d) {
  double Q = kInvFact[kTop];
#pragma unroll
  for (int n = kTop - 1; n >= 2; --n) Q = __fma_rn(Q, d, kInvFact[n]);
  return __dmul_rn(__dmul_rn(d, d), Q);
}
__device__ __forceinline__ double k3_small(double d) { return k3_series<9>(d); }
__device__ __forceinline__ double k3_mid(double d) { return k3_series<15>(d); }
__device__ __forceinline__ double k3_medium(double d) { return k3_series<23>(d); }

// The short and mid series of one token in a single Horner chain: the mid prefix (n = 15..10)
// runs for every token, then a tiny token (|d| <= 2^-6) restarts from fma(0, d, c9) = c9, which
// is exactly the short series' start; n = 8..2 are the same ops for both.  Bit-identical to
// k3_small (tiny) / k3_mid (otherwise).
__device__ __forceinline__ double k3_small_or_mid(double d, bool tiny) {
  double P = kInvFact[15];
#pragma unroll
  for (int n = 14; n >= 10; --n) P = __fma_rn(P, d, kInvFact[n]);
  P = __fma_rn(tiny ? 0.0 : P, d, kInvFact[9]);
#pragma unroll
  for (int n = 8; n >= 2; --n) P = __fma_rn(P, d, kInvFact[n]);
  return __dmul_rn(__dmul_rn(d, d), P);
}

// Cody-Waite e^d for -700 <= d <= 709: k = rint(d log2 e), r = (d - k ln2_hi) - k ln2_lo,
// degree-13 Taylor (Horner), * 2^k.
__device__ __forceinline__ double exp_cw(double d) {
  const double k = rint(__dmul_rn(d, kLog2e));
  const double r = __dsub_rn(__dsub_rn(d, __dmul_rn(k, kLn2Hi)), __dmul_rn(k, kLn2Lo));
  double p = kInvFact[13];
#pragma unroll
  for (int n = 12; n >= 0; --n) p = __dadd_rn(__dmul_rn(p, r), kInvFact[n]);
  const long long ki = static_cast<long long>(k);  // in [-1010, 1023]: 2^k is a normal double
  return __dmul_rn(p, __longlong_as_double((ki + 1023) << 52));
}

// e^d.  |d| <= 2^-2: (1 + d) + K3(d) with the K3 branch's own series (e^d = 1 + d + K3, the K3
// the caller needs anyway).  Otherwise Cody-Waite (exp_cw); +inf above 709, 0 below -700.
__device__ __forceinline__ double exp_from_k3_small(double d, double k3s) { return __dadd_rn(__dadd_rn(1.0, d), k3s); }
__device__ __forceinline__ double exp_c(double d) {
  if (d > 709.0) return CUDART_INF;
  if (d < -700.0) return 0.0;
  const double ad = fabs(d);
  if (ad <= kSmall) return exp_from_k3_small(d, k3_small(d));
  if (ad <= kMid) return exp_from_k3_small(d, k3_mid(d));
  return exp_cw(d);
}

// K3 = e^d - 1 - d = d^2 P(d): Horner series of (e^d - 1 - d) / d^2 with RN(1/n!), n = 2..9 for
// |d| <= 2^-6, n = 2..15 for |d| <= 2^-2, n = 2..23 for |d| <= 1; (exp_c(d) - 1) - d otherwise.
__device__ __forceinline__ double k3_c(double d) {
  const double ad = fabs(d);
  if (ad <= kSmall) return k3_small(d);
  if (ad <= kMid) return k3_mid(d);
  if (ad <= 1.0) return k3_medium(d);
  return __dsub_rn(__dsub_rn(exp_c(d), 1.0), d);
}

// X = rint(K 2^52); |K| > 2^10 or NaN/inf saturates to sign(K) 2^62.
__device__ __forceinline__ long long fixed_point(double K, bool& sat) {
  if (!(fabs(K) <= 1024.0)) {
    sat = true;
    return signbit(K) ? -kSatX : kSatX;
  }
  sat = false;
  return __double2ll_rn(__dmul_rn(K, kTwo52));
}

__device__ __forceinline__ void atomic_add_i128(int64_t* p, __int128 v) {
  const unsigned long long lo = static_cast<unsigned long long>(v);
  unsigned long long hi = static_cast<unsigned long long>(v >> 64);
  if (lo != 0) {
    const unsigned long long old = atomicAdd(reinterpret_cast<unsigned long long*>(p), lo);
    if (old + lo < old) hi += 1;  // carry out of the low word
  }
  if (hi != 0) atomicAdd(reinterpret_cast<unsigned long long*>(p + 1), hi);
}

__device__ __forceinline__ __int128 shfl_down_i128(__int128 v, int off) {
  long long lo = static_cast<long long>(static_cast<unsigned long long>(v));
  long long hi = static_cast<long long>(v >> 64);
  lo = __shfl_down_sync(0xffffffffu, lo, off);
  hi = __shfl_down_sync(0xffffffffu, hi, off);
  return (static_cast<__int128>(hi) << 64) | static_cast<__int128>(static_cast<unsigned long long>(lo));
}
__device__ __forceinline__ __int128 warp_sum_i128(__int128 v) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v += shfl_down_i128(v, off);
  return v;
}
__device__ __forceinline__ long long warp_sum_i64(long long v) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v += __shfl_down_sync(0xffffffffu, v, off);
  return v;
}
__device__ __forceinline__ unsigned long long warp_max_u64(unsigned long long v) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    const unsigned long long o = __shfl_down_sync(0xffffffffu, v, off);
    v = o > v ? o : v;
  }
  return v;
}

struct SeqAcc {
  long long sid;  // sequence id (LLONG_MAX: none)
  __int128 x;
  long long t, nsat;
};

__device__ __forceinline__ void flush_seq(tim_seq_partial* seqp, const SeqAcc& a) {
  if (a.t == 0 && a.x == 0 && a.nsat == 0) return;
  tim_seq_partial* d = seqp + a.sid;
  atomic_add_i128(&d->x_lo, a.x);
  if (a.t) atomicAdd(reinterpret_cast<unsigned long long*>(&d->n_tok), static_cast<unsigned long long>(a.t));
  if (a.nsat) atomicAdd(reinterpret_cast<unsigned long long*>(&d->n_sat), static_cast<unsigned long long>(a.nsat));
}

// sequence containing global token g: last s with cu[s] <= g
__device__ __forceinline__ long long seq_of(const int64_t* cu, long long n_seq, long long g) {
  long long lo = 0, hi = n_seq;  // invariant cu[lo] <= g (cu[0] == 0), answer in [lo, hi)
  while (hi - lo > 1) {
    const long long mid = (lo + hi) >> 1;
    if (__ldg(cu + mid) <= g) lo = mid; else hi = mid;
  }
  return lo;
}

// The shard [tok_begin, tok_begin + n) must lie inside the global sequences [cu[0], cu[n_seq]).
// A token outside is a data error (reading U13b): its global index (the first one outside) goes
// to the status through bad_inv (the max of kBadSentinel - index, i.e. the min index wins).
__device__ __forceinline__ void shard_range_check(const int64_t* cu, long long n_seq, long long tok_begin,
                                                  long long n, unsigned long long& bad_inv) {
  if (n <= 0) return;
  const long long c0 = __ldg(cu), c1 = __ldg(cu + n_seq);
  long long first = -1;
  if (tok_begin < c0) first = tok_begin;
  else if (tok_begin + n > c1) first = tok_begin > c1 ? tok_begin : c1;
  if (first >= 0) {
    const unsigned long long b = kBadSentinel - static_cast<unsigned long long>(first);
    bad_inv = b > bad_inv ? b : bad_inv;
  }
}

// exact int128 -> double, round to nearest even
__device__ __forceinline__ double i128_to_double(__int128 x) {
  const bool neg = x < 0;
  unsigned __int128 u = neg ? static_cast<unsigned __int128>(-x) : static_cast<unsigned __int128>(x);
  const unsigned long long hi = static_cast<unsigned long long>(u >> 64);
  double r;
  if (hi == 0) {
    r = __ull2double_rn(static_cast<unsigned long long>(u));
  } else {
    const int sh = 64 - __clzll(hi);  // bits above the low 64
    unsigned long long top = static_cast<unsigned long long>(u >> sh);
    const unsigned __int128 rem = u & ((static_cast<unsigned __int128>(1) << sh) - 1);
    if (rem != 0) top |= 1ull;  // sticky: bit 0 lies 11 bits below the rounding position
    r = __dmul_rn(__ull2double_rn(top), __longlong_as_double(static_cast<long long>(sh + 1023) << 52));
  }
  return neg ? -r : r;
}

__device__ __forceinline__ __int128 ld_i128(const int64_t* p) {
  return (static_cast<__int128>(p[1]) << 64) | static_cast<__int128>(static_cast<unsigned long long>(p[0]));
}

// floor(tau * 2^52 * T) exactly: tau = mant * 2^e (frexp), M = mant * 2^53 an integer,
// tau 2^52 T = M T 2^(e-1).  |tau| < 2^10 => e <= 11, M T < 2^84: fits int128.
__device__ __forceinline__ __int128 seq_threshold(double tau, long long T) {
  int e;
  const double mant = frexp(tau, &e);
  const long long M = static_cast<long long>(__dmul_rn(mant, 0x1p53));
  const __int128 MT = static_cast<__int128>(M) * T;
  const int sh = e - 1;
  return sh >= 0 ? (MT << sh) : (MT >> (-sh));  // arithmetic shift = floor
}


// Sequence keep (C.3 step 9): T_s = 0 keeps, a saturated token rejects, else the exact int128
// compare X_s <= floor(tau 2^52) (SUM) or floor(tau 2^52 T_s) (MEAN).
__device__ __forceinline__ bool seq_keep_decision(double tau_seq, int seq_agg, __int128 X, long long T,
                                                  long long nsat) {
  if (T == 0) return true;
  if (nsat > 0) return false;
  return X <= seq_threshold(tau_seq, seq_agg == TIM_AGG_MEAN ? T : 1);
}

}  // namespace tim
