// correct.cu -- mismatch statistics and TIS / RS corrections.
//
// Real-number semantics from PAPER.md: delta_t (§2), r_corr = e^delta (§4.2),
// w = min(r_corr, tau_tok) (L_TIS P:497-507), K1 = -log r, K3 = (r-1) - log r (§4.1),
// S_seq = sum_t K(q_t) and 1[S_seq <= tau_seq] (L_RS P:509-547, App. A.4).
//
// Integer outputs (masks, counts, sequence decisions) are bit-exact by construction through
// the decision-path arithmetic contract: every fp64 op is an
// explicit round-to-nearest intrinsic (__dadd_rn / __dsub_rn / __dmul_rn: never contracted to
// FMA), no transcendental from libm sits on the decision path, the per-token K values are turned
// into exact 2^-52 fixed point and all sums are int128 integer sums -- exact, so independent of
// the reduction order, of atomics order, of sharding and of the GPU count.
//
// Layout: structure-of-arrays fp32 / u8 token vectors, one warp owns 128 consecutive tokens
// (4 per lane, 16-B vector loads and stores), so every load and store is fully coalesced.
#include <cuda_runtime.h>
#include <math_constants.h>

#include <cstdint>

#include "contract.cuh"
#include "ptx.cuh"
#include "tim_internal.h"

namespace tim {

#ifndef TIM_CORR_MINB
#define TIM_CORR_MINB 5
#endif
constexpr int kTpl = 4;                 // tokens per lane (one float4 of num / den, one u32 of resp)
constexpr int kWarpTok = 32 * kTpl;     // tokens per warp chunk
constexpr int kLocalThreads = 128;
constexpr int kLocalWarps = kLocalThreads / 32;
#ifndef TIM_CORR_PLAIN_STORES
#define TIM_CORR_PLAIN_STORES 1  // 0: st.global.cs stores (3% slower end to end)
#endif
#ifndef TIM_ZERO_PLAIN_STORES
#define TIM_ZERO_PLAIN_STORES 0  // 1: plain stores in the zeroing pass (0.5% slower)
#endif
#ifndef TIM_CORR_LOAD_HINT
#define TIM_CORR_LOAD_HINT 0  // 1: cp.async reads with an L2 evict_first policy (1.2% slower)
#endif
#ifndef TIM_CORR_STAGES
#define TIM_CORR_STAGES 4
#endif
constexpr int kStages = TIM_CORR_STAGES;  // per-warp TMA ring: chunks of num / den in flight
constexpr int kFoldChunks = 16;        // the exact fp64 chunk sums are folded into int128 this often

// Per-thread state that the fast path does not touch every chunk, in shared memory so the hot
// loop keeps its registers for the loads in flight and the Horner chains: the int128 sums, the
// sequence walk, and the counters of the (out-of-line) mixed-chunk path.
struct LaneState {
  __int128 s_abs, s_k1, s_k3, seq_x;
  unsigned long long bad_inv;
  long long c_sat, seq_nsat;
  long long sid, next_b, seq_t;
  double mx;
  unsigned c_resp, c_trunc, c_rej, pad;
  long long pad2;
};
static_assert(sizeof(LaneState) % 16 == 0, "LaneState alignment");

struct Chunk {
  float4 num, den;
  uint32_t resp;
};

__device__ __forceinline__ Chunk load_chunk(const LocalParams& p, long long i0) {
  Chunk c;
  if (p.vec && i0 + kTpl <= p.n) {
    c.num = __ldcs(reinterpret_cast<const float4*>(p.num + i0));
    c.den = __ldcs(reinterpret_cast<const float4*>(p.den + i0));
    c.resp = p.resp ? __ldcs(reinterpret_cast<const unsigned int*>(p.resp + i0)) : 0x01010101u;
  } else {
    float nv[4], dv[4];
    uint32_t r = 0;
#pragma unroll
    for (int k = 0; k < kTpl; ++k) {
      const long long i = i0 + k;
      nv[k] = i < p.n ? p.num[i] : 0.f;
      dv[k] = i < p.n ? p.den[i] : 0.f;
      r |= static_cast<uint32_t>(i < p.n ? (p.resp ? (p.resp[i] != 0) : 1) : 0) << (8 * k);
    }
    c.num = make_float4(nv[0], nv[1], nv[2], nv[3]);
    c.den = make_float4(dv[0], dv[1], dv[2], dv[3]);
    c.resp = r;
  }
  return c;
}

__device__ __forceinline__ void store_chunk(const LocalParams& p, long long i0, bool full, const float* w_out,
                                            const float* c_out, uint32_t kbits) {
  if (full) {
#if TIM_CORR_PLAIN_STORES  // plain stores: measured 3% faster end to end than st.global.cs
    *reinterpret_cast<float4*>(p.tis_w + i0) = make_float4(w_out[0], w_out[1], w_out[2], w_out[3]);
    *reinterpret_cast<float4*>(p.coeff + i0) = make_float4(c_out[0], c_out[1], c_out[2], c_out[3]);
    *reinterpret_cast<unsigned int*>(p.tok_keep + i0) = kbits;
#else
    __stcs(reinterpret_cast<float4*>(p.tis_w + i0), make_float4(w_out[0], w_out[1], w_out[2], w_out[3]));
    __stcs(reinterpret_cast<float4*>(p.coeff + i0), make_float4(c_out[0], c_out[1], c_out[2], c_out[3]));
    __stcs(reinterpret_cast<unsigned int*>(p.tok_keep + i0), kbits);
#endif
  } else {
#pragma unroll
    for (int k = 0; k < kTpl; ++k) {
      const long long i = i0 + k;
      if (i < p.n) {
        p.tis_w[i] = w_out[k];
        p.coeff[i] = c_out[k];
        p.tok_keep[i] = (kbits >> (8 * k)) & 0xffu;
      }
    }
  }
}

// K3 and e^delta of a token outside the short-polynomial range (rare; out of line so the
// chunk loop keeps its registers and stays in the instruction cache).
__device__ __noinline__ double2 k3_exp_full(double d) {
  if (fabs(d) <= kMid) {  // series branches: e^d = (1 + d) + K3 with the same series
    const double k3 = fabs(d) <= kSmall ? k3_small(d) : k3_mid(d);
    return make_double2(k3, exp_from_k3_small(d, k3));
  }
  return make_double2(k3_c(d), exp_c(d));
}

// Fast-path register state of a lane: exact fp64 sums of quantised values (each an integer with
// |X| <= 2^46, so 16 chunks of four sum exactly, < 2^52), max |delta| and counters.
struct FastAcc {
  double k1, k3, ab, seq, mx;
  unsigned resp, trunc, rej, seq_t;
};

// A chunk that the fast body cannot take (a sequence or prompt / response boundary inside it, a
// partial or unaligned chunk, a non-interior configuration): per-token response masks, the short
// contract series in lock-step for every token with |delta| <= 2^-6 of a whole lane (four tokens
// before the lane's next sequence boundary), and the remaining (slow) tokens afterwards with the
// full contract per lane, int128 sums and the sequence walk in the lane's shared-memory state.
template <bool kOut, int kSeqK, bool kTis, bool kTokRs>
__device__ __forceinline__ void masked_body(const LocalParams& p, LaneState& st, FastAcc& fa, const uint32_t resp_bits,
                                            const long long i0, const bool full, const bool lane_whole,
                                            const double (&dv)[kTpl]) {
  constexpr bool kSeq = kSeqK != TIM_SEQ_NONE;
  constexpr bool seq_k1 = kSeqK == TIM_SEQ_K1;
  const CorrectDevCfg& cfg = p.cfg;
  const float cap_f = __double2float_rn(cfg.tis_cap);
  unsigned slow = 0;
  double ds[kTpl], k3s[kTpl];
#pragma unroll
  for (int k = 0; k < kTpl; ++k) {
    const bool sm = fabs(dv[k]) <= kSmall;  // false for NaN / inf
    if (!sm || !lane_whole) slow |= 1u << k;
    ds[k] = sm ? dv[k] : 0.0;  // slow small tokens reuse their k3s
  }
  {  // short K3 series, four independent Horner chains
    double q[kTpl];
#pragma unroll
    for (int k = 0; k < kTpl; ++k) q[k] = kInvFact[9];
#pragma unroll
    for (int n = 8; n >= 2; --n)
#pragma unroll
      for (int k = 0; k < kTpl; ++k) q[k] = __fma_rn(q[k], ds[k], kInvFact[n]);
#pragma unroll
    for (int k = 0; k < kTpl; ++k) k3s[k] = __dmul_rn(__dmul_rn(ds[k], ds[k]), q[k]);
  }
  float w_out[kTpl], c_out[kTpl];
  uint32_t kbits = 0;
  double cmx = 0.0;
  unsigned cn = 0, ctr = 0, crj = 0, cst = 0;
#pragma unroll
  for (int k = 0; k < kTpl; ++k) {
    const double d = ds[k];
    const bool resp = ((resp_bits >> (8 * k)) & 0xffu) != 0u;
    const bool use = resp && !((slow >> k) & 1u);
    bool trunc = false;
    float w = 1.f;
    if (kTis) {  // (float) min(e, cap) == min((float) e, (float) cap): rounding is monotonic
      trunc = d > cfg.log_tis_cap;
      w = trunc ? cap_f : fminf(__double2float_rn(exp_from_k3_small(d, k3s[k])), cap_f);
    }
    const bool keep = kTokRs ? (cfg.log_lo <= d && d <= cfg.log_hi) : true;
    w_out[k] = w;
    c_out[k] = (resp && keep) ? w : 0.f;
    kbits |= static_cast<uint32_t>(keep) << (8 * k);
    const double dz = use ? d : 0.0;  // unused tokens add exactly 0
    const double kz = use ? k3s[k] : 0.0;
    const double x1 = rint(__dmul_rn(-dz, kTwo52));  // exact scaling, then round to integer
    const double x3 = rint(__dmul_rn(kz, kTwo52));
    fa.k1 = __dadd_rn(fa.k1, x1);
    fa.k3 = __dadd_rn(fa.k3, x3);
    fa.ab = __dadd_rn(fa.ab, fabs(x1));
    cmx = fabs(dz) > cmx ? fabs(dz) : cmx;
    cn += use ? 1u : 0u;
    if (kTis) ctr += (use && trunc) ? 1u : 0u;
    if (kTokRs) crj += (use && !keep) ? 1u : 0u;
    if (kSeq) {
      const double xq = seq_k1 ? x1 : x3;
      if (kTokRs) {
        fa.seq = __dadd_rn(fa.seq, keep ? xq : 0.0);
        cst += (use && keep) ? 1u : 0u;
      } else {
        fa.seq = __dadd_rn(fa.seq, xq);
        cst += use ? 1u : 0u;
      }
    }
  }
  fa.mx = cmx > fa.mx ? cmx : fa.mx;
  fa.resp += cn;
  fa.trunc += ctr;
  fa.rej += crj;
  if (kSeq) fa.seq_t += cst;

  if (slow) {  // rare: the full contract per token, in the slow tokens' lanes only
    if (kSeq) {  // the lane may leave its sequence below: its pending sums go with it
      st.seq_x += __double2ll_rn(fa.seq);
      st.seq_t += fa.seq_t;
      fa.seq = 0.0;
      fa.seq_t = 0;
    }
#pragma unroll
    for (int k = 0; k < kTpl; ++k) {
      if (!((slow >> k) & 1u)) continue;
      const long long i = i0 + k;
      if (i >= p.n) continue;
      const long long g = p.tok_begin + i;
      const double d = dv[k];
      if (kSeq) {
        // crossed into a later sequence (skips empty ones); bounded by the last sequence so a
        // shard reaching past cu[n_seq] (a data error, flagged by the range check) stays in bounds
        while (g >= st.next_b && st.sid + 1 < p.n_seq) {
          SeqAcc a;
          a.sid = st.sid;
          a.x = st.seq_x;
          a.t = st.seq_t;
          a.nsat = st.seq_nsat;
          flush_seq(p.seqp, a);
          st.seq_x = 0;
          st.seq_nsat = 0;
          st.seq_t = 0;
          st.sid += 1;
          st.next_b = __ldg(p.cu + st.sid + 1);
        }
      }
      if (!isfinite(d)) {  // C.3.2 data error: excluded from every sum, outputs NaN / 0
        const unsigned long long b = kBadSentinel - static_cast<unsigned long long>(g);
        st.bad_inv = b > st.bad_inv ? b : st.bad_inv;
        w_out[k] = CUDART_NAN_F;
        c_out[k] = 0.f;
        kbits &= ~(0xffu << (8 * k));
        continue;
      }
      const bool resp = (resp_bits >> (8 * k)) & 0xffu;
      const bool sm = fabs(d) <= kSmall;
      double k3, e;
      if (sm) {
        k3 = k3s[k];
        e = exp_from_k3_small(d, k3);
      } else {
        const double2 ke = k3_exp_full(d);
        k3 = ke.x;
        e = ke.y;
      }
      const bool trunc = kTis && d > cfg.log_tis_cap;
      if (kTis) w_out[k] = __double2float_rn(trunc ? cfg.tis_cap : fmin(e, cfg.tis_cap));
      const bool keep = kTokRs ? (cfg.log_lo <= d && d <= cfg.log_hi) : true;
      c_out[k] = (resp && keep) ? w_out[k] : 0.f;
      kbits = (kbits & ~(0xffu << (8 * k))) | (static_cast<uint32_t>(keep) << (8 * k));
      if (!resp) continue;
      bool sat1, sat3;
      const long long x1 = fixed_point(-d, sat1);
      const long long x3 = fixed_point(k3, sat3);
      st.c_resp += 1;
      st.c_trunc += trunc ? 1u : 0u;
      st.c_rej += keep ? 0u : 1u;
      st.s_abs += x1 < 0 ? -x1 : x1;  // rint is odd-symmetric: X(|delta|) = |X(-delta)|
      st.s_k1 += x1;
      st.s_k3 += x3;
      st.mx = fmax(st.mx, fabs(d));
      if (kSeq && keep) {
        const bool satq = seq_k1 ? sat1 : sat3;
        st.seq_x += seq_k1 ? x1 : x3;
        st.seq_t += 1;
        st.seq_nsat += satq ? 1 : 0;
        st.c_sat += satq ? 1 : 0;
      }
    }
  }
  if (kOut) store_chunk(p, i0, full, w_out, c_out, kbits);
}

// The few tokens of a fast-body chunk that the lock-step body took as delta = 0 (|delta| > 2^-6,
// or non-finite), redone in their own lanes: the full contract, int128 sums in the lane's
// shared-memory state, and corrections of what the lock-step body counted for them (a response
// token, kept, one more contributing token of the sequence).  The chunk lies inside the warp's
// current sequence, so there is no sequence walk; the scalar stores follow the chunk's vector
// store in program order.
template <bool kOut, int kSeqK, bool kTis, bool kTokRs>
__device__ __forceinline__ void fix_slow(const LocalParams& p, LaneState& st, const unsigned slow, const long long i0,
                                         const bool sum_on, const double (&dv)[kTpl]) {
  constexpr bool kSeq = kSeqK != TIM_SEQ_NONE;
  constexpr bool seq_k1 = kSeqK == TIM_SEQ_K1;
  const CorrectDevCfg& cfg = p.cfg;
#pragma unroll
  for (int k = 0; k < kTpl; ++k) {
    if (!((slow >> k) & 1u)) continue;
    const long long i = i0 + k;
    const double d = dv[k];
    float w = 1.f, c = 0.f;
    uint8_t keep8 = 0;
    if (!isfinite(d)) {  // C.3.2 data error: out of every sum and count, outputs NaN / 0
      const unsigned long long b = kBadSentinel - static_cast<unsigned long long>(p.tok_begin + i);
      st.bad_inv = b > st.bad_inv ? b : st.bad_inv;
      w = CUDART_NAN_F;
      if (sum_on) {
        st.c_resp -= 1u;
        if (kSeq) st.seq_t -= 1;
      }
    } else {
      const double2 ke = k3_exp_full(d);
      const bool trunc = kTis && d > cfg.log_tis_cap;
      if (kTis) w = __double2float_rn(trunc ? cfg.tis_cap : fmin(ke.y, cfg.tis_cap));
      const bool keep = kTokRs ? (cfg.log_lo <= d && d <= cfg.log_hi) : true;
      c = (sum_on && keep) ? w : 0.f;
      keep8 = keep ? 1 : 0;
      if (sum_on) {
        bool sat1, sat3;
        const long long x1 = fixed_point(-d, sat1);
        const long long x3 = fixed_point(ke.x, sat3);
        st.c_trunc += trunc ? 1u : 0u;
        st.c_rej += keep ? 0u : 1u;
        st.s_abs += x1 < 0 ? -x1 : x1;
        st.s_k1 += x1;
        st.s_k3 += x3;
        st.mx = fmax(st.mx, fabs(d));
        if (kSeq) {
          if (keep) {
            const bool satq = seq_k1 ? sat1 : sat3;
            st.seq_x += seq_k1 ? x1 : x3;
            st.seq_nsat += satq ? 1 : 0;
            st.c_sat += satq ? 1 : 0;
          } else {
            st.seq_t -= 1;
          }
        }
      }
    }
    if (kOut) {
      p.tis_w[i] = w;
      p.coeff[i] = c;
      p.tok_keep[i] = keep8;
    }
  }
}

// The select-free body of a chunk inside one sequence whose response mask is warp-uniform
// (sum_on: every token a response token, or none), under an interior configuration
// (LocalParams::interior): every token with |delta| <= 2^-6 runs the short contract series in
// lock-step (one fused multiply-add per Horner step) and is neither truncated nor token-rejected,
// and its weight is (float) e^delta.  A token outside that range enters as delta = 0, which adds
// exactly 0 to every sum, and fix_slow then redoes it.
template <bool kOut, int kSeqK, bool kTis, bool kTokRs>
__device__ __forceinline__ void fast_body(const LocalParams& p, LaneState& st, FastAcc& fa, const long long i0,
                                          const bool sum_on, const double (&dv)[kTpl]) {
  constexpr bool kSeq = kSeqK != TIM_SEQ_NONE;
  constexpr bool seq_k1 = kSeqK == TIM_SEQ_K1;
  double ds[kTpl];
  unsigned slow = 0;
#pragma unroll
  for (int k = 0; k < kTpl; ++k) {
    const bool sm = fabs(dv[k]) <= kSmall;  // false for NaN
    slow |= sm ? 0u : (1u << k);
    ds[k] = sm ? dv[k] : 0.0;
  }
  double k3s[kTpl] = {0.0, 0.0, 0.0, 0.0};
  if (kTis || sum_on) {  // short K3 series, four independent Horner chains
    double q[kTpl];
#pragma unroll
    for (int k = 0; k < kTpl; ++k) q[k] = kInvFact[9];
#pragma unroll
    for (int n = 8; n >= 2; --n)
#pragma unroll
      for (int k = 0; k < kTpl; ++k) q[k] = __fma_rn(q[k], ds[k], kInvFact[n]);
#pragma unroll
    for (int k = 0; k < kTpl; ++k) k3s[k] = __dmul_rn(__dmul_rn(ds[k], ds[k]), q[k]);
  }
  float w_out[kTpl], c_out[kTpl];
#pragma unroll
  for (int k = 0; k < kTpl; ++k) {
    w_out[k] = kTis ? __double2float_rn(exp_from_k3_small(ds[k], k3s[k])) : 1.f;
    c_out[k] = sum_on ? w_out[k] : 0.f;
  }
  if (sum_on) {
#pragma unroll
    for (int k = 0; k < kTpl; ++k) {
      const double x1 = rint(__dmul_rn(-ds[k], kTwo52));  // exact scaling, then round to integer
      const double x3 = rint(__dmul_rn(k3s[k], kTwo52));
      fa.k1 = __dadd_rn(fa.k1, x1);
      fa.k3 = __dadd_rn(fa.k3, x3);
      fa.ab = __dadd_rn(fa.ab, fabs(x1));
      if (kSeq) fa.seq = __dadd_rn(fa.seq, seq_k1 ? x1 : x3);
    }
    // running max |delta| as compare-and-select (ds is never NaN here, so fmax's NaN handling --
    // five instructions per step -- is not needed; the same value results)
    double amx = fa.mx;
#pragma unroll
    for (int k = 0; k < kTpl; ++k) {
      const double a = fabs(ds[k]);
      amx = a > amx ? a : amx;
    }
    fa.mx = amx;
    fa.resp += kTpl;
    if (kSeq) fa.seq_t += kTpl;
  }
  if (kOut) store_chunk(p, i0, true, w_out, c_out, 0x01010101u);
  if (slow) fix_slow<kOut, kSeqK, kTis, kTokRs>(p, st, slow, i0, sum_on, dv);
}

// Segmented warp flush of per-lane pending sequence sums (sequence ids non-decreasing in lane
// order): the head lane of each run of equal ids adds the run's total with one set of atomics.
__device__ __forceinline__ void seq_flush_segmented(tim_seq_partial* seqp, SeqAcc acc, const int lane) {
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const long long osid = __shfl_down_sync(0xffffffffu, acc.sid, off);
    const __int128 ox = shfl_down_i128(acc.x, off);
    const long long ot = __shfl_down_sync(0xffffffffu, acc.t, off);
    const long long on = __shfl_down_sync(0xffffffffu, acc.nsat, off);
    if (lane + off < 32 && osid == acc.sid) {
      acc.x += ox;
      acc.t += ot;
      acc.nsat += on;
    }
  }
  // lane l now holds the sum of lanes [l, l+2^k) with the same id, so the head of each run
  // (first lane of that id) holds the whole run because runs are contiguous.
  const long long prev_sid = __shfl_up_sync(0xffffffffu, acc.sid, 1);
  const bool head = lane == 0 || prev_sid != acc.sid;
  if (head && acc.sid != LLONG_MAX) flush_seq(seqp, acc);
}

// Pass 1 (a5).  Every warp owns a contiguous run of 128-token chunks (four tokens per lane).
// The warp streams its chunks' num / den (and the response mask when 16-B aligned) through a
// kStages-deep ring in shared memory (1-D bulk copies issued by one elected lane, completion on
// one mbarrier per stage), so the bytes in flight do not cost registers.  The warp keeps a
// warp-uniform sequence cursor (w_sid, w_next = cu[w_sid + 1]): a chunk that starts at or after
// w_next first flushes the warp's pending sums of w_sid (one warp reduction, one set of atomics)
// and advances the cursor.  A chunk inside w_sid with a warp-uniform response mask takes
// fast_body; any other chunk (a sequence boundary or a prompt / response boundary inside it, a
// non-interior configuration) takes the masked body with per-lane sequence walks, after which the
// lanes are brought back onto one cursor.
template <bool kOut, int kSeqK, bool kTis, bool kTokRs>
__device__ __forceinline__ void pass1_body(const LocalParams& p) {
  constexpr bool kSeq = kSeqK != TIM_SEQ_NONE;  // kSeqK: the sequence score (TIM_SEQ_K1 / TIM_SEQ_K3)
  __shared__ LaneState sh_state[kLocalThreads];
  __shared__ __align__(128) float ring[kLocalWarps][kStages][2][kWarpTok];
  __shared__ __align__(128) uint32_t ring_resp[kLocalWarps][kStages][kWarpTok / 4];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const long long warp_g = (static_cast<long long>(blockIdx.x) * kLocalThreads + threadIdx.x) >> 5;
  const long long nwarps = (static_cast<long long>(gridDim.x) * kLocalThreads) >> 5;
  const long long n_chunks = (p.n + kWarpTok - 1) / kWarpTok;
  LaneState& st = sh_state[threadIdx.x];
  st.s_abs = 0;
  st.s_k1 = 0;
  st.s_k3 = 0;
  st.seq_x = 0;
  st.bad_inv = 0;
  st.c_sat = 0;
  st.seq_nsat = 0;
  st.seq_t = 0;
  st.mx = 0.0;
  st.c_resp = st.c_trunc = st.c_rej = 0;

  const long long cpw = (n_chunks + nwarps - 1) / nwarps;
  const long long c_begin = warp_g * cpw;
  const long long c_end = c_begin + cpw < n_chunks ? c_begin + cpw : n_chunks;
  long long w_sid = 0, w_next = LLONG_MAX;  // warp-uniform sequence cursor
  if (kSeq && c_begin < c_end) {
    w_sid = seq_of(p.cu, p.n_seq, p.tok_begin + c_begin * kWarpTok);
    w_next = __ldg(p.cu + w_sid + 1);
  }
  st.sid = w_sid;  // the masked body's per-lane walk starts from the cursor
  st.next_b = w_next;

  if (blockIdx.x == 0 && threadIdx.x == 0) shard_range_check(p.cu, p.n_seq, p.tok_begin, p.n, st.bad_inv);

  FastAcc fa;
  fa.k1 = fa.k3 = fa.ab = fa.seq = fa.mx = 0.0;
  fa.resp = fa.trunc = fa.rej = fa.seq_t = 0;
  auto fold = [&]() {  // fp64 sums -> int128
    st.s_abs += __double2ll_rn(fa.ab);
    st.s_k1 += __double2ll_rn(fa.k1);
    st.s_k3 += __double2ll_rn(fa.k3);
    if (kSeq) st.seq_x += __double2ll_rn(fa.seq);
    fa.ab = fa.k1 = fa.k3 = fa.seq = 0.0;
  };
  auto pending = [&]() {  // this lane's unflushed sums of sequence st.sid
    SeqAcc a;
    a.sid = st.sid;
    a.x = st.seq_x + __double2ll_rn(fa.seq);
    a.t = st.seq_t + static_cast<long long>(fa.seq_t);
    a.nsat = st.seq_nsat;
    return a;
  };
  auto clear_pending = [&]() {
    st.seq_x = 0;
    st.seq_t = 0;
    st.seq_nsat = 0;
    fa.seq = 0.0;
    fa.seq_t = 0;
  };

  const long long n_vec = p.vec ? p.n / kWarpTok : 0;  // whole, vector-accessible chunks
  long long c_mid = c_end < n_vec ? c_end : n_vec;
  if (c_mid < c_begin) c_mid = c_begin;
  // per-lane cp.async ring: lane l copies (and later reads) only its own 4 tokens of each chunk,
  // so completion is per thread (commit / wait groups) -- no mbarrier, no warp synchronisation
  const uint32_t ring0 = smem_u32(&ring[wib][0][0][lane * kTpl]);
  const uint32_t resp0 = smem_u32(&ring_resp[wib][0][lane]);
  [[maybe_unused]] const uint64_t pol = policy_evict_first();
  const bool has_resp = p.resp != nullptr;
  auto issue = [&](int j, long long c) {  // chunk c into stage j (one commit group, possibly empty)
    if (c < c_mid) {
      const long long i = c * kWarpTok + lane * kTpl;
      const uint32_t dst = ring0 + j * (2 * kWarpTok * 4);
#if TIM_CORR_LOAD_HINT
      cp_async_16_hint(dst, p.num + i, pol);
      cp_async_16_hint(dst + kWarpTok * 4, p.den + i, pol);
#else
      cp_async_16(dst, p.num + i);
      cp_async_16(dst + kWarpTok * 4, p.den + i);
#endif
      if (has_resp) cp_async_4(resp0 + j * kWarpTok, p.resp + i);
    }
    cp_async_commit();
  };
  for (int j = 0; j < kStages; ++j) issue(j, c_begin + j);
  int cnt = 0, j = 0;
  for (long long c = c_begin; c < c_mid; ++c) {
    const long long i0 = c * kWarpTok + lane * kTpl;
    cp_async_wait<kStages - 1>();  // this lane's copies of chunk c have landed
    const float4 numv = *reinterpret_cast<const float4*>(&ring[wib][j][0][lane * kTpl]);
    const float4 denv = *reinterpret_cast<const float4*>(&ring[wib][j][1][lane * kTpl]);
    const uint32_t resp = has_resp ? ring_resp[wib][j][lane] : 0x01010101u;
    double dv[kTpl];
    dv[0] = __dsub_rn(static_cast<double>(numv.x), static_cast<double>(denv.x));
    dv[1] = __dsub_rn(static_cast<double>(numv.y), static_cast<double>(denv.y));
    dv[2] = __dsub_rn(static_cast<double>(numv.z), static_cast<double>(denv.z));
    dv[3] = __dsub_rn(static_cast<double>(numv.w), static_cast<double>(denv.w));
    issue(j, c + kStages);  // the lane has read stage j: refill it (its own slots only)
    if (++j == kStages) j = 0;
    const long long g0 = p.tok_begin + c * kWarpTok;
    bool fast = p.interior != 0;  // warp-uniform
    if (kSeq && fast) {
      if (g0 >= w_next) {  // the chunk starts past the cursor's sequence: flush it, advance
        SeqAcc a = pending();
        a.x = warp_sum_i128(a.x);
        a.t = warp_sum_i64(a.t);
        a.nsat = warp_sum_i64(a.nsat);
        if (lane == 0) flush_seq(p.seqp, a);
        clear_pending();
        while (g0 >= w_next && w_sid + 1 < p.n_seq) {  // skips empty sequences; bounded
          ++w_sid;
          w_next = __ldg(p.cu + w_sid + 1);
        }
        st.sid = w_sid;
        st.next_b = w_next;
      }
      fast = g0 + (kWarpTok - 1) < w_next;  // no boundary inside the chunk
    }
    const bool f_all = fast && __all_sync(0xffffffffu, resp == 0x01010101u);
    const bool f_none = fast && !f_all && __all_sync(0xffffffffu, resp == 0u);
    if (f_all || f_none) {
      fast_body<kOut, kSeqK, kTis, kTokRs>(p, st, fa, i0, f_all, dv);
    } else {
      const bool lane_whole = !(kSeq && p.tok_begin + i0 + (kTpl - 1) >= st.next_b);
      masked_body<kOut, kSeqK, kTis, kTokRs>(p, st, fa, resp, i0, true, lane_whole, dv);
      if (kSeq && p.interior) {  // back onto one cursor: lane 31 holds the furthest sequence
        const long long ms = __shfl_sync(0xffffffffu, st.sid, 31);
        if (__any_sync(0xffffffffu, st.sid != ms)) {
          seq_flush_segmented(p.seqp, pending(), lane);
          clear_pending();
        }
        w_sid = ms;
        w_next = __shfl_sync(0xffffffffu, st.next_b, 31);
        st.sid = w_sid;
        st.next_b = w_next;
      }
    }
    if (++cnt == kFoldChunks) {
      fold();
      cnt = 0;
    }
  }
  // unaligned arrays, or the partial last chunk: element-wise loads, the masked body
  for (long long ch = c_mid; ch < c_end; ++ch) {
    const long long i0 = ch * kWarpTok + lane * kTpl;
    const Chunk cc = load_chunk(p, i0);
    const bool full = p.vec && i0 + kTpl <= p.n;
    double dv[kTpl];
    dv[0] = __dsub_rn(static_cast<double>(cc.num.x), static_cast<double>(cc.den.x));
    dv[1] = __dsub_rn(static_cast<double>(cc.num.y), static_cast<double>(cc.den.y));
    dv[2] = __dsub_rn(static_cast<double>(cc.num.z), static_cast<double>(cc.den.z));
    dv[3] = __dsub_rn(static_cast<double>(cc.num.w), static_cast<double>(cc.den.w));
    const bool lane_whole = full && !(kSeq && p.tok_begin + i0 + (kTpl - 1) >= st.next_b);
    masked_body<kOut, kSeqK, kTis, kTokRs>(p, st, fa, cc.resp, i0, full, lane_whole, dv);
    fold();
  }
  fold();
  st.mx = fa.mx > st.mx ? fa.mx : st.mx;
  st.c_resp += fa.resp;
  st.c_trunc += fa.trunc;
  st.c_rej += fa.rej;
  st.seq_t += fa.seq_t;

  __int128 s_abs = st.s_abs, s_k1 = st.s_k1, s_k3 = st.s_k3;
  unsigned long long maxbits = static_cast<unsigned long long>(__double_as_longlong(st.mx));
  unsigned long long bad_inv = st.bad_inv;
  long long c_sat = st.c_sat;
  const unsigned c_resp_t = st.c_resp, c_trunc_t = st.c_trunc, c_rej_t = st.c_rej;

  if (kSeq) {
    SeqAcc acc;
    acc.sid = st.sid;
    acc.x = st.seq_x;
    acc.t = st.seq_t;
    acc.nsat = st.seq_nsat;
    seq_flush_segmented(p.seqp, acc, lane);
  }

  // block reduction of the global statistics, then one set of integer atomics per block
  __shared__ long long sh_cnt[4][kLocalThreads / 32];
  __shared__ long long sh_sum[6][kLocalThreads / 32];
  __shared__ unsigned long long sh_max[kLocalThreads / 32], sh_bad[kLocalThreads / 32];
  const int w = threadIdx.x >> 5;
  const long long n_resp = warp_sum_i64(static_cast<long long>(c_resp_t));
  const long long n_trunc = warp_sum_i64(static_cast<long long>(c_trunc_t));
  const long long n_rej = warp_sum_i64(static_cast<long long>(c_rej_t));
  c_sat = warp_sum_i64(c_sat);
  s_abs = warp_sum_i128(s_abs);
  s_k1 = warp_sum_i128(s_k1);
  s_k3 = warp_sum_i128(s_k3);
  maxbits = warp_max_u64(maxbits);
  bad_inv = warp_max_u64(bad_inv);
  if (lane == 0) {
    sh_cnt[0][w] = n_resp;
    sh_cnt[1][w] = n_trunc;
    sh_cnt[2][w] = n_rej;
    sh_cnt[3][w] = c_sat;
    sh_sum[0][w] = static_cast<long long>(static_cast<unsigned long long>(s_abs));
    sh_sum[1][w] = static_cast<long long>(s_abs >> 64);
    sh_sum[2][w] = static_cast<long long>(static_cast<unsigned long long>(s_k1));
    sh_sum[3][w] = static_cast<long long>(s_k1 >> 64);
    sh_sum[4][w] = static_cast<long long>(static_cast<unsigned long long>(s_k3));
    sh_sum[5][w] = static_cast<long long>(s_k3 >> 64);
    sh_max[w] = maxbits;
    sh_bad[w] = bad_inv;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    long long cnt[4] = {0, 0, 0, 0};
    __int128 sums[3] = {0, 0, 0};
    unsigned long long mxb = 0, bd = 0;
    for (int i = 0; i < kLocalThreads / 32; ++i) {
      for (int k = 0; k < 4; ++k) cnt[k] += sh_cnt[k][i];
      for (int k = 0; k < 3; ++k)
        sums[k] += (static_cast<__int128>(sh_sum[2 * k + 1][i]) << 64) |
                   static_cast<__int128>(static_cast<unsigned long long>(sh_sum[2 * k][i]));
      mxb = sh_max[i] > mxb ? sh_max[i] : mxb;
      bd = sh_bad[i] > bd ? sh_bad[i] : bd;
    }
    tim_partial_header* h = p.hdr;
    if (blockIdx.x == 0)
      atomicAdd(reinterpret_cast<unsigned long long*>(&h->n_tok), static_cast<unsigned long long>(p.n));
    if (cnt[0]) atomicAdd(reinterpret_cast<unsigned long long*>(&h->n_resp_tok), static_cast<unsigned long long>(cnt[0]));
    if (cnt[1]) atomicAdd(reinterpret_cast<unsigned long long*>(&h->n_truncated), static_cast<unsigned long long>(cnt[1]));
    if (cnt[2]) atomicAdd(reinterpret_cast<unsigned long long*>(&h->n_tok_rejected), static_cast<unsigned long long>(cnt[2]));
    if (cnt[3]) atomicAdd(reinterpret_cast<unsigned long long*>(&h->n_saturated), static_cast<unsigned long long>(cnt[3]));
    atomic_add_i128(h->sum_abs_delta, sums[0]);
    atomic_add_i128(h->sum_k1, sums[1]);
    atomic_add_i128(h->sum_k3, sums[2]);
    if (mxb) atomicMax(reinterpret_cast<unsigned long long*>(&h->max_abs_delta_bits), mxb);
    if (bd) atomicMax(reinterpret_cast<unsigned long long*>(&h->reserved[0]), bd);
  }
  // status commit by the last block (ticket in hdr->reserved[1], bad index in reserved[0])
  commit_status_last_block(reinterpret_cast<WsHeader*>(&p.hdr->reserved[0]), p.dstatus);
}

template <bool kOut, int kSeqK, bool kTis, bool kTokRs>
__global__ void __launch_bounds__(kLocalThreads, TIM_CORR_MINB) correct_local_kernel(LocalParams p) {
  pass1_body<kOut, kSeqK, kTis, kTokRs>(p);
}

constexpr int kFinishThreads = 1024;

// a7 + a8 on the gathered partial blocks: one thread per sequence (grid-stride), the last block
// to finish (ticket in p.scratch) writes the statistics.
__device__ __forceinline__ void finish_body(const FinishParams& p) {
  const CorrectDevCfg cfg = p.cfg;
  __shared__ int sh_rej[kFinishThreads / 32];
  int rej = 0;
  constexpr int kU = 4;  // sequences per thread per round: their partial loads are issued together
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  for (long long s0 = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; s0 < p.n_seq; s0 += kU * stride) {
    __int128 X[kU];
    long long T[kU], nsat[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const long long s = s0 + u * stride;
      X[u] = 0;
      T[u] = nsat[u] = 0;
      if (s >= p.n_seq) continue;
      for (int r = 0; r < p.nranks; ++r) {  // fixed rank order (exact anyway)
        const tim_seq_partial* sp = reinterpret_cast<const tim_seq_partial*>(
            p.gathered + r * p.block_bytes + sizeof(tim_partial_header)) + s;
        const longlong2 xv = *reinterpret_cast<const longlong2*>(sp);       // {x_lo, x_hi}
        const longlong2 tv = *(reinterpret_cast<const longlong2*>(sp) + 1);  // {n_tok, n_sat}
        X[u] += (static_cast<__int128>(xv.y) << 64) | static_cast<__int128>(static_cast<unsigned long long>(xv.x));
        T[u] += tv.x;
        nsat[u] += tv.y;
      }
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const long long s = s0 + u * stride;
      if (s >= p.n_seq) continue;
      uint8_t keep = 1;
      double score = 0.0;
      if (cfg.seq_rs != TIM_SEQ_NONE) {
        score = __dmul_rn(i128_to_double(X[u]), 0x1p-52);
        if (cfg.seq_agg == TIM_AGG_MEAN) score = T[u] > 0 ? __ddiv_rn(score, static_cast<double>(T[u])) : 0.0;
        keep = seq_keep_decision(cfg.tau_seq, cfg.seq_agg, X[u], T[u], nsat[u]) ? 1 : 0;
      }
      rej += keep ? 0 : 1;
      if (p.seq_keep) p.seq_keep[s] = keep;
      if (p.seq_score) p.seq_score[s] = score;
    }
  }
  for (int off = 16; off > 0; off >>= 1) rej += __shfl_down_sync(0xffffffffu, rej, off);
  if ((threadIdx.x & 31) == 0) sh_rej[threadIdx.x >> 5] = rej;
  __syncthreads();
  // several blocks (p.scratch = {ticket, rejections}, zeroed): the last block to finish writes the stats
  __shared__ int last;
  long long n_rej = 0;
  if (threadIdx.x == 0) {
    for (int i = 0; i < static_cast<int>(blockDim.x) / 32; ++i) n_rej += sh_rej[i];
    last = 1;
    if (gridDim.x > 1) {
      atomicAdd(&p.scratch[1], static_cast<unsigned long long>(n_rej));
      __threadfence();
      last = atomicAdd(&p.scratch[0], 1ull) == gridDim.x - 1;
      if (last) n_rej = static_cast<long long>(atomicAdd(&p.scratch[1], 0ull));
    }
  }
  __syncthreads();
  if (threadIdx.x == 0 && last && p.stats) {
    long long cnt[5] = {0, 0, 0, 0, 0};
    __int128 sums[3] = {0, 0, 0};
    unsigned long long mx = 0;
    for (int r = 0; r < p.nranks; ++r) {
      const tim_partial_header* h = reinterpret_cast<const tim_partial_header*>(p.gathered + r * p.block_bytes);
      cnt[0] += h->n_tok;
      cnt[1] += h->n_resp_tok;
      cnt[2] += h->n_truncated;
      cnt[3] += h->n_tok_rejected;
      cnt[4] += h->n_saturated;
      sums[0] += ld_i128(h->sum_abs_delta);
      sums[1] += ld_i128(h->sum_k1);
      sums[2] += ld_i128(h->sum_k3);
      mx = h->max_abs_delta_bits > mx ? h->max_abs_delta_bits : mx;
    }
    tim_stats* st = p.stats;
    st->n_tok = cnt[0];
    st->n_resp_tok = cnt[1];
    st->n_seq = p.n_seq;
    st->n_truncated = cnt[2];
    st->n_tok_rejected = cnt[3];
    st->n_seq_rejected = n_rej;
    st->n_saturated = cnt[4];
    st->sum_abs_delta_fx[0] = static_cast<int64_t>(static_cast<unsigned long long>(sums[0]));
    st->sum_abs_delta_fx[1] = static_cast<int64_t>(sums[0] >> 64);
    st->sum_k1_fx[0] = static_cast<int64_t>(static_cast<unsigned long long>(sums[1]));
    st->sum_k1_fx[1] = static_cast<int64_t>(sums[1] >> 64);
    st->sum_k3_fx[0] = static_cast<int64_t>(static_cast<unsigned long long>(sums[2]));
    st->sum_k3_fx[1] = static_cast<int64_t>(sums[2] >> 64);
    st->max_abs_delta = __longlong_as_double(static_cast<long long>(mx));
    st->mean_abs_delta = 0.0;
    st->mean_k1 = 0.0;
    st->mean_k3 = 0.0;
  }
}

__global__ void __launch_bounds__(kFinishThreads) correct_finish_kernel(FinishParams p) { finish_body(p); }

// Zero the coefficient of this rank's tokens that belong to rejected sequences (one block per
// sequence, grid-stride; 16-B stores between the scalar head and tail).
__device__ __forceinline__ void zero_body(const ZeroParams& p) {
  const long long te = p.tok_begin + p.n;
  for (long long s = blockIdx.x; s < p.n_seq; s += gridDim.x) {
    if (p.seq_keep[s]) continue;
    const long long c0 = p.cu[s], c1 = p.cu[s + 1], tb = p.tok_begin;
    const long long a = (c0 > tb ? c0 : tb) - tb;  // local token range [a, b)
    const long long b = (c1 < te ? c1 : te) - tb;
    if (a >= b) continue;
    float* c = p.coeff;
    long long va = (a + 3) & ~3ll, vb = b & ~3ll;  // float4-aligned middle when coeff is 16-B aligned
    if (va > vb || (reinterpret_cast<uintptr_t>(c) & 15u) != 0) va = vb = b;
    for (long long i = a + threadIdx.x; i < va; i += blockDim.x) c[i] = 0.f;
    for (long long i = vb + threadIdx.x; i < b; i += blockDim.x) c[i] = 0.f;
    for (long long i = va + 4 * threadIdx.x; i < vb; i += 4 * blockDim.x) {
#if TIM_ZERO_PLAIN_STORES
      *reinterpret_cast<float4*>(c + i) = make_float4(0.f, 0.f, 0.f, 0.f);
#else
      __stcs(reinterpret_cast<float4*>(c + i), make_float4(0.f, 0.f, 0.f, 0.f));
#endif
    }
  }
}

__global__ void __launch_bounds__(256) correct_zero_kernel(ZeroParams p) { zero_body(p); }

// Grid-wide barrier of a co-resident (cooperative) grid: one counter, zeroed before the launch,
// reaches `round` x gridDim.x after the `round`-th barrier.
__device__ __forceinline__ void grid_barrier(unsigned int* counter, unsigned int round) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(counter, 1u);
    const unsigned int target = round * gridDim.x;
    while (atomicAdd(counter, 0u) < target) __nanosleep(64);
    __threadfence();
  }
  __syncthreads();
}

// a5 -> a7 -> a8 in ONE launch when P = 1 (SURVEY.md §8(a) a7 "fused into pass 1 when P = 1"):
// pass 1, a grid barrier, the sequence decisions and statistics on the local partial block, a
// second barrier, the coefficient zeroing of rejected sequences.  Launched cooperatively (every
// block resident), so the barriers cannot deadlock; the counter is WsHeader::pad of the local
// block's header (zeroed with the block).
template <bool kOut, int kSeqK, bool kTis, bool kTokRs>
__global__ void __launch_bounds__(kLocalThreads, TIM_CORR_MINB) correct_fused_kernel(LocalParams p, FinishParams f,
                                                                                      ZeroParams z) {
  pass1_body<kOut, kSeqK, kTis, kTokRs>(p);
  unsigned int* bar = &reinterpret_cast<WsHeader*>(&p.hdr->reserved[0])->pad;
  grid_barrier(bar, 1u);
  finish_body(f);
  if (kSeqK != TIM_SEQ_NONE && kOut) {
    grid_barrier(bar, 2u);
    // every warp zeroes the rejected tokens of the token range it ran pass 1 on (balanced over
    // the whole grid), walking the sequences that overlap it
    const int lane = threadIdx.x & 31;
    const long long warp_g = (static_cast<long long>(blockIdx.x) * kLocalThreads + threadIdx.x) >> 5;
    const long long nwarps = (static_cast<long long>(gridDim.x) * kLocalThreads) >> 5;
    const long long n_chunks = (p.n + kWarpTok - 1) / kWarpTok;
    const long long cpw = (n_chunks + nwarps - 1) / nwarps;
    const long long t0 = warp_g * cpw * kWarpTok;
    long long t1 = t0 + cpw * kWarpTok;
    if (t1 > p.n) t1 = p.n;
    if (t0 >= t1) return;
    const long long tb = p.tok_begin;
    long long g = tb + t0;
    long long sq = seq_of(p.cu, p.n_seq, g);
    float* c = p.coeff;
    while (g < tb + t1) {
      const long long sb = __ldg(p.cu + sq), se = __ldg(p.cu + sq + 1);
      const long long a = (g > sb ? g : sb) - tb;
      const long long b = (se < tb + t1 ? se : tb + t1) - tb;
      if (a < b && !z.seq_keep[sq]) {
        long long va = (a + 3) & ~3ll, vb = b & ~3ll;  // coeff is 16-B aligned (tim_correct checks)
        if (va > vb) va = vb = b;
        for (long long i = a + lane; i < va; i += 32) c[i] = 0.f;
        for (long long i = vb + lane; i < b; i += 32) c[i] = 0.f;
        for (long long i = va + 4 * lane; i < vb; i += 128)
          __stcs(reinterpret_cast<float4*>(c + i), make_float4(0.f, 0.f, 0.f, 0.f));
      }
      if (sq + 1 >= p.n_seq) break;
      g = g > se ? g : se;
      ++sq;
    }
  }
}

cudaError_t launch_correct_local(const LocalParams& p_in, int num_sms, cudaStream_t stream) {
  LocalParams p = p_in;
  {  // interior: |delta| <= 2^-6 is never truncated (e^(2^-6) < 1.0158 <= tau) nor token-rejected
    const CorrectDevCfg& c = p.cfg;
    p.interior = (!c.tis || (c.log_tis_cap > kSmall && c.tis_cap >= 1.0158)) &&
                 (!c.tok_rs || (c.log_lo <= -kSmall && c.log_hi >= kSmall));
  }
  const long long chunks = (p.n + kWarpTok - 1) / kWarpTok;
  const long long warps_per_block = kLocalThreads / 32;
  long long blocks = (chunks + warps_per_block - 1) / warps_per_block;
  const long long cap = static_cast<long long>(num_sms) * TIM_CORR_MINB;  // one resident wave
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  const bool out = p.tis_w != nullptr;
  const int sk = p.cfg.seq_rs;
  const int v = (out ? 8 : 0) | (p.cfg.tis ? 2 : 0) | (p.cfg.tok_rs ? 1 : 0);
#define TIM_CORR_CASE(o, t, r)                                                                   \
  case (o ? 8 : 0) | (t ? 2 : 0) | (r ? 1 : 0):                                                  \
    if (sk == TIM_SEQ_K1)                                                                        \
      correct_local_kernel<o, TIM_SEQ_K1, t, r><<<blocks, kLocalThreads, 0, stream>>>(p);        \
    else if (sk == TIM_SEQ_K3)                                                                   \
      correct_local_kernel<o, TIM_SEQ_K3, t, r><<<blocks, kLocalThreads, 0, stream>>>(p);        \
    else                                                                                         \
      correct_local_kernel<o, TIM_SEQ_NONE, t, r><<<blocks, kLocalThreads, 0, stream>>>(p);      \
    break;
  switch (v) {
    TIM_CORR_CASE(true, true, true) TIM_CORR_CASE(true, true, false)
    TIM_CORR_CASE(true, false, true) TIM_CORR_CASE(true, false, false)
    TIM_CORR_CASE(false, true, true) TIM_CORR_CASE(false, true, false)
    TIM_CORR_CASE(false, false, true) TIM_CORR_CASE(false, false, false)
  }
#undef TIM_CORR_CASE
  return cudaGetLastError();
}

template <bool kOut, int kSeqK, bool kTis, bool kTokRs>
static cudaError_t launch_fused_t(const LocalParams& p, const FinishParams& f, const ZeroParams& z, int num_sms,
                                  cudaStream_t stream) {
  auto kern = correct_fused_kernel<kOut, kSeqK, kTis, kTokRs>;
  int per_sm = 0;  // co-resident blocks per SM (the launch fails rather than deadlock if this lies)
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kLocalThreads, 0);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) return cudaErrorLaunchOutOfResources;
  const long long chunks = (p.n + kWarpTok - 1) / kWarpTok;
  long long blocks = (chunks + kLocalWarps - 1) / kLocalWarps;
  const long long cap = static_cast<long long>(num_sms) * per_sm;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  LocalParams pp = p;
  FinishParams ff = f;
  ZeroParams zz = z;
  void* args[] = {&pp, &ff, &zz};
  return cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(kern), dim3(static_cast<unsigned>(blocks)),
                                     dim3(kLocalThreads), args, 0, stream);
}

cudaError_t launch_correct_fused(const LocalParams& p_in, const FinishParams& f, const ZeroParams& z, int num_sms,
                                 cudaStream_t stream) {
  LocalParams p = p_in;
  {
    const CorrectDevCfg& c = p.cfg;
    p.interior = (!c.tis || (c.log_tis_cap > kSmall && c.tis_cap >= 1.0158)) &&
                 (!c.tok_rs || (c.log_lo <= -kSmall && c.log_hi >= kSmall));
  }
  const bool out = p.tis_w != nullptr;
  const int sk = p.cfg.seq_rs;
  const int v = (out ? 8 : 0) | (p.cfg.tis ? 2 : 0) | (p.cfg.tok_rs ? 1 : 0);
#define TIM_FUSED_CASE(o, t, r)                                                                        \
  case (o ? 8 : 0) | (t ? 2 : 0) | (r ? 1 : 0):                                                        \
    if (sk == TIM_SEQ_K1) return launch_fused_t<o, TIM_SEQ_K1, t, r>(p, f, z, num_sms, stream);         \
    if (sk == TIM_SEQ_K3) return launch_fused_t<o, TIM_SEQ_K3, t, r>(p, f, z, num_sms, stream);         \
    return launch_fused_t<o, TIM_SEQ_NONE, t, r>(p, f, z, num_sms, stream);
  switch (v) {
    TIM_FUSED_CASE(true, true, true) TIM_FUSED_CASE(true, true, false)
    TIM_FUSED_CASE(true, false, true) TIM_FUSED_CASE(true, false, false)
    TIM_FUSED_CASE(false, true, true) TIM_FUSED_CASE(false, true, false)
    TIM_FUSED_CASE(false, false, true) TIM_FUSED_CASE(false, false, false)
  }
#undef TIM_FUSED_CASE
  return cudaErrorInvalidValue;
}

cudaError_t launch_correct_finish(const FinishParams& p, int num_sms, cudaStream_t stream) {
  if (p.scratch == nullptr) {  // no zeroed scratch: one block
    correct_finish_kernel<<<1, kFinishThreads, 0, stream>>>(p);
  } else {
    long long blocks = (p.n_seq + 255) / 256;
    if (blocks > num_sms) blocks = num_sms;
    if (blocks < 1) blocks = 1;
    correct_finish_kernel<<<static_cast<int>(blocks), 256, 0, stream>>>(p);
  }
  return cudaGetLastError();
}

cudaError_t launch_correct_zero(const ZeroParams& p, cudaStream_t stream) {
  long long blocks = p.n_seq < 4096 ? p.n_seq : 4096;
  if (blocks < 1) return cudaSuccess;
  correct_zero_kernel<<<static_cast<int>(blocks), 256, 0, stream>>>(p);
  return cudaGetLastError();
}

}  // namespace tim
