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
#include "tim_internal.h"

namespace tim {

#ifndef TIM_CORR_MINB
#define TIM_CORR_MINB 3
#endif
constexpr int kTpl = 4;                 // tokens per lane (one float4 of num / den, one u32 of resp)
constexpr int kWarpTok = 32 * kTpl;     // tokens per warp chunk
constexpr int kLocalThreads = 256;
constexpr int kFlushChunks = 4096;      // fast-path int64 sums are folded into int128 this often

// Per-thread rarely-touched state (int128 sums of the slow path, data errors), in shared memory
// so the hot loop keeps its registers for the loads in flight and the Horner chains.
struct SlowAcc {
  __int128 s_abs, s_k1, s_k3, seq_x;
  unsigned long long bad_inv;
  long long c_sat, seq_nsat;
  long long pad;
};

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

// Pass 1 (a5).  Every warp owns a contiguous run of 128-token chunks (4 tokens per lane, the
// next chunk's loads in flight while the current one computes).  Fast path, all lanes in
// lockstep: tokens with |delta| <= 2^-6 (finite by construction) use the short contract
// polynomials; their K values cannot saturate (|K| <= 2^-6), so they accumulate in int64
// (|X| <= 2^46, folded into int128 every kFlushChunks chunks).  Slow path, per lane and rare:
// larger or non-finite delta, a partial chunk, or a sequence boundary inside the lane's four
// tokens -- the full per-token contract with int128 sums and the sequence walk.
template <bool kOut, bool kSeq, bool kTis, bool kTokRs>
__global__ void __launch_bounds__(kLocalThreads, TIM_CORR_MINB) correct_local_kernel(LocalParams p) {
  __shared__ SlowAcc sh_slow[kLocalThreads];
  const int lane = threadIdx.x & 31;
  const long long warp_g = (static_cast<long long>(blockIdx.x) * kLocalThreads + threadIdx.x) >> 5;
  const long long nwarps = (static_cast<long long>(gridDim.x) * kLocalThreads) >> 5;
  const long long n_chunks = (p.n + kWarpTok - 1) / kWarpTok;
  const CorrectDevCfg cfg = p.cfg;
  SlowAcc& sa = sh_slow[threadIdx.x];
  sa.s_abs = 0;
  sa.s_k1 = 0;
  sa.s_k3 = 0;
  sa.seq_x = 0;
  sa.bad_inv = 0;
  sa.c_sat = 0;
  sa.seq_nsat = 0;

  unsigned c_resp = 0, c_trunc = 0, c_rej = 0;
  long long f_abs = 0, f_k1 = 0, f_k3 = 0, f_seq = 0;  // fast-path exact sums
  double mx = 0.0;                                     // max |delta| (finite response tokens)
  long long seq_t = 0;

  const long long cpw = (n_chunks + nwarps - 1) / nwarps;
  const long long c_begin = warp_g * cpw;
  const long long c_end = c_begin + cpw < n_chunks ? c_begin + cpw : n_chunks;
  long long sid = LLONG_MAX, next_b = LLONG_MAX;
  if (kSeq && c_begin < c_end && c_begin * kWarpTok + lane * kTpl < p.n) {
    sid = seq_of(p.cu, p.n_seq, p.tok_begin + c_begin * kWarpTok + lane * kTpl);
    next_b = __ldg(p.cu + sid + 1);
  }
  const bool seq_k1 = cfg.seq_rs == TIM_SEQ_K1;
  const float cap_f = __double2float_rn(cfg.tis_cap);

  Chunk nxt;
  if (c_begin < c_end) nxt = load_chunk(p, c_begin * kWarpTok + lane * kTpl);
  for (long long ch = c_begin; ch < c_end; ++ch) {
    const long long i0 = ch * kWarpTok + lane * kTpl;
    const Chunk cur = nxt;
    if (ch + 1 < c_end) nxt = load_chunk(p, i0 + kWarpTok);
    const float num[4] = {cur.num.x, cur.num.y, cur.num.z, cur.num.w};
    const float den[4] = {cur.den.x, cur.den.y, cur.den.z, cur.den.w};

    double dv[kTpl], ds[kTpl], k3s[kTpl];
    const bool full = p.vec && i0 + kTpl <= p.n;
    unsigned slow = full ? 0u : 0xFu;
    if (kSeq && p.tok_begin + i0 + (kTpl - 1) >= next_b) slow = 0xFu;
#pragma unroll
    for (int k = 0; k < kTpl; ++k) {
      dv[k] = __dsub_rn(static_cast<double>(num[k]), static_cast<double>(den[k]));
      const bool sm = fabs(dv[k]) <= kSmall;  // false for NaN / inf
      if (!sm) slow |= 1u << k;
      ds[k] = sm ? dv[k] : 0.0;
    }
    // short K3 series of the four tokens in lockstep (independent Horner chains)
    double q[kTpl];
#pragma unroll
    for (int k = 0; k < kTpl; ++k) q[k] = kInvFact[9];
#pragma unroll
    for (int n = 8; n >= 2; --n)
#pragma unroll
      for (int k = 0; k < kTpl; ++k) q[k] = __dadd_rn(__dmul_rn(q[k], ds[k]), kInvFact[n]);
#pragma unroll
    for (int k = 0; k < kTpl; ++k) k3s[k] = __dmul_rn(__dmul_rn(ds[k], ds[k]), q[k]);

    float w_out[kTpl], c_out[kTpl];
    uint32_t kbits = 0;
    // this chunk's exact sums in fp64: every X is an integer with |X| <= 2^46, so the sums of
    // four are exact doubles; one conversion per sum per chunk
    double ck1 = 0.0, ck3 = 0.0, cabs = 0.0, cseq = 0.0, cmx = 0.0;
    unsigned cn = 0, ctr = 0, crj = 0, cst = 0;
#pragma unroll
    for (int k = 0; k < kTpl; ++k) {
      const double d = ds[k];
      const bool resp = (cur.resp >> (8 * k)) & 0xffu;
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
      const double dz = use ? d : 0.0;  // unused tokens contribute exactly 0 to every sum
      const double kz = use ? k3s[k] : 0.0;
      const double x1 = rint(__dmul_rn(-dz, kTwo52));  // exact scaling, then round to integer
      const double x3 = rint(__dmul_rn(kz, kTwo52));
      ck1 = __dadd_rn(ck1, x1);
      ck3 = __dadd_rn(ck3, x3);
      cabs = __dadd_rn(cabs, fabs(x1));
      const double ad = fabs(dz);
      cmx = ad > cmx ? ad : cmx;
      cn += use ? 1u : 0u;
      if (kTis) ctr += (use && trunc) ? 1u : 0u;
      if (kTokRs) crj += (use && !keep) ? 1u : 0u;
      if (kSeq) {
        if (kTokRs) cseq = __dadd_rn(cseq, keep ? (seq_k1 ? x1 : x3) : 0.0);
        cst += (use && keep) ? 1u : 0u;
      }
    }
    const long long ik1 = __double2ll_rn(ck1), ik3 = __double2ll_rn(ck3);
    f_k1 += ik1;
    f_k3 += ik3;
    f_abs += __double2ll_rn(cabs);
    mx = cmx > mx ? cmx : mx;
    c_resp += cn;
    c_trunc += ctr;
    c_rej += crj;
    if (kSeq) {
      f_seq += kTokRs ? __double2ll_rn(cseq) : (seq_k1 ? ik1 : ik3);
      seq_t += cst;
    }

    if (slow) {  // rare: the full contract per token, in the slow tokens' lanes only
#pragma unroll
      for (int k = 0; k < kTpl; ++k) {
        if (!((slow >> k) & 1u)) continue;
        const long long i = i0 + k;
        if (i >= p.n) continue;
        const long long g = p.tok_begin + i;
        const double d = dv[k];
        if (kSeq) {
          while (g >= next_b) {  // crossed into a later sequence (skips empty ones)
            SeqAcc a;
            a.sid = sid;
            a.x = sa.seq_x + static_cast<__int128>(f_seq);
            a.t = seq_t;
            a.nsat = sa.seq_nsat;
            flush_seq(p.seqp, a);
            sa.seq_x = 0;
            sa.seq_nsat = 0;
            f_seq = 0;
            seq_t = 0;
            sid += 1;
            next_b = __ldg(p.cu + sid + 1);
          }
        }
        if (!isfinite(d)) {  // C.3.2 data error: excluded from every sum, outputs NaN / 0
          const unsigned long long b = kBadSentinel - static_cast<unsigned long long>(g);
          sa.bad_inv = b > sa.bad_inv ? b : sa.bad_inv;
          w_out[k] = CUDART_NAN_F;
          c_out[k] = 0.f;
          kbits &= ~(0xffu << (8 * k));
          continue;
        }
        const bool resp = (cur.resp >> (8 * k)) & 0xffu;
        const bool sm = fabs(d) <= kSmall;
        const double k3 = sm ? k3s[k] : k3_c(d);
        const bool trunc = kTis && d > cfg.log_tis_cap;
        if (kTis) {
          const double e = sm ? exp_from_k3_small(d, k3) : exp_c(d);
          w_out[k] = __double2float_rn(trunc ? cfg.tis_cap : fmin(e, cfg.tis_cap));
        }
        const bool keep = kTokRs ? (cfg.log_lo <= d && d <= cfg.log_hi) : true;
        c_out[k] = (resp && keep) ? w_out[k] : 0.f;
        kbits = (kbits & ~(0xffu << (8 * k))) | (static_cast<uint32_t>(keep) << (8 * k));
        if (!resp) continue;
        bool sat1, sat3;
        const long long x1 = fixed_point(-d, sat1);
        const long long x3 = fixed_point(k3, sat3);
        c_resp += 1;
        c_trunc += trunc ? 1u : 0u;
        c_rej += keep ? 0u : 1u;
        sa.s_abs += x1 < 0 ? -x1 : x1;  // rint is odd-symmetric: X(|delta|) = |X(-delta)|
        sa.s_k1 += x1;
        sa.s_k3 += x3;
        mx = fmax(mx, fabs(d));
        if (kSeq && keep) {
          const bool satq = seq_k1 ? sat1 : sat3;
          sa.seq_x += seq_k1 ? x1 : x3;
          seq_t += 1;
          sa.seq_nsat += satq ? 1 : 0;
          sa.c_sat += satq ? 1 : 0;
        }
      }
    }

    if (kOut) {
      if (full) {
        __stcs(reinterpret_cast<float4*>(p.tis_w + i0), make_float4(w_out[0], w_out[1], w_out[2], w_out[3]));
        __stcs(reinterpret_cast<float4*>(p.coeff + i0), make_float4(c_out[0], c_out[1], c_out[2], c_out[3]));
        __stcs(reinterpret_cast<unsigned int*>(p.tok_keep + i0), kbits);
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
    if (((ch - c_begin) & (kFlushChunks - 1)) == kFlushChunks - 1) {
      sa.s_abs += f_abs;
      sa.s_k1 += f_k1;
      sa.s_k3 += f_k3;
      sa.seq_x += f_seq;
      f_abs = f_k1 = f_k3 = f_seq = 0;
    }
  }

  __int128 s_abs = sa.s_abs + f_abs, s_k1 = sa.s_k1 + f_k1, s_k3 = sa.s_k3 + f_k3;
  unsigned long long maxbits = static_cast<unsigned long long>(__double_as_longlong(mx));
  unsigned long long bad_inv = sa.bad_inv;
  long long c_sat = sa.c_sat;

  if (kSeq) {
    SeqAcc acc;
    acc.sid = sid;
    acc.x = sa.seq_x + static_cast<__int128>(f_seq);
    acc.t = seq_t;
    acc.nsat = sa.seq_nsat;
    // segmented warp reduction of the open segments (sequence ids are non-decreasing in lane order)
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
    if (head && acc.sid != LLONG_MAX) flush_seq(p.seqp, acc);
  }

  // block reduction of the global statistics, then one set of integer atomics per block
  __shared__ long long sh_cnt[4][kLocalThreads / 32];
  __shared__ long long sh_sum[6][kLocalThreads / 32];
  __shared__ unsigned long long sh_max[kLocalThreads / 32], sh_bad[kLocalThreads / 32];
  const int w = threadIdx.x >> 5;
  const long long n_resp = warp_sum_i64(static_cast<long long>(c_resp));
  const long long n_trunc = warp_sum_i64(static_cast<long long>(c_trunc));
  const long long n_rej = warp_sum_i64(static_cast<long long>(c_rej));
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

constexpr int kFinishThreads = 1024;

__global__ void __launch_bounds__(kFinishThreads) correct_finish_kernel(FinishParams p) {
  const CorrectDevCfg cfg = p.cfg;
  __shared__ int sh_rej[kFinishThreads / 32];
  int rej = 0;
  for (long long s = threadIdx.x; s < p.n_seq; s += blockDim.x) {
    __int128 X = 0;
    long long T = 0, nsat = 0;
    for (int r = 0; r < p.nranks; ++r) {  // fixed rank order (exact anyway)
      const tim_seq_partial* sp = reinterpret_cast<const tim_seq_partial*>(
          p.gathered + r * p.block_bytes + sizeof(tim_partial_header)) + s;
      X += ld_i128(&sp->x_lo);
      T += sp->n_tok;
      nsat += sp->n_sat;
    }
    uint8_t keep = 1;
    double score = 0.0;
    if (cfg.seq_rs != TIM_SEQ_NONE) {
      score = __dmul_rn(i128_to_double(X), 0x1p-52);
      if (cfg.seq_agg == TIM_AGG_MEAN) score = T > 0 ? __ddiv_rn(score, static_cast<double>(T)) : 0.0;
      if (T == 0) keep = 1;
      else if (nsat > 0) keep = 0;
      else keep = X <= seq_threshold(cfg.tau_seq, cfg.seq_agg == TIM_AGG_MEAN ? T : 1) ? 1 : 0;
    }
    rej += keep ? 0 : 1;
    if (p.seq_keep) p.seq_keep[s] = keep;
    if (p.seq_score) p.seq_score[s] = score;
  }
  for (int off = 16; off > 0; off >>= 1) rej += __shfl_down_sync(0xffffffffu, rej, off);
  if ((threadIdx.x & 31) == 0) sh_rej[threadIdx.x >> 5] = rej;
  __syncthreads();
  if (threadIdx.x == 0 && p.stats) {
    long long n_rej = 0;
    for (int i = 0; i < kFinishThreads / 32; ++i) n_rej += sh_rej[i];
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

// Zero the coefficient of this rank's tokens that belong to rejected sequences.
__global__ void __launch_bounds__(256) correct_zero_kernel(ZeroParams p) {
  const long long te = p.tok_begin + p.n;
  for (long long s = blockIdx.x; s < p.n_seq; s += gridDim.x) {
    if (p.seq_keep[s]) continue;
    const long long c0 = p.cu[s], c1 = p.cu[s + 1], tb = p.tok_begin;
    const long long a = c0 > tb ? c0 : tb;
    const long long b = c1 < te ? c1 : te;
    for (long long g = a + threadIdx.x; g < b; g += blockDim.x) p.coeff[g - p.tok_begin] = 0.f;
  }
}

cudaError_t launch_correct_local(const LocalParams& p, int num_sms, cudaStream_t stream) {
  const long long chunks = (p.n + kWarpTok - 1) / kWarpTok;
  const long long warps_per_block = kLocalThreads / 32;
  long long blocks = (chunks + warps_per_block - 1) / warps_per_block;
  const long long cap = static_cast<long long>(num_sms) * TIM_CORR_MINB;  // one resident wave
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  const bool out = p.tis_w != nullptr;
  const bool seq = p.cfg.seq_rs != TIM_SEQ_NONE;
  const int v = (out ? 8 : 0) | (seq ? 4 : 0) | (p.cfg.tis ? 2 : 0) | (p.cfg.tok_rs ? 1 : 0);
  switch (v) {
#define TIM_CORR_CASE(o, s, t, r) \
  case (o ? 8 : 0) | (s ? 4 : 0) | (t ? 2 : 0) | (r ? 1 : 0): \
    correct_local_kernel<o, s, t, r><<<blocks, kLocalThreads, 0, stream>>>(p); break;
    TIM_CORR_CASE(true, true, true, true) TIM_CORR_CASE(true, true, true, false)
    TIM_CORR_CASE(true, true, false, true) TIM_CORR_CASE(true, true, false, false)
    TIM_CORR_CASE(true, false, true, true) TIM_CORR_CASE(true, false, true, false)
    TIM_CORR_CASE(true, false, false, true) TIM_CORR_CASE(true, false, false, false)
    TIM_CORR_CASE(false, true, true, true) TIM_CORR_CASE(false, true, true, false)
    TIM_CORR_CASE(false, true, false, true) TIM_CORR_CASE(false, true, false, false)
    TIM_CORR_CASE(false, false, true, true) TIM_CORR_CASE(false, false, true, false)
    TIM_CORR_CASE(false, false, false, true) TIM_CORR_CASE(false, false, false, false)
#undef TIM_CORR_CASE
  }
  return cudaGetLastError();
}

cudaError_t launch_correct_finish(const FinishParams& p, cudaStream_t stream) {
  correct_finish_kernel<<<1, kFinishThreads, 0, stream>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_correct_zero(const ZeroParams& p, cudaStream_t stream) {
  long long blocks = p.n_seq < 4096 ? p.n_seq : 4096;
  if (blocks < 1) return cudaSuccess;
  correct_zero_kernel<<<static_cast<int>(blocks), 256, 0, stream>>>(p);
  return cudaGetLastError();
}

}  // namespace tim
