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
// Layout: structure-of-arrays fp32 / u8 token vectors, one warp owns 256 consecutive tokens
// (8 per lane, 32-B vector loads), so every load and store is fully coalesced.
#include <cuda_runtime.h>
#include <math_constants.h>

#include <cstdint>

#include "contract.cuh"
#include "tim_internal.h"

namespace tim {

#ifndef TIM_CORR_TPL
#define TIM_CORR_TPL 4
#endif
#ifndef TIM_CORR_MINB
#define TIM_CORR_MINB 3
#endif
constexpr int kTpl = TIM_CORR_TPL;      // tokens per lane
constexpr int kWarpTok = 32 * kTpl;     // tokens per warp chunk
constexpr int kLocalThreads = 256;

template <bool kOut, bool kSeq>
__global__ void __launch_bounds__(kLocalThreads, TIM_CORR_MINB) correct_local_kernel(LocalParams p) {
  const int lane = threadIdx.x & 31;
  const long long warp_g = (static_cast<long long>(blockIdx.x) * kLocalThreads + threadIdx.x) >> 5;
  const long long nwarps = (static_cast<long long>(gridDim.x) * kLocalThreads) >> 5;
  const long long n_chunks = (p.n + kWarpTok - 1) / kWarpTok;
  const CorrectDevCfg cfg = p.cfg;

  long long c_resp = 0, c_trunc = 0, c_rej = 0, c_sat = 0;
  __int128 s_abs = 0, s_k1 = 0, s_k3 = 0;
  unsigned long long maxbits = 0;
  unsigned long long bad_inv = 0;

  // every warp owns a contiguous run of chunks: one binary search per lane per run, then the
  // per-lane sequence accumulator walks forward (flushing only when it crosses a boundary)
  const long long cpw = (n_chunks + nwarps - 1) / nwarps;
  const long long c_begin = warp_g * cpw;
  const long long c_end = c_begin + cpw < n_chunks ? c_begin + cpw : n_chunks;
  SeqAcc acc;
  acc.sid = LLONG_MAX;
  acc.x = 0;
  acc.t = 0;
  acc.nsat = 0;
  long long next_b = LLONG_MAX;
  if (kSeq && c_begin < c_end && c_begin * kWarpTok + lane * kTpl < p.n) {
    acc.sid = seq_of(p.cu, p.n_seq, p.tok_begin + c_begin * kWarpTok + lane * kTpl);
    next_b = __ldg(p.cu + acc.sid + 1);
  }

  for (long long ch = c_begin; ch < c_end; ++ch) {
    const long long i0 = ch * kWarpTok + lane * kTpl;
    float num[kTpl], den[kTpl];
    uint8_t rs[kTpl];
    const bool full = (kTpl % 4 == 0) && i0 + kTpl <= p.n;  // vector path needs whole float4s
    if (full) {
#pragma unroll
      for (int v = 0; v < kTpl / 4; ++v) {
        const float4 a = __ldg(reinterpret_cast<const float4*>(p.num + i0) + v);
        const float4 b = __ldg(reinterpret_cast<const float4*>(p.den + i0) + v);
        num[4 * v] = a.x; num[4 * v + 1] = a.y; num[4 * v + 2] = a.z; num[4 * v + 3] = a.w;
        den[4 * v] = b.x; den[4 * v + 1] = b.y; den[4 * v + 2] = b.z; den[4 * v + 3] = b.w;
      }
      if (p.resp) {
#pragma unroll
        for (int v = 0; v < kTpl / 4; ++v) {
          const uint32_t m = __ldg(reinterpret_cast<const uint32_t*>(p.resp + i0) + v);
#pragma unroll
          for (int k = 0; k < 4; ++k) rs[4 * v + k] = (m >> (8 * k)) & 0xff;
        }
      } else {
#pragma unroll
        for (int k = 0; k < kTpl; ++k) rs[k] = 1;
      }
    } else {
#pragma unroll
      for (int k = 0; k < kTpl; ++k) {
        const long long i = i0 + k;
        num[k] = i < p.n ? p.num[i] : 0.f;
        den[k] = i < p.n ? p.den[i] : 0.f;
        rs[k] = i < p.n ? (p.resp ? p.resp[i] : 1) : 0;
      }
    }

    // (1) delta for the lane's 8 tokens; (2) the short small-|delta| polynomials of all 8 tokens in
    // lockstep (8 independent Horner chains: latency hidden by ILP); (3) the rare tokens outside
    // [-2^-6, 2^-6] take the long contract paths.  Same op sequence per token as exp_c / k3_c.
    double dv[kTpl], ds[kTpl], ev[kTpl], k3v[kTpl];
    unsigned big_mask = 0;
#pragma unroll
    for (int k = 0; k < kTpl; ++k) {
      dv[k] = __dsub_rn(static_cast<double>(num[k]), static_cast<double>(den[k]));
      const bool ok = i0 + k < p.n && isfinite(dv[k]);
      const bool sm = ok && fabs(dv[k]) <= kSmall;
      if (ok && !sm) big_mask |= 1u << k;
      ds[k] = sm ? dv[k] : 0.0;
      k3v[k] = kInvFact[9];
      ev[k] = kInvFact[7];
    }
#pragma unroll
    for (int n = 8; n >= 2; --n)
#pragma unroll
      for (int k = 0; k < kTpl; ++k) k3v[k] = __dadd_rn(__dmul_rn(k3v[k], ds[k]), kInvFact[n]);
#pragma unroll
    for (int k = 0; k < kTpl; ++k) k3v[k] = __dmul_rn(__dmul_rn(ds[k], ds[k]), k3v[k]);
    if (cfg.tis) {
#pragma unroll
      for (int n = 6; n >= 0; --n)
#pragma unroll
        for (int k = 0; k < kTpl; ++k) ev[k] = __dadd_rn(__dmul_rn(ev[k], ds[k]), kInvFact[n]);
    }
    if (big_mask) {
#pragma unroll
      for (int k = 0; k < kTpl; ++k) {
        if ((big_mask >> k) & 1u) {
          k3v[k] = k3_c(dv[k]);
          if (cfg.tis) ev[k] = exp_c(dv[k]);
        }
      }
    }

    float w_out[kTpl], c_out[kTpl];
    uint8_t k_out[kTpl];
#pragma unroll
    for (int k = 0; k < kTpl; ++k) {
      const long long i = i0 + k;
      w_out[k] = 1.f;
      c_out[k] = 0.f;
      k_out[k] = 1;
      if (i >= p.n) continue;
      const long long g = p.tok_begin + i;
      const double d = dv[k];
      if (!isfinite(d)) {  // C.3.2 data error: excluded from every sum, outputs NaN / 0
        const unsigned long long b = kBadSentinel - static_cast<unsigned long long>(g);
        bad_inv = b > bad_inv ? b : bad_inv;
        w_out[k] = CUDART_NAN_F;
        k_out[k] = 0;
        continue;
      }
      const bool resp = rs[k] != 0;
      const bool trunc = cfg.tis && d > cfg.log_tis_cap;
      if (cfg.tis) {
        const double w = trunc ? cfg.tis_cap : fmin(ev[k], cfg.tis_cap);
        w_out[k] = __double2float_rn(w);
      }
      const bool keep = cfg.tok_rs ? (cfg.log_lo <= d && d <= cfg.log_hi) : true;
      k_out[k] = keep ? 1 : 0;
      c_out[k] = (resp && keep) ? w_out[k] : 0.f;

      bool sat1, sat3;
      const long long x1 = fixed_point(-d, sat1);
      const double k3 = k3v[k];
      const long long x3 = fixed_point(k3, sat3);
      if (resp) {
        // rint is odd-symmetric and |K1| = |delta| saturate together: X(|delta|) = |X(-delta)|
        const long long xa = x1 < 0 ? -x1 : x1;
        c_resp += 1;
        c_trunc += trunc ? 1 : 0;
        c_rej += keep ? 0 : 1;
        s_abs += xa;
        s_k1 += x1;
        s_k3 += x3;
        const unsigned long long bits = static_cast<unsigned long long>(__double_as_longlong(fabs(d)));
        maxbits = bits > maxbits ? bits : maxbits;
      }
      if (kSeq) {
        while (g >= next_b) {  // crossed into a later sequence (skips empty ones)
          flush_seq(p.seqp, acc);
          acc.x = 0;
          acc.t = 0;
          acc.nsat = 0;
          acc.sid += 1;
          next_b = __ldg(p.cu + acc.sid + 1);
        }
        if (resp && keep) {
          const bool satq = cfg.seq_rs == TIM_SEQ_K1 ? sat1 : sat3;
          acc.x += cfg.seq_rs == TIM_SEQ_K1 ? x1 : x3;
          acc.t += 1;
          acc.nsat += satq ? 1 : 0;
          c_sat += satq ? 1 : 0;
        }
      }
    }

    if (kOut) {
      if (full) {
        float4* pw = reinterpret_cast<float4*>(p.tis_w + i0);
        float4* pc = reinterpret_cast<float4*>(p.coeff + i0);
#pragma unroll
        for (int v = 0; v < kTpl / 4; ++v) {
          pw[v] = make_float4(w_out[4 * v], w_out[4 * v + 1], w_out[4 * v + 2], w_out[4 * v + 3]);
          pc[v] = make_float4(c_out[4 * v], c_out[4 * v + 1], c_out[4 * v + 2], c_out[4 * v + 3]);
          reinterpret_cast<uint32_t*>(p.tok_keep + i0)[v] =
              k_out[4 * v] | (k_out[4 * v + 1] << 8) | (k_out[4 * v + 2] << 16) |
              (static_cast<uint32_t>(k_out[4 * v + 3]) << 24);
        }
      } else {
#pragma unroll
        for (int k = 0; k < kTpl; ++k) {
          const long long i = i0 + k;
          if (i < p.n) {
            p.tis_w[i] = w_out[k];
            p.coeff[i] = c_out[k];
            p.tok_keep[i] = k_out[k];
          }
        }
      }
    }

  }

  if (kSeq) {
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
    // note: lane l now holds the sum of lanes [l, l+2^k) with the same id, so the head of each
    // run (first lane of that id) holds the whole run because runs are contiguous.
    const long long prev_sid = __shfl_up_sync(0xffffffffu, acc.sid, 1);
    const bool head = lane == 0 || prev_sid != acc.sid;
    if (head && acc.sid != LLONG_MAX) flush_seq(p.seqp, acc);
  }

  // block reduction of the global statistics, then one set of integer atomics per block
  __shared__ long long sh_cnt[4][kLocalThreads / 32];
  __shared__ long long sh_sum[6][kLocalThreads / 32];
  __shared__ unsigned long long sh_max[kLocalThreads / 32], sh_bad[kLocalThreads / 32];
  const int w = threadIdx.x >> 5;
  c_resp = warp_sum_i64(c_resp);
  c_trunc = warp_sum_i64(c_trunc);
  c_rej = warp_sum_i64(c_rej);
  c_sat = warp_sum_i64(c_sat);
  s_abs = warp_sum_i128(s_abs);
  s_k1 = warp_sum_i128(s_k1);
  s_k3 = warp_sum_i128(s_k3);
  maxbits = warp_max_u64(maxbits);
  bad_inv = warp_max_u64(bad_inv);
  if (lane == 0) {
    sh_cnt[0][w] = c_resp;
    sh_cnt[1][w] = c_trunc;
    sh_cnt[2][w] = c_rej;
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
    unsigned long long mx = 0, bd = 0;
    for (int i = 0; i < kLocalThreads / 32; ++i) {
      for (int k = 0; k < 4; ++k) cnt[k] += sh_cnt[k][i];
      for (int k = 0; k < 3; ++k)
        sums[k] += (static_cast<__int128>(sh_sum[2 * k + 1][i]) << 64) |
                   static_cast<__int128>(static_cast<unsigned long long>(sh_sum[2 * k][i]));
      mx = sh_max[i] > mx ? sh_max[i] : mx;
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
    if (mx) atomicMax(reinterpret_cast<unsigned long long*>(&h->max_abs_delta_bits), mx);
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
  if (out && seq) correct_local_kernel<true, true><<<blocks, kLocalThreads, 0, stream>>>(p);
  else if (out) correct_local_kernel<true, false><<<blocks, kLocalThreads, 0, stream>>>(p);
  else if (seq) correct_local_kernel<false, true><<<blocks, kLocalThreads, 0, stream>>>(p);
  else correct_local_kernel<false, false><<<blocks, kLocalThreads, 0, stream>>>(p);
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
