// ppo.cu -- NEXT-2: fused PPO / GRPO surrogate and the paper's loss diagnostics.
//
// Per token (PAPER.md eq:ppo_loss P:352-360, eq:ppo_ratio P:361-373, App. A.4):
//   r = exp_c(lp_cur - lp_old)  (C.3 contract), clipped <=> A > 0 ? r > clip_hi : (A < 0 && r < clip_lo)
//   loss = -(w * (clipped ? clip * A : r * A)), w = correction coefficient (or response mask)
//   grad = d loss / d lp_cur = clipped ? 0 : loss  (score-function gradient)
//   C(r) = -(r - 1) A histogrammed by sign(A); K1 / K3 on r
// Per sequence: exact int128 sum of the 2^-52 fixed-point loss (token sum over the response,
// P:384); the batch loss = sum of sequence sums / sequences with a contributing token.
// Bandwidth-bound: reads 3 fp32 + (fp32 coeff | u8 mask), writes 2 fp32 + u8 per token.
#include <cuda_runtime.h>
#include <math_constants.h>

#include <atomic>
#include <cstdint>
#include <type_traits>

#include "contract.cuh"
#include "ptx.cuh"
#include "tim_internal.h"

namespace tim {

constexpr int kPpoTpl = 4;                  // tokens per lane: one float4 of each input
constexpr int kPpoWarpTok = 32 * kPpoTpl;
#ifndef TIM_PPO_THREADS
#define TIM_PPO_THREADS 128
#endif
#ifndef TIM_PPO_MINB
#define TIM_PPO_MINB 4
#endif
#ifndef TIM_PPO_PLAIN_STORES
#define TIM_PPO_PLAIN_STORES 0  // 1: plain stores instead of st.global.cs (0.7% slower here)
#endif
#ifndef TIM_PPO_LOAD_HINT
#define TIM_PPO_LOAD_HINT 0  // 1: cp.async reads with an L2 evict_first policy (0.6% slower)
#endif
#ifndef TIM_PPO_STAGES
#define TIM_PPO_STAGES 4
#endif
constexpr int kPpoStages = TIM_PPO_STAGES;  // per-warp cp.async ring depth (chunks in flight)
constexpr int kPpoStageBytes = 4 * 512;     // cur, old, adv, coeff (or the u8 mask): 128 tokens each
constexpr int kPpoThreads = TIM_PPO_THREADS;
constexpr int kPpoMinB = TIM_PPO_MINB;
constexpr int kMaxHistBins = 1024;
constexpr long long kPpoFold = 1024;       // chunks per int64 K1 / K3 fold: 2^10 x 2^52 < 2^63
constexpr double kPpoFastLoss = 256.0;      // fast path: |loss| <= 2^8, so |X| <= 2^60 and four fit int64

struct PpoCold {
  __int128 s_loss, s_k1, s_k3;
};

struct PpoChunk {
  float4 cur, old, adv, w;  // w = coeff, or the response mask as 0 / 1
};

// Weight source, a kernel template argument (no per-chunk pointer tests): the correction
// coefficient, the u8 response mask, or none (every token weight 1).
enum PpoWeight : int { kWCoeff = 0, kWResp = 1, kWNone = 2 };

template <int kW>
__device__ __forceinline__ PpoChunk ppo_load(const PpoLocalParams& p, long long i0) {
  PpoChunk c;
  if (p.vec && i0 + kPpoTpl <= p.n) {
    c.cur = __ldcs(reinterpret_cast<const float4*>(p.cur + i0));
    c.old = __ldcs(reinterpret_cast<const float4*>(p.old + i0));
    c.adv = __ldcs(reinterpret_cast<const float4*>(p.adv + i0));
    if (kW == kWCoeff) {
      c.w = __ldcs(reinterpret_cast<const float4*>(p.coeff + i0));
    } else if (kW == kWResp) {
      const uint32_t m = __ldcs(reinterpret_cast<const unsigned int*>(p.resp + i0));
      c.w = make_float4((m & 0xffu) ? 1.f : 0.f, (m & 0xff00u) ? 1.f : 0.f, (m & 0xff0000u) ? 1.f : 0.f,
                        (m & 0xff000000u) ? 1.f : 0.f);
    } else {
      c.w = make_float4(1.f, 1.f, 1.f, 1.f);
    }
  } else {
    float v[4][4];
#pragma unroll
    for (int k = 0; k < kPpoTpl; ++k) {
      const long long i = i0 + k;
      const bool in = i < p.n;
      v[0][k] = in ? p.cur[i] : 0.f;
      v[1][k] = in ? p.old[i] : 0.f;
      v[2][k] = in ? p.adv[i] : 0.f;
      v[3][k] = !in ? 0.f : (kW == kWCoeff ? p.coeff[i] : ((kW == kWResp ? p.resp[i] != 0 : true) ? 1.f : 0.f));
    }
    c.cur = make_float4(v[0][0], v[0][1], v[0][2], v[0][3]);
    c.old = make_float4(v[1][0], v[1][1], v[1][2], v[1][3]);
    c.adv = make_float4(v[2][0], v[2][1], v[2][2], v[2][3]);
    c.w = make_float4(v[3][0], v[3][1], v[3][2], v[3][3]);
  }
  return c;
}

// dynamic shared memory: [2][bins + 2] int histogram, 32 per-lane sink slots (the lock-step path's
// atomics for A = 0 tokens land there, so the atomic needs no branch), then the per-warp rings
// (16-B aligned)
__host__ __device__ constexpr size_t ppo_hist_bytes(int bins) {
  return (sizeof(int) * (2 * static_cast<size_t>(bins + 2) + 32) + 15) & ~size_t(15);
}

// Slot of C(r) = -(r - 1) A: 0 below hist_lo, bins + 1 at or above the top edge, else floor + 1.
// Branch-free: clamping the saturated integer floor to [-1, bins] gives the same slot for every
// non-NaN C (C is never NaN for a counted token: r is finite or +inf, A finite and nonzero).
__device__ __forceinline__ int hist_slot(const PpoLocalParams& p, double r, double A) {
  const double C = __dmul_rn(-__dsub_rn(r, 1.0), A);
  // floor and convert in one (cvt.rmi.s32.f64 saturates out-of-range values and infinities)
  const int raw = __double2int_rd(__dmul_rn(__dsub_rn(C, p.hist_lo), p.hist_inv_width));
  return min(max(raw, -1), p.bins) + 1;
}

// loss = -(w * (clipped ? clip * A : r * A)): one product of the selected factor, bit-identical
__device__ __forceinline__ double ppo_token_loss(const PpoLocalParams& p, double r, double A, float w,
                                                 bool& clipped) {
  const bool pos = A > 0.0;
  clipped = (pos & (r > p.clip_hi)) | ((A < 0.0) & (r < p.clip_lo));  // no short-circuit branch
  const double f = clipped ? (pos ? p.clip_hi : p.clip_lo) : r;
  return -__dmul_rn(static_cast<double>(w), __dmul_rn(f, A));
}

// 4 tokens per lane, next chunk prefetched, a lock-step fast path (|delta| <= 2^-2, |loss| <=
// 2^8: the short / mid contract series in one Horner chain per token, exact int64 chunk sums
// folded into int128 per chunk) and a rare per-lane slow path with the full contract (larger delta
// or loss, non-finite input, partial or unaligned chunk, sequence boundary inside the lane's
// tokens).
template <int kW>
__global__ void __launch_bounds__(kPpoThreads, kPpoMinB) ppo_local_kernel(PpoLocalParams p) {
  extern __shared__ __align__(16) int sh_hist[];  // [2][bins + 2], then the rings
  const int nslot = p.bins + 2;
  for (int i = threadIdx.x; i < 2 * nslot; i += blockDim.x) sh_hist[i] = 0;
  __syncthreads();

  const int lane = threadIdx.x & 31;
  const long long warp_g = (static_cast<long long>(blockIdx.x) * kPpoThreads + threadIdx.x) >> 5;
  const long long nwarps = (static_cast<long long>(gridDim.x) * kPpoThreads) >> 5;
  const long long n_chunks = (p.n + kPpoWarpTok - 1) / kPpoWarpTok;
  const long long cpw = (n_chunks + nwarps - 1) / nwarps;
  const long long c_begin = warp_g * cpw;
  const long long c_end = c_begin + cpw < n_chunks ? c_begin + cpw : n_chunks;

  unsigned c_contrib = 0, c_clip = 0, c_zero = 0, c_sat = 0;
  // s_loss collects each flushed sequence segment (acc.x), so the hot path adds the chunk's loss
  // once (to acc.x); the lock-step path's K1 / K3 chunk sums (|X| <= 2^52 per chunk) go to int64
  // lane accumulators folded into the int128 sums every kPpoFold chunks.
  // the int128 sums are touched only at folds, flushes and in the slow path: per-thread shared
  // memory, so the hot loop keeps its registers
  __shared__ PpoCold sh_cold[kPpoThreads];
  PpoCold& cold = sh_cold[threadIdx.x];
  cold.s_loss = 0;
  cold.s_k1 = 0;
  cold.s_k3 = 0;
  long long f_k1 = 0, f_k3 = 0;
  auto fold = [&]() {
    cold.s_k1 += f_k1;
    cold.s_k3 += f_k3;
    f_k1 = 0;
    f_k3 = 0;
  };
  unsigned long long bad_inv = 0;

  SeqAcc acc;
  acc.sid = LLONG_MAX;
  acc.x = 0;
  acc.t = 0;
  acc.nsat = 0;
  long long next_b = LLONG_MAX;
  if (c_begin < c_end && c_begin * kPpoWarpTok + lane * kPpoTpl < p.n) {
    acc.sid = seq_of(p.cu, p.n_seq, p.tok_begin + c_begin * kPpoWarpTok + lane * kPpoTpl);
    next_b = __ldg(p.cu + acc.sid + 1);
  }
  // i0 >= seq_lim <=> the lane's tokens reach the start of the next sequence
  long long seq_lim = next_b - p.tok_begin - (kPpoTpl - 1);

  if (blockIdx.x == 0 && threadIdx.x == 0) shard_range_check(p.cu, p.n_seq, p.tok_begin, p.n, bad_inv);

  // kFull: a whole vector chunk (the ring loop) -- known at compile time there
  auto body = [&](const PpoChunk& cur, const long long i0, auto full_tag) {
    const float cu_[4] = {cur.cur.x, cur.cur.y, cur.cur.z, cur.cur.w};
    const float ol_[4] = {cur.old.x, cur.old.y, cur.old.z, cur.old.w};
    const float ad_[4] = {cur.adv.x, cur.adv.y, cur.adv.z, cur.adv.w};
    const float wv_[4] = {cur.w.x, cur.w.y, cur.w.z, cur.w.w};
    const bool full = decltype(full_tag)::value || (p.vec && i0 + kPpoTpl <= p.n);

    // fast tokens: |delta| <= 2^-2 (finite): the short (|delta| <= 2^-6) and the mid contract
    // series in one lock-step Horner chain per token (k3_small_or_mid), e^delta = (1 + delta) + K3.
    // A slow token (|delta| > 2^-2, non-finite) runs the chain too; every result of it is masked
    // out of the sums below and overwritten by the slow path.
    // The slow decision is per lane: one slow token sends the lane's four tokens to the slow path
    // (rare, and the slow path is the full contract, so the results are the same).
    double dv[kPpoTpl], k3f[kPpoTpl];
    bool lane_slow = !full || i0 >= seq_lim;
#pragma unroll
    for (int k = 0; k < kPpoTpl; ++k) {
      dv[k] = __dsub_rn(static_cast<double>(cu_[k]), static_cast<double>(ol_[k]));
      lane_slow |= !(fabs(dv[k]) <= kMid);  // true for NaN / inf
    }
#pragma unroll
    for (int k = 0; k < kPpoTpl; ++k) k3f[k] = k3_small_or_mid(dv[k], fabs(dv[k]) <= kSmall);

    float l_out[kPpoTpl], g_out[kPpoTpl];
    uint32_t cbits = 0;
    double loss_[kPpoTpl], r_[kPpoTpl];
#pragma unroll
    for (int k = 0; k < kPpoTpl; ++k) {
      const double r = exp_from_k3_small(dv[k], k3f[k]);
      bool clipped;
      const double loss = ppo_token_loss(p, r, static_cast<double>(ad_[k]), wv_[k], clipped);
      lane_slow |= !(fabs(loss) <= kPpoFastLoss);
      const float lf = __double2float_rn(loss);
      l_out[k] = lf;
      g_out[k] = clipped ? 0.f : lf;
      cbits |= static_cast<uint32_t>(clipped) << (8 * k);
      loss_[k] = loss;
      r_[k] = r;
    }
    const unsigned slow = lane_slow ? 0xFu : 0u;
    long long cl = 0, ck1 = 0, ck3 = 0;  // chunk sums: |X| <= 2^60 (loss), 2^52 (K1, K3)
    unsigned cn = 0, ccl = 0, cz = 0;
    // warp-uniform: every token of the chunk fast and weighted (the common case inside the
    // response) -> the sums without per-token masks
    const bool lane_clean = slow == 0u && wv_[0] != 0.f && wv_[1] != 0.f && wv_[2] != 0.f && wv_[3] != 0.f;
    if (__all_sync(0xffffffffu, lane_clean)) {
#pragma unroll
      for (int k = 0; k < kPpoTpl; ++k) {
        const double A = static_cast<double>(ad_[k]);
        cl += __double2ll_rn(__dmul_rn(loss_[k], kTwo52));
        ck1 += __double2ll_rn(__dmul_rn(-dv[k], kTwo52));
        ck3 += __double2ll_rn(__dmul_rn(k3f[k], kTwo52));
        ccl += (cbits >> (8 * k)) & 1u;
        cz += A == 0.0 ? 1u : 0u;
        const int hs = hist_slot(p, r_[k], A);  // computed for every token: no branch
        const int slot = A == 0.0 ? 2 * nslot + lane : (A > 0.0 ? 0 : nslot) + hs;
        atomicAdd(&sh_hist[slot], 1);  // A = 0: the lane's sink slot
      }
      cn = kPpoTpl;
    } else {
#pragma unroll
      for (int k = 0; k < kPpoTpl; ++k) {
        const double A = static_cast<double>(ad_[k]);
        const bool use = wv_[k] != 0.f && !((slow >> k) & 1u);
        const double lz = use ? loss_[k] : 0.0;
        const double dz = use ? dv[k] : 0.0;
        const double kz = use ? k3f[k] : 0.0;
        cl += __double2ll_rn(__dmul_rn(lz, kTwo52));
        ck1 += __double2ll_rn(__dmul_rn(-dz, kTwo52));
        ck3 += __double2ll_rn(__dmul_rn(kz, kTwo52));
        cn += use ? 1u : 0u;
        ccl += (use && ((cbits >> (8 * k)) & 1u)) ? 1u : 0u;
        cz += (use && A == 0.0) ? 1u : 0u;
        const int slot = (A > 0.0 ? 0 : nslot) + hist_slot(p, r_[k], A);
        if (use && A != 0.0) atomicAdd(&sh_hist[slot], 1);
      }
    }
    acc.x += cl;
    acc.t += cn;
    f_k1 += ck1;
    f_k3 += ck3;
    c_contrib += cn;
    c_clip += ccl;
    c_zero += cz;

    if (slow) {  // rare: the full contract per token in the slow tokens' lanes
#pragma unroll
      for (int k = 0; k < kPpoTpl; ++k) {
        if (!((slow >> k) & 1u)) continue;
        const long long i = i0 + k;
        if (i >= p.n) continue;
        const long long g = p.tok_begin + i;
        const double d = dv[k];
        while (g >= next_b && acc.sid + 1 < p.n_seq) {  // leave the sequence(s) walked past (bounded)
          flush_seq(p.seqp, acc);
          cold.s_loss += acc.x;
          acc.x = 0;
          acc.t = 0;
          acc.nsat = 0;
          acc.sid += 1;
          next_b = __ldg(p.cu + acc.sid + 1);
          seq_lim = next_b - p.tok_begin - (kPpoTpl - 1);
        }
        // data error (U13): a non-finite log-prob, advantage or weight -- loss NaN, grad 0, the
        // token excluded from the histogram and every sum
        if (!isfinite(d) || !isfinite(ad_[k]) || !isfinite(wv_[k])) {
          const unsigned long long b = kBadSentinel - static_cast<unsigned long long>(g);
          bad_inv = b > bad_inv ? b : bad_inv;
          l_out[k] = CUDART_NAN_F;
          g_out[k] = 0.f;
          cbits &= ~(0xffu << (8 * k));
          continue;
        }
        const double k3 = k3_c(d);
        const double r = exp_c(d);
        const double A = static_cast<double>(ad_[k]);
        bool clipped;
        const double loss = ppo_token_loss(p, r, A, wv_[k], clipped);
        l_out[k] = __double2float_rn(loss);
        g_out[k] = clipped ? 0.f : l_out[k];
        cbits = (cbits & ~(0xffu << (8 * k))) | (static_cast<uint32_t>(clipped) << (8 * k));
        if (wv_[k] == 0.f) continue;
        bool sat, sat1, sat3;
        const long long X = fixed_point(loss, sat);
        const long long X1 = fixed_point(-d, sat1);
        const long long X3 = fixed_point(k3, sat3);
        c_contrib += 1;
        c_clip += clipped ? 1u : 0u;
        c_sat += sat ? 1u : 0u;
        cold.s_k1 += X1;
        cold.s_k3 += X3;
        acc.x += X;
        acc.t += 1;
        acc.nsat += sat ? 1 : 0;
        if (A == 0.0) c_zero += 1;
        else atomicAdd(&sh_hist[(A > 0.0 ? 0 : nslot) + hist_slot(p, r, A)], 1);
      }
    }

    if (full) {
#if TIM_PPO_PLAIN_STORES
      *reinterpret_cast<float4*>(p.loss + i0) = make_float4(l_out[0], l_out[1], l_out[2], l_out[3]);
      *reinterpret_cast<float4*>(p.grad + i0) = make_float4(g_out[0], g_out[1], g_out[2], g_out[3]);
      *reinterpret_cast<unsigned int*>(p.clipped + i0) = cbits;
#else
      __stcs(reinterpret_cast<float4*>(p.loss + i0), make_float4(l_out[0], l_out[1], l_out[2], l_out[3]));
      __stcs(reinterpret_cast<float4*>(p.grad + i0), make_float4(g_out[0], g_out[1], g_out[2], g_out[3]));
      __stcs(reinterpret_cast<unsigned int*>(p.clipped + i0), cbits);
#endif
    } else {
#pragma unroll
      for (int k = 0; k < kPpoTpl; ++k) {
        const long long i = i0 + k;
        if (i < p.n) {
          p.loss[i] = l_out[k];
          p.grad[i] = g_out[k];
          p.clipped[i] = (cbits >> (8 * k)) & 0xffu;
        }
      }
    }
  };

  // whole vector chunks stream through a per-lane cp.async ring in shared memory (lane l copies and
  // later reads only its own 4 tokens' slots: completion per thread by commit / wait groups, no
  // barrier, and the bytes in flight cost no registers); the rest takes element-wise loads
  const long long n_vec = p.vec ? p.n / kPpoWarpTok : 0;
  long long c_mid = c_end < n_vec ? c_end : n_vec;
  if (c_mid < c_begin) c_mid = c_begin;
  const int wib = threadIdx.x >> 5;
  uint8_t* ring = reinterpret_cast<uint8_t*>(sh_hist) + ppo_hist_bytes(p.bins) + wib * kPpoStages * kPpoStageBytes;
  const uint32_t ring16 = smem_u32(ring) + lane * 16;
  const uint32_t ring4 = smem_u32(ring) + 3 * 512 + lane * 4;
  [[maybe_unused]] const uint64_t pol = policy_evict_first();
  auto issue = [&](int j, long long c) {  // chunk c into stage j (one commit group, possibly empty)
    if (c < c_mid) {
      const long long i = c * kPpoWarpTok + lane * kPpoTpl;
      const uint32_t d = ring16 + j * kPpoStageBytes;
#if TIM_PPO_LOAD_HINT
      cp_async_16_hint(d, p.cur + i, pol);
      cp_async_16_hint(d + 512, p.old + i, pol);
      cp_async_16_hint(d + 1024, p.adv + i, pol);
      if (kW == kWCoeff) cp_async_16_hint(d + 1536, p.coeff + i, pol);
#else
      cp_async_16(d, p.cur + i);
      cp_async_16(d + 512, p.old + i);
      cp_async_16(d + 1024, p.adv + i);
      if (kW == kWCoeff) cp_async_16(d + 1536, p.coeff + i);
#endif
      else if (kW == kWResp) cp_async_4(ring4 + j * kPpoStageBytes, p.resp + i);
    }
    cp_async_commit();
  };
  for (int j = 0; j < kPpoStages; ++j) issue(j, c_begin + j);
  int j = 0;
  for (long long cb = c_begin; cb < c_mid; cb += kPpoFold) {
  const long long ce = cb + kPpoFold < c_mid ? cb + kPpoFold : c_mid;
  for (long long ch = cb; ch < ce; ++ch) {
    cp_async_wait<kPpoStages - 1>();  // this lane's copies of chunk ch have landed
    const uint8_t* st = ring + j * kPpoStageBytes;
    PpoChunk c;
    c.cur = *reinterpret_cast<const float4*>(st + lane * 16);
    c.old = *reinterpret_cast<const float4*>(st + 512 + lane * 16);
    c.adv = *reinterpret_cast<const float4*>(st + 1024 + lane * 16);
    if (kW == kWCoeff) {
      c.w = *reinterpret_cast<const float4*>(st + 1536 + lane * 16);
    } else if (kW == kWResp) {
      const uint32_t m = *reinterpret_cast<const uint32_t*>(st + 1536 + lane * 4);
      c.w = make_float4((m & 0xffu) ? 1.f : 0.f, (m & 0xff00u) ? 1.f : 0.f, (m & 0xff0000u) ? 1.f : 0.f,
                        (m & 0xff000000u) ? 1.f : 0.f);
    } else {
      c.w = make_float4(1.f, 1.f, 1.f, 1.f);
    }
    issue(j, ch + kPpoStages);  // the lane has read stage j: refill it
    if (++j == kPpoStages) j = 0;
    body(c, ch * kPpoWarpTok + lane * kPpoTpl, std::true_type{});
  }
  fold();
  }
  for (long long ch = c_mid; ch < c_end; ++ch) {
    const long long i0 = ch * kPpoWarpTok + lane * kPpoTpl;
    body(ppo_load<kW>(p, i0), i0, std::false_type{});
  }
  fold();
  __int128 s_loss = cold.s_loss + acc.x;  // + this lane's open segment
  __int128 s_k1 = cold.s_k1, s_k3 = cold.s_k3;
  // the open sequence segments of the warp (ids are non-decreasing in lane order)
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
  const long long prev_sid = __shfl_up_sync(0xffffffffu, acc.sid, 1);
  if ((lane == 0 || prev_sid != acc.sid) && acc.sid != LLONG_MAX) flush_seq(p.seqp, acc);

  // global counters: warp reduce, then integer atomics (exact)
  const long long n_contrib = warp_sum_i64(c_contrib);
  const long long n_clip = warp_sum_i64(c_clip);
  const long long n_zero = warp_sum_i64(c_zero);
  const long long n_sat = warp_sum_i64(c_sat);
  s_loss = warp_sum_i128(s_loss);
  s_k1 = warp_sum_i128(s_k1);
  s_k3 = warp_sum_i128(s_k3);
  bad_inv = warp_max_u64(bad_inv);
  tim_ppo_partial_header* h = p.hdr;
  if (lane == 0) {
    if (n_contrib) atomicAdd(reinterpret_cast<unsigned long long*>(&h->n_contrib), static_cast<unsigned long long>(n_contrib));
    if (n_clip) atomicAdd(reinterpret_cast<unsigned long long*>(&h->n_clipped), static_cast<unsigned long long>(n_clip));
    if (n_zero) atomicAdd(reinterpret_cast<unsigned long long*>(&h->n_zero_adv), static_cast<unsigned long long>(n_zero));
    if (n_sat) atomicAdd(reinterpret_cast<unsigned long long*>(&h->n_saturated), static_cast<unsigned long long>(n_sat));
    atomic_add_i128(h->sum_loss, s_loss);
    atomic_add_i128(h->sum_k1, s_k1);
    atomic_add_i128(h->sum_k3, s_k3);
    if (bad_inv) atomicMax(reinterpret_cast<unsigned long long*>(&h->reserved[0]), bad_inv);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0)
    atomicAdd(reinterpret_cast<unsigned long long*>(&h->n_tok), static_cast<unsigned long long>(p.n));
  __syncthreads();
  for (int i = threadIdx.x; i < 2 * nslot; i += blockDim.x)
    if (sh_hist[i]) atomicAdd(reinterpret_cast<unsigned long long*>(p.hist + i), static_cast<unsigned long long>(sh_hist[i]));
  commit_status_last_block(reinterpret_cast<WsHeader*>(&h->reserved[0]), p.dstatus);
}

constexpr int kPpoFinishThreads = 1024;

__global__ void __launch_bounds__(kPpoFinishThreads) ppo_finish_kernel(PpoFinishParams p) {
  __shared__ long long sh_nc[kPpoFinishThreads / 32];
  long long nc = 0;
  const int nslot = p.bins + 2;
  const int64_t seq_off = static_cast<int64_t>(sizeof(tim_ppo_partial_header)) + 16ll * nslot;
  const long long tid = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  for (long long s = tid; s < p.n_seq; s += stride) {
    __int128 X = 0;
    long long T = 0;
    for (int r = 0; r < p.nranks; ++r) {
      const tim_seq_partial* sp =
          reinterpret_cast<const tim_seq_partial*>(p.gathered + r * p.block_bytes + seq_off) + s;
      X += ld_i128(&sp->x_lo);
      T += sp->n_tok;
    }
    nc += T > 0 ? 1 : 0;
    if (p.seq_loss) p.seq_loss[s] = __dmul_rn(i128_to_double(X), 0x1p-52);
  }
  if (p.hist) {
    for (long long i = tid; i < 2 * nslot; i += stride) {
      long long v = 0;
      for (int r = 0; r < p.nranks; ++r)
        v += reinterpret_cast<const int64_t*>(p.gathered + r * p.block_bytes + sizeof(tim_ppo_partial_header))[i];
      p.hist[i] = v;
    }
  }
  for (int off = 16; off > 0; off >>= 1) nc += __shfl_down_sync(0xffffffffu, nc, off);
  if ((threadIdx.x & 31) == 0) sh_nc[threadIdx.x >> 5] = nc;
  __syncthreads();
  // several blocks (p.scratch = {ticket, contributing sequences}, zeroed): the last block writes the stats
  __shared__ int last;
  long long n_seq_contrib = 0;
  if (threadIdx.x == 0) {
    for (int i = 0; i < static_cast<int>(blockDim.x) / 32; ++i) n_seq_contrib += sh_nc[i];
    last = 1;
    if (gridDim.x > 1) {
      atomicAdd(&p.scratch[1], static_cast<unsigned long long>(n_seq_contrib));
      __threadfence();
      last = atomicAdd(&p.scratch[0], 1ull) == gridDim.x - 1;
      if (last) n_seq_contrib = static_cast<long long>(atomicAdd(&p.scratch[1], 0ull));
    }
  }
  __syncthreads();
  if (threadIdx.x == 0 && last && p.stats) {
    long long cnt[5] = {0, 0, 0, 0, 0};
    __int128 sums[3] = {0, 0, 0};
    for (int r = 0; r < p.nranks; ++r) {
      const tim_ppo_partial_header* h = reinterpret_cast<const tim_ppo_partial_header*>(p.gathered + r * p.block_bytes);
      cnt[0] += h->n_tok;
      cnt[1] += h->n_contrib;
      cnt[2] += h->n_clipped;
      cnt[3] += h->n_zero_adv;
      cnt[4] += h->n_saturated;
      sums[0] += ld_i128(h->sum_loss);
      sums[1] += ld_i128(h->sum_k1);
      sums[2] += ld_i128(h->sum_k3);
    }
    tim_ppo_stats* st = p.stats;
    st->n_tok = cnt[0];
    st->n_contrib = cnt[1];
    st->n_clipped = cnt[2];
    st->n_zero_adv = cnt[3];
    st->n_saturated = cnt[4];
    st->n_seq = p.n_seq;
    st->n_seq_contrib = n_seq_contrib;
    int64_t* dst[3] = {st->sum_loss_fx, st->sum_k1_fx, st->sum_k3_fx};
    for (int k = 0; k < 3; ++k) {
      dst[k][0] = static_cast<int64_t>(static_cast<unsigned long long>(sums[k]));
      dst[k][1] = static_cast<int64_t>(sums[k] >> 64);
    }
    st->batch_loss = 0.0;
    st->clip_frac = 0.0;
    st->mean_k1 = 0.0;
    st->mean_k3 = 0.0;
  }
}

int ppo_max_hist_bins() { return kMaxHistBins; }

cudaError_t launch_ppo_local(const PpoLocalParams& p, int num_sms, cudaStream_t stream) {
  const long long chunks = (p.n + kPpoWarpTok - 1) / kPpoWarpTok;
  long long blocks = (chunks + kPpoThreads / 32 - 1) / (kPpoThreads / 32);
  const long long cap = static_cast<long long>(num_sms) * kPpoMinB;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  const size_t smem = ppo_hist_bytes(p.bins) + static_cast<size_t>(kPpoThreads / 32) * kPpoStages * kPpoStageBytes;
  const int mode = p.coeff ? kWCoeff : (p.resp ? kWResp : kWNone);
  auto kern = mode == kWCoeff ? ppo_local_kernel<kWCoeff> : (mode == kWResp ? ppo_local_kernel<kWResp> : ppo_local_kernel<kWNone>);
  if (smem > 48 * 1024) {  // the attribute is per device and kernel: set it for the current device
    static std::atomic<bool> attr_set[3][kMaxDevices];
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    if (dev < 0 || dev >= kMaxDevices) return cudaErrorInvalidDevice;
    if (!attr_set[mode][dev].load()) {
      e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
      if (e != cudaSuccess) return e;
      attr_set[mode][dev].store(true);
    }
  }
  kern<<<static_cast<int>(blocks), kPpoThreads, smem, stream>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_ppo_finish(const PpoFinishParams& p, int num_sms, cudaStream_t stream) {
  if (p.scratch == nullptr) {  // no zeroed scratch: one block
    ppo_finish_kernel<<<1, kPpoFinishThreads, 0, stream>>>(p);
  } else {
    long long blocks = (p.n_seq + 255) / 256;
    if (blocks > num_sms) blocks = num_sms;
    if (blocks < 1) blocks = 1;
    ppo_finish_kernel<<<static_cast<int>(blocks), 256, 0, stream>>>(p);
  }
  return cudaGetLastError();
}

}  // namespace tim
