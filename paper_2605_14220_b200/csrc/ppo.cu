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

#include <cstdint>

#include "contract.cuh"
#include "tim_internal.h"

namespace tim {

constexpr int kPpoTpl = 8;
constexpr int kPpoWarpTok = 32 * kPpoTpl;
constexpr int kPpoThreads = 256;
constexpr int kMaxHistBins = 1024;

__global__ void __launch_bounds__(kPpoThreads, 2) ppo_local_kernel(PpoLocalParams p) {
  extern __shared__ int sh_hist[];  // [2][bins + 2]
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

  long long c_contrib = 0, c_clip = 0, c_zero = 0, c_sat = 0;
  __int128 s_loss = 0, s_k1 = 0, s_k3 = 0;
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

  for (long long ch = c_begin; ch < c_end; ++ch) {
    const long long i0 = ch * kPpoWarpTok + lane * kPpoTpl;
    double dv[kPpoTpl], rv[kPpoTpl];
    float adv[kPpoTpl], wv[kPpoTpl];
    bool cb[kPpoTpl];
    unsigned big_mask = 0;
#pragma unroll
    for (int k = 0; k < kPpoTpl; ++k) {
      const long long i = i0 + k;
      const bool in = i < p.n;
      const float cur = in ? __ldg(p.cur + i) : 0.f;
      const float old = in ? __ldg(p.old + i) : 0.f;
      adv[k] = in ? __ldg(p.adv + i) : 0.f;
      if (p.coeff) {
        wv[k] = in ? __ldg(p.coeff + i) : 0.f;
        cb[k] = wv[k] != 0.f;
      } else {
        cb[k] = in && (p.resp ? __ldg(p.resp + i) != 0 : true);
        wv[k] = cb[k] ? 1.f : 0.f;
      }
      dv[k] = __dsub_rn(static_cast<double>(cur), static_cast<double>(old));
      const bool ok = in && isfinite(dv[k]);
      const bool sm = ok && fabs(dv[k]) <= kSmall;
      if (ok && !sm) big_mask |= 1u << k;
      const double ds = sm ? dv[k] : 0.0;
      rv[k] = exp_from_k3_small(ds, k3_small(ds));
    }
    if (big_mask) {
#pragma unroll
      for (int k = 0; k < kPpoTpl; ++k)
        if ((big_mask >> k) & 1u) rv[k] = exp_c(dv[k]);
    }

#pragma unroll
    for (int k = 0; k < kPpoTpl; ++k) {
      const long long i = i0 + k;
      if (i >= p.n) continue;
      const long long g = p.tok_begin + i;
      const double d = dv[k];
      if (!isfinite(d)) {
        const unsigned long long b = kBadSentinel - static_cast<unsigned long long>(g);
        bad_inv = b > bad_inv ? b : bad_inv;
        p.loss[i] = CUDART_NAN_F;
        p.grad[i] = 0.f;
        p.clipped[i] = 0;
        continue;
      }
      const double r = rv[k];
      const double A = static_cast<double>(adv[k]);
      const bool clipped = (A > 0.0 && r > p.clip_hi) || (A < 0.0 && r < p.clip_lo);
      const double sv = clipped ? __dmul_rn(A > 0.0 ? p.clip_hi : p.clip_lo, A) : __dmul_rn(r, A);
      const double loss = -__dmul_rn(static_cast<double>(wv[k]), sv);
      p.loss[i] = __double2float_rn(loss);
      p.grad[i] = clipped ? 0.f : __double2float_rn(loss);
      p.clipped[i] = clipped ? 1 : 0;
      // leave the sequence(s) the lane has walked past
      while (g >= next_b) {
        flush_seq(p.seqp, acc);
        acc.x = 0;
        acc.t = 0;
        acc.nsat = 0;
        acc.sid += 1;
        next_b = __ldg(p.cu + acc.sid + 1);
      }
      if (!cb[k]) continue;
      bool sat, sat1, sat3;
      const long long X = fixed_point(loss, sat);
      const long long X1 = fixed_point(-d, sat1);
      const long long X3 = fixed_point(k3_c(d), sat3);
      c_contrib += 1;
      c_clip += clipped ? 1 : 0;
      c_sat += sat ? 1 : 0;
      s_loss += X;
      s_k1 += X1;
      s_k3 += X3;
      acc.x += X;
      acc.t += 1;
      acc.nsat += sat ? 1 : 0;
      if (A == 0.0) {
        c_zero += 1;
      } else {
        const double C = __dmul_rn(-__dsub_rn(r, 1.0), A);
        const double raw = floor(__dmul_rn(__dsub_rn(C, p.hist_lo), p.hist_inv_width));
        const int slot = raw < 0.0 ? 0 : (raw >= static_cast<double>(p.bins) ? p.bins + 1 : static_cast<int>(raw) + 1);
        atomicAdd(&sh_hist[(A > 0.0 ? 0 : nslot) + slot], 1);
      }
    }
  }

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
  c_contrib = warp_sum_i64(c_contrib);
  c_clip = warp_sum_i64(c_clip);
  c_zero = warp_sum_i64(c_zero);
  c_sat = warp_sum_i64(c_sat);
  s_loss = warp_sum_i128(s_loss);
  s_k1 = warp_sum_i128(s_k1);
  s_k3 = warp_sum_i128(s_k3);
  bad_inv = warp_max_u64(bad_inv);
  tim_ppo_partial_header* h = p.hdr;
  if (lane == 0) {
    if (c_contrib) atomicAdd(reinterpret_cast<unsigned long long*>(&h->n_contrib), static_cast<unsigned long long>(c_contrib));
    if (c_clip) atomicAdd(reinterpret_cast<unsigned long long*>(&h->n_clipped), static_cast<unsigned long long>(c_clip));
    if (c_zero) atomicAdd(reinterpret_cast<unsigned long long*>(&h->n_zero_adv), static_cast<unsigned long long>(c_zero));
    if (c_sat) atomicAdd(reinterpret_cast<unsigned long long*>(&h->n_saturated), static_cast<unsigned long long>(c_sat));
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
  for (long long s = threadIdx.x; s < p.n_seq; s += blockDim.x) {
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
    for (int i = threadIdx.x; i < 2 * nslot; i += blockDim.x) {
      long long v = 0;
      for (int r = 0; r < p.nranks; ++r)
        v += reinterpret_cast<const int64_t*>(p.gathered + r * p.block_bytes + sizeof(tim_ppo_partial_header))[i];
      p.hist[i] = v;
    }
  }
  for (int off = 16; off > 0; off >>= 1) nc += __shfl_down_sync(0xffffffffu, nc, off);
  if ((threadIdx.x & 31) == 0) sh_nc[threadIdx.x >> 5] = nc;
  __syncthreads();
  if (threadIdx.x == 0 && p.stats) {
    long long n_seq_contrib = 0;
    for (int i = 0; i < kPpoFinishThreads / 32; ++i) n_seq_contrib += sh_nc[i];
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
  const long long cap = static_cast<long long>(num_sms) * 2;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  const size_t smem = sizeof(int) * 2 * (p.bins + 2);
  ppo_local_kernel<<<static_cast<int>(blocks), kPpoThreads, smem, stream>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_ppo_finish(const PpoFinishParams& p, cudaStream_t stream) {
  ppo_finish_kernel<<<1, kPpoFinishThreads, 0, stream>>>(p);
  return cudaGetLastError();
}

}  // namespace tim
