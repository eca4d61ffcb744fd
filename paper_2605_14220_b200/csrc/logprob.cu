// logprob.cu -- tim_logprob device code.
//
// a2  lm_head contraction z = H W^T on the 5th-gen tensor cores: tcgen05.mma kind::f16,
//     bf16 x bf16 -> fp32 accumulators in TMEM (never rounded to bf16), operands staged in
//     shared memory by TMA (128-byte swizzle), a CTA pair (cta_group::2) computes a 256-token x
//     256-vocab tile; K ascending in steps of 16 from a zeroed accumulator.
// a3  fused epilogue: each epilogue thread owns one token row (TMEM lane), reads 32 columns
//     at a time with tcgen05.ld and keeps an online (max m, sum-exp s, sum p*(y-m) u, gathered
//     y_a) in registers -- log2 domain, y = z * log2(e) / T.  Logits never reach HBM.
// a4  fixed-order vocab-slice merge (merge kernel): slices 0..S_v-1 in order, fp64.
//
// Batch invariance (§3.1): a token row's arithmetic depends only on its
// own H row, W and constants of (V, d): the vocab tile (256), the slice split S_v(V), the K
// order and the MMA shape.  Which CTA, which row slot, how many rows, SMs or GPUs -- none
// of these enter the arithmetic of a row.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <math_constants.h>

#include <atomic>
#include <cstdint>

#include "ptx.cuh"
#include "tim_internal.h"

namespace tim {

constexpr int kBlockK = 64;        // K elements per pipeline stage (128 B rows -> SW128)
constexpr int kUmmaK = 16;         // K per tcgen05.mma kind::f16
constexpr int kCtaM = 128;         // token rows per CTA (= TMEM lanes)
constexpr int kTileN = 256;        // vocab columns per tile (MMA N)
constexpr int kEpiWarps = 4;
constexpr int kThreads = 64 + 32 * kEpiWarps;
constexpr float kLog2eF = 1.44269504088896340736f;

template <bool kPair>
struct KCfg {
  static constexpr int kBRows = kPair ? 128 : 256;  // W rows staged per CTA
  static constexpr int kABytes = kCtaM * kBlockK * 2;
  static constexpr int kBBytes = kBRows * kBlockK * 2;
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kStages = kPair ? 6 : 4;
  static constexpr int kUnitM = kPair ? 2 * kCtaM : kCtaM;
  static constexpr int kSmemBytes = kStages * kStageBytes + 1024 + 256;
  static constexpr int kCtaGroup = kPair ? 2 : 1;
};

__device__ __forceinline__ float chunk_max32(const float (&y)[32]) {
  float a[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) a[i] = fmaxf(y[i], y[i + 16]);
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = fmaxf(a[i], a[i + 8]);
#pragma unroll
  for (int i = 0; i < 4; ++i) a[i] = fmaxf(a[i], a[i + 4]);
  return fmaxf(fmaxf(a[0], a[2]), fmaxf(a[1], a[3]));
}

// Online update of the row state with 32 consecutive columns (fixed order, fixed tree).
// Log2 domain with c = RN(log2(e) / T) > 0.  The running max is kept on the raw fp32 accumulators
// (mz), and t = RN(RN(z - mz) c) is the column's log2 weight relative to it: the column holding
// the max has t = 0 exactly, so its weight is ex2(0) = 1 exactly and a one-column vocabulary gives
// logp = 0 and H = 0 exactly (reading U16).  (Subtract-then-scale cannot be contracted
// into an FMA; ptxas does contract a packed mul.rn.f32x2 + add.rn.f32x2 pair, so y - m formed as
// RN(z c) - m would silently become fma(z, c, -m).)  The slice partial stores m = RN(mz c), the
// same rounding as the gathered y_a = RN(z_a c).  Per logit FMNMX(3) + FADD + FMUL + MUFU.EX2 +
// FADD + FFMA, in packed pairs.
template <bool kTail>
__device__ __forceinline__ void epi_chunk(const uint32_t (&r)[32], float c, int col0, int vocab, int64_t a,
                                          float& mz, float& s, float& u, float& ya) {
  float z[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    z[i] = __uint_as_float(r[i]);
    if (kTail && col0 + i >= vocab) z[i] = -CUDART_INF_F;
  }
  const float zmax = chunk_max32(z);
  const int64_t rel = a - col0;
  if (static_cast<uint64_t>(rel) < 32u) {
#pragma unroll
    for (int i = 0; i < 32; ++i)
      if (rel == i) ya = z[i] * c;
  }
  if (zmax > mz) {
    const float dm = __fmul_rn(__fsub_rn(mz, zmax), c);  // -inf on the first chunk of a slice
    const float sc = ex2_approx(dm);
    u = (s > 0.f) ? sc * fmaf(s, dm, u) : 0.f;
    s = s * sc;
    mz = zmax;
  }
  // four partial sums per quantity (column i goes to i mod 4, ascending i), two at a time in
  // packed fp32 pairs: the same per-lane operations as four scalar chains
  float2 s01 = make_float2(0.f, 0.f), s23 = s01, u01 = s01, u23 = s01;
  const float2 c2 = make_float2(c, c), nmz2 = make_float2(-mz, -mz);
#pragma unroll
  for (int i = 0; i < 32; i += 2) {
    float2 t = fmul2(fadd2(make_float2(z[i], z[i + 1]), nmz2), c2);
    if (kTail) {  // masked column: e = 0, e * t = 0 (no -inf * 0)
      t.x = fmaxf(t.x, -256.f);
      t.y = fmaxf(t.y, -256.f);
    }
    const float2 e = make_float2(ex2_approx(t.x), ex2_approx(t.y));
    if ((i & 3) == 0) {
      s01 = fadd2(s01, e);
      u01 = ffma2(e, t, u01);
    } else {
      s23 = fadd2(s23, e);
      u23 = ffma2(e, t, u23);
    }
  }
  s += (s01.x + s01.y) + (s23.x + s23.y);
  u += (u01.x + u01.y) + (u23.x + u23.y);
}

// First vocab tile of local slice j: global slice slice0 + j of the fixed split of n_vt tiles into
// n_slices_total slices (a function of V only -- the numerics contract).  A tensor-parallel rank
// runs a contiguous subset of the slices against its shard of W (rows from w_row0 on).
__device__ __forceinline__ int slice_tile(const LogprobParams& p, int j) {
  return ((p.slice0 + j) * p.n_vt) / p.n_slices_total;
}

__device__ __forceinline__ uint64_t make_policy(int kind) {
  return kind == 3 ? policy_evict_last() : kind == 2 ? policy_evict_first() : policy_evict_normal();
}

// ---------------------------------------------------------------- sampling twin (NEXT-1) --
// Counter-based Philox4x32-10 (Salmon et al., SC'11): multipliers 0xD2511F53 / 0xCD9E8D57,
// Weyl key increments 0x9E3779B9 / 0xBB67AE85.
// The key schedule (k0 + r W0, k1 + r W1) is the same for every block of the kernel: it is
// expanded once (PhiloxKeys, warp-uniform) instead of per call.
struct PhiloxKeys {
  uint32_t k0[10], k1[10];
  __device__ __forceinline__ PhiloxKeys(uint32_t a, uint32_t b) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
      k0[r] = a;
      k1[r] = b;
      a += 0x9E3779B9u;
      b += 0xBB67AE85u;
    }
  }
};
__device__ __forceinline__ uint4 philox4x32_10(uint4 c, const PhiloxKeys& k) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t hi0 = __umulhi(0xD2511F53u, c.x), lo0 = 0xD2511F53u * c.x;
    const uint32_t hi1 = __umulhi(0xCD9E8D57u, c.z), lo1 = 0xCD9E8D57u * c.z;
    c = make_uint4(hi1 ^ c.y ^ k.k0[r], lo1, hi0 ^ c.w ^ k.k1[r], lo0);
  }
  return c;
}
__device__ __forceinline__ float lg2_approx(float x) {
  float y;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// Gumbel-max over 32 columns in the log2 domain: score = y - log2(-log2 u) (the Gumbel noise in
// log2 units up to a constant), u = ((x >> 9) + 1/2) 2^-23 from Philox block (col / 4, 0, key
// lo, key hi) under the seed.  y = RN(z c) exactly as tim_logprob's gather, so the sampled
// token's log-prob is bit-identical to tim_logprob's.  Strict '>' in ascending column order:
// ties go to the lowest column.
template <bool kTail>
__device__ __forceinline__ void gumbel_chunk(const uint32_t (&r)[32], float c, int col0, int vocab,
                                             const PhiloxKeys& keys, uint32_t rk_lo, uint32_t rk_hi, float& best_s,
                                             float& best_y, int& best_col) {
#pragma unroll
  for (int g = 0; g < 8; ++g) {
    const uint4 x = philox4x32_10(make_uint4(static_cast<uint32_t>(col0 >> 2) + g, 0u, rk_lo, rk_hi), keys);
    const uint32_t xs[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
    for (int q = 0; q < 4; q += 2) {
      const int i = 4 * g + q;
      // u = ((x >> 9) + 1/2) 2^-23 exactly: 1.f with the 23 mantissa bits (x >> 9), minus
      // (1 - 2^-24) (Sterbenz: exact) -- no int->float conversion on the XU pipe.  Two columns
      // per packed fp32 op (each lane the scalar IEEE op).
      const float2 u = fsub2(make_float2(__uint_as_float(0x3f800000u | (xs[q] >> 9)),
                                         __uint_as_float(0x3f800000u | (xs[q + 1] >> 9))),
                             make_float2(0x1.fffffep-1f, 0x1.fffffep-1f));
      const float2 y = fmul2(make_float2(__uint_as_float(r[i]), __uint_as_float(r[i + 1])), make_float2(c, c));
      const float2 sc = fsub2(y, make_float2(lg2_approx(-lg2_approx(u.x)), lg2_approx(-lg2_approx(u.y))));
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        float sch = h ? sc.y : sc.x;
        if (kTail && col0 + i + h >= vocab) sch = -CUDART_INF_F;
        if (sch > best_s) {
          best_s = sch;
          best_y = h ? y.y : y.x;
          best_col = col0 + i + h;
        }
      }
    }
  }
}

// Static unit schedule (changes only WHICH pair runs a unit, never any row's arithmetic).
// Pairs form groups of G (G | S_v): in full round r, group q owns M-tile r*ngrp + q and its
// member g sweeps slices [g S_v/G, (g+1) S_v/G) -- vocab tiles in ascending order, so all pairs
// with the same g read the same W tile at the same step, and the ngrp live H tiles (1 MB each at
// d = 2048: G = 1; 2 MB at d = 4096: G = 2 keeps 74 MB live) stay hot in L2 for the whole sweep.
// The remaining M-tiles are split into (M-tile, slice) units dealt round-robin, slice-major.
struct UnitSched {
  int rounds, rem, ncl, S, G, ngrp, per_round;
  __device__ UnitSched(int n_mt, int n_slices, int n_clusters, int group)
      : ncl(n_clusters), S(n_slices), G(group) {
    ngrp = n_clusters / group;
    rounds = n_mt / ngrp;
    rem = n_mt - rounds * ngrp;
    per_round = n_slices / group;
  }
  __device__ __forceinline__ bool unit(int c, int k, int& mt, int& j) const {
    const int kfull = c < ngrp * G ? rounds * per_round : 0;
    if (k < kfull) {
      mt = (k / per_round) * ngrp + c / G;
      j = (c % G) * per_round + k % per_round;
      return true;
    }
    const int q = c + (k - kfull) * ncl;
    if (q >= rem * S) return false;
    j = q / rem;
    mt = rounds * ngrp + q % rem;
    return true;
  }
  // unit k is the last one pair c runs on its current M-tile (full rounds only)
  __device__ __forceinline__ bool last_of_mtile(int c, int k) const {
    return c < ngrp * G && k < rounds * per_round && (k % per_round) == per_round - 1;
  }
};

__device__ __forceinline__ void st_relaxed_gpu(uint32_t* p, uint32_t v) {
  asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_relaxed_gpu(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// Whole producer warp: wait (at most ~200 us) until every pair has issued `target` tiles.
// Returns the observed minimum.  Only a throttle -- never needed for correctness.
__device__ __noinline__ uint32_t wait_progress(const uint32_t* prog, uint32_t ncl, uint32_t target, int lane) {
  const uint64_t t0 = globaltimer_ns();
  uint32_t mn;
  while (true) {
    mn = 0xFFFFFFFFu;
    for (uint32_t c = lane; c < ncl; c += 32) {
      const uint32_t v = ld_relaxed_gpu(prog + c);
      mn = v < mn ? v : mn;
    }
    mn = __reduce_min_sync(0xffffffffu, mn);
    if (mn >= target || globaltimer_ns() - t0 > 200000ull) break;
    __nanosleep(256);
  }
  return mn;
}

// kNP = CTA pairs per cluster: 1 (cluster of 2) or 2 (cluster of 4: the two pairs own different
// M-tiles, sweep the same vocab tiles in lock-step and share every W tile through TMA multicast).
// ------------------------------------------------------------ head backward (NEXT-3) --
// G[t, v] = dL/dz[t, v] = (1/T) [ g (1[v = a] - p) - e p (ln p + H) ] for L = sum_t g_t logp_t +
// e_t H_t, with p = 2^(y - lse2) from the forward's log2-sum-exp; written as bf16 to the G block
// (row-major, ld = p.g_ld) for the two library GEMMs dH = G W and dW = G^T H: each warp stages
// its 32 rows x 32 columns in shared memory and one lane writes the tile with a TMA store
// (tmap_g), instead of 32 scattered 64-B row segments per chunk.
// G[t, v] = (g (1[v = a] - p) - e p (ln p + H)) / T per logit, with the row constants folded
// (gA = -e ln2 / T, gB = (-g - e H) / T, gS = g / T):  G = p (gA log2 p + gB) + 1[v = a] gS --
// two FFMAs, an EX2 and a select per logit; `rel` = a - col0 when a falls in this chunk, else -1.
__device__ __forceinline__ void grad_chunk(const uint32_t (&r)[32], float c, int rel, float gA, float gB, float gS,
                                           float lse2, uint32_t stage, int lane) {
  uint32_t packed[16];
#pragma unroll
  for (int i = 0; i < 32; i += 2) {
    float gv[2];
    const float2 t = ffma2(make_float2(__uint_as_float(r[i]), __uint_as_float(r[i + 1])), make_float2(c, c),
                           make_float2(-lse2, -lse2));  // log2 p
    const float2 pr = make_float2(ex2_approx(t.x), ex2_approx(t.y));
    const float2 g2 = ffma2(pr, ffma2(t, make_float2(gA, gA), make_float2(gB, gB)),
                            make_float2(rel == i ? gS : 0.f, rel == i + 1 ? gS : 0.f));
    gv[0] = g2.x;
    gv[1] = g2.y;
    const __nv_bfloat162 b = __floats2bfloat162_rn(gv[0], gv[1]);
    packed[i / 2] = *reinterpret_cast<const uint32_t*>(&b);
  }
  // this row's 64 B into the warp's 32 x 32 bf16 staging tile, 16-B chunks swizzled as the
  // tensor map's SWIZZLE_64B expects (chunk ^ ((row >> 1) & 3)): conflict-free shared stores
#pragma unroll
  for (int v = 0; v < 4; ++v) {
    const uint32_t addr = stage + lane * 64 + ((v ^ ((lane >> 1) & 3)) << 4);
    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(packed[4 * v]), "r"(packed[4 * v + 1]),
                 "r"(packed[4 * v + 2]), "r"(packed[4 * v + 3])
                 : "memory");
  }
}

template <bool kPair, bool kDebug, bool kSample, int kNP, bool kGrad = false>
__global__ void __launch_bounds__(kThreads, 1)
    logprob_fwd_kernel(const __grid_constant__ CUtensorMap tmap_h, const __grid_constant__ CUtensorMap tmap_w,
                       const __grid_constant__ CUtensorMap tmap_g, LogprobParams p) {
  using C = KCfg<kPair>;
  static_assert(kNP == 1 || (kPair && kNP == 2), "multicast clusters are built from CTA pairs");
#ifndef TIM_EPI_PREFETCH
#define TIM_EPI_PREFETCH 0
#endif
  // software-pipelined TMEM loads in the epilogue (0 = off, the default: measured slower for the
  // sampling twin and neutral for the forward); 1 = sampling twin, 2 = also the forward
  constexpr bool kPrefetch = !kGrad && !kDebug && (kSample ? TIM_EPI_PREFETCH >= 1 : TIM_EPI_PREFETCH >= 2);
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* smem_a = smem;
  uint8_t* smem_b = smem + C::kStages * C::kABytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::kStages * C::kStageBytes);
  uint64_t* full = bars;
  uint64_t* empty = bars + C::kStages;
  uint64_t* tfull = bars + 2 * C::kStages;
  uint64_t* tempty = bars + 2 * C::kStages + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * C::kStages + 4);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = kPair ? cluster_ctarank() : 0u;
  const uint32_t prank = rank & 1u;      // rank inside the CTA pair
  const uint32_t pid = rank >> 1;        // pair inside the cluster
  const uint32_t pl = rank & ~1u;        // rank of this pair's leader CTA
  const bool leader = prank == 0;
  if (blockIdx.x == 0 && threadIdx.x == 0 && p.clk) {  // the SM clock actually sustained (diagnostics)
    p.clk[0] = static_cast<unsigned long long>(clock64());
    p.clk[1] = globaltimer_ns();
  }
  const uint32_t cid = kPair ? cluster_id_x() : blockIdx.x;
  const uint32_t ncl = kPair ? ncluster_x() : gridDim.x;
  // Die-aware grouping (G > 1, schedule only -- no row's arithmetic depends on it): the pair takes
  // a virtual cluster id from its die's end of [0, ncl) -- die 0 counts up from 0, die 1 down from
  // ncl - 1 -- so consecutive virtual ids, which form the M-tile groups, sit on one die (at most one
  // group straddles) and each group's H tile lives in one die's L2.  Any die split is a valid
  // permutation of [0, ncl).  The id goes to both CTAs of the pair through shared::cluster.
  const bool remap = kPair && kNP == 1 && p.die_ok && p.group > 1;
  uint32_t* vslot = reinterpret_cast<uint32_t*>(bars + 2 * C::kStages + 4) + 1;

  if (threadIdx.x == 0) {
    for (int s = 0; s < C::kStages; ++s) {
      mbar_init(smem_u32(&full[s]), 1);
      mbar_init(smem_u32(&empty[s]), kNP);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(smem_u32(&tfull[a]), 1);
      mbar_init(smem_u32(&tempty[a]), kPair ? 2 * kEpiWarps : kEpiWarps);
    }
    fence_mbar_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmap_h);
    tma_prefetch(&tmap_w);
  }
  if (warp == 1) tmem_alloc<C::kCtaGroup>(smem_u32(tmem_slot), 512);
  if (remap && leader && threadIdx.x == 0) {
    const uint32_t sm = smid_reg();
    const uint32_t die = static_cast<uint32_t>(p.die_mask[(sm >> 6) & 3] >> (sm & 63)) & 1u;
    const uint32_t v = die == 0 ? atomicAdd(p.die_counter, 1u) : ncl - 1u - atomicAdd(p.die_counter + 1, 1u);
    *vslot = v;  // the peer CTA reads it through shared::cluster after the cluster barrier
  }
  tc_fence_before();
  if (kPair) cluster_sync(); else __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // the pair's id in the unit schedule: the leader CTA's slot (a DSMEM read, after the barrier
  // that guarantees the peer CTA has started and the leader's write is visible)
  const uint32_t vcid = !remap ? cid : (leader ? *vslot : ld_shared_cluster_u32(mapa(smem_u32(vslot), pl)));

  const int n_slices = p.n_slices;
  const int nkb = p.hidden / kBlockK;
  const UnitSched sched((p.n_mt + kNP - 1) / kNP, n_slices, ncl, p.group);

  if (warp == 0) {
    // ===================== TMA producer (whole warp; lane 0 issues) =====================
    uint32_t stage = 0, phase = 0;
    const uint64_t pol_h = make_policy(p.h_policy), pol_w = make_policy(p.w_policy);
    const bool hints = p.h_policy != 0 || p.w_policy != 0;
    const bool publish = kPair && rank == 0 && p.sync_slack > 0 && p.progress != nullptr;
    bool gate = publish;
    uint32_t step = 0, known_min = 0;
    int dm, j;
    for (int k = 0; sched.unit(vcid, k, dm, j); ++k) {
      const int mt = dm * kNP + pid;
      const int m0 = mt * C::kUnitM + prank * kCtaM;
      const int t0 = slice_tile(p, j), t1 = slice_tile(p, j + 1);
      for (int vt = t0; vt < t1; ++vt, ++step) {
        // bound the drift between pairs sweeping the same W tiles (performance only:
        // the wait is time-limited, results never depend on it)
        if (gate && static_cast<uint64_t>(step) > static_cast<uint64_t>(known_min) + p.sync_slack) {
          known_min = wait_progress(p.progress, ncl, step - p.sync_slack, lane);
          // a pair that never shows up (not co-resident: another kernel holds SMs, or a cluster
          // shape the GPU cannot place everywhere) must not throttle us: stop gating after a
          // timed-out wait
          if (known_min + p.sync_slack < step) {
            gate = false;
            if (lane == 0 && p.gate_stats) atomicAdd(p.gate_stats, 1ull);  // diagnostics: gates given up
          }
        }
        const int n0 = vt * kTileN - p.w_row0 + prank * C::kBRows + (kNP == 2 ? pid * (C::kBRows / 2) : 0);
        for (int kb = 0; kb < nkb; ++kb) {
          if (p.sleep_waits & 1) mbar_wait_sleep(smem_u32(&empty[stage]), phase ^ 1);
          else mbar_wait(smem_u32(&empty[stage]), phase ^ 1);
          if (kPair && kNP == 1 && hints) {
            // the default path, warp-wide: one elected lane issues (no single-lane issue loops)
            const uint32_t fb_local = smem_u32(&full[stage]);
            if (leader) mbar_arrive_expect_tx_elect(fb_local, 2 * C::kStageBytes);
            const uint32_t fb = mapa(fb_local, 0);
            tma_load_2d_pair_hint_elect(smem_u32(smem_a + stage * C::kABytes), &tmap_h, fb, kb * kBlockK, m0, pol_h);
            tma_load_2d_pair_hint_elect(smem_u32(smem_b + stage * C::kBBytes), &tmap_w, fb, kb * kBlockK, n0, pol_w);
          } else if (lane == 0) {
            const uint32_t fb_local = smem_u32(&full[stage]);
            const uint32_t a_dst = smem_u32(smem_a + stage * C::kABytes);
            const uint32_t b_dst = smem_u32(smem_b + stage * C::kBBytes);
            if (kNP == 2) {
              // own H rows -> own smem; half of the W half-tile this CTA and its counterpart in the
              // other pair both need -> multicast into both.  Bytes land on each destination's
              // pair-leader barrier (peer bit cleared), 64 KB per pair per stage as before.
              if (leader) mbar_arrive_expect_tx(fb_local, 2 * C::kStageBytes);
              const uint32_t fb_pair = fb_local & 0xFEFFFFFFu;
              const uint16_t mc = static_cast<uint16_t>((1u << prank) | (1u << (prank + 2)));
              tma_load_2d_pair_hint(a_dst, &tmap_h, mapa(fb_local, pl), kb * kBlockK, m0, pol_h);
              tma_load_2d_pair_mc_hint(b_dst + pid * (C::kBBytes / 2), &tmap_w, fb_pair, mc, kb * kBlockK, n0,
                                       pol_w);
            } else if (kPair) {
              if (leader) mbar_arrive_expect_tx(fb_local, 2 * C::kStageBytes);
              const uint32_t fb = mapa(fb_local, 0);
              if (hints) {
                tma_load_2d_pair_hint(a_dst, &tmap_h, fb, kb * kBlockK, m0, pol_h);
                tma_load_2d_pair_hint(b_dst, &tmap_w, fb, kb * kBlockK, n0, pol_w);
              } else {
                tma_load_2d_pair(a_dst, &tmap_h, fb, kb * kBlockK, m0);
                tma_load_2d_pair(b_dst, &tmap_w, fb, kb * kBlockK, n0);
              }
            } else {
              mbar_arrive_expect_tx(fb_local, C::kStageBytes);
              tma_load_2d(a_dst, &tmap_h, fb_local, kb * kBlockK, m0);
              tma_load_2d(b_dst, &tmap_w, fb_local, kb * kBlockK, n0);
            }
          }
          __syncwarp();
          if (++stage == C::kStages) { stage = 0; phase ^= 1; }
        }
        if (publish && lane == 0) st_relaxed_gpu(p.progress + vcid, step + 1);
      }
      // This CTA has issued its last load of the M-tile (end of its slice range in a full round):
      // demote its H rows from evict_last to evict_normal so dead tiles do not crowd W out of L2.
      if (p.demote && sched.last_of_mtile(vcid, k)) {
        const int rows = min(kCtaM, p.n_tok - m0);
        const int lines_per_row = p.hidden / 64;  // 128-B lines of one bf16 row
        const uint8_t* base = static_cast<const uint8_t*>(p.hidden_ptr);
        for (int e = lane; e < rows * lines_per_row; e += 32) {
          const int rr = e / lines_per_row, ll = e % lines_per_row;
          l2_demote(base + static_cast<int64_t>(m0 + rr) * p.ld_hidden_bytes + ll * 128);
        }
      }
    }
    if (publish && lane == 0) st_relaxed_gpu(p.progress + vcid, 0xFFFFFFFFu);
  } else if (warp == 1) {
    // ===================== MMA issuer (the leader CTA's warp 1) =====================
    // The whole warp runs the loop (warp-uniform waits and descriptors); one lane issues each
    // tcgen05 instruction (elect.sync).  Shared-memory descriptors advance by constants: stage s
    // and K-step kk of operand A start at a0 + s * kABytes + kk * 32 bytes, i.e. the descriptor's
    // address field (bits 0-13, address >> 4) plus s * kABytes / 16 + 2 kk.
    if (leader) {
      const uint32_t idesc = umma_idesc_bf16_f32(kPair ? 256 : 128, kTileN);
      const uint16_t mask_empty = kNP == 2 ? 0xF : (kPair ? 0x3 : 0x1);
      const uint16_t mask_full = static_cast<uint16_t>((kPair ? 0x3 : 0x1) << pl);
      const uint64_t desc_a0 = umma_desc_sw128(smem_u32(smem_a));
      const uint64_t desc_b0 = umma_desc_sw128(smem_u32(smem_b));
      uint32_t stage = 0, phase = 0, acc = 0, aphase = 0;
      int dm, j;
      for (int k = 0; sched.unit(vcid, k, dm, j); ++k) {
        const int t0 = slice_tile(p, j), t1 = slice_tile(p, j + 1);
        for (int vt = t0; vt < t1; ++vt) {
          if (p.sleep_waits & 4) mbar_wait_sleep(smem_u32(&tempty[acc]), aphase ^ 1);
          else mbar_wait(smem_u32(&tempty[acc]), aphase ^ 1);
          tc_fence_after();
          const uint32_t d_tmem = tmem_base + acc * kTileN;
          for (int kb = 0; kb < nkb; ++kb) {
            if (p.sleep_waits & 4) mbar_wait_sleep(smem_u32(&full[stage]), phase);
            else mbar_wait(smem_u32(&full[stage]), phase);
            tc_fence_after();
            const uint64_t da = desc_a0 + stage * (C::kABytes >> 4);
            const uint64_t db = desc_b0 + stage * (C::kBBytes >> 4);
#pragma unroll
            for (int kk = 0; kk < kBlockK / kUmmaK; ++kk)
              umma_bf16_elect<C::kCtaGroup>(d_tmem, da + 2 * kk, db + 2 * kk, idesc, (kb | kk) != 0);
            umma_commit_mc_elect<C::kCtaGroup>(smem_u32(&empty[stage]), mask_empty);
            if (++stage == C::kStages) { stage = 0; phase ^= 1; }
          }
          umma_commit_mc_elect<C::kCtaGroup>(smem_u32(&tfull[acc]), mask_full);
          acc ^= 1;
          if (acc == 0) aphase ^= 1;
        }
      }
    }
  } else {
    // ===================== epilogue warps: TMEM -> registers -> online LSE =====================
    const int q = warp & 3;  // TMEM lane quadrant this warp may access
    const int row_in_cta = q * 32 + lane;
    const uint32_t tempty_leader = kPair ? mapa(smem_u32(tempty), pl) : smem_u32(tempty);
    uint32_t acc = 0, aphase = 0;
    // gradient mode: two 2-KB staging tiles per epilogue warp (1024-B aligned for the swizzle)
    const uint32_t gstage0 =
        kGrad ? ((smem_u32(smem + C::kStages * C::kStageBytes + 256) + 1023u) & ~1023u) + (warp - 2) * 4096u : 0u;
    int gbuf = 0;
    int dm, j;
    for (int k = 0; sched.unit(vcid, k, dm, j); ++k) {
      const int mt = dm * kNP + pid;
      const int row = mt * C::kUnitM + prank * kCtaM + row_in_cta;
      const bool valid = row < p.n_tok;
      const int64_t a = (valid && p.ids) ? __ldg(p.ids + row) : int64_t(-1);
      const float T = (valid && p.temps) ? __ldg(p.temps + row) : p.temperature;
      const float c = __fdiv_rn(kLog2eF, T);
      float m = -CUDART_INF_F, s = 0.f, uu = 0.f, ya = -CUDART_INF_F;  // m: running max of the raw z
      float gA = 0.f, gB = 0.f, gS = 0.f, lse2 = 0.f;  // gradient mode (NEXT-3): grad_chunk's row constants
      if (kGrad && valid) {
        const float gl = __ldg(p.grad_logp + row);
        const float ge = p.grad_ent ? __ldg(p.grad_ent + row) : 0.f;
        const float gH = __ldg(p.ent_in + row);
        const float invT = __fdiv_rn(1.0f, T);
        constexpr float kLn2 = 0.69314718055994530942f;
        lse2 = __ldg(p.lse2_in + row);
        gA = -ge * kLn2 * invT;
        gB = (-gl - ge * gH) * invT;
        gS = gl * invT;
      }
      float best_s = -CUDART_INF_F, best_y = -CUDART_INF_F;
      int best_col = -1;
      uint32_t rk_lo = 0, rk_hi = 0;
      if (kSample && valid) {
        const uint64_t rk = __ldg(reinterpret_cast<const unsigned long long*>(p.row_keys) + row);
        rk_lo = static_cast<uint32_t>(rk);
        rk_hi = static_cast<uint32_t>(rk >> 32);
      }
      const int t0 = slice_tile(p, j), t1 = slice_tile(p, j + 1);
      for (int vt = t0; vt < t1; ++vt) {
        if (p.sleep_waits & 2) mbar_wait_sleep(smem_u32(&tfull[acc]), aphase);
        else mbar_wait(smem_u32(&tfull[acc]), aphase);
        tc_fence_after();
        const uint32_t taddr = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + acc * kTileN;
        const bool tail_tile = (vt + 1) * kTileN > p.vocab;
        auto chunk = [&](const uint32_t (&r)[32], int ch) {
          const int col0 = vt * kTileN + ch * 32;
          if (kDebug && valid) {
            float* dst = p.debug_logits + static_cast<int64_t>(row) * p.debug_ld + col0;
#pragma unroll
            for (int i = 0; i < 32; ++i)
              if (col0 + i < p.vocab) dst[i] = __uint_as_float(r[i]);
          }
          if (kGrad) {
            const uint32_t stage = gstage0 + gbuf * 2048u;
            if (lane == 0) bulk_wait_group_read<1>();  // this buffer's previous store has read it
            __syncwarp();
            const int64_t rel64 = a - col0;
            grad_chunk(r, c, static_cast<uint64_t>(rel64) < 32u ? static_cast<int>(rel64) : -1, gA, gB, gS, lse2,
                       stage, lane);
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) {
              // G streams out (4 GiB per block): evict_first keeps the W slice resident in L2
              tma_store_2d_hint(&tmap_g, stage, col0 - p.g_col0, row - lane, policy_evict_first());
              bulk_commit_group();
            }
            gbuf ^= 1;
          } else if (tail_tile)
            epi_chunk<true>(r, c, col0, p.vocab, a, m, s, uu, ya);
          else
            epi_chunk<false>(r, c, col0, p.vocab, a, m, s, uu, ya);
          if (kSample) {
            const PhiloxKeys keys(static_cast<uint32_t>(p.seed), static_cast<uint32_t>(p.seed >> 32));
            if (tail_tile)
              gumbel_chunk<true>(r, c, col0, p.vocab, keys, rk_lo, rk_hi, best_s, best_y, best_col);
            else
              gumbel_chunk<false>(r, c, col0, p.vocab, keys, rk_lo, rk_hi, best_s, best_y, best_col);
          }
        };
        auto release = [&]() {  // every TMEM load of this tile has landed: the MMA may overwrite it
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive_cluster(tempty_leader + acc * 8);
        };
        if constexpr (kPrefetch) {
          // the next chunk's TMEM load is in flight while this chunk computes
          uint32_t ra[32], rb[32];
          tmem_ld_32x32b_x32(taddr, ra);
#pragma unroll 1
          for (int ch = 0; ch < kTileN / 32; ch += 2) {
            tmem_ld_wait_regs(ra);
            tmem_ld_32x32b_x32(taddr + (ch + 1) * 32, rb);
            chunk(ra, ch);
            tmem_ld_wait_regs(rb);
            if (ch + 2 < kTileN / 32) tmem_ld_32x32b_x32(taddr + (ch + 2) * 32, ra);
            else release();
            chunk(rb, ch + 1);
          }
        } else {
#pragma unroll 1
          for (int ch = 0; ch < kTileN / 32; ++ch) {
            uint32_t r[32];
            tmem_ld_32x32b_x32(taddr + ch * 32, r);
            tmem_ld_wait();
            if (ch == kTileN / 32 - 1) release();
            chunk(r, ch);
          }
        }
        acc ^= 1;
        if (acc == 0) aphase ^= 1;
      }
      if (valid && !kGrad) {
        // m = RN(mz c): the slice max in log2 units, rounded like the gathered y_a
        p.partials[static_cast<int64_t>(j) * p.n_tok + row] = make_float4(__fmul_rn(m, c), s, uu, ya);
        if (kSample)
          p.partials2[static_cast<int64_t>(j) * p.n_tok + row] =
              make_float4(best_s, best_y, __int_as_float(best_col), 0.f);
      }
    }
  }

  if (blockIdx.x == 0 && threadIdx.x == 0 && p.clk) {
    p.clk[2] = static_cast<unsigned long long>(clock64());
    p.clk[3] = globaltimer_ns();
  }
  if (kGrad && warp >= 2 && lane == 0) bulk_wait_group_all();  // the G tiles are written
  __syncwarp();
  tc_fence_before();
  if (kPair) cluster_sync(); else __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<C::kCtaGroup>(tmem_base, 512);
  }
}

// a4: fixed-order merge of the S_v slice partials of every token (fp64), id / temperature checks.
__global__ void __launch_bounds__(256) logprob_merge_kernel(MergeParams p) {
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t < p.n_tok) {
    double M = -CUDART_INF;
    for (int j = 0; j < p.n_slices; ++j) M = fmax(M, static_cast<double>(p.partials[j * p.n_tok + t].x));
    double S = 0.0, U = 0.0, ya = -CUDART_INF;
    for (int j = 0; j < p.n_slices; ++j) {
      const float4 q = p.partials[j * p.n_tok + t];
      const double dm = static_cast<double>(q.x) - M;
      const double w = exp2(dm);
      S = S + static_cast<double>(q.y) * w;
      U = U + w * (static_cast<double>(q.z) + static_cast<double>(q.y) * dm);
      if (q.w > -CUDART_INF_F) ya = static_cast<double>(q.w);
    }
    const int64_t a = p.ids[t];
    bool bad = a < 0 || a >= p.vocab;
    if (p.temps) {
      const float T = p.temps[t];
      bad = bad || !(T > 0.f) || !isfinite(T);
    }
    const double l2s = log2(S);
    const double kLn2 = 0.69314718055994530942;
    if (p.lse2_out) p.lse2_out[t] = static_cast<float>(M + l2s);
    p.logp[t] = bad ? CUDART_NAN_F : static_cast<float>(kLn2 * ((ya - M) - l2s));
    if (p.entropy) p.entropy[t] = static_cast<float>(kLn2 * (l2s - U / S));
    if (bad) atomicMax(reinterpret_cast<unsigned long long*>(&p.ws->bad_inv),
                       static_cast<unsigned long long>(kBadSentinel - (t + p.index_base)));
  }
  commit_status_last_block(p.ws, p.dstatus);
}

// a4 for the sampling twin: same merge; the sampled column is the best Gumbel score over the
// slices in slice order (strict '>': ties go to the lowest slice, i.e. the lowest column), and
// its log-prob uses that column's y exactly as tim_logprob's gather would.
__global__ void __launch_bounds__(256) sample_merge_kernel(MergeParams p) {
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t < p.n_tok) {
    double M = -CUDART_INF;
    for (int j = 0; j < p.n_slices; ++j) M = fmax(M, static_cast<double>(p.partials[j * p.n_tok + t].x));
    double S = 0.0, U = 0.0;
    float bs = -CUDART_INF_F, by = -CUDART_INF_F;
    int bc = -1;
    for (int j = 0; j < p.n_slices; ++j) {
      const float4 q = p.partials[j * p.n_tok + t];
      const double dm = static_cast<double>(q.x) - M;
      const double w = exp2(dm);
      S = S + static_cast<double>(q.y) * w;
      U = U + w * (static_cast<double>(q.z) + static_cast<double>(q.y) * dm);
      const float4 g = p.partials2[j * p.n_tok + t];
      if (g.x > bs) {
        bs = g.x;
        by = g.y;
        bc = __float_as_int(g.z);
      }
    }
    bool bad = bc < 0;
    if (p.temps) {
      const float T = p.temps[t];
      bad = bad || !(T > 0.f) || !isfinite(T);
    }
    const double l2s = log2(S);
    const double kLn2 = 0.69314718055994530942;
    p.ids_out[t] = bad ? -1 : bc;
    p.logp[t] = bad ? CUDART_NAN_F : static_cast<float>(kLn2 * ((static_cast<double>(by) - M) - l2s));
    if (p.entropy) p.entropy[t] = static_cast<float>(kLn2 * (l2s - U / S));
    if (bad) atomicMax(reinterpret_cast<unsigned long long*>(&p.ws->bad_inv),
                       static_cast<unsigned long long>(kBadSentinel - t));
  }
  commit_status_last_block(p.ws, p.dstatus);
}

template <bool kPair, bool kDebug, bool kSample, int kNP, bool kGrad = false>
static cudaError_t launch_fwd(const CUtensorMap& th, const CUtensorMap& tw, const LogprobParams& p, int grid,
                              cudaStream_t stream, const CUtensorMap* tg = nullptr) {
  using C = KCfg<kPair>;
  auto kern = logprob_fwd_kernel<kPair, kDebug, kSample, kNP, kGrad>;
  // gradient mode: + 1 KB alignment slack and 4 warps x 2 x 2 KB G staging tiles
  constexpr int kSmem = C::kSmemBytes + (kGrad ? 1024 + kEpiWarps * 4096 : 0);
  // the attribute is per device: a process driving several GPUs sets it once on each
  static std::atomic<bool> attr_set[kMaxDevices];
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev < 0 || dev >= kMaxDevices) return cudaErrorInvalidDevice;
  if (!attr_set[dev].load()) {
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
    if (e != cudaSuccess) return e;
    attr_set[dev].store(true);
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = kSmem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = kPair ? 2 * kNP : 1;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, th, tw, tg ? *tg : th, p);
}

int fwd_unit_rows(bool pair) { return pair ? KCfg<true>::kUnitM : KCfg<false>::kUnitM; }
int fwd_w_box_rows(bool pair) { return pair ? KCfg<true>::kBRows : KCfg<false>::kBRows; }

// Small-batch H staging (api.cu small_pad_rows): rows [0, n_tok) copied, rows [n_tok, n_rows)
// zeroed, one block per row, 16-B vectors.  Pure data movement.
__global__ void __launch_bounds__(256) pad_rows_kernel(const uint8_t* __restrict__ src, int64_t ld_src_bytes,
                                                       uint8_t* __restrict__ dst, int row_bytes, int n_tok) {
  const int row = blockIdx.x;
  uint4* d = reinterpret_cast<uint4*>(dst + static_cast<int64_t>(row) * row_bytes);
  const uint4* sp = reinterpret_cast<const uint4*>(src + static_cast<int64_t>(row) * ld_src_bytes);
  for (int i = threadIdx.x; i < row_bytes / 16; i += blockDim.x)
    d[i] = row < n_tok ? __ldg(sp + i) : make_uint4(0u, 0u, 0u, 0u);
}
cudaError_t launch_pad_rows(const void* src, int64_t ld_src_bytes, void* dst, int row_bytes, int n_tok, int n_rows,
                            cudaStream_t stream) {
  pad_rows_kernel<<<n_rows, 256, 0, stream>>>(static_cast<const uint8_t*>(src), ld_src_bytes,
                                              static_cast<uint8_t*>(dst), row_bytes, n_tok);
  return cudaGetLastError();
}

cudaError_t launch_head_grad(const CUtensorMap& th, const CUtensorMap& tw, const CUtensorMap& tg,
                             const LogprobParams& p, int grid, cudaStream_t stream) {
  return launch_fwd<true, false, false, 1, true>(th, tw, p, grid, stream, &tg);
}

cudaError_t launch_logprob_fwd(bool pair, bool debug, bool sample, bool quad, const CUtensorMap& th,
                               const CUtensorMap& tw, const LogprobParams& p, int grid, cudaStream_t stream) {
  if (quad) return sample ? launch_fwd<true, false, true, 2>(th, tw, p, grid, stream)
                          : (debug ? launch_fwd<true, true, false, 2>(th, tw, p, grid, stream)
                                   : launch_fwd<true, false, false, 2>(th, tw, p, grid, stream));
  if (sample) return pair ? launch_fwd<true, false, true, 1>(th, tw, p, grid, stream)
                          : launch_fwd<false, false, true, 1>(th, tw, p, grid, stream);
  if (pair) return debug ? launch_fwd<true, true, false, 1>(th, tw, p, grid, stream)
                         : launch_fwd<true, false, false, 1>(th, tw, p, grid, stream);
  return debug ? launch_fwd<false, true, false, 1>(th, tw, p, grid, stream)
               : launch_fwd<false, false, false, 1>(th, tw, p, grid, stream);
}

// One CTA per SM (the caller's shared-memory request keeps a second CTA off every SM): time 64
// dependent ld.global.cg of each zero-filled line after 4 warm-up loads (the chain's address
// depends on the loaded value, so nothing overlaps).
__global__ void __launch_bounds__(32) die_probe_kernel(const uint64_t* lines, int nlines, int stride_u64,
                                                       uint32_t* lat, uint32_t* smid) {
  if (threadIdx.x != 0) return;
  for (int l = 0; l < nlines; ++l) {
    const uint64_t* line = lines + static_cast<int64_t>(l) * stride_u64;
    uint64_t v = 0;
#pragma unroll 1
    for (int i = 0; i < 4; ++i) {
      uint64_t x;
      asm volatile("ld.global.cg.u64 %0, [%1];" : "=l"(x) : "l"(line + v));
      v += x;
    }
    const long long t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < 64; ++i) {
      uint64_t x;
      asm volatile("ld.global.cg.u64 %0, [%1];" : "=l"(x) : "l"(line + v));
      v += x;
    }
    const long long t1 = clock64();
    lat[blockIdx.x * nlines + l] = static_cast<uint32_t>((t1 - t0) / 64) + static_cast<uint32_t>(v);
  }
  smid[blockIdx.x] = smid_reg();
}

cudaError_t launch_die_probe(const uint64_t* lines, int nlines, int stride_u64, uint32_t* lat, uint32_t* smid,
                             int grid, cudaStream_t stream) {
  constexpr int kSmem = 160 * 1024;  // more than half of an SM's shared memory: one CTA per SM
  cudaError_t e = cudaFuncSetAttribute(die_probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
  if (e != cudaSuccess) return e;
  die_probe_kernel<<<grid, 32, kSmem, stream>>>(lines, nlines, stride_u64, lat, smid);
  return cudaGetLastError();
}

cudaError_t launch_sample_merge(const MergeParams& p, cudaStream_t stream) {
  const int blocks = static_cast<int>((p.n_tok + 255) / 256);
  sample_merge_kernel<<<blocks, 256, 0, stream>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_logprob_merge(const MergeParams& p, cudaStream_t stream) {
  const int blocks = static_cast<int>((p.n_tok + 255) / 256);
  logprob_merge_kernel<<<blocks, 256, 0, stream>>>(p);
  return cudaGetLastError();
}

}  // namespace tim
