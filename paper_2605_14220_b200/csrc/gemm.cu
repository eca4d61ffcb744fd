// gemm.cu -- the two GEMMs of the head backward (§3 P:474-478,
// the score-function gradient that flows through log pi_theta of the recomputed tokens):
//
//   dH[t, :] = sum_v G[t, v] W[v, :]      A = G   [tok x V]  K-major (K = V contiguous)
//                                         B = W   [V x d]    MN-major (N = d contiguous)
//   dW[v, :] += sum_t G[t, v] H[t, :]     A = G^T [V x tok]  MN-major (M = V contiguous in G)
//                                         B = H   [tok x d]  MN-major
//
// Hand-written tcgen05 kernel (no library GEMM): a persistent CTA pair (cta_group::2) owns a
// 256 x 256 output tile, operands staged by TMA (128-B swizzle; MN-major operands as 64-element
// x 64-K boxes whose 8-row K groups are 1024 B apart (SBO) and whose two 64-element MN chunks are
// 8 KB apart (LBO)), 6-stage shared-memory ring, tcgen05.mma kind::f16 M = 256 N = 256 K = 16
// into fp32 TMEM accumulators (two 256-column buffers: the MMA fills one while the epilogue
// drains the other), epilogue tcgen05.ld 32x32b -> registers -> global.
//
// Numerics.  Every output element is ONE fp32 tensor-core accumulation over K in ascending order
// from a zeroed accumulator, in K = 16 steps: a constant of (V, d) for dH -- so dH[t] depends only
// on row t of G and on W, never on the batch, the token block, the row slot or the grid (batch
// invariant, like the forward) -- and of the token-block size for dW.  dW accumulates the token
// blocks in block order through red.global.add (one add per element per launch, launches ordered
// on the stream): deterministic run to run.
#include <cuda.h>
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>

#include "ptx.cuh"
#include "tim_internal.h"

namespace tim {

namespace {

constexpr int kGBlockK = 64;    // K per pipeline stage
constexpr int kGUmmaK = 16;     // K per tcgen05.mma kind::f16
constexpr int kGCtaM = 128;     // output rows per CTA (TMEM lanes)
constexpr int kGTileN = 256;    // output columns per tile (MMA N; each CTA stages half of B)
constexpr int kGStages = 6;
constexpr int kGABytes = kGCtaM * kGBlockK * 2;          // 16 KB
constexpr int kGBBytes = (kGTileN / 2) * kGBlockK * 2;   // 16 KB
constexpr int kGStageBytes = kGABytes + kGBBytes;
constexpr int kGEpiWarps = 4;
constexpr int kGThreads = 64 + 32 * kGEpiWarps;
constexpr int kGSmemBytes = kGStages * kGStageBytes + 1024 + 256;
constexpr int kMnChunkBytes = 64 * kGBlockK * 2;          // one 64-element x 64-K MN-major box: 8 KB

// UMMA shared-memory descriptor of an MN-major operand in the 128-byte swizzle canonical layout
// (PTX ISA tcgen05 "matrix descriptors"; the canonical MN-major SW128 layout is, in 16-byte units,
// ((8, n), (8, k)) : ((1, LBO), (8, SBO))): 64 contiguous MN elements per 128-B row, 8 K rows per
// 1024-B swizzle atom, K groups SBO = 1024 B apart, MN chunks of 64 elements LBO apart.
__device__ __forceinline__ uint64_t umma_desc_sw128_mn(uint32_t smem_addr, uint32_t lbo_bytes) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((smem_addr >> 4) & 0x3FFFu);
  d |= static_cast<uint64_t>((lbo_bytes >> 4) & 0x3FFFu) << 16;
  d |= static_cast<uint64_t>(1024u >> 4) << 32;
  d |= static_cast<uint64_t>(1u) << 46;   // version 1 (sm_100)
  d |= static_cast<uint64_t>(2u) << 61;   // SWIZZLE_128B
  return d;
}

__device__ __forceinline__ void st_relaxed_u32(uint32_t* p, uint32_t v) {
  asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_relaxed_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint64_t gtimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// Whole producer warp: wait (at most ~200 us) until every pair has issued `target` k-blocks;
// returns the observed minimum.  A throttle only -- results never depend on it.
__device__ __noinline__ uint32_t gemm_wait_progress(const uint32_t* prog, uint32_t ncl, uint32_t target, int lane) {
  const uint64_t t0 = gtimer_ns();
  uint32_t mn;
  while (true) {
    mn = 0xFFFFFFFFu;
    for (uint32_t c = lane; c < ncl; c += 32) {
      const uint32_t v = ld_relaxed_u32(prog + c);
      mn = v < mn ? v : mn;
    }
    mn = __reduce_min_sync(0xffffffffu, mn);
    if (mn >= target || gtimer_ns() - t0 > 200000ull) break;
    __nanosleep(128);
  }
  return mn;
}

__device__ __forceinline__ uint64_t gemm_policy(int kind) {
  return kind == 3 ? policy_evict_last() : kind == 2 ? policy_evict_first() : policy_evict_normal();
}

__device__ __forceinline__ void red_add_v4(float* p, float a, float b, float c, float d) {
  asm volatile("red.relaxed.gpu.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(a), "f"(b), "f"(c), "f"(d)
               : "memory");
}
__device__ __forceinline__ void st_v4(float* p, float a, float b, float c, float d) {
  asm volatile("st.global.cs.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(a), "f"(b), "f"(c), "f"(d) : "memory");
}

// kAMN: operand A is MN-major (dW: A = G^T); otherwise K-major (dH: A = G).  B is always MN-major.
// kRed: accumulate into C with red.global.add (dW) instead of storing (dH).
template <bool kAMN, bool kRed>
__global__ void __launch_bounds__(kGThreads, 1)
    bwd_gemm_kernel(const __grid_constant__ CUtensorMap tmap_a, const __grid_constant__ CUtensorMap tmap_b,
                    BwdGemmParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* smem_a = smem;
  uint8_t* smem_b = smem + kGStages * kGABytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kGStages * kGStageBytes);
  uint64_t* full = bars;
  uint64_t* empty = bars + kGStages;
  uint64_t* tfull = bars + 2 * kGStages;
  uint64_t* tempty = bars + 2 * kGStages + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * kGStages + 4);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t prank = cluster_ctarank() & 1u;
  const bool leader = prank == 0;
  const uint32_t cid = cluster_id_x();
  const uint32_t ncl = ncluster_x();
  // die-aware virtual cluster ids (the forward kernel's scheme, logprob.cu): consecutive tiles
  // share an A stream (one M-tile, all N-tiles), so their pairs should share a die's L2
  const bool remap = p.die_ok != 0;
  uint32_t* vslot = tmem_slot + 1;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kGStages; ++s) {
      mbar_init(smem_u32(&full[s]), 1);
      mbar_init(smem_u32(&empty[s]), 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(smem_u32(&tfull[a]), 1);
      mbar_init(smem_u32(&tempty[a]), 2 * kGEpiWarps);
    }
    fence_mbar_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmap_a);
    tma_prefetch(&tmap_b);
  }
  if (warp == 1) tmem_alloc<2>(smem_u32(tmem_slot), 512);
  if (remap && leader && threadIdx.x == 0) {
    const uint32_t sm = smid_reg();
    const uint32_t die = static_cast<uint32_t>(p.die_mask[(sm >> 6) & 3] >> (sm & 63)) & 1u;
    const uint32_t v = die == 0 ? atomicAdd(p.die_counter, 1u) : ncl - 1u - atomicAdd(p.die_counter + 1, 1u);
    *vslot = v;  // the peer CTA reads it through shared::cluster after the cluster barrier
  }
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const uint32_t vcid =
      !remap ? cid : (leader ? *vslot : ld_shared_cluster_u32(mapa(smem_u32(vslot), cluster_ctarank() & ~1u)));

  const int n_nt = (p.n + kGTileN - 1) / kGTileN;
  const int n_tiles = ((p.m + 2 * kGCtaM - 1) / (2 * kGCtaM)) * n_nt;
  const int nkb = (p.k + kGBlockK - 1) / kGBlockK;

  if (warp == 0) {
    // ===================== TMA producer (whole warp; one elected lane issues) =====================
    uint32_t stage = 0, phase = 0;
    // L2 policies of the two operand streams (host-chosen, tim_debug_set_gemm_policy)
    const uint64_t pol_a = gemm_policy(p.a_policy);
    const uint64_t pol_b = gemm_policy(p.b_policy);
    // progress gate (performance only): the pairs sharing an A or B stream read the same k-block
    // within `sync_slack` k-blocks of each other, so a stream is fetched from DRAM about once per
    // wave instead of once per pair (ncu, dH at C1's 14080-token block: DRAM 22 -> 8.3 GB)
    const bool publish = prank == 0 && p.sync_slack > 0 && p.progress != nullptr;
    bool gate = publish;
    uint32_t step = 0, known_min = 0;
    for (int tile = static_cast<int>(vcid); tile < n_tiles; tile += static_cast<int>(ncl)) {
      const int mt = tile / n_nt, nt = tile % n_nt;
      const int m0 = mt * 2 * kGCtaM + static_cast<int>(prank) * kGCtaM;   // this CTA's A rows
      const int n0 = nt * kGTileN + static_cast<int>(prank) * (kGTileN / 2);  // this CTA's half of B
      for (int kb = 0; kb < nkb; ++kb, ++step) {
        if (gate && (step & 7u) == 0u) {
          if (lane == 0) st_relaxed_u32(p.progress + vcid, step);
          if (step > known_min + static_cast<uint32_t>(p.sync_slack)) {
            known_min = gemm_wait_progress(p.progress, ncl, step - p.sync_slack, lane);
            if (known_min + static_cast<uint32_t>(p.sync_slack) < step) gate = false;  // a pair never showed up
          }
        }
        mbar_wait(smem_u32(&empty[stage]), phase ^ 1);
        const uint32_t fb_local = smem_u32(&full[stage]);
        if (leader) mbar_arrive_expect_tx_elect(fb_local, 2 * kGStageBytes);
        const uint32_t fb = mapa(fb_local, 0);
        const uint32_t a_dst = smem_u32(smem_a + stage * kGABytes);
        const uint32_t b_dst = smem_u32(smem_b + stage * kGBBytes);
        const int k0 = kb * kGBlockK;
        if (kAMN) {  // G^T: box {64 vocab columns, 64 token rows} x 2
          tma_load_2d_pair_hint_elect(a_dst, &tmap_a, fb, m0, k0, pol_a);
          tma_load_2d_pair_hint_elect(a_dst + kMnChunkBytes, &tmap_a, fb, m0 + 64, k0, pol_a);
        } else {     // G: box {64 K columns, 128 token rows}
          tma_load_2d_pair_hint_elect(a_dst, &tmap_a, fb, k0, m0, pol_a);
        }
        tma_load_2d_pair_hint_elect(b_dst, &tmap_b, fb, n0, k0, pol_b);
        tma_load_2d_pair_hint_elect(b_dst + kMnChunkBytes, &tmap_b, fb, n0 + 64, k0, pol_b);
        __syncwarp();
        if (++stage == kGStages) { stage = 0; phase ^= 1; }
      }
    }
    if (publish && lane == 0) st_relaxed_u32(p.progress + vcid, 0xFFFFFFFFu);
  } else if (warp == 1) {
    // ===================== MMA issuer (the leader CTA's warp 1) =====================
    if (leader) {
      const uint32_t idesc = umma_idesc_bf16_f32(256, kGTileN) | (kAMN ? (1u << 15) : 0u) | (1u << 16);
      const uint64_t desc_a0 = kAMN ? umma_desc_sw128_mn(smem_u32(smem_a), kMnChunkBytes) : umma_desc_sw128(smem_u32(smem_a));
      const uint64_t desc_b0 = umma_desc_sw128_mn(smem_u32(smem_b), kMnChunkBytes);
      // K step of 16 inside a stage: K-major A advances 32 B along its 128-B rows (+2 in 16-B
      // units); MN-major operands advance 16 K rows = 2048 B (+128)
      constexpr uint32_t kAStep = kAMN ? 128u : 2u;
      constexpr uint32_t kBStep = 128u;
      uint32_t stage = 0, phase = 0, acc = 0, aphase = 0;
      for (int tile = static_cast<int>(vcid); tile < n_tiles; tile += static_cast<int>(ncl)) {
        mbar_wait(smem_u32(&tempty[acc]), aphase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * kGTileN;
        for (int kb = 0; kb < nkb; ++kb) {
          mbar_wait(smem_u32(&full[stage]), phase);
          tc_fence_after();
          const uint64_t da = desc_a0 + stage * (kGABytes >> 4);
          const uint64_t db = desc_b0 + stage * (kGBBytes >> 4);
#pragma unroll
          for (int kk = 0; kk < kGBlockK / kGUmmaK; ++kk)
            umma_bf16_elect<2>(d_tmem, da + kAStep * kk, db + kBStep * kk, idesc, (kb | kk) != 0);
          umma_commit_mc_elect<2>(smem_u32(&empty[stage]), 0x3);
          if (++stage == kGStages) { stage = 0; phase ^= 1; }
        }
        umma_commit_mc_elect<2>(smem_u32(&tfull[acc]), 0x3);
        acc ^= 1;
        if (acc == 0) aphase ^= 1;
      }
    }
  } else {
    // ===================== epilogue warps: TMEM -> registers -> global =====================
    const int q = warp & 3;
    const int row_in_cta = q * 32 + lane;
    const uint32_t tempty_leader = mapa(smem_u32(tempty), 0);
    uint32_t acc = 0, aphase = 0;
    for (int tile = static_cast<int>(vcid); tile < n_tiles; tile += static_cast<int>(ncl)) {
      const int mt = tile / n_nt, nt = tile % n_nt;
      const int row = mt * 2 * kGCtaM + static_cast<int>(prank) * kGCtaM + row_in_cta;
      const bool valid = row < p.m;
      float* crow = p.c + static_cast<int64_t>(valid ? row : 0) * p.ldc;
      mbar_wait(smem_u32(&tfull[acc]), aphase);
      tc_fence_after();
      const uint32_t taddr = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + acc * kGTileN;
#pragma unroll 1
      for (int ch = 0; ch < kGTileN / 32; ++ch) {
        uint32_t r[32];
        tmem_ld_32x32b_x32(taddr + ch * 32, r);
        tmem_ld_wait();
        if (ch == kGTileN / 32 - 1) {  // every TMEM load of this tile has landed: the MMA may reuse it
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive_cluster(tempty_leader + acc * 8);
        }
        const int col0 = nt * kGTileN + ch * 32;
        if (valid && col0 < p.n) {  // n % 64 == 0: a 32-column chunk is wholly in or out
          float* dst = crow + col0;
#pragma unroll
          for (int i = 0; i < 32; i += 4) {
            if (kRed)
              red_add_v4(dst + i, __uint_as_float(r[i]), __uint_as_float(r[i + 1]), __uint_as_float(r[i + 2]),
                         __uint_as_float(r[i + 3]));
            else
              st_v4(dst + i, __uint_as_float(r[i]), __uint_as_float(r[i + 1]), __uint_as_float(r[i + 2]),
                    __uint_as_float(r[i + 3]));
          }
        }
      }
      acc ^= 1;
      if (acc == 0) aphase ^= 1;
    }
  }

  __syncwarp();
  tc_fence_before();
  cluster_sync();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<2>(tmem_base, 512);
  }
}

template <bool kAMN, bool kRed>
cudaError_t launch_gemm(const CUtensorMap& ta, const CUtensorMap& tb, const BwdGemmParams& p, int max_pairs,
                        cudaStream_t stream) {
  auto kern = bwd_gemm_kernel<kAMN, kRed>;
  static std::atomic<bool> attr_set[kMaxDevices];
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev < 0 || dev >= kMaxDevices) return cudaErrorInvalidDevice;
  if (!attr_set[dev].load()) {
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kGSmemBytes);
    if (e != cudaSuccess) return e;
    attr_set[dev].store(true);
  }
  const long long tiles =
      static_cast<long long>((p.m + 2 * kGCtaM - 1) / (2 * kGCtaM)) * ((p.n + kGTileN - 1) / kGTileN);
  const long long pairs = tiles < max_pairs ? tiles : max_pairs;
  if (pairs < 1) return cudaSuccess;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(2 * pairs));
  cfg.blockDim = dim3(kGThreads);
  cfg.dynamicSmemBytes = kGSmemBytes;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, ta, tb, p);
}

}  // namespace

cudaError_t launch_bwd_gemm_dh(const CUtensorMap& tg_kmajor, const CUtensorMap& tw_mn, const BwdGemmParams& p,
                               int max_pairs, cudaStream_t stream) {
  return launch_gemm<false, false>(tg_kmajor, tw_mn, p, max_pairs, stream);
}

cudaError_t launch_bwd_gemm_dw(const CUtensorMap& tg_mn, const CUtensorMap& th_mn, const BwdGemmParams& p,
                               int max_pairs, cudaStream_t stream) {
  return launch_gemm<true, true>(tg_mn, th_mn, p, max_pairs, stream);
}

}  // namespace tim
