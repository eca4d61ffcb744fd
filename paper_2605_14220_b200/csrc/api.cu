// api.cu -- the C ABI of libtim.so (include/tim.h): argument validation, workspace layout,
// TMA tensor-map encoding, launch configuration, NCCL exchange, status mapping.
// Every argument error returns synchronously before anything is enqueued.
#include <cuda.h>
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <atomic>
#include <mutex>
#include <vector>

#include "../../include/tim.h"
#include "../../include/tim_debug.h"
#include "tim_internal.h"

using namespace tim;

namespace {

// ------------------------------------------------------------------ device --
struct DevInfo {
  bool ok = false;
  bool sm100 = false;
  int num_sms = 0;
  int max_pair_clusters = 0;
  int max_single_ctas = 0;
  int l2_bytes = 0;
  int dev_id = 0;
  std::atomic<int> die_state{0};  // SM -> die map: 0 not probed yet, 1 valid, -1 unavailable
  uint64_t die_mask[4] = {0, 0, 0, 0};
};
constexpr int kMaxDev = 64;
DevInfo g_dev[kMaxDev];
std::mutex g_mu;

// Debug / tuning knobs (tim_debug.h).  None of them changes a result bit; they are atomics set by
// the tim_debug_* calls and snapshotted ONCE at the start of every library call (Knobs), so a call
// never sees a mix of old and new settings and the hot path reads no mutable global.
std::atomic<int> g_use_pair{1};      // cta_group::2 kernel (the numerics contract) vs ::1 bring-up
std::atomic<int> g_pad_small{1};     // small-batch H staging
std::atomic<int> g_max_clusters{0};  // SM cap to emulate smaller GPUs
std::atomic<int> g_h_policy{3};      // H tiles: evict_last (re-read for every vocab tile of the sweep)
std::atomic<int> g_w_policy{2};      // W tiles: evict_first (shared by all pairs within a few tiles, then dead)
std::atomic<int> g_sleep_waits{0};   // spinning mbarrier waits: +0.7-1% vs nanosleep (profiles/r01_sleep_waits_ab.txt)
std::atomic<int> g_sync_slack{4};    // pairs stay within 4 vocab tiles of each other: W window ~4 MB in L2
std::atomic<int> g_group{0};         // pairs per M-tile group (0 = automatic from the L2 size)
std::atomic<int> g_demote{0};        // demote finished H tiles to evict_normal (applypriority)
std::atomic<int> g_quad{0};          // 2-pair clusters sharing W tiles through TMA multicast
// backward GEMMs: pairs stay within 128 k-blocks of each other; L2 policies dH A / B, dW A / B
// (H evict_last: the <= 115 MB token block is re-read by every wave).  Interleaved A/B over slack
// {0, 32, 128} x policies: within 3-5%, this the fastest (profiles/r02_gemm_knobs_ab.txt).
std::atomic<int> g_gemm_slack{128};
std::atomic<int> g_gemm_pol[4] = {{1}, {1}, {1}, {3}};
std::atomic<int> g_die_groups{1};     // die-aware M-tile groups (G > 1); 0 = cluster-id order
std::atomic<int> g_split_correct{1};  // P = 1 tim_correct: 1 = local + finish + zero launches (default: 2.5%
                                      // faster than the fused cooperative launch, profiles/r02_correction_fused_ab.txt)

struct Knobs {
  int use_pair, pad_small, max_clusters, h_policy, w_policy, sleep_waits, sync_slack, group, demote, quad, gemm_slack;
  int gemm_pol[4];
  int split_correct;
  int die_groups;
};
Knobs knobs() {
  return Knobs{g_use_pair.load(), g_pad_small.load(), g_max_clusters.load(), g_h_policy.load(), g_w_policy.load(),
               g_sleep_waits.load(), g_sync_slack.load(), g_group.load(), g_demote.load(), g_quad.load(),
               g_gemm_slack.load(), {g_gemm_pol[0].load(), g_gemm_pol[1].load(), g_gemm_pol[2].load(),
                                     g_gemm_pol[3].load()}, g_split_correct.load(), g_die_groups.load()};
}

tim_status device_info(DevInfo** out) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDev) return TIM_ERR_CUDA;
  std::lock_guard<std::mutex> lk(g_mu);
  DevInfo& d = g_dev[dev];
  if (!d.ok) {
    int maj = 0, min = 0;
    if (cudaDeviceGetAttribute(&maj, cudaDevAttrComputeCapabilityMajor, dev) != cudaSuccess) return TIM_ERR_CUDA;
    if (cudaDeviceGetAttribute(&min, cudaDevAttrComputeCapabilityMinor, dev) != cudaSuccess) return TIM_ERR_CUDA;
    if (cudaDeviceGetAttribute(&d.num_sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return TIM_ERR_CUDA;
    d.sm100 = (maj == 10 && min == 0);
    d.dev_id = dev;
    d.max_pair_clusters = d.num_sms / 2;
    d.max_single_ctas = d.num_sms;
    if (cudaDeviceGetAttribute(&d.l2_bytes, cudaDevAttrL2CacheSize, dev) != cudaSuccess) return TIM_ERR_CUDA;
    d.ok = true;
  }
  *out = &d;
  return d.sm100 ? TIM_OK : TIM_ERR_UNSUPPORTED;
}

// SM -> die map of this device, probed once (B200: two dies whose L2 halves each cache what their
// own SMs read; which SMs sit on which die depends on the chip's floorsweeping).  One CTA per SM
// times dependent L2 loads of 16 lines 512 KB apart; a line is homed on one die, so its latency
// splits the SMs into near (~270 cycles) and far (~300) sets.  Per line an Otsu threshold; the
// lines' patterns are oriented against the clearest one and summed (weighted by agreement), so a
// few noisy samples cannot flip an SM.  Only the schedule uses the map (which pairs share an
// M-tile): a wrong bit costs L2 locality, never a result bit.  Skipped while the caller's stream
// is capturing a graph (allocation and synchronisation are not capturable); tried again later.
std::mutex g_die_mu;
static double otsu_threshold(std::vector<double> v, double* sep) {
  std::sort(v.begin(), v.end());
  const int n = static_cast<int>(v.size());
  double tot = 0;
  for (double x : v) tot += x;
  double best = -1, thr = v[n / 2], left = 0;
  for (int k = 1; k < n; ++k) {
    left += v[k - 1];
    const double w0 = static_cast<double>(k) / n, w1 = 1.0 - w0;
    const double m0 = left / k, m1 = (tot - left) / (n - k);
    const double b = w0 * w1 * (m0 - m1) * (m0 - m1);
    if (b > best) { best = b; thr = 0.5 * (v[k - 1] + v[k]); }
  }
  *sep = best;
  return thr;
}
static void ensure_die_map(DevInfo* d, cudaStream_t caller) {
  if (d->die_state.load() != 0) return;
  std::lock_guard<std::mutex> lk(g_die_mu);
  if (d->die_state.load() != 0) return;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(caller, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) {
    cudaGetLastError();
    return;
  }
  constexpr int kLines = 16, kStride = 65536;  // u64 words between lines (512 KB)
  const int n = d->num_sms;
  uint64_t* lines = nullptr;
  uint32_t *lat = nullptr, *smid = nullptr;
  cudaStream_t ps = nullptr;
  std::vector<uint32_t> hl(static_cast<size_t>(n) * kLines), hs(n);
  bool ok = cudaMalloc(&lines, sizeof(uint64_t) * kLines * kStride) == cudaSuccess &&
            cudaMalloc(&lat, sizeof(uint32_t) * n * kLines) == cudaSuccess &&
            cudaMalloc(&smid, sizeof(uint32_t) * n) == cudaSuccess &&
            cudaStreamCreateWithFlags(&ps, cudaStreamNonBlocking) == cudaSuccess &&
            cudaMemsetAsync(lines, 0, sizeof(uint64_t) * kLines * kStride, ps) == cudaSuccess &&
            launch_die_probe(lines, kLines, kStride, lat, smid, n, ps) == cudaSuccess &&
            cudaMemcpyAsync(hl.data(), lat, hl.size() * 4, cudaMemcpyDeviceToHost, ps) == cudaSuccess &&
            cudaMemcpyAsync(hs.data(), smid, hs.size() * 4, cudaMemcpyDeviceToHost, ps) == cudaSuccess &&
            cudaStreamSynchronize(ps) == cudaSuccess;
  if (ps) cudaStreamDestroy(ps);
  cudaFree(lines);
  cudaFree(lat);
  cudaFree(smid);
  cudaGetLastError();
  // every CTA on its own SM, smid < 256
  std::vector<int> seen(256, 0);
  for (int b = 0; ok && b < n; ++b) ok = hs[b] < 256 && !seen[hs[b]]++;
  if (ok) {
    std::vector<double> thr(kLines), sep(kLines);
    std::vector<std::vector<int>> cls(kLines, std::vector<int>(n));
    int r = 0;
    for (int l = 0; l < kLines; ++l) {
      std::vector<double> v(n);
      for (int b = 0; b < n; ++b) v[b] = hl[b * kLines + l];
      thr[l] = otsu_threshold(v, &sep[l]);
      for (int b = 0; b < n; ++b) cls[l][b] = v[b] > thr[l];
      if (sep[l] > sep[r]) r = l;
    }
    std::vector<double> score(n, 0.0);
    for (int l = 0; l < kLines; ++l) {
      int agree = 0;
      for (int b = 0; b < n; ++b) agree += cls[l][b] == cls[r][b];
      const double a = static_cast<double>(agree) / n;
      const double w = (a >= 0.5 ? 1.0 : -1.0) * std::fabs(2.0 * a - 1.0);
      for (int b = 0; b < n; ++b) score[b] += w * (hl[b * kLines + l] - thr[l]);
    }
    // the two SMs of a TPC (smid 2k, 2k + 1: where a CTA pair lands) share a die -- pool their
    // scores, and refuse the map when too many pairs disagree (a noisy probe must not group worse
    // than the cluster-id order does)
    std::vector<double> by_smid(256, 0.0);
    std::vector<int> have(256, 0);
    for (int b = 0; b < n; ++b) {
      by_smid[hs[b]] = score[b];
      have[hs[b]] = 1;
    }
    int n1 = 0, pairs = 0, disagree = 0;
    uint64_t mask[4] = {0, 0, 0, 0};
    for (int s0 = 0; s0 < 256; s0 += 2) {
      if (!have[s0] && !have[s0 + 1]) continue;
      const double t = by_smid[s0] + by_smid[s0 + 1];
      if (have[s0] && have[s0 + 1]) {
        ++pairs;
        disagree += (by_smid[s0] > 0) != (by_smid[s0 + 1] > 0);
      }
      for (int k = 0; k < 2; ++k)
        if (have[s0 + k] && t > 0) {
          ++n1;
          mask[(s0 + k) >> 6] |= 1ull << ((s0 + k) & 63);
        }
    }
    ok = n1 >= 0.3 * n && n1 <= 0.7 * n && std::sqrt(sep[r]) >= 5.0 &&  // two dies, >= ~10 cycles apart
         disagree * 10 <= pairs;                                           // <= 10% of TPCs split
    if (ok) std::memcpy(d->die_mask, mask, sizeof(mask));
  }
  d->die_state.store(ok ? 1 : -1);
}

static void set_gemm_die(DevInfo* d, BwdGemmParams& gp, int max_pairs, cudaStream_t s) {
  gp.die_ok = 0;
  if (max_pairs + 2 > kMaxProgress || !gp.progress) return;
  ensure_die_map(d, s);
  if (d->die_state.load() != 1) return;
  gp.die_ok = 1;
  std::memcpy(gp.die_mask, d->die_mask, sizeof(gp.die_mask));
  gp.die_counter = gp.progress + kMaxProgress - 2;  // zeroed with the gate counters
}

// Fill the kernel's die-grouping fields (G > 1, CTA pairs, the whole grid's clusters fit the
// progress area's spare words).
static void set_die_grouping(DevInfo* d, LogprobParams& p, int64_t clusters, cudaStream_t s) {
  p.die_ok = 0;
  if (p.group <= 1 || clusters + 2 > kMaxProgress || !p.progress) return;
  ensure_die_map(d, s);
  if (d->die_state.load() != 1) return;
  p.die_ok = 1;
  std::memcpy(p.die_mask, d->die_mask, sizeof(p.die_mask));
  p.die_counter = p.progress + kMaxProgress - 2;  // zeroed with the progress counters
}

// ------------------------------------------------------------- tensor maps --
typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                     const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                     CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
PFN_encodeTiled get_encode() {
  static PFN_encodeTiled fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_encodeTiled>(p);
  });
  return fn;
}

// 2-D bf16 [rows, cols] (cols contiguous), row pitch `pitch_elems`; box = 64 cols x box_rows, SW128
bool encode_bf16_2d(CUtensorMap* m, const void* base, uint64_t rows, uint64_t cols, uint64_t pitch_elems,
                    uint32_t box_rows) {
  PFN_encodeTiled enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {pitch_elems * 2};
  cuuint32_t box[2] = {64, box_rows};
  cuuint32_t estr[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// G block [rows][pitch] bf16 as the gradient epilogue's TMA store target: 32 x 32 tiles, 64-B swizzle
bool encode_g_store(CUtensorMap* m, void* base, uint64_t rows, uint64_t cols, uint64_t pitch_elems) {
  PFN_encodeTiled enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {pitch_elems * 2};
  cuuint32_t box[2] = {32, 32};
  cuuint32_t estr[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, base, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
             CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

inline bool aligned(const void* p, uintptr_t a) { return (reinterpret_cast<uintptr_t>(p) & (a - 1)) == 0; }

// int128 {lo, hi} -> double, round to nearest even (bits below 64 significant ones fold into a sticky bit)
double i128_host_to_double(const int64_t* v) {
  const __int128 x = (static_cast<__int128>(v[1]) << 64) | static_cast<__int128>(static_cast<uint64_t>(v[0]));
  const bool neg = x < 0;
  const unsigned __int128 u = neg ? static_cast<unsigned __int128>(-x) : static_cast<unsigned __int128>(x);
  const uint64_t hi = static_cast<uint64_t>(u >> 64);
  double r;
  if (hi == 0) {
    r = static_cast<double>(static_cast<uint64_t>(u));  // RN (default rounding mode)
  } else {
    const int sh = 64 - __builtin_clzll(hi);
    uint64_t top = static_cast<uint64_t>(u >> sh);
    if ((u & ((static_cast<unsigned __int128>(1) << sh) - 1)) != 0) top |= 1u;
    r = std::ldexp(static_cast<double>(top), sh);
  }
  return neg ? -r : r;
}

#ifndef TIM_MAX_SLICES
#define TIM_MAX_SLICES 64
#endif
constexpr int kMaxSlices = TIM_MAX_SLICES;
inline int32_t n_vocab_tiles(int32_t vocab) { return (vocab + 255) / 256; }
inline int32_t vocab_slices(int32_t vocab) {
  const int32_t nvt = n_vocab_tiles(vocab);
  return nvt < kMaxSlices ? nvt : kMaxSlices;
}

int pick_group(const DevInfo* dev, bool pair, int n_slices, int64_t groups, int32_t d, int forced) {
  int g = 1;
  if (pair && forced > 0) {
    if (n_slices % forced == 0 && groups >= forced) g = forced;
  } else if (pair) {
    const double h_tile = 256.0 * d * 2.0;
    while (g < 8 && n_slices % (g * 2) == 0 && groups >= g * 2 &&
           (static_cast<double>(groups) / g) * h_tile > 0.75 * dev->l2_bytes)
      g *= 2;
  }
  return g;
}

// Small batches whose last 128-row H box is mostly out of bounds (n_tok < 256, n_tok % 128 in
// [1, 32]): the kernel would re-load that box (TMA zero-fills the missing rows) for every vocab tile
// and K step, and such boxes are slow to fill (C1's head, interleaved in one process: N = 1
// 0.26 ms, N = 16 0.17-0.22 ms, N = 64 0.13 ms).  Their rows are copied into a zero-padded buffer
// of whole boxes at the end of the workspace first (one small kernel, ~4 us: N = 1 0.16 ms, N = 16
// 0.13-0.16 ms); above 32 rows the copy costs more than it saves.  Rows are independent, so no
// result bit changes (tested).
static int64_t small_pad_rows(int64_t n_tok) {
  if (n_tok <= 0 || n_tok >= 256 || n_tok % 128 == 0 || n_tok % 128 > 32) return 0;
  return (n_tok + 127) / 128 * 128;
}
static size_t small_pad_bytes(int64_t n_tok, int32_t hidden) {
  const int64_t r = small_pad_rows(n_tok);
  if (r == 0 || hidden < 1) return 0;
  return 256 + static_cast<size_t>(r) * static_cast<size_t>(hidden) * 2u;  // + alignment slack
}

tim_status logprob_impl(const void* hidden, int64_t ld_hidden, const void* weight, int32_t d, int32_t vocab,
                        const int64_t* ids, int64_t n_tok, float temperature, const float* temps, float* logp,
                        float* ent, void* ws, size_t ws_bytes, tim_device_status* dstatus, void* stream,
                        float* debug_logits, int64_t debug_ld, const uint64_t* row_keys = nullptr,
                        uint64_t seed = 0, int64_t* ids_out = nullptr, int32_t tp = 1, int32_t tp_rank = 0,
                        void* tp_partial_out = nullptr, float* lse2_out = nullptr, int64_t index_base = 0,
                        bool pad_small = true) {
  const Knobs kn = knobs();
  const bool sample = row_keys != nullptr;
  const bool tp_mode = tp_partial_out != nullptr;  // vocab-parallel rank: partials only, no merge
  if (!weight) return TIM_ERR_NULL;
  if (n_tok < 0 || n_tok >= (int64_t(1) << 31)) return TIM_ERR_SHAPE;
  if (d < 64 || d > 16384 || d % 64 != 0) return TIM_ERR_SHAPE;
  if (vocab < 1 || vocab > (1 << 24)) return TIM_ERR_SHAPE;
  if (ld_hidden < d) return TIM_ERR_SHAPE;
  if (!(temperature > 0.f) || !std::isfinite(temperature)) return TIM_ERR_VALUE;
  if (!aligned(weight, 16) || (ld_hidden * 2) % 16 != 0) return TIM_ERR_ALIGN;
  if (n_tok == 0) return TIM_OK;  // empty batch: pointers may be NULL, nothing is launched
  if (!hidden || (!tp_mode && !logp) || (sample ? !ids_out : !ids)) return TIM_ERR_NULL;
  if (!aligned(hidden, 16)) return TIM_ERR_ALIGN;
  if (!ws) return TIM_ERR_NULL;
  if (!aligned(ws, 16)) return TIM_ERR_ALIGN;
  const bool pad = pad_small && kn.pad_small && !tp_mode && small_pad_rows(n_tok) > 0;
  const size_t ws_need = tp_mode ? kWsHeaderBytes
                                 : (sample ? tim_sample_workspace_bytes(n_tok, d, vocab)
                                           : tim_logprob_workspace_bytes(n_tok, d, vocab)) -
                                       (pad ? 0 : small_pad_bytes(n_tok, d));
  if (ws_bytes < ws_need) return TIM_ERR_WORKSPACE;
  // fixed split of the full vocabulary; a tensor-parallel rank owns slices [s0, s1) = W rows [row0, row1)
  const int32_t S_total = vocab_slices(vocab);
  if (tp < 1 || S_total % tp != 0 || tp_rank < 0 || tp_rank >= tp) return TIM_ERR_SHAPE;
  if (tp_mode && !aligned(tp_partial_out, 16)) return TIM_ERR_ALIGN;
  const int32_t s0 = tp_rank * (S_total / tp), s1 = s0 + S_total / tp;
  const int32_t nvt = n_vocab_tiles(vocab);
  const int32_t row0 = tp_mode ? ((s0 * nvt) / S_total) * 256 : 0;
  const int32_t row1 = tp_mode ? std::min(((s1 * nvt) / S_total) * 256, vocab) : vocab;
  DevInfo* dev = nullptr;
  tim_status st = device_info(&dev);
  if (st != TIM_OK) return st;

  const bool pair = kn.use_pair != 0;
  // 2-pair multicast clusters when the live H tiles of all pairs fit in L2 (d <= 2048 on B200);
  // otherwise 1-pair clusters with M-tile groups (below).  Never changes a result bit.
  const bool quad = pair && kn.quad != 0 && dev->max_pair_clusters >= 2 &&
                    dev->max_pair_clusters * 256.0 * d * 2.0 <= 0.75 * dev->l2_bytes;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  uint8_t* wsb = static_cast<uint8_t*>(ws);
  const void* h_tma = hidden;
  int64_t h_ld = ld_hidden, h_rows = n_tok;
  if (pad) {
    const size_t off = (ws_need - small_pad_bytes(n_tok, d) + 255) & ~size_t(255);
    uint8_t* hp = wsb + off;
    h_rows = small_pad_rows(n_tok);
    h_ld = d;
    const size_t row_b = static_cast<size_t>(d) * 2u;
    if (launch_pad_rows(hidden, ld_hidden * 2, hp, static_cast<int>(row_b), static_cast<int>(n_tok),
                        static_cast<int>(h_rows), s) != cudaSuccess)
      return TIM_ERR_CUDA;
    h_tma = hp;
  }
  CUtensorMap th, tw;
  if (!encode_bf16_2d(&th, h_tma, h_rows, d, h_ld, 128)) return TIM_ERR_CUDA;
  if (!encode_bf16_2d(&tw, weight, row1 - row0, d, d, quad ? fwd_w_box_rows(pair) / 2 : fwd_w_box_rows(pair)))
    return TIM_ERR_CUDA;

  WsHeader* hdr = reinterpret_cast<WsHeader*>(wsb);
  float4* partials = tp_mode ? static_cast<float4*>(tp_partial_out) : reinterpret_cast<float4*>(wsb + kWsHeaderBytes);
  if (cudaMemsetAsync(hdr, 0, kWsHeaderBytes, s) != cudaSuccess) return TIM_ERR_CUDA;

  LogprobParams p{};
  p.ids = ids;
  p.temps = temps;
  p.temperature = temperature;
  p.partials = partials;
  p.n_tok = static_cast<int>(n_tok);
  p.vocab = vocab;
  p.hidden = d;
  const int unit = fwd_unit_rows(pair);
  p.n_mt = static_cast<int>((n_tok + unit - 1) / unit);
  p.n_vt = nvt;
  p.n_slices = s1 - s0;
  p.n_slices_total = S_total;
  p.slice0 = s0;
  p.w_row0 = row0;
  p.debug_logits = debug_logits;
  p.debug_ld = debug_ld;
  p.h_policy = kn.h_policy;
  p.w_policy = kn.w_policy;
  p.sleep_waits = kn.sleep_waits;
  p.progress = reinterpret_cast<uint32_t*>(wsb + kWsProgressOffset);
  p.sync_slack = kn.sync_slack;
  p.hidden_ptr = h_tma;
  p.ld_hidden_bytes = h_ld * 2;
  p.demote = kn.demote;
  p.gate_stats = &hdr->reserved[5];  // read back by the diagnostics scripts (zeroed with the header)
  p.clk = &hdr->reserved[1];         // reserved[1..4]: SM clock inside the kernel (bench.py reads it)
  p.row_keys = row_keys;
  p.seed = seed;
  p.partials2 = sample ? partials + static_cast<size_t>(vocab_slices(vocab)) * static_cast<size_t>(n_tok) : nullptr;
  const int64_t n_units = static_cast<int64_t>(quad ? (p.n_mt + 1) / 2 : p.n_mt) * p.n_slices;
  int64_t ctas_cap = quad ? dev->max_pair_clusters / 2 : (pair ? dev->max_pair_clusters : dev->max_single_ctas);
  if (kn.max_clusters > 0 && kn.max_clusters < ctas_cap) ctas_cap = kn.max_clusters;
  const int64_t groups = n_units < ctas_cap ? n_units : ctas_cap;
  const int grid = static_cast<int>(groups * (quad ? 4 : (pair ? 2 : 1)));
  // Pairs sharing an M-tile: smallest G in {1, 2, 4, 8} (dividing S_v, <= #pairs) whose live H
  // tiles (one 256-row tile per group) fit in ~75% of L2.  Performance only: which pair runs
  // which (M-tile, slice) unit never changes a row's arithmetic.
  p.group = quad ? 1 : pick_group(dev, pair, p.n_slices, groups, d, kn.group);
  if (pair && !quad && kn.die_groups) set_die_grouping(dev, p, groups, s);
  if (launch_logprob_fwd(pair, debug_logits != nullptr, sample, quad, th, tw, p, grid, s) != cudaSuccess)
    return TIM_ERR_CUDA;
  if (tp_mode) return TIM_OK;  // the caller all-gathers the slice partials, then tim_logprob_tp_merge

  MergeParams mp{};
  mp.partials = partials;
  mp.ids = ids;
  mp.temps = temps;
  mp.logp = logp;
  mp.entropy = ent;
  mp.n_tok = n_tok;
  mp.vocab = vocab;
  mp.n_slices = p.n_slices;
  mp.ws = hdr;
  mp.dstatus = dstatus;
  mp.partials2 = p.partials2;
  mp.ids_out = ids_out;
  mp.lse2_out = lse2_out;
  mp.index_base = index_base;
  if ((sample ? launch_sample_merge(mp, s) : launch_logprob_merge(mp, s)) != cudaSuccess) return TIM_ERR_CUDA;
  return TIM_OK;
}

// ----------------------------------------------------------------- correct --
tim_status check_cfg(const tim_correct_cfg* c) {
  if (!c) return TIM_ERR_NULL;
  if (c->tis != 0 && c->tis != 1) return TIM_ERR_VALUE;
  if (c->tok_rs != 0 && c->tok_rs != 1) return TIM_ERR_VALUE;
  if (c->seq_rs != TIM_SEQ_NONE && c->seq_rs != TIM_SEQ_K1 && c->seq_rs != TIM_SEQ_K3) return TIM_ERR_VALUE;
  if (c->seq_agg != TIM_AGG_SUM && c->seq_agg != TIM_AGG_MEAN) return TIM_ERR_VALUE;
  if (c->tis && (!(c->tis_cap > 0.0) || !std::isfinite(c->tis_cap) || !std::isfinite(c->log_tis_cap)))
    return TIM_ERR_VALUE;
  if (c->tok_rs && (std::isnan(c->log_tok_lo) || std::isnan(c->log_tok_hi) || c->log_tok_lo > c->log_tok_hi))
    return TIM_ERR_VALUE;
  if (c->seq_rs != TIM_SEQ_NONE && (!std::isfinite(c->tau_seq) || std::fabs(c->tau_seq) >= 1024.0))
    return TIM_ERR_VALUE;
  return TIM_OK;
}

CorrectDevCfg dev_cfg(const tim_correct_cfg* c) {
  CorrectDevCfg d{};
  d.tis = c->tis;
  d.tok_rs = c->tok_rs;
  d.seq_rs = c->seq_rs;
  d.seq_agg = c->seq_agg;
  d.tis_cap = c->tis_cap;
  d.log_tis_cap = c->log_tis_cap;
  d.log_lo = c->log_tok_lo;
  d.log_hi = c->log_tok_hi;
  d.tau_seq = c->tau_seq;
  return d;
}

tim_status check_common(const float* num, const float* den, const int64_t* cu, int64_t n_seq, int64_t tok_begin,
                        int64_t n_local, const uint8_t* resp) {
  if (!cu) return TIM_ERR_NULL;
  if (n_local > 0 && (!num || !den)) return TIM_ERR_NULL;
  if (n_seq < 0 || n_seq >= (int64_t(1) << 40) || n_local < 0 || tok_begin < 0) return TIM_ERR_SHAPE;
  if (n_local > 0 && n_seq == 0) return TIM_ERR_SHAPE;
  if (!aligned(num, 4) || !aligned(den, 4)) return TIM_ERR_ALIGN;  // 16-B aligned arrays take the vector path
  return TIM_OK;
}

// ------------------------------------------------------------------ NCCL --
typedef struct { char internal[128]; } nccl_uid;
typedef void* nccl_comm_t;
typedef int (*PFN_getUniqueId)(nccl_uid*);
typedef int (*PFN_commInitRank)(nccl_comm_t*, int, nccl_uid, int);
typedef int (*PFN_allGather)(const void*, void*, size_t, int, nccl_comm_t, cudaStream_t);
typedef int (*PFN_commDestroy)(nccl_comm_t);
struct NcclApi {
  bool ok = false;
  PFN_getUniqueId get_uid = nullptr;
  PFN_commInitRank init_rank = nullptr;
  PFN_allGather all_gather = nullptr;
  PFN_commDestroy destroy = nullptr;
};
NcclApi* nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
    api.get_uid = reinterpret_cast<PFN_getUniqueId>(dlsym(h, "ncclGetUniqueId"));
    api.init_rank = reinterpret_cast<PFN_commInitRank>(dlsym(h, "ncclCommInitRank"));
    api.all_gather = reinterpret_cast<PFN_allGather>(dlsym(h, "ncclAllGather"));
    api.destroy = reinterpret_cast<PFN_commDestroy>(dlsym(h, "ncclCommDestroy"));
    api.ok = api.get_uid && api.init_rank && api.all_gather && api.destroy;
  });
  return &api;
}
constexpr int kNcclInt8 = 0;

}  // namespace

struct tim_comm {
  nccl_comm_t comm;
  int nranks;
  int rank;
};

// ======================================================================= C ABI ==
extern "C" {

const char* tim_status_string(tim_status s) {
  switch (s) {
    case TIM_OK: return "TIM_OK";
    case TIM_ERR_NULL: return "TIM_ERR_NULL: a required pointer is NULL";
    case TIM_ERR_SHAPE: return "TIM_ERR_SHAPE: size out of range or inconsistent";
    case TIM_ERR_ALIGN: return "TIM_ERR_ALIGN: pointer / pitch violates the 16-byte (TMA) alignment";
    case TIM_ERR_VALUE: return "TIM_ERR_VALUE: scalar parameter out of range";
    case TIM_ERR_WORKSPACE: return "TIM_ERR_WORKSPACE: workspace too small";
    case TIM_ERR_CUDA: return "TIM_ERR_CUDA: CUDA call failed";
    case TIM_ERR_NCCL: return "TIM_ERR_NCCL: NCCL unavailable or failed";
    case TIM_ERR_UNSUPPORTED: return "TIM_ERR_UNSUPPORTED: requires an sm_100 (B200) device";
    case TIM_ERR_DATA: return "TIM_ERR_DATA: device-side data error (see first_bad_index)";
  }
  return "unknown tim_status";
}

int tim_abi_version(void) { return TIM_ABI_VERSION; }

int32_t tim_logprob_vocab_slices(int32_t vocab) { return vocab < 1 ? 0 : vocab_slices(vocab); }

size_t tim_logprob_workspace_bytes(int64_t n_tok, int32_t hidden, int32_t vocab) {
  if (n_tok < 0 || vocab < 1) return 0;
  return kWsHeaderBytes + static_cast<size_t>(vocab_slices(vocab)) * static_cast<size_t>(n_tok) * 16u +
         small_pad_bytes(n_tok, hidden);
}

tim_status tim_logprob(const void* hidden_bf16, int64_t ld_hidden, const void* weight_bf16, int32_t hidden,
                       int32_t vocab, const int64_t* token_ids, int64_t n_tok, float temperature,
                       const float* temperatures_or_null, float* logp_out, float* entropy_out_or_null,
                       void* workspace, size_t workspace_bytes, tim_device_status* dstatus, void* stream) {
  return logprob_impl(hidden_bf16, ld_hidden, weight_bf16, hidden, vocab, token_ids, n_tok, temperature,
                      temperatures_or_null, logp_out, entropy_out_or_null, workspace, workspace_bytes, dstatus,
                      stream, nullptr, 0);
}

size_t tim_sample_workspace_bytes(int64_t n_tok, int32_t hidden, int32_t vocab) {
  if (n_tok < 0 || vocab < 1) return 0;
  return kWsHeaderBytes + 2u * static_cast<size_t>(vocab_slices(vocab)) * static_cast<size_t>(n_tok) * 16u +
         small_pad_bytes(n_tok, hidden);
}

tim_status tim_sample(const void* hidden_bf16, int64_t ld_hidden, const void* weight_bf16, int32_t hidden,
                      int32_t vocab, const uint64_t* row_keys, int64_t n_tok, uint64_t seed, float temperature,
                      const float* temperatures_or_null, int64_t* ids_out, float* logp_out,
                      float* entropy_out_or_null, void* workspace, size_t workspace_bytes,
                      tim_device_status* dstatus, void* stream) {
  if (n_tok > 0 && !row_keys) return TIM_ERR_NULL;
  if (n_tok == 0) row_keys = nullptr;
  const uint64_t dummy = 0;
  return logprob_impl(hidden_bf16, ld_hidden, weight_bf16, hidden, vocab, nullptr, n_tok, temperature,
                      temperatures_or_null, logp_out, entropy_out_or_null, workspace, workspace_bytes, dstatus,
                      stream, nullptr, 0, n_tok > 0 ? row_keys : &dummy, seed, ids_out);
}

tim_status tim_stats_finalize(tim_stats* h) {
  if (!h) return TIM_ERR_NULL;
  auto to_d = [](const int64_t* v) {
    const __int128 x = (static_cast<__int128>(v[1]) << 64) | static_cast<__int128>(static_cast<uint64_t>(v[0]));
    const bool neg = x < 0;
    unsigned __int128 u = neg ? static_cast<unsigned __int128>(-x) : static_cast<unsigned __int128>(x);
    const uint64_t hi = static_cast<uint64_t>(u >> 64);
    double r;
    if (hi == 0) {
      r = static_cast<double>(static_cast<uint64_t>(u));  // RN (default rounding mode)
    } else {
      const int sh = 64 - __builtin_clzll(hi);
      uint64_t top = static_cast<uint64_t>(u >> sh);
      if ((u & ((static_cast<unsigned __int128>(1) << sh) - 1)) != 0) top |= 1u;
      r = std::ldexp(static_cast<double>(top), sh);
    }
    return neg ? -r : r;
  };
  const double n = static_cast<double>(h->n_resp_tok);
  const double sc = std::ldexp(1.0, -52);
  h->mean_abs_delta = h->n_resp_tok ? (to_d(h->sum_abs_delta_fx) * sc) / n : 0.0;
  h->mean_k1 = h->n_resp_tok ? (to_d(h->sum_k1_fx) * sc) / n : 0.0;
  h->mean_k3 = h->n_resp_tok ? (to_d(h->sum_k3_fx) * sc) / n : 0.0;
  return TIM_OK;
}

size_t tim_correct_partial_bytes(int64_t n_seq) {
  if (n_seq < 0) return 0;
  return sizeof(tim_partial_header) + static_cast<size_t>(n_seq) * sizeof(tim_seq_partial);
}

size_t tim_correct_workspace_bytes(int64_t n_tok_local, int64_t n_seq, int32_t nranks) {
  (void)n_tok_local;
  if (n_seq < 0 || nranks < 1) return 0;
  const size_t b = (tim_correct_partial_bytes(n_seq) + 255) & ~size_t(255);
  return b * (1 + static_cast<size_t>(nranks));  // local block + the all-gathered blocks
}

// Validate pass-1 arguments, zero the partial block and fill the kernel parameters.
static tim_status prep_correct_local(const float* num, const float* den, const int64_t* cu, int64_t n_seq,
                                     int64_t tok_begin, int64_t n_local, const uint8_t* resp,
                                     const tim_correct_cfg* cfg, float* tis_w, uint8_t* tok_keep, float* coeff,
                                     void* partial_out, tim_device_status* dstatus, void* stream, LocalParams* out,
                                     DevInfo** dev_out) {
  tim_status st = check_common(num, den, cu, n_seq, tok_begin, n_local, resp);
  if (st != TIM_OK) return st;
  if ((st = check_cfg(cfg)) != TIM_OK) return st;
  const bool any_out = tis_w || tok_keep || coeff;
  if (!partial_out) return TIM_ERR_NULL;
  if (any_out && !(tis_w && tok_keep && coeff)) return TIM_ERR_NULL;
  if (any_out && (!aligned(tis_w, 16) || !aligned(coeff, 16) || !aligned(tok_keep, 8))) return TIM_ERR_ALIGN;
  if (!aligned(partial_out, 16)) return TIM_ERR_ALIGN;
  if ((st = device_info(dev_out)) != TIM_OK) return st;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (cudaMemsetAsync(partial_out, 0, tim_correct_partial_bytes(n_seq), s) != cudaSuccess) return TIM_ERR_CUDA;
  LocalParams& p = *out;
  p = LocalParams{};
  p.num = num;
  p.den = den;
  p.cu = cu;
  p.n_seq = n_seq;
  p.tok_begin = tok_begin;
  p.n = n_local;
  p.resp = resp;
  p.tis_w = tis_w;
  p.tok_keep = tok_keep;
  p.coeff = coeff;
  p.hdr = static_cast<tim_partial_header*>(partial_out);
  p.seqp = reinterpret_cast<tim_seq_partial*>(static_cast<uint8_t*>(partial_out) + sizeof(tim_partial_header));
  p.cfg = dev_cfg(cfg);
  p.dstatus = dstatus;
  p.vec = aligned(num, 16) && aligned(den, 16) && aligned(resp, 4) && aligned(tis_w, 16) && aligned(coeff, 16) &&
          aligned(tok_keep, 4);
  return TIM_OK;
}

tim_status tim_correct_local(const float* num, const float* den, const int64_t* cu, int64_t n_seq,
                             int64_t tok_begin, int64_t n_local, const uint8_t* resp, const tim_correct_cfg* cfg,
                             float* tis_w, uint8_t* tok_keep, float* coeff, void* partial_out,
                             tim_device_status* dstatus, void* stream) {
  LocalParams p{};
  DevInfo* dev = nullptr;
  const tim_status st = prep_correct_local(num, den, cu, n_seq, tok_begin, n_local, resp, cfg, tis_w, tok_keep, coeff,
                                           partial_out, dstatus, stream, &p, &dev);
  if (st != TIM_OK || n_local == 0) return st;
  return launch_correct_local(p, dev->num_sms, reinterpret_cast<cudaStream_t>(stream)) == cudaSuccess ? TIM_OK
                                                                                                       : TIM_ERR_CUDA;
}

// scratch: 2 zeroed words for a multi-block finish (or null: one block)
static tim_status correct_finish_impl(const void* gathered, int32_t nranks, const int64_t* cu, int64_t n_seq,
                                      int64_t tok_begin, int64_t n_local, const tim_correct_cfg* cfg, float* coeff,
                                      uint8_t* seq_keep, double* seq_score, tim_stats* stats,
                                      unsigned long long* scratch, void* stream) {
  if (!gathered || !cu) return TIM_ERR_NULL;
  if (nranks < 1 || n_seq < 0 || n_local < 0 || tok_begin < 0) return TIM_ERR_SHAPE;
  tim_status st = check_cfg(cfg);
  if (st != TIM_OK) return st;
  if (cfg->seq_rs != TIM_SEQ_NONE && n_local > 0 && !coeff) return TIM_ERR_NULL;
  if (!aligned(gathered, 16)) return TIM_ERR_ALIGN;
  DevInfo* dev = nullptr;
  if ((st = device_info(&dev)) != TIM_OK) return st;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  FinishParams f{};
  f.gathered = static_cast<const uint8_t*>(gathered);
  f.block_bytes = static_cast<int64_t>(tim_correct_partial_bytes(n_seq));
  f.nranks = nranks;
  f.n_seq = n_seq;
  f.cfg = dev_cfg(cfg);
  f.seq_keep = seq_keep;
  f.seq_score = seq_score;
  f.stats = stats;
  f.scratch = scratch;
  if (launch_correct_finish(f, dev->num_sms, s) != cudaSuccess) return TIM_ERR_CUDA;
  if (cfg->seq_rs != TIM_SEQ_NONE && n_local > 0 && n_seq > 0) {
    if (!seq_keep) return TIM_ERR_NULL;
    ZeroParams z{};
    z.cu = cu;
    z.n_seq = n_seq;
    z.tok_begin = tok_begin;
    z.n = n_local;
    z.seq_keep = seq_keep;
    z.coeff = coeff;
    if (launch_correct_zero(z, s) != cudaSuccess) return TIM_ERR_CUDA;
  }
  return TIM_OK;
}

tim_status tim_correct_finish(const void* gathered, int32_t nranks, const int64_t* cu, int64_t n_seq,
                              int64_t tok_begin, int64_t n_local, const tim_correct_cfg* cfg, float* coeff,
                              uint8_t* seq_keep, double* seq_score, tim_stats* stats, void* stream) {
  return correct_finish_impl(gathered, nranks, cu, n_seq, tok_begin, n_local, cfg, coeff, seq_keep, seq_score, stats,
                             nullptr, stream);
}

static tim_status correct_impl(const float* num, const float* den, const int64_t* cu, int64_t n_seq,
                               int64_t tok_begin, int64_t n_local, const uint8_t* resp, const tim_correct_cfg* cfg,
                               tim_comm* comm, float* tis_w, uint8_t* tok_keep, uint8_t* seq_keep, float* coeff,
                               double* seq_score, tim_stats* stats, void* ws, size_t ws_bytes,
                               tim_device_status* dstatus, void* stream) {
  tim_status st = check_common(num, den, cu, n_seq, tok_begin, n_local, resp);
  if (st != TIM_OK) return st;
  if ((st = check_cfg(cfg)) != TIM_OK) return st;
  const int nranks = comm ? comm->nranks : 1;
  if (!ws) return TIM_ERR_NULL;
  if (!aligned(ws, 256)) return TIM_ERR_ALIGN;
  if (ws_bytes < tim_correct_workspace_bytes(n_local, n_seq, nranks)) return TIM_ERR_WORKSPACE;
  if (seq_keep == nullptr && cfg->seq_rs != TIM_SEQ_NONE && tis_w) return TIM_ERR_NULL;
  uint8_t* local = static_cast<uint8_t*>(ws);
  const size_t blk = (tim_correct_partial_bytes(n_seq) + 255) & ~size_t(255);
  // the local block's header reserved[2..3] (zeroed with the block; pass 1 uses [0..1]) serve as
  // the finish pass's {ticket, rejections}
  unsigned long long* scratch =
      reinterpret_cast<unsigned long long*>(&reinterpret_cast<tim_partial_header*>(local)->reserved[2]);
  if (comm == nullptr && n_local > 0 && !knobs().split_correct) {
    // P = 1: pass 1, decisions / stats and the zeroing of rejected sequences in ONE cooperative
    // launch (a7 "fused into pass 1 when P = 1")
    LocalParams p{};
    DevInfo* dev = nullptr;
    if ((st = prep_correct_local(num, den, cu, n_seq, tok_begin, n_local, resp, cfg, tis_w, tok_keep, coeff, local,
                                 dstatus, stream, &p, &dev)) != TIM_OK)
      return st;
    if (cfg->seq_rs != TIM_SEQ_NONE && tis_w && !seq_keep) return TIM_ERR_NULL;
    FinishParams f{};
    f.gathered = local;
    f.block_bytes = static_cast<int64_t>(tim_correct_partial_bytes(n_seq));
    f.nranks = 1;
    f.n_seq = n_seq;
    f.cfg = dev_cfg(cfg);
    f.seq_keep = seq_keep;
    f.seq_score = seq_score;
    f.stats = stats;
    f.scratch = scratch;
    ZeroParams z{};
    z.cu = cu;
    z.n_seq = n_seq;
    z.tok_begin = tok_begin;
    z.n = n_local;
    z.seq_keep = seq_keep;
    z.coeff = coeff;
    return launch_correct_fused(p, f, z, dev->num_sms, reinterpret_cast<cudaStream_t>(stream)) == cudaSuccess
               ? TIM_OK
               : TIM_ERR_CUDA;
  }
  if ((st = tim_correct_local(num, den, cu, n_seq, tok_begin, n_local, resp, cfg, tis_w, tok_keep, coeff, local,
                              dstatus, stream)) != TIM_OK)
    return st;
  const void* gathered = local;
  if (comm != nullptr) {  // NCCL all-gather of the exact partial blocks (also for a 1-rank comm)
    NcclApi* api = nccl();
    if (!api->ok) return TIM_ERR_NCCL;
    uint8_t* g = local + blk;
    // the gathered buffer is [nranks][partial_bytes] with no padding between blocks
    if (api->all_gather(local, g, tim_correct_partial_bytes(n_seq), kNcclInt8, comm->comm,
                        reinterpret_cast<cudaStream_t>(stream)) != 0)
      return TIM_ERR_NCCL;
    gathered = g;
  }
  return correct_finish_impl(gathered, nranks, cu, n_seq, tok_begin, n_local, cfg, coeff, seq_keep, seq_score, stats,
                             scratch, stream);
}

tim_status tim_mismatch_stats(const float* num, const float* den, const int64_t* cu, int64_t n_seq,
                              int64_t tok_begin, int64_t n_local, const uint8_t* resp, tim_comm* comm,
                              tim_stats* stats_dev, void* ws, size_t ws_bytes, tim_device_status* dstatus,
                              void* stream) {
  if (!stats_dev) return TIM_ERR_NULL;
  tim_correct_cfg cfg{};
  cfg.tis = 0;
  cfg.tok_rs = 0;
  cfg.seq_rs = TIM_SEQ_NONE;
  cfg.seq_agg = TIM_AGG_SUM;
  return correct_impl(num, den, cu, n_seq, tok_begin, n_local, resp, &cfg, comm, nullptr, nullptr, nullptr, nullptr,
                      nullptr, stats_dev, ws, ws_bytes, dstatus, stream);
}

tim_status tim_correct(const float* num, const float* den, const int64_t* cu, int64_t n_seq, int64_t tok_begin,
                       int64_t n_local, const uint8_t* resp, const tim_correct_cfg* cfg, tim_comm* comm,
                       float* tis_w, uint8_t* tok_keep, uint8_t* seq_keep, float* coeff, double* seq_score,
                       tim_stats* stats_dev, void* ws, size_t ws_bytes, tim_device_status* dstatus,
                       void* stream) {
  if (!tis_w || !tok_keep || !coeff || !seq_keep) return TIM_ERR_NULL;
  return correct_impl(num, den, cu, n_seq, tok_begin, n_local, resp, cfg, comm, tis_w, tok_keep, seq_keep, coeff,
                      seq_score, stats_dev, ws, ws_bytes, dstatus, stream);
}

tim_status tim_comm_unique_id(void* out) {
  if (!out) return TIM_ERR_NULL;
  NcclApi* api = nccl();
  if (!api->ok) return TIM_ERR_NCCL;
  nccl_uid id;
  if (api->get_uid(&id) != 0) return TIM_ERR_NCCL;
  std::memcpy(out, &id, sizeof(id));
  return TIM_OK;
}

tim_status tim_comm_init(const void* uid, int32_t nranks, int32_t rank, tim_comm** out) {
  if (!uid || !out) return TIM_ERR_NULL;
  if (nranks < 1 || rank < 0 || rank >= nranks) return TIM_ERR_SHAPE;
  NcclApi* api = nccl();
  if (!api->ok) return TIM_ERR_NCCL;
  nccl_uid id;
  std::memcpy(&id, uid, sizeof(id));
  nccl_comm_t c = nullptr;
  if (api->init_rank(&c, nranks, id, rank) != 0) return TIM_ERR_NCCL;
  tim_comm* t = new tim_comm{c, nranks, rank};
  *out = t;
  return TIM_OK;
}

tim_status tim_comm_destroy(tim_comm* comm) {
  if (!comm) return TIM_ERR_NULL;
  NcclApi* api = nccl();
  if (api->ok && comm->comm) api->destroy(comm->comm);
  delete comm;
  return TIM_OK;
}

// ------------------------------------------------ vocab-parallel (TP) head (NEXT-4) --
tim_status tim_l2_persisting(int64_t bytes, int64_t* granted_bytes) {
  if (bytes < 0) return TIM_ERR_VALUE;
  int dev = 0, mx = 0;
  if (cudaGetDevice(&dev) != cudaSuccess ||
      cudaDeviceGetAttribute(&mx, cudaDevAttrMaxPersistingL2CacheSize, dev) != cudaSuccess)
    return TIM_ERR_CUDA;
  const size_t want = static_cast<size_t>(bytes < mx ? bytes : mx);
  size_t got = 0;
  if (cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, want) != cudaSuccess ||
      cudaDeviceGetLimit(&got, cudaLimitPersistingL2CacheSize) != cudaSuccess)
    return TIM_ERR_CUDA;
  if (granted_bytes) *granted_bytes = static_cast<int64_t>(got);
  return TIM_OK;
}

tim_status tim_tp_vocab_range(int32_t vocab, int32_t tp, int32_t rank, int32_t* begin, int32_t* end) {
  if (!begin || !end) return TIM_ERR_NULL;
  if (vocab < 1 || tp < 1 || rank < 0 || rank >= tp) return TIM_ERR_SHAPE;
  const int32_t S = vocab_slices(vocab);
  if (S % tp != 0) return TIM_ERR_SHAPE;
  const int32_t nvt = n_vocab_tiles(vocab);
  const int32_t s0 = rank * (S / tp), s1 = s0 + S / tp;
  *begin = ((s0 * nvt) / S) * 256;
  *end = std::min(((s1 * nvt) / S) * 256, vocab);
  return TIM_OK;
}

size_t tim_logprob_tp_partial_bytes(int64_t n_tok, int32_t vocab, int32_t tp) {
  if (n_tok < 0 || vocab < 1 || tp < 1 || vocab_slices(vocab) % tp != 0) return 0;
  return static_cast<size_t>(vocab_slices(vocab) / tp) * static_cast<size_t>(n_tok) * 16u;
}

tim_status tim_logprob_tp_partial(const void* hidden_bf16, int64_t ld_hidden, const void* weight_shard_bf16,
                                  int32_t hidden, int32_t vocab, int32_t tp, int32_t rank, const int64_t* token_ids,
                                  int64_t n_tok, float temperature, const float* temperatures_or_null,
                                  void* partial_out, void* workspace, size_t workspace_bytes, void* stream) {
  if (n_tok > 0 && !partial_out) return TIM_ERR_NULL;
  return logprob_impl(hidden_bf16, ld_hidden, weight_shard_bf16, hidden, vocab, token_ids, n_tok, temperature,
                      temperatures_or_null, nullptr, nullptr, workspace, workspace_bytes, nullptr, stream, nullptr, 0,
                      nullptr, 0, nullptr, tp, rank, partial_out);
}

tim_status tim_logprob_tp_merge(const void* gathered_partials, int64_t n_tok, int32_t vocab, const int64_t* token_ids,
                                const float* temperatures_or_null, float* logp_out, float* entropy_out_or_null,
                                void* workspace, size_t workspace_bytes, tim_device_status* dstatus, void* stream) {
  if (n_tok < 0 || vocab < 1) return TIM_ERR_SHAPE;
  if (n_tok == 0) return TIM_OK;
  if (!gathered_partials || !token_ids || !logp_out || !workspace) return TIM_ERR_NULL;
  if (!aligned(gathered_partials, 16) || !aligned(workspace, 16)) return TIM_ERR_ALIGN;
  if (workspace_bytes < kWsHeaderBytes) return TIM_ERR_WORKSPACE;
  DevInfo* dev = nullptr;
  tim_status st = device_info(&dev);
  if (st != TIM_OK) return st;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  WsHeader* hdr = static_cast<WsHeader*>(workspace);
  if (cudaMemsetAsync(hdr, 0, kWsHeaderBytes, s) != cudaSuccess) return TIM_ERR_CUDA;
  MergeParams mp{};
  mp.partials = static_cast<const float4*>(gathered_partials);
  mp.ids = token_ids;
  mp.temps = temperatures_or_null;
  mp.logp = logp_out;
  mp.entropy = entropy_out_or_null;
  mp.n_tok = n_tok;
  mp.vocab = vocab;
  mp.n_slices = vocab_slices(vocab);
  mp.ws = hdr;
  mp.dstatus = dstatus;
  return launch_logprob_merge(mp, s) == cudaSuccess ? TIM_OK : TIM_ERR_CUDA;
}

size_t tim_logprob_tp_workspace_bytes(int64_t n_tok, int32_t vocab, int32_t tp) {
  const size_t part = tim_logprob_tp_partial_bytes(n_tok, vocab, tp);
  if (n_tok < 0 || vocab < 1 || tp < 1 || vocab_slices(vocab) % tp != 0) return 0;
  return kWsHeaderBytes + part + part * static_cast<size_t>(tp);  // header, local block, gathered blocks
}

tim_status tim_logprob_tp(const void* hidden_bf16, int64_t ld_hidden, const void* weight_shard_bf16, int32_t hidden,
                          int32_t vocab, tim_comm* comm, const int64_t* token_ids, int64_t n_tok, float temperature,
                          const float* temperatures_or_null, float* logp_out, float* entropy_out_or_null,
                          void* workspace, size_t workspace_bytes, tim_device_status* dstatus, void* stream) {
  if (!comm) return TIM_ERR_NULL;
  const int32_t tp = comm->nranks;
  if (n_tok < 0 || vocab < 1 || vocab_slices(vocab) % tp != 0) return TIM_ERR_SHAPE;
  if (n_tok == 0) return TIM_OK;
  if (!workspace || !logp_out) return TIM_ERR_NULL;
  if (!aligned(workspace, 256)) return TIM_ERR_ALIGN;
  if (workspace_bytes < tim_logprob_tp_workspace_bytes(n_tok, vocab, tp)) return TIM_ERR_WORKSPACE;
  const size_t part = tim_logprob_tp_partial_bytes(n_tok, vocab, tp);
  uint8_t* ws = static_cast<uint8_t*>(workspace);
  uint8_t* local = ws + kWsHeaderBytes;
  uint8_t* gathered = local + part;
  tim_status st = tim_logprob_tp_partial(hidden_bf16, ld_hidden, weight_shard_bf16, hidden, vocab, tp, comm->rank,
                                         token_ids, n_tok, temperature, temperatures_or_null, local, ws,
                                         kWsHeaderBytes, stream);
  if (st != TIM_OK) return st;
  NcclApi* api = nccl();
  if (!api->ok) return TIM_ERR_NCCL;
  // [tp][S_v / tp][n_tok] in rank order = the full slice-major [S_v][n_tok] array
  if (api->all_gather(local, gathered, part, kNcclInt8, comm->comm, reinterpret_cast<cudaStream_t>(stream)) != 0)
    return TIM_ERR_NCCL;
  return tim_logprob_tp_merge(gathered, n_tok, vocab, token_ids, temperatures_or_null, logp_out, entropy_out_or_null,
                              ws, kWsHeaderBytes, dstatus, stream);
}

// --------------------------------------------------------------- RMSNorm (NEXT-4) --
tim_status tim_rmsnorm(const void* hidden, int64_t ld_hidden, const void* gamma, float eps, int32_t d, int64_t n_tok,
                       void* out, void* stream) {
  if (n_tok < 0 || d < 64 || d > 16384 || d % 64 != 0 || ld_hidden < d) return TIM_ERR_SHAPE;
  if (!(eps >= 0.f) || !std::isfinite(eps)) return TIM_ERR_VALUE;
  if (n_tok == 0) return TIM_OK;
  if (!hidden || !gamma || !out) return TIM_ERR_NULL;
  if (!aligned(hidden, 16) || !aligned(gamma, 16) || !aligned(out, 16) || ld_hidden % 8 != 0) return TIM_ERR_ALIGN;
  DevInfo* dev = nullptr;
  tim_status st = device_info(&dev);
  if (st != TIM_OK) return st;
  RmsNormParams p{};
  p.h = static_cast<const uint16_t*>(hidden);
  p.ld = ld_hidden;
  p.gamma = static_cast<const uint16_t*>(gamma);
  p.eps = eps;
  p.d = d;
  p.n = n_tok;
  p.out = static_cast<uint16_t*>(out);
  return launch_rmsnorm(p, reinterpret_cast<cudaStream_t>(stream)) == cudaSuccess ? TIM_OK : TIM_ERR_CUDA;
}

size_t tim_logprob_rmsnorm_workspace_bytes(int64_t n_tok, int32_t hidden, int32_t vocab) {
  if (n_tok < 0 || hidden < 1 || vocab < 1) return 0;
  const size_t x = (static_cast<size_t>(n_tok) * static_cast<size_t>(hidden) * 2u + 255) & ~size_t(255);
  return x + tim_logprob_workspace_bytes(n_tok, hidden, vocab);
}

tim_status tim_logprob_rmsnorm(const void* hidden, int64_t ld_hidden, const void* gamma, float eps, const void* weight,
                               int32_t d, int32_t vocab, const int64_t* ids, int64_t n_tok, float temperature,
                               const float* temps, float* logp, float* ent, void* ws, size_t ws_bytes,
                               tim_device_status* dstatus, void* stream) {
  if (n_tok > 0 && !ws) return TIM_ERR_NULL;
  if (n_tok > 0 && !aligned(ws, 256)) return TIM_ERR_ALIGN;
  if (n_tok > 0 && ws_bytes < tim_logprob_rmsnorm_workspace_bytes(n_tok, d, vocab)) return TIM_ERR_WORKSPACE;
  const size_t xb = (static_cast<size_t>(n_tok) * static_cast<size_t>(d) * 2u + 255) & ~size_t(255);
  void* x = ws;
  tim_status st = tim_rmsnorm(hidden, ld_hidden, gamma, eps, d, n_tok, x, stream);
  if (st != TIM_OK) return st;
  return tim_logprob(n_tok ? x : nullptr, d, weight, d, vocab, ids, n_tok, temperature, temps, logp, ent,
                     n_tok ? static_cast<uint8_t*>(ws) + xb : nullptr, n_tok ? ws_bytes - xb : 0, dstatus, stream);
}

// ------------------------------------------------------------------ head backward (NEXT-3) --
static int64_t bwd_g_ld(int32_t vocab) { return (static_cast<int64_t>(vocab) + 7) & ~int64_t(7); }
static int64_t bwd_block_rows(int64_t n_tok, int32_t vocab) {
  constexpr double kGBudget = 4294967296.0;  // bf16 G block <= 4 GiB
  int64_t nb = static_cast<int64_t>(kGBudget / (2.0 * static_cast<double>(bwd_g_ld(vocab))));
  nb = nb / 256 * 256;
  if (nb < 256) nb = 256;
  const int64_t need = (n_tok + 255) / 256 * 256;
  return need < nb ? need : nb;
}
static size_t al256(size_t x) { return (x + 255) & ~size_t(255); }

size_t tim_head_backward_workspace_bytes(int64_t n_tok, int32_t hidden, int32_t vocab) {
  if (n_tok < 0 || vocab < 1) return 0;
  if (n_tok == 0) return 0;
  const int64_t nb = bwd_block_rows(n_tok, vocab);
  return al256(tim_logprob_workspace_bytes(nb, hidden, vocab)) + 3 * al256(static_cast<size_t>(nb) * 4u) +
         static_cast<size_t>(nb) * static_cast<size_t>(bwd_g_ld(vocab)) * 2u;
}

tim_status tim_logprob_saved(const void* hidden_bf16, int64_t ld_hidden, const void* weight_bf16, int32_t hidden,
                             int32_t vocab, const int64_t* token_ids, int64_t n_tok, float temperature,
                             const float* temperatures_or_null, float* logp_out, float* entropy_out,
                             float* lse2_out, void* workspace, size_t workspace_bytes, tim_device_status* dstatus,
                             void* stream) {
  if (n_tok > 0 && (!entropy_out || !lse2_out)) return TIM_ERR_NULL;
  return logprob_impl(hidden_bf16, ld_hidden, weight_bf16, hidden, vocab, token_ids, n_tok, temperature,
                      temperatures_or_null, logp_out, entropy_out, workspace, workspace_bytes, dstatus, stream,
                      nullptr, 0, nullptr, 0, nullptr, 1, 0, nullptr, lse2_out, 0);
}

// ent_saved / lse2_saved null: run the forward per token block (tim_head_backward); else take the
// forward's per-token entropy and log2-sum-exp from the caller (tim_head_backward_saved).
static tim_status head_backward_impl(const void* hidden_bf16, int64_t ld_hidden, const void* weight_bf16, int32_t d,
                                     int32_t vocab, const int64_t* token_ids, int64_t n_tok, float temperature,
                                     const float* temps, const float* ent_saved, const float* lse2_saved,
                                     const float* grad_logp, const float* grad_ent_or_null,
                                     float* dhidden_or_null, float* dweight_or_null, void* ws, size_t ws_bytes,
                                     tim_device_status* dstatus, void* stream) {
  const Knobs kn = knobs();
  const bool saved = ent_saved != nullptr;
  if (!weight_bf16) return TIM_ERR_NULL;
  if (n_tok < 0 || n_tok >= (int64_t(1) << 31)) return TIM_ERR_SHAPE;
  if (d < 64 || d > 16384 || d % 64 != 0) return TIM_ERR_SHAPE;
  if (vocab < 1 || vocab > (1 << 24)) return TIM_ERR_SHAPE;
  if (ld_hidden < d) return TIM_ERR_SHAPE;
  if (!(temperature > 0.f) || !std::isfinite(temperature)) return TIM_ERR_VALUE;
  if (!aligned(weight_bf16, 16) || (ld_hidden * 2) % 16 != 0) return TIM_ERR_ALIGN;
  if (!dhidden_or_null && !dweight_or_null) return TIM_ERR_NULL;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (dweight_or_null && !aligned(dweight_or_null, 16)) return TIM_ERR_ALIGN;
  if (n_tok == 0) {  // dL/dW of an empty batch is 0; nothing else to do
    if (dweight_or_null &&
        cudaMemsetAsync(dweight_or_null, 0, static_cast<size_t>(vocab) * d * 4u, s) != cudaSuccess)
      return TIM_ERR_CUDA;
    return TIM_OK;
  }
  if (!hidden_bf16 || !token_ids || !grad_logp || !ws) return TIM_ERR_NULL;
  if (saved && !lse2_saved) return TIM_ERR_NULL;
  if (!aligned(hidden_bf16, 16) || !aligned(ws, 256)) return TIM_ERR_ALIGN;
  if (dhidden_or_null && !aligned(dhidden_or_null, 16)) return TIM_ERR_ALIGN;
  if (ws_bytes < tim_head_backward_workspace_bytes(n_tok, d, vocab)) return TIM_ERR_WORKSPACE;
  DevInfo* dev = nullptr;
  tim_status st = device_info(&dev);
  if (st != TIM_OK) return st;

  const int64_t nb = bwd_block_rows(n_tok, vocab), g_ld = bwd_g_ld(vocab);
  uint8_t* w8 = static_cast<uint8_t*>(ws);
  const size_t fwd_bytes = al256(tim_logprob_workspace_bytes(nb, d, vocab));
  uint8_t* fwd_ws = w8;
  float* logp = reinterpret_cast<float*>(w8 + fwd_bytes);
  float* ent_ws = reinterpret_cast<float*>(w8 + fwd_bytes + al256(nb * 4));
  float* lse2_ws = reinterpret_cast<float*>(w8 + fwd_bytes + 2 * al256(nb * 4));
  uint16_t* G = reinterpret_cast<uint16_t*>(w8 + fwd_bytes + 3 * al256(nb * 4));
  const int32_t S = vocab_slices(vocab);
  const int32_t nvt = n_vocab_tiles(vocab);
  CUtensorMap tw;
  if (!encode_bf16_2d(&tw, weight_bf16, vocab, d, d, fwd_w_box_rows(true))) return TIM_ERR_CUDA;
  if (dweight_or_null &&
      cudaMemsetAsync(dweight_or_null, 0, static_cast<size_t>(vocab) * d * 4u, s) != cudaSuccess)
    return TIM_ERR_CUDA;

  for (int64_t b0 = 0; b0 < n_tok; b0 += nb) {
    const int64_t nbc = (n_tok - b0 < nb) ? n_tok - b0 : nb;
    const void* hb = static_cast<const uint8_t*>(hidden_bf16) + b0 * ld_hidden * 2;
    const float* tb = temps ? temps + b0 : nullptr;
    // (1) forward: logp, H, log2-sum-exp of the block (the same kernel and numerics as tim_logprob),
    //     unless the caller saved them (tim_logprob_saved; batch-invariant, so the same values)
    const float* ent = saved ? ent_saved + b0 : ent_ws;
    const float* lse2 = saved ? lse2_saved + b0 : lse2_ws;
    if (!saved) {
      st = logprob_impl(hb, ld_hidden, weight_bf16, d, vocab, token_ids + b0, nbc, temperature, tb, logp, ent_ws,
                        fwd_ws, fwd_bytes, dstatus, stream, nullptr, 0, nullptr, 0, nullptr, 1, 0, nullptr, lse2_ws,
                        b0, /*pad_small=*/false);
      if (st != TIM_OK) return st;
    }
    // (2) recompute the logits tile by tile; the epilogue writes G = dL/dz (bf16) instead of LSE partials
    CUtensorMap th;
    if (!encode_bf16_2d(&th, hb, nbc, d, ld_hidden, 128)) return TIM_ERR_CUDA;
    if (cudaMemsetAsync(fwd_ws, 0, kWsHeaderBytes, s) != cudaSuccess) return TIM_ERR_CUDA;
    LogprobParams p{};
    p.ids = token_ids + b0;
    p.temps = tb;
    p.temperature = temperature;
    p.partials = reinterpret_cast<float4*>(fwd_ws + kWsHeaderBytes);  // not written in gradient mode
    p.n_tok = static_cast<int>(nbc);
    p.vocab = vocab;
    p.hidden = d;
    p.n_mt = static_cast<int>((nbc + fwd_unit_rows(true) - 1) / fwd_unit_rows(true));
    p.n_vt = nvt;
    p.n_slices = S;
    p.n_slices_total = S;
    p.h_policy = kn.h_policy;
    p.w_policy = kn.w_policy;
    p.sleep_waits = kn.sleep_waits;
    p.progress = reinterpret_cast<uint32_t*>(fwd_ws + kWsProgressOffset);
    p.sync_slack = kn.sync_slack;
    p.hidden_ptr = hb;
    p.ld_hidden_bytes = ld_hidden * 2;
    p.grad_logp = grad_logp + b0;
    p.grad_ent = grad_ent_or_null ? grad_ent_or_null + b0 : nullptr;
    p.ent_in = ent;
    p.lse2_in = lse2;
    p.g_out = G;
    p.g_ld = g_ld;
    p.g_col0 = 0;
    const int64_t n_units = static_cast<int64_t>(p.n_mt) * S;
    int64_t cap = dev->max_pair_clusters;
    if (kn.max_clusters > 0 && kn.max_clusters < cap) cap = kn.max_clusters;
    const int64_t groups = n_units < cap ? n_units : cap;
    p.group = pick_group(dev, true, S, groups, d, kn.group);
    if (kn.die_groups) set_die_grouping(dev, p, groups, s);
    CUtensorMap tg;
    if (!encode_g_store(&tg, G, nbc, vocab, g_ld)) return TIM_ERR_CUDA;
    if (launch_head_grad(th, tw, tg, p, static_cast<int>(groups * 2), s) != cudaSuccess) return TIM_ERR_CUDA;
    // (3) dH[b] = G W and (4) dW += G^T H[b]: the hand-written tcgen05 GEMMs (gemm.cu).  dH's K
    //     order (ascending V in steps of 16) is a constant of (V, d): batch-invariant rows.
    int max_pairs = dev->max_pair_clusters;
    if (kn.max_clusters > 0 && kn.max_clusters < max_pairs) max_pairs = kn.max_clusters;
    uint32_t* prog = reinterpret_cast<uint32_t*>(fwd_ws + kWsProgressOffset);  // per-pair gate counters
    if (dhidden_or_null) {
      CUtensorMap ta, tb;
      if (!encode_bf16_2d(&ta, G, nbc, vocab, g_ld, 128)) return TIM_ERR_CUDA;        // A = G, K-major
      if (!encode_bf16_2d(&tb, weight_bf16, vocab, d, d, 64)) return TIM_ERR_CUDA;    // B = W, MN-major
      if (cudaMemsetAsync(prog, 0, kWsHeaderBytes - kWsProgressOffset, s) != cudaSuccess) return TIM_ERR_CUDA;
      BwdGemmParams gp{dhidden_or_null + b0 * d, d, static_cast<int>(nbc), d, vocab, prog, kn.gemm_slack,
                       kn.gemm_pol[0], kn.gemm_pol[1]};
      if (kn.die_groups) set_gemm_die(dev, gp, max_pairs, s);
      if (launch_bwd_gemm_dh(ta, tb, gp, max_pairs, s) != cudaSuccess) return TIM_ERR_CUDA;
    }
    if (dweight_or_null) {
      CUtensorMap ta, tb;
      if (!encode_bf16_2d(&ta, G, nbc, vocab, g_ld, 64)) return TIM_ERR_CUDA;         // A = G^T, MN-major
      if (!encode_bf16_2d(&tb, hb, nbc, d, ld_hidden, 64)) return TIM_ERR_CUDA;       // B = H, MN-major
      if (cudaMemsetAsync(prog, 0, kWsHeaderBytes - kWsProgressOffset, s) != cudaSuccess) return TIM_ERR_CUDA;
      BwdGemmParams gp{dweight_or_null, d, vocab, d, static_cast<int>(nbc), prog, kn.gemm_slack, kn.gemm_pol[2],
                       kn.gemm_pol[3]};
      if (kn.die_groups) set_gemm_die(dev, gp, max_pairs, s);
      if (launch_bwd_gemm_dw(ta, tb, gp, max_pairs, s) != cudaSuccess) return TIM_ERR_CUDA;
    }
  }
  return TIM_OK;
}

tim_status tim_head_backward(const void* hidden_bf16, int64_t ld_hidden, const void* weight_bf16, int32_t d,
                             int32_t vocab, const int64_t* token_ids, int64_t n_tok, float temperature,
                             const float* temps, const float* grad_logp, const float* grad_ent_or_null,
                             float* dhidden_or_null, float* dweight_or_null, void* ws, size_t ws_bytes,
                             tim_device_status* dstatus, void* stream) {
  return head_backward_impl(hidden_bf16, ld_hidden, weight_bf16, d, vocab, token_ids, n_tok, temperature, temps,
                            nullptr, nullptr, grad_logp, grad_ent_or_null, dhidden_or_null, dweight_or_null, ws,
                            ws_bytes, dstatus, stream);
}

tim_status tim_head_backward_saved(const void* hidden_bf16, int64_t ld_hidden, const void* weight_bf16, int32_t d,
                                   int32_t vocab, const int64_t* token_ids, int64_t n_tok, float temperature,
                                   const float* temps, const float* entropy_saved, const float* lse2_saved,
                                   const float* grad_logp, const float* grad_ent_or_null, float* dhidden_or_null,
                                   float* dweight_or_null, void* ws, size_t ws_bytes, tim_device_status* dstatus,
                                   void* stream) {
  if (n_tok > 0 && (!entropy_saved || !lse2_saved)) return TIM_ERR_NULL;
  return head_backward_impl(hidden_bf16, ld_hidden, weight_bf16, d, vocab, token_ids, n_tok, temperature, temps,
                            entropy_saved, lse2_saved, grad_logp, grad_ent_or_null, dhidden_or_null,
                            dweight_or_null, ws, ws_bytes, dstatus, stream);
}

// ------------------------------------------------------------------ PPO (NEXT-2) --
static tim_status check_ppo_cfg(const tim_ppo_cfg* c) {
  if (!c) return TIM_ERR_NULL;
  if (!std::isfinite(c->clip_lo) || !std::isfinite(c->clip_hi) || !(c->clip_lo <= c->clip_hi)) return TIM_ERR_VALUE;
  if (!std::isfinite(c->hist_lo) || !std::isfinite(c->hist_inv_width) || !(c->hist_inv_width > 0.0))
    return TIM_ERR_VALUE;
  if (c->hist_bins < 1 || c->hist_bins > ppo_max_hist_bins()) return TIM_ERR_VALUE;
  return TIM_OK;
}

size_t tim_ppo_partial_bytes(int64_t n_seq, int32_t hist_bins) {
  if (n_seq < 0 || hist_bins < 1) return 0;
  return sizeof(tim_ppo_partial_header) + 16u * static_cast<size_t>(hist_bins + 2) +
         static_cast<size_t>(n_seq) * sizeof(tim_seq_partial);
}

size_t tim_ppo_workspace_bytes(int64_t n_seq, int32_t hist_bins, int32_t nranks) {
  if (n_seq < 0 || hist_bins < 1 || nranks < 1) return 0;
  const size_t b = (tim_ppo_partial_bytes(n_seq, hist_bins) + 255) & ~size_t(255);
  return b * (1 + static_cast<size_t>(nranks));
}

tim_status tim_ppo_local(const float* cur, const float* old, const float* adv, const float* coeff, const uint8_t* resp,
                         const int64_t* cu, int64_t n_seq, int64_t tok_begin, int64_t n_local, const tim_ppo_cfg* cfg,
                         float* loss, float* grad, uint8_t* clipped, void* partial_out, tim_device_status* dstatus,
                         void* stream) {
  tim_status st = check_common(cur, old, cu, n_seq, tok_begin, n_local, resp);
  if (st != TIM_OK) return st;
  if ((st = check_ppo_cfg(cfg)) != TIM_OK) return st;
  if (!partial_out) return TIM_ERR_NULL;
  if (n_local > 0 && (!adv || !loss || !grad || !clipped)) return TIM_ERR_NULL;
  if (!aligned(partial_out, 16)) return TIM_ERR_ALIGN;
  DevInfo* dev = nullptr;
  if ((st = device_info(&dev)) != TIM_OK) return st;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (cudaMemsetAsync(partial_out, 0, tim_ppo_partial_bytes(n_seq, cfg->hist_bins), s) != cudaSuccess)
    return TIM_ERR_CUDA;
  if (n_local == 0) return TIM_OK;
  PpoLocalParams p{};
  p.cur = cur;
  p.old = old;
  p.adv = adv;
  p.coeff = coeff;
  p.resp = resp;
  p.cu = cu;
  p.n_seq = n_seq;
  p.tok_begin = tok_begin;
  p.n = n_local;
  p.clip_lo = cfg->clip_lo;
  p.clip_hi = cfg->clip_hi;
  p.hist_lo = cfg->hist_lo;
  p.hist_inv_width = cfg->hist_inv_width;
  p.bins = cfg->hist_bins;
  p.bins_d = static_cast<double>(cfg->hist_bins);
  p.loss = loss;
  p.grad = grad;
  p.clipped = clipped;
  uint8_t* blk = static_cast<uint8_t*>(partial_out);
  p.hdr = reinterpret_cast<tim_ppo_partial_header*>(blk);
  p.hist = reinterpret_cast<int64_t*>(blk + sizeof(tim_ppo_partial_header));
  p.seqp = reinterpret_cast<tim_seq_partial*>(blk + sizeof(tim_ppo_partial_header) +
                                              16u * static_cast<size_t>(cfg->hist_bins + 2));
  p.dstatus = dstatus;
  p.vec = aligned(cur, 16) && aligned(old, 16) && aligned(adv, 16) && aligned(coeff, 16) && aligned(loss, 16) && aligned(grad, 16) && aligned(clipped, 4) &&
          aligned(resp, 4);
  return launch_ppo_local(p, dev->num_sms, s) == cudaSuccess ? TIM_OK : TIM_ERR_CUDA;
}

static tim_status ppo_finish_impl(const void* gathered, int32_t nranks, int64_t n_seq, const tim_ppo_cfg* cfg,
                                  double* seq_loss, int64_t* hist, tim_ppo_stats* stats, unsigned long long* scratch,
                                  void* stream) {
  if (!gathered) return TIM_ERR_NULL;
  if (nranks < 1 || n_seq < 0) return TIM_ERR_SHAPE;
  tim_status st = check_ppo_cfg(cfg);
  if (st != TIM_OK) return st;
  if (!aligned(gathered, 16)) return TIM_ERR_ALIGN;
  DevInfo* dev = nullptr;
  if ((st = device_info(&dev)) != TIM_OK) return st;
  PpoFinishParams f{};
  f.gathered = static_cast<const uint8_t*>(gathered);
  f.block_bytes = static_cast<int64_t>(tim_ppo_partial_bytes(n_seq, cfg->hist_bins));
  f.nranks = nranks;
  f.n_seq = n_seq;
  f.bins = cfg->hist_bins;
  f.seq_loss = seq_loss;
  f.hist = hist;
  f.stats = stats;
  f.scratch = scratch;
  return launch_ppo_finish(f, dev->num_sms, reinterpret_cast<cudaStream_t>(stream)) == cudaSuccess ? TIM_OK
                                                                                                   : TIM_ERR_CUDA;
}

tim_status tim_ppo_finish(const void* gathered, int32_t nranks, int64_t n_seq, const tim_ppo_cfg* cfg,
                          double* seq_loss, int64_t* hist, tim_ppo_stats* stats, void* stream) {
  return ppo_finish_impl(gathered, nranks, n_seq, cfg, seq_loss, hist, stats, nullptr, stream);
}

tim_status tim_ppo_loss(const float* cur, const float* old, const float* adv, const float* coeff, const uint8_t* resp,
                        const int64_t* cu, int64_t n_seq, int64_t tok_begin, int64_t n_local, const tim_ppo_cfg* cfg,
                        tim_comm* comm, float* loss, float* grad, uint8_t* clipped, double* seq_loss, int64_t* hist,
                        tim_ppo_stats* stats, void* ws, size_t ws_bytes, tim_device_status* dstatus, void* stream) {
  tim_status st = check_ppo_cfg(cfg);
  if (st != TIM_OK) return st;
  const int nranks = comm ? comm->nranks : 1;
  if (!ws) return TIM_ERR_NULL;
  if (!aligned(ws, 256)) return TIM_ERR_ALIGN;
  if (ws_bytes < tim_ppo_workspace_bytes(n_seq, cfg->hist_bins, nranks)) return TIM_ERR_WORKSPACE;
  uint8_t* local = static_cast<uint8_t*>(ws);
  const size_t blk = (tim_ppo_partial_bytes(n_seq, cfg->hist_bins) + 255) & ~size_t(255);
  if ((st = tim_ppo_local(cur, old, adv, coeff, resp, cu, n_seq, tok_begin, n_local, cfg, loss, grad, clipped, local,
                          dstatus, stream)) != TIM_OK)
    return st;
  const void* gathered = local;
  if (comm != nullptr) {
    NcclApi* api = nccl();
    if (!api->ok) return TIM_ERR_NCCL;
    if (api->all_gather(local, local + blk, tim_ppo_partial_bytes(n_seq, cfg->hist_bins), kNcclInt8, comm->comm,
                        reinterpret_cast<cudaStream_t>(stream)) != 0)
      return TIM_ERR_NCCL;
    gathered = local + blk;
  }
  // the local block's header reserved[2..3] (zeroed with the block; pass 1 uses [0..1]) serve as
  // the finish pass's {ticket, contributing sequences}
  unsigned long long* scratch =
      reinterpret_cast<unsigned long long*>(&reinterpret_cast<tim_ppo_partial_header*>(local)->reserved[2]);
  return ppo_finish_impl(gathered, nranks, n_seq, cfg, seq_loss, hist, stats, scratch, stream);
}

tim_status tim_ppo_stats_finalize(tim_ppo_stats* h) {
  if (!h) return TIM_ERR_NULL;
  const double sc = std::ldexp(1.0, -52);
  const double nc = static_cast<double>(h->n_contrib);
  h->batch_loss = h->n_seq_contrib ? (i128_host_to_double(h->sum_loss_fx) * sc) / static_cast<double>(h->n_seq_contrib)
                                   : 0.0;
  h->clip_frac = h->n_contrib ? static_cast<double>(h->n_clipped) / nc : 0.0;
  h->mean_k1 = h->n_contrib ? (i128_host_to_double(h->sum_k1_fx) * sc) / nc : 0.0;
  h->mean_k3 = h->n_contrib ? (i128_host_to_double(h->sum_k3_fx) * sc) / nc : 0.0;
  return TIM_OK;
}

// ---------------------------------------------------------------- debug ABI --
tim_status tim_debug_logprob_logits(const void* hidden_bf16, int64_t ld_hidden, const void* weight_bf16,
                                    int32_t hidden, int32_t vocab, const int64_t* token_ids, int64_t n_tok,
                                    float* logits_out, int64_t ld_logits, float* logp_out, float* entropy_out,
                                    void* workspace, size_t workspace_bytes, void* stream) {
  if (!logits_out) return TIM_ERR_NULL;
  if (ld_logits < vocab) return TIM_ERR_SHAPE;
  return logprob_impl(hidden_bf16, ld_hidden, weight_bf16, hidden, vocab, token_ids, n_tok, 1.0f, nullptr, logp_out,
                      entropy_out, workspace, workspace_bytes, nullptr, stream, logits_out, ld_logits);
}

tim_status tim_debug_set_pad_small(int32_t enable) {
  if (enable != 0 && enable != 1) return TIM_ERR_VALUE;
  g_pad_small = enable;
  return TIM_OK;
}

tim_status tim_debug_set_kernel(int32_t use_pair, int32_t max_ctas_or_clusters) {
  if (use_pair != 0 && use_pair != 1) return TIM_ERR_VALUE;
  if (max_ctas_or_clusters < 0) return TIM_ERR_VALUE;
  g_use_pair = use_pair;
  g_max_clusters = max_ctas_or_clusters;
  return TIM_OK;
}

tim_status tim_debug_set_cluster(int32_t pairs_per_cluster) {
  if (pairs_per_cluster != 1 && pairs_per_cluster != 2) return TIM_ERR_VALUE;
  g_quad = pairs_per_cluster == 2;
  return TIM_OK;
}

tim_status tim_debug_set_schedule(int32_t group, int32_t demote) {
  if (group != 0 && group != 1 && group != 2 && group != 4 && group != 8) return TIM_ERR_VALUE;
  g_group = group;
  g_demote = demote != 0;
  return TIM_OK;
}

tim_status tim_debug_set_gemm_slack(int32_t k_blocks) {
  if (k_blocks < 0) return TIM_ERR_VALUE;
  g_gemm_slack = k_blocks;
  return TIM_OK;
}

tim_status tim_debug_set_gemm_policy(int32_t dh_a, int32_t dh_b, int32_t dw_a, int32_t dw_b) {
  const int32_t v[4] = {dh_a, dh_b, dw_a, dw_b};
  for (int i = 0; i < 4; ++i)
    if (v[i] < 1 || v[i] > 3) return TIM_ERR_VALUE;
  for (int i = 0; i < 4; ++i) g_gemm_pol[i] = v[i];
  return TIM_OK;
}

tim_status tim_debug_set_die_groups(int32_t enable) {
  if (enable != 0 && enable != 1) return TIM_ERR_VALUE;
  g_die_groups = enable;
  return TIM_OK;
}

tim_status tim_debug_die_map(int32_t* state_out, uint64_t* mask_out4) {
  if (!state_out || !mask_out4) return TIM_ERR_NULL;
  DevInfo* dev = nullptr;
  const tim_status st = device_info(&dev);
  if (st != TIM_OK) return st;
  ensure_die_map(dev, nullptr);
  *state_out = dev->die_state.load();
  std::memcpy(mask_out4, dev->die_mask, sizeof(dev->die_mask));
  return TIM_OK;
}

tim_status tim_debug_set_correct_split(int32_t split) {
  if (split != 0 && split != 1) return TIM_ERR_VALUE;
  g_split_correct = split;
  return TIM_OK;
}

tim_status tim_debug_set_tuning(int32_t h_policy, int32_t w_policy, int32_t sleep_waits, int32_t sync_slack) {
  if (sync_slack < 0) return TIM_ERR_VALUE;
  if (h_policy < 0 || h_policy > 3 || w_policy < 0 || w_policy > 3) return TIM_ERR_VALUE;
  if (sleep_waits < 0 || sleep_waits > 7) return TIM_ERR_VALUE;
  g_sync_slack = sync_slack;
  g_h_policy = h_policy;
  g_w_policy = w_policy;
  g_sleep_waits = sleep_waits;  // bit 0 producer, bit 1 epilogue, bit 2 MMA issuer (3 = the round-1 'sleep')
  return TIM_OK;
}

}  // extern "C"
