// tim_internal.h -- shared declarations between the C-ABI host layer and the kernels.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "../../include/tim.h"

namespace tim {

// Per-call workspace header (memset to 0 before every call).
struct WsHeader {
  unsigned long long bad_inv;  // max over bad tokens of (kBadSentinel - index); 0 = no error
  unsigned int counter;        // "last block" ticket
  unsigned int pad;            // the fused correction's grid-barrier counter (correct.cu)
  unsigned long long reserved[6];
};
static_assert(sizeof(WsHeader) == 64, "WsHeader size");
constexpr unsigned long long kBadSentinel = 1ull << 62;
constexpr int kMaxDevices = 64;  // devices per process the library keeps per-device state for
constexpr size_t kWsHeaderBytes = 1024;      // WsHeader + per-pair progress counters
constexpr size_t kWsProgressOffset = 64;
constexpr int kMaxProgress = (kWsHeaderBytes - kWsProgressOffset) / 4;

struct LogprobParams {
  const int64_t* ids;
  const float* temps;
  float temperature;
  float4* partials;  // [n_slices][n_tok]
  int n_tok;
  int vocab;
  int hidden;
  int n_mt;
  int n_vt;
  int n_slices;         // slices this launch runs (all of them unless tensor-parallel)
  int n_slices_total;   // S_v of the full vocabulary
  int slice0;           // first global slice of this launch
  int w_row0;           // first W row present in the weight tensor (tensor-parallel shard)
  float* debug_logits;  // test-only raw fp32 accumulators [n_tok][debug_ld]
  int64_t debug_ld;
  int h_policy;         // L2 eviction policy of H / W tile loads: 0 none, 1 normal, 2 first, 3 last
  int w_policy;
  int sleep_waits;      // mbarrier waits that sleep (suspend-time hint) instead of polling: bit 0 producer, 1 epilogue, 2 MMA
  uint32_t* progress;   // [clusters] tiles issued per CTA pair (workspace, zeroed per call)
  int sync_slack;       // max tiles a pair may run ahead of the slowest pair (0 = no throttle)
  int group;            // pairs sharing one M-tile (split its slices) so the live H tiles fit in L2
  const uint64_t* row_keys;  // sampling twin: per-row Philox counter (e.g. sequence << 32 | position)
  uint64_t seed;             // sampling twin: Philox key
  float4* partials2;         // sampling twin: {best score, its y, its column, 0} [n_slices][n_tok]
  const void* hidden_ptr;    // H base (for L2 priority demotion of finished M-tiles)
  int64_t ld_hidden_bytes;
  int demote;                // demote finished H tiles to evict_normal
  unsigned long long* gate_stats;  // diagnostics: number of progress gates given up (timed out)
  unsigned long long* clk;         // diagnostics: {clock64, globaltimer} at CTA 0's start and end
  // head backward (NEXT-3) gradient epilogue
  const float* grad_logp;    // [n_tok] dL/dlogp
  const float* grad_ent;     // [n_tok] dL/dH or null
  const float* ent_in;       // [n_tok] entropy (nats) from the forward
  const float* lse2_in;      // [n_tok] log2-sum-exp of y = z log2(e) / T from the forward
  uint16_t* g_out;           // bf16 G block of the current slice, [n_tok][g_ld]
  int64_t g_ld;
  int g_col0;                // first vocab column of the G block
  // die-aware grouping (G > 1): SM -> die bits from the per-device probe; the pairs of one M-tile
  // group are taken from the same die so that the group's H tile is not cached in both dies' L2
  int die_ok;
  uint64_t die_mask[4];      // bit s = die of SM s (smid < 256)
  uint32_t* die_counter;     // 2 words in the zeroed workspace header: clusters seen per die
};

struct MergeParams {
  const float4* partials;
  const int64_t* ids;
  const float* temps;
  float* logp;
  float* entropy;
  int64_t n_tok;
  int vocab;
  int n_slices;
  WsHeader* ws;
  tim_device_status* dstatus;
  const float4* partials2;  // sampling twin
  int64_t* ids_out;         // sampling twin
  float* lse2_out;          // head backward: per-token log2-sum-exp (may be null)
  int64_t index_base;       // added to a bad token's index in the status (token-blocked callers)
};

// Commit the call's data-error state to the caller's status word; executed by the last block
// of a grid to finish (ticket in ws->counter).  Deterministic: min index wins.
__device__ __forceinline__ void commit_status_last_block(WsHeader* ws, tim_device_status* st) {
  __shared__ int last;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned int ticket = atomicAdd(&ws->counter, 1u);
    last = (ticket == gridDim.x * gridDim.y * gridDim.z - 1);
  }
  __syncthreads();
  if (last && threadIdx.x == 0 && st != nullptr) {
    __threadfence();
    const unsigned long long b = atomicAdd(&ws->bad_inv, 0ull);
    if (b != 0) {
      const int64_t idx = static_cast<int64_t>(kBadSentinel - b);
      volatile tim_device_status* vs = st;
      if (vs->code == 0) {
        vs->first_bad_index = idx;
        vs->code = TIM_ERR_DATA;
      } else if (idx < vs->first_bad_index) {
        vs->first_bad_index = idx;
      }
    }
  }
}

// logprob.cu
int fwd_unit_rows(bool pair);
int fwd_w_box_rows(bool pair);
cudaError_t launch_logprob_fwd(bool pair, bool debug, bool sample, bool quad, const CUtensorMap& th,
                               const CUtensorMap& tw, const LogprobParams& p, int grid, cudaStream_t stream);
cudaError_t launch_logprob_merge(const MergeParams& p, cudaStream_t stream);
cudaError_t launch_pad_rows(const void* src, int64_t ld_src_bytes, void* dst, int row_bytes, int n_tok, int n_rows,
                            cudaStream_t stream);
cudaError_t launch_head_grad(const CUtensorMap& th, const CUtensorMap& tw, const CUtensorMap& tg,
                             const LogprobParams& p, int grid, cudaStream_t stream);
cudaError_t launch_sample_merge(const MergeParams& p, cudaStream_t stream);
// one-time per-device probe: CTA b runs on SM smid[b] and times dependent L2 loads of `nlines`
// zero-filled 128-B lines `stride_u64` words apart -> lat[b * nlines + l] (cycles per load)
cudaError_t launch_die_probe(const uint64_t* lines, int nlines, int stride_u64, uint32_t* lat, uint32_t* smid,
                             int grid, cudaStream_t stream);

// gemm.cu -- head-backward GEMMs C[m, n] (fp32, row pitch ldc) = A[m, k] B[k, n] (bf16 operands
// through TMA tensor maps): dH stores, dW accumulates (red.global.add)
struct BwdGemmParams {
  float* c;
  int64_t ldc;
  int m, n, k;
  uint32_t* progress;  // [pairs] k-blocks issued per CTA pair (zeroed per launch), or null: no gate
  int sync_slack;      // max k-blocks a pair may run ahead of the slowest (0 = no gate)
  int a_policy, b_policy;  // L2 policy of the A / B tile loads: 1 normal, 2 evict_first, 3 evict_last
  // die-aware tile order (as LogprobParams): the pairs sharing an operand stream sit on one die
  int die_ok;
  uint64_t die_mask[4];
  uint32_t* die_counter;
};
cudaError_t launch_bwd_gemm_dh(const CUtensorMap& tg_kmajor, const CUtensorMap& tw_mn, const BwdGemmParams& p,
                               int max_pairs, cudaStream_t stream);
cudaError_t launch_bwd_gemm_dw(const CUtensorMap& tg_mn, const CUtensorMap& th_mn, const BwdGemmParams& p,
                               int max_pairs, cudaStream_t stream);

// correct.cu
struct CorrectDevCfg {
  int tis, tok_rs, seq_rs, seq_agg;
  double tis_cap, log_tis_cap, log_lo, log_hi, tau_seq;
};
struct LocalParams {
  const float* num;
  const float* den;
  const int64_t* cu;
  int64_t n_seq;
  int64_t tok_begin;
  int64_t n;
  const uint8_t* resp;
  float* tis_w;       // may be null (stats only)
  uint8_t* tok_keep;  // may be null
  float* coeff;       // may be null
  tim_partial_header* hdr;
  tim_seq_partial* seqp;
  CorrectDevCfg cfg;
  tim_device_status* dstatus;
  int vec;            // every per-token array allows 16-B (4-B for u8) vector accesses
  int interior;       // set by the launcher: no token with |delta| <= 2^-6 can be truncated or
                      // token-rejected and min(e^delta, tau) = e^delta there (select-free fast body)
};
struct FinishParams {
  const uint8_t* gathered;  // [nranks][block_bytes]
  int64_t block_bytes;
  int nranks;
  int64_t n_seq;
  CorrectDevCfg cfg;
  uint8_t* seq_keep;     // may be null
  double* seq_score;     // may be null
  tim_stats* stats;      // may be null
  unsigned long long* scratch;  // {ticket, rejections}, zeroed, or null (then one block)
};
struct ZeroParams {
  const int64_t* cu;
  int64_t n_seq;
  int64_t tok_begin;
  int64_t n;
  const uint8_t* seq_keep;
  float* coeff;
};
// ppo.cu
struct PpoLocalParams {
  const float* cur;
  const float* old;
  const float* adv;
  const float* coeff;    // may be null (then resp / all)
  const uint8_t* resp;   // may be null
  const int64_t* cu;
  int64_t n_seq;
  int64_t tok_begin;
  int64_t n;
  double clip_lo, clip_hi, hist_lo, hist_inv_width;
  double bins_d;         // (double) bins, for the branch-free histogram slot
  int bins;
  float* loss;
  float* grad;
  uint8_t* clipped;
  tim_ppo_partial_header* hdr;
  int64_t* hist;         // [2][bins + 2] inside the partial block
  tim_seq_partial* seqp;
  tim_device_status* dstatus;
  int vec;               // every per-token array allows 16-B (4-B for u8) vector accesses
};
struct PpoFinishParams {
  const uint8_t* gathered;
  int64_t block_bytes;
  int nranks;
  int64_t n_seq;
  int bins;
  double* seq_loss;      // may be null
  int64_t* hist;         // may be null
  tim_ppo_stats* stats;  // may be null
  unsigned long long* scratch;  // {ticket, contributing sequences}, zeroed, or null (then one block)
};
int ppo_max_hist_bins();

// rmsnorm.cu
struct RmsNormParams {
  const uint16_t* h;      // bf16 [n][ld] (pre-norm hidden states)
  int64_t ld;
  const uint16_t* gamma;  // bf16 [d]
  float eps;
  int d;
  int64_t n;
  uint16_t* out;          // bf16 [n][d]
};
cudaError_t launch_rmsnorm(const RmsNormParams& p, cudaStream_t stream);
cudaError_t launch_ppo_local(const PpoLocalParams& p, int num_sms, cudaStream_t stream);
cudaError_t launch_ppo_finish(const PpoFinishParams& p, int num_sms, cudaStream_t stream);

cudaError_t launch_correct_local(const LocalParams& p, int num_sms, cudaStream_t stream);
cudaError_t launch_correct_finish(const FinishParams& p, int num_sms, cudaStream_t stream);
cudaError_t launch_correct_zero(const ZeroParams& p, cudaStream_t stream);
// P = 1: pass 1 + decisions / stats + zeroing in one cooperative launch (grid barriers on the
// local block header's WsHeader::pad word, zeroed with the block)
cudaError_t launch_correct_fused(const LocalParams& p, const FinishParams& f, const ZeroParams& z, int num_sms,
                                 cudaStream_t stream);

}  // namespace tim
