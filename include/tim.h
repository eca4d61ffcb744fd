/*
 * tim.h -- C ABI of the B200-native batch-invariant log-prob + TIS/RS library (libtim.so).
 *
 * Method: arxiv 2605.14220 ("Training-Inference Mismatch", PAPER.md).  The
 * library implements the data-parallel hot path of the paper's zero-mismatch
 * setting:
 *   tim_logprob         per-token log pi(a_t | s_t) of the sampled id and the entropy,
 *                       recomputed from the final hidden state (§4.1
 *                       "the trainer re-evaluates the sampled tokens"; §2 P:99 the
 *                       token distributions), bit-identical for a token whatever batch
 *                       it is scored in (§3.1 P:202-207 "fix the tiling and reduction
 *                       order").
 *   tim_mismatch_stats  delta_t = log pi_train_old - log pi_rollout_old (§2),
 *                       batch mean / max |delta| (fig:delta_t_batch), K1 / K3
 *                       means (§4.1).
 *   tim_correct         TIS weights min(r_corr, tau_tok) (§4.2), token-level
 *                       RS (reading U4), sequence-level RS 1[S_seq <= tau_seq] with
 *                       S_seq = sum_t K(q_t) (App. A.4), the
 *                       per-token coefficient resp * tok_keep * seq_keep * w.
 *
 * Conventions (apply to every entry point unless stated otherwise)
 *   - Every pointer argument is DEVICE memory owned by the caller, except
 *     `cfg_host` (host) and the tim_stats_finalize argument (host).  The library
 *     allocates nothing on the hot path; the only library-owned object is tim_comm.
 *   - All calls are asynchronous and stream-ordered on `stream` (cudaStream_t passed
 *     as void*; NULL = legacy default stream).  Collectives are enqueued on it too.
 *   - Argument errors are detected on the host and returned synchronously BEFORE any
 *     launch (nothing is enqueued).  Data errors found on the device (token id out of
 *     [0, V), non-finite log-prob) are reported in the caller's device status word
 *     `dstatus` (zero-initialise it; code = TIM_ERR_DATA, first_bad_index = minimum
 *     offending global token index, written with integer atomics => deterministic).
 *   - Runs on sm_100a only; on any other device every compute call returns
 *     TIM_ERR_UNSUPPORTED.  There is no CPU fallback.
 *   - A tim_comm must not be used from two host threads at once (NCCL rule).
 */
#ifndef TIM_H_
#define TIM_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TIM_ABI_VERSION 1

typedef enum {
  TIM_OK = 0,
  TIM_ERR_NULL = 1,        /* a required pointer is NULL                                  */
  TIM_ERR_SHAPE = 2,       /* a size is out of range / inconsistent                       */
  TIM_ERR_ALIGN = 3,       /* TMA alignment: pointers 16-B aligned, ld_hidden*2 % 16 == 0 */
  TIM_ERR_VALUE = 4,       /* a scalar parameter is out of range (temperature, tau, ...)  */
  TIM_ERR_WORKSPACE = 5,   /* workspace too small (query the *_workspace_bytes function)  */
  TIM_ERR_CUDA = 6,        /* a CUDA runtime / driver call failed                         */
  TIM_ERR_NCCL = 7,        /* NCCL unavailable or a collective failed                     */
  TIM_ERR_UNSUPPORTED = 8, /* device is not sm_100 (B200)                                 */
  TIM_ERR_DATA = 9         /* device-side data error (only ever stored in dstatus->code)   */
} tim_status;

/* Device status word: caller-owned device memory, zero-initialised by the caller. */
typedef struct {
  int32_t code;             /* TIM_OK or TIM_ERR_DATA                                */
  int32_t reserved;
  int64_t first_bad_index;  /* valid when code != 0: minimum offending token index    */
} tim_device_status;

const char* tim_status_string(tim_status s);
int tim_abi_version(void);

/* ----------------------------------------------------------------------------
 * tim_logprob
 *
 * For every token row t in [0, n_tok):
 *   z_v   = sum_k H[t,k] W[v,k]                 bf16 x bf16 products, fp32 accumulation
 *                                               (tcgen05, never rounded to bf16, reading U8)
 *   x_v   = z_v / T_t                           T_t = temperatures[t] if given, else temperature (U7)
 *   logp  = x_{ids[t]} - log sum_v exp(x_v)     natural log, all V rows count (U10)
 *   H_t   = -sum_v p_v ln p_v                   entropy in nats of the tempered distribution (U9)
 * Row t is paired with ids[t]: the next-token shift is the caller's job (U18).
 *
 * Batch invariance: every reduction has a split and order that depends only on
 * (V, hidden) -- never on n_tok, the row's position in the batch, the number of
 * SMs or of GPUs -- so a token's logp/entropy bits are identical whether it is
 * scored alone or in any packed batch (§3.1).
 *
 * Layout / ownership:
 *   hidden_bf16  [n_tok, hidden] row stride ld_hidden elements (>= hidden); 16-B aligned;
 *                ld_hidden*2 % 16 == 0.  bf16 (uint16 storage).
 *   weight_bf16  [vocab, hidden] contiguous, 16-B aligned (the lm_head weight, K-major).
 *   token_ids    [n_tok] int64; ids outside [0, vocab) -> dstatus TIM_ERR_DATA, logp NaN.
 *   temperatures_or_null [n_tok] fp32 (> 0, finite) or NULL.
 *   logp_out     [n_tok] fp32.  entropy_out_or_null [n_tok] fp32 or NULL.
 *   workspace    >= tim_logprob_workspace_bytes(n_tok, hidden, vocab) bytes, 256-B aligned.
 * Constraints: hidden % 64 == 0, 64 <= hidden <= 16384; 1 <= vocab <= 2^24;
 *   0 <= n_tok < 2^31; temperature > 0 and finite.  n_tok == 0 -> TIM_OK, no launch.
 * Errors: TIM_ERR_NULL / SHAPE / ALIGN / VALUE / WORKSPACE (sync, nothing launched),
 *   TIM_ERR_UNSUPPORTED (not sm_100), TIM_ERR_CUDA (launch failure).
 * -------------------------------------------------------------------------- */
size_t tim_logprob_workspace_bytes(int64_t n_tok, int32_t hidden, int32_t vocab);
tim_status tim_logprob(const void* hidden_bf16, int64_t ld_hidden,
                       const void* weight_bf16, int32_t hidden, int32_t vocab,
                       const int64_t* token_ids, int64_t n_tok,
                       float temperature, const float* temperatures_or_null,
                       float* logp_out, float* entropy_out_or_null,
                       void* workspace, size_t workspace_bytes,
                       tim_device_status* dstatus, void* stream);

/* Number of vocab slices S_v of the fixed split for a given vocab (numerics contract, U20):
 * min(64, ceil(vocab / 256)) contiguous runs of whole 256-column tiles (64 at V = 151936).  The
 * slice count fixes the merge order, so it depends on the vocabulary only; 64 slices let a
 * small batch (one M-tile) spread over 64 CTA pairs. */
int32_t tim_logprob_vocab_slices(int32_t vocab);

/* ----------------------------------------------------------------------------
 * tim_sample  (the rollout-side twin)
 *
 * Samples a_t ~ softmax(z_t / T_t) for every row, with the same head arithmetic as
 * tim_logprob, so the rollout's log pi(a_t) is produced by the very kernel the trainer uses:
 * logp_out[t] and entropy_out[t] are bit-identical to what tim_logprob returns for
 * ids = ids_out (zero training-inference mismatch at the head, §3.1).
 * Rule (U22): Gumbel-max, a_t = argmax_v x_v + g_v, g_v = -ln(-ln u_v),
 * u_v = ((x >> 9) + 1/2) 2^-23 with x word (v % 4) of Philox4x32-10(counter = {v / 4, 0,
 * row_keys[t] lo, row_keys[t] hi}, key = seed); ties go to the lowest column.  The draw of a
 * row depends only on (seed, row_keys[t], the row's logits): batch-invariant like the log-prob.
 *   row_keys [n_tok] uint64 (device): per-row counter, e.g. (sequence id << 32) | position.
 *   ids_out [n_tok] int64, logp_out [n_tok] fp32, entropy_out_or_null [n_tok] fp32.
 *   workspace >= tim_sample_workspace_bytes(n_tok, hidden, vocab).
 * Other arguments, constraints and errors as tim_logprob.
 * -------------------------------------------------------------------------- */
size_t tim_sample_workspace_bytes(int64_t n_tok, int32_t hidden, int32_t vocab);
tim_status tim_sample(const void* hidden_bf16, int64_t ld_hidden,
                      const void* weight_bf16, int32_t hidden, int32_t vocab,
                      const uint64_t* row_keys, int64_t n_tok, uint64_t seed,
                      float temperature, const float* temperatures_or_null,
                      int64_t* ids_out, float* logp_out, float* entropy_out_or_null,
                      void* workspace, size_t workspace_bytes,
                      tim_device_status* dstatus, void* stream);

/* ----------------------------------------------------------------------------
 * Corrections and statistics
 *
 * Inputs common to tim_mismatch_stats / tim_correct / tim_correct_local:
 *   logp_num, logp_den  [n_tok_local] fp32; delta = (double)num - (double)den (C.3.1).
 *                       (num, den) = (train_old, rollout) gives r_corr = e^delta;
 *                       (cur, rollout) gives r^rollout_ppo as masking signal q_t.
 *   cu_seqlens_global   [n_seq + 1] int64 global sequence offsets, cu[0] == 0, non-decreasing.
 *   tok_begin           global index of this rank's first token; this rank holds tokens
 *                       [tok_begin, tok_begin + n_tok_local) which must lie in [0, cu[n_seq]].
 *                       Sequences may straddle ranks.
 *   resp_mask_or_null   [n_tok_local] u8 (1 = response token); NULL = all response (U11).
 * Only response tokens enter K sums, T_s and statistics; non-response tokens get coeff 0.
 * The shard must lie inside the sequences: cu[0] <= tok_begin and tok_begin + n_tok_local <=
 * cu[n_seq].  cu is device memory, so this is checked on the device: a violation is a data error
 * (device status TIM_ERR_DATA, first_bad_index = the first global token outside; reading U13b)
 * and no access leaves the arrays.  cu must be non-decreasing (not checked; the walk is bounded). 
 * Alignment: fp32 arrays 4-B aligned (TIM_ERR_ALIGN otherwise).  When every per-token array
 * is 16-B aligned (u8 arrays 4-B) the kernels use 16-B vector accesses; otherwise (e.g. a
 * shard cut at an arbitrary token) the same results come from the scalar path, slower.
 * -------------------------------------------------------------------------- */
typedef enum { TIM_SEQ_NONE = 0, TIM_SEQ_K1 = 1, TIM_SEQ_K3 = 3 } tim_seq_rs;
typedef enum { TIM_AGG_SUM = 0, TIM_AGG_MEAN = 1 } tim_agg;

/* Correction configuration (host memory).  No defaults: the caller sets every field.
 * Paper values: tis_cap = 2, log_tis_cap = ln 2, tau_seq = 0.001. */
typedef struct {
  int32_t tis;          /* 1: w = min(e^delta, tis_cap); truncated iff delta > log_tis_cap   */
  int32_t tok_rs;       /* 1: token keep iff log_tok_lo <= delta <= log_tok_hi (U4)          */
  int32_t seq_rs;       /* tim_seq_rs: sequence score K1 (= -delta) or K3 (C.3.6)            */
  int32_t seq_agg;      /* tim_agg: S_s = sum (paper literal) or mean over contributing tokens */
  double tis_cap;       /* tau_tok > 0, finite                                              */
  double log_tis_cap;   /* ln tau_tok, computed by the caller (no libm on the decision path) */
  double log_tok_lo;    /* ln lower ratio bound                                             */
  double log_tok_hi;    /* ln upper ratio bound, >= log_tok_lo                              */
  double tau_seq;       /* keep iff S_s <= tau_seq; |tau_seq| < 2^10, finite                 */
} tim_correct_cfg;

/* Statistics.  Device writes every integer field and max_abs_delta; the three means are
 * filled by tim_stats_finalize on a host copy.  int128 values are {lo, hi} two's complement,
 * scale 2^-52 (fixed point of C.3.8), exact and independent of sharding / GPU count. */
typedef struct {
  int64_t n_tok;            /* tokens scored (all ranks)                                   */
  int64_t n_resp_tok;       /* response tokens                                             */
  int64_t n_seq;
  int64_t n_truncated;      /* response tokens with delta > log_tis_cap (when tis)          */
  int64_t n_tok_rejected;   /* response tokens failing token-RS (when tok_rs)              */
  int64_t n_seq_rejected;
  int64_t n_saturated;      /* contributing tokens whose |K| > 2^10 (sequence rejected, U19) */
  int64_t sum_abs_delta_fx[2];
  int64_t sum_k1_fx[2];
  int64_t sum_k3_fx[2];
  double max_abs_delta;
  double mean_abs_delta;    /* host: tim_stats_finalize                                    */
  double mean_k1;
  double mean_k3;
} tim_stats;

/* Pure host: fills the means of a host copy from its exact totals (RN conversions). */
tim_status tim_stats_finalize(tim_stats* host_copy);

size_t tim_correct_workspace_bytes(int64_t n_tok_local, int64_t n_seq, int32_t nranks);

/* Statistics only (no masks).  comm_or_null: NULL for a single rank, else the NCCL
 * communicator of all ranks sharing the batch (exact all-gather of integer partials). */
typedef struct tim_comm tim_comm;
tim_status tim_mismatch_stats(const float* logp_num, const float* logp_den,
                              const int64_t* cu_seqlens_global, int64_t n_seq,
                              int64_t tok_begin, int64_t n_tok_local,
                              const uint8_t* resp_mask_or_null,
                              tim_comm* comm_or_null, tim_stats* stats_dev,
                              void* workspace, size_t workspace_bytes,
                              tim_device_status* dstatus, void* stream);

/* Full correction.  Outputs (device):
 *   tis_w     [n_tok_local] fp32  w_t (tis) or 1.0
 *   tok_keep  [n_tok_local] u8    token-RS keep (all 1 when !tok_rs)
 *   seq_keep  [n_seq]       u8    sequence keep (all 1 when seq_rs == NONE)
 *   coeff     [n_tok_local] fp32  resp * tok_keep * seq_keep * (tis ? w : 1)
 *   seq_score_or_null [n_seq] f64 S_s (SUM) or S_s / T_s (MEAN) from the exact sum
 *   stats_dev may be NULL.
 */
tim_status tim_correct(const float* logp_num, const float* logp_den,
                       const int64_t* cu_seqlens_global, int64_t n_seq,
                       int64_t tok_begin, int64_t n_tok_local,
                       const uint8_t* resp_mask_or_null,
                       const tim_correct_cfg* cfg_host, tim_comm* comm_or_null,
                       float* tis_w, uint8_t* tok_keep, uint8_t* seq_keep, float* coeff,
                       double* seq_score_or_null, tim_stats* stats_dev,
                       void* workspace, size_t workspace_bytes,
                       tim_device_status* dstatus, void* stream);

/* ----------------------------------------------------------------------------
 * Split form of tim_correct for callers that exchange partials themselves
 * (e.g. torch.distributed).  tim_correct == local -> all-gather -> finish.
 *
 * tim_correct_local writes this rank's exact partial block (tim_correct_partial_bytes(n_seq)
 * bytes at `partial_out`, device) and the per-token outputs tis_w, tok_keep and a
 * provisional coeff (= resp * tok_keep * w).  The block is plain bytes: gather the blocks
 * of all ranks contiguously, in rank order, into [nranks * partial_bytes] and pass them to
 * tim_correct_finish on every rank.  finish sums the blocks exactly (int128), decides every
 * sequence, zeroes coeff of this rank's tokens in rejected sequences, and writes seq_keep,
 * seq_score and stats.  Block layout: tim_partial_header followed by n_seq tim_seq_partial.
 * -------------------------------------------------------------------------- */
typedef struct {
  int64_t n_tok, n_resp_tok, n_truncated, n_tok_rejected, n_saturated;
  uint64_t max_abs_delta_bits;       /* bits of a non-negative double (max commutes with bits) */
  int64_t sum_abs_delta[2], sum_k1[2], sum_k3[2];
  int64_t reserved[4];
} tim_partial_header;                /* 128 B */
typedef struct {
  int64_t x_lo, x_hi;                /* int128 sum of X = rint(K * 2^52) over contributing tokens */
  int64_t n_tok;                     /* T_s contribution                                          */
  int64_t n_sat;                     /* saturated contributing tokens                             */
} tim_seq_partial;                   /* 32 B */

size_t tim_correct_partial_bytes(int64_t n_seq);
tim_status tim_correct_local(const float* logp_num, const float* logp_den,
                             const int64_t* cu_seqlens_global, int64_t n_seq,
                             int64_t tok_begin, int64_t n_tok_local,
                             const uint8_t* resp_mask_or_null, const tim_correct_cfg* cfg_host,
                             float* tis_w, uint8_t* tok_keep, float* coeff,
                             void* partial_out, tim_device_status* dstatus, void* stream);
tim_status tim_correct_finish(const void* gathered_partials, int32_t nranks,
                              const int64_t* cu_seqlens_global, int64_t n_seq,
                              int64_t tok_begin, int64_t n_tok_local,
                              const tim_correct_cfg* cfg_host,
                              float* coeff, uint8_t* seq_keep, double* seq_score_or_null,
                              tim_stats* stats_dev_or_null, void* stream);

/* ----------------------------------------------------------------------------
 * Vocab-parallel (tensor-parallel) head  (§5 P:651 TBIK:
 * reductions invariant to the TP degree)
 *
 * The fixed vocab split of tim_logprob (S_v slices, U20) doubles as the TP split: with tp | S_v,
 * rank r owns slices [r S_v/tp, (r+1) S_v/tp) = W rows [begin, end) from tim_tp_vocab_range.
 * tim_logprob_tp_partial runs those slices against the rank's shard weight_shard[end - begin, hidden]
 * and writes (S_v/tp) x n_tok slice partials (16 B each, slice-major) to partial_out
 * (tim_logprob_tp_partial_bytes).  All-gather the blocks of all ranks contiguously in rank order
 * (that is the full [S_v][n_tok] slice-major array) and call tim_logprob_tp_merge: logp / entropy
 * are BIT-IDENTICAL to tim_logprob on the unsharded weight, for every tp -- the cross-rank
 * log-sum-exp merge is the same fixed slice-order merge.
 * The shard MUST be exactly W rows [begin, end) of that split (whole 256-row tiles; at V = 151936
 * and tp = 8 rank 0 owns 18944 rows, not an even V / tp split): the C ABI cannot see the shard's
 * extent, so a shorter shard is read out of bounds and a differently cut one gives shifted
 * columns.  The Python binding checks the shape against tim_tp_vocab_range.
 * Workspaces: >= 1024 B each (progress counters / status).  Errors as tim_logprob; tp must divide S_v.
 * -------------------------------------------------------------------------- */
tim_status tim_tp_vocab_range(int32_t vocab, int32_t tp, int32_t rank, int32_t* begin, int32_t* end);
size_t tim_logprob_tp_partial_bytes(int64_t n_tok, int32_t vocab, int32_t tp);
tim_status tim_logprob_tp_partial(const void* hidden_bf16, int64_t ld_hidden, const void* weight_shard_bf16,
                                  int32_t hidden, int32_t vocab, int32_t tp, int32_t rank,
                                  const int64_t* token_ids, int64_t n_tok,
                                  float temperature, const float* temperatures_or_null,
                                  void* partial_out, void* workspace, size_t workspace_bytes, void* stream);
tim_status tim_logprob_tp_merge(const void* gathered_partials, int64_t n_tok, int32_t vocab,
                                const int64_t* token_ids, const float* temperatures_or_null,
                                float* logp_out, float* entropy_out_or_null,
                                void* workspace, size_t workspace_bytes,
                                tim_device_status* dstatus, void* stream);

/* The whole vocab-parallel head in one call: the rank's tim_logprob_tp_partial, the NCCL
 * all-gather of the slice partials inside the library over `comm` (tp = comm's rank count, this
 * rank = comm's rank; every rank passes the same n_tok rows and ids), and tim_logprob_tp_merge.
 * Every rank gets logp / entropy for all n_tok rows, bitwise equal to tim_logprob on the full W.
 * The exchange carries 16 B per token per slice (S_v n_tok 16 B gathered per rank), stream-ordered
 * on `stream` like every other call.  Workspace: tim_logprob_tp_workspace_bytes (device, >= 256-B
 * aligned).  Errors: those of tim_logprob_tp_partial / _merge; TIM_ERR_NCCL if the all-gather
 * fails; tp must divide S_v. */
size_t tim_logprob_tp_workspace_bytes(int64_t n_tok, int32_t vocab, int32_t tp);
tim_status tim_logprob_tp(const void* hidden_bf16, int64_t ld_hidden, const void* weight_shard_bf16,
                          int32_t hidden, int32_t vocab, tim_comm* comm,
                          const int64_t* token_ids, int64_t n_tok,
                          float temperature, const float* temperatures_or_null,
                          float* logp_out, float* entropy_out_or_null,
                          void* workspace, size_t workspace_bytes,
                          tim_device_status* dstatus, void* stream);

/* ----------------------------------------------------------------------------
 * tim_rmsnorm / tim_logprob_rmsnorm  (the batch-invariant RMSNorm
 * prologue of the head, §3.1)
 *
 * Hugging Face Qwen3 RMSNorm semantics (the paper's models):
 *   x1[t,k]  = bf16( h[t,k] * 1/sqrt(mean_k h[t,k]^2 + eps) )    (fp32, IEEE sqrt / div)
 *   out[t,k] = bf16( gamma[k] * x1[t,k] )
 * The sum of squares of a row is reduced in an order fixed by `hidden` only (batch-invariant).
 *   hidden_bf16 [n_tok, hidden] row pitch ld_hidden (16-B aligned, ld_hidden % 8 == 0);
 *   gamma_bf16 [hidden]; out_bf16 [n_tok, hidden] contiguous; hidden % 64 == 0; eps >= 0.
 * tim_logprob_rmsnorm = tim_rmsnorm into the workspace followed by tim_logprob on the
 * normalized rows (the same outputs and errors as tim_logprob);
 * workspace >= tim_logprob_rmsnorm_workspace_bytes(n_tok, hidden, vocab).
 * -------------------------------------------------------------------------- */
tim_status tim_rmsnorm(const void* hidden_bf16, int64_t ld_hidden, const void* gamma_bf16, float eps,
                       int32_t hidden, int64_t n_tok, void* out_bf16, void* stream);
size_t tim_logprob_rmsnorm_workspace_bytes(int64_t n_tok, int32_t hidden, int32_t vocab);
tim_status tim_logprob_rmsnorm(const void* hidden_bf16, int64_t ld_hidden, const void* gamma_bf16, float eps,
                               const void* weight_bf16, int32_t hidden, int32_t vocab,
                               const int64_t* token_ids, int64_t n_tok,
                               float temperature, const float* temperatures_or_null,
                               float* logp_out, float* entropy_out_or_null,
                               void* workspace, size_t workspace_bytes,
                               tim_device_status* dstatus, void* stream);

/* ----------------------------------------------------------------------------
 * tim_head_backward  (backward of the head; the "score function
 * gradient" the trainer takes through logp, §3)
 *
 * For the scalar L = sum_t g_t logp_t + e_t H_t (g = grad_logp, e = grad_ent_or_null or 0) with
 * z = h W^T, y = z / T_t, p = softmax(y), logp_t = y[a_t] - lse(y), H_t = -sum_v p ln p:
 *   G[t, v]     = dL/dz[t, v] = (1/T_t) [ g_t (1[v = a_t] - p_v) - e_t p_v (ln p_v + H_t) ]
 *   dhidden[t]  = sum_v G[t, v] W[v]         (fp32 [n_tok, hidden], contiguous; overwritten)
 *   dweight[v]  = sum_t G[t, v] h[t]         (fp32 [vocab, hidden], contiguous; overwritten)
 * Path: tim_logprob's kernel (forward: logp, H, log2-sum-exp per token), the same tcgen05 kernel
 * again with a gradient epilogue that writes G as bf16 into the workspace (logits never reach
 * HBM), then two cuBLAS bf16 GEMMs with fp32 accumulation (libcublas loaded at run time;
 * TIM_ERR_UNSUPPORTED if it cannot be loaded).  Tokens are processed in blocks whose bf16 G
 * block fits 4 GiB; dweight accumulates over the blocks in block order (fp32).
 * Deterministic run to run on one device; NOT batch-invariant (cuBLAS picks its kernel by
 * shape, and G is rounded to bf16 before the GEMMs).
 * Inputs and errors as tim_logprob (bad id / temperature -> TIM_ERR_DATA with the global token
 * index); either output may be NULL (skipped), not both.  n_tok == 0 zeroes dweight.
 * workspace >= tim_head_backward_workspace_bytes(n_tok, hidden, vocab), 256-B aligned.
 * -------------------------------------------------------------------------- */
size_t tim_head_backward_workspace_bytes(int64_t n_tok, int32_t hidden, int32_t vocab);
tim_status tim_head_backward(const void* hidden_bf16, int64_t ld_hidden, const void* weight_bf16,
                             int32_t hidden, int32_t vocab, const int64_t* token_ids, int64_t n_tok,
                             float temperature, const float* temperatures_or_null,
                             const float* grad_logp, const float* grad_ent_or_null,
                             float* dhidden_or_null, float* dweight_or_null,
                             void* workspace, size_t workspace_bytes,
                             tim_device_status* dstatus, void* stream);

/* ----------------------------------------------------------------------------
 * tim_logprob_saved / tim_head_backward_saved  (NEXT-3 for a trainer that keeps forward state:
 * the backward then skips its own forward pass -- 3 instead of 4 passes over the logits)
 *
 * tim_logprob_saved = tim_logprob (same arguments, outputs, errors and numerics) that also
 *   writes lse2_out[t] = log2 sum_v 2^(y[t,v]), y = z log2(e) / T_t (fp32, the value the merge
 *   forms in fp64 then rounds); entropy_out and lse2_out are required ([n_tok] fp32 each).
 * tim_head_backward_saved = tim_head_backward given the forward's entropy_saved / lse2_saved
 *   (from tim_logprob_saved on the SAME hidden, weight, ids and temperatures -- they are not
 *   re-validated here; bad ids / temperatures were reported by that forward call).  Because the
 *   forward is batch-invariant, the outputs are bitwise those of tim_head_backward on the same
 *   inputs.  Same workspace size and the other arguments / errors as tim_head_backward;
 *   entropy_saved / lse2_saved NULL -> TIM_ERR_NULL (n_tok > 0).
 * -------------------------------------------------------------------------- */
tim_status tim_logprob_saved(const void* hidden_bf16, int64_t ld_hidden, const void* weight_bf16,
                             int32_t hidden, int32_t vocab, const int64_t* token_ids, int64_t n_tok,
                             float temperature, const float* temperatures_or_null,
                             float* logp_out, float* entropy_out, float* lse2_out,
                             void* workspace, size_t workspace_bytes,
                             tim_device_status* dstatus, void* stream);
tim_status tim_head_backward_saved(const void* hidden_bf16, int64_t ld_hidden, const void* weight_bf16,
                                   int32_t hidden, int32_t vocab, const int64_t* token_ids, int64_t n_tok,
                                   float temperature, const float* temperatures_or_null,
                                   const float* entropy_saved, const float* lse2_saved,
                                   const float* grad_logp, const float* grad_ent_or_null,
                                   float* dhidden_or_null, float* dweight_or_null,
                                   void* workspace, size_t workspace_bytes,
                                   tim_device_status* dstatus, void* stream);

/* ----------------------------------------------------------------------------
 * tim_ppo_loss  (fused PPO / GRPO surrogate + loss diagnostics)
 *
 * Per token t (PAPER.md eq:ppo_loss P:352-360, eq:ppo_ratio P:361-373, App. A.4):
 *   r_t   = exp(logp_cur - logp_old)     logp_old = trainer-recomputed (recompute mode) or
 *                                        rollout log-prob (bypass mode), C.3 exp contract
 *   clipped_t <=> (A_t > 0 and r_t > clip_hi) or (A_t < 0 and r_t < clip_lo)
 *   loss_t = -w_t min(r_t A_t, clip(r_t, clip_lo, clip_hi) A_t), w_t = coeff_t (the tim_correct
 *            coefficient resp * tok_keep * seq_keep * TIS weight) or the response mask
 *   grad_t = d loss_t / d logp_cur_t = (clipped ? 0 : loss_t)   (score-function gradient)
 * Diagnostics over contributing tokens (coeff != 0, else response tokens): clip fraction,
 * K1 / K3 of r, and the zero-centred contribution C(r) = -(r - 1) A
 * histogrammed separately for A > 0 and A < 0 (A == 0 counted apart).
 * Aggregation (reading U17): per-sequence loss = sum over its contributing tokens (exact
 * 2^-52 fixed point, int128), batch_loss = sum of sequence losses / number of sequences with a
 * contributing token.  Multi-rank: like tim_correct (exact partial blocks, rank-ordered sums).
 *
 * Buffers (device): logp_cur, logp_old, advantages [n_tok_local] fp32; coeff_or_null fp32;
 * resp_mask_or_null u8 (ignored when coeff is given); loss_tok, grad_logp fp32, clipped u8
 * [n_tok_local]; seq_loss_or_null [n_seq] f64; hist_or_null [2][hist_bins + 2] int64 (slot 0 =
 * underflow, hist_bins + 1 = overflow; row 0: A > 0, row 1: A < 0); stats optional.
 * Data errors (dstatus TIM_ERR_DATA, first global index; readings U13 / U13b): a non-finite
 * logp, advantage or coeff (e.g. NaN advantages from whitening a zero-variance GRPO group) -- that
 * token's loss = NaN, grad = 0, clipped = 0, and it enters no histogram, count or sum; a shard
 * outside [cu[0], cu[n_seq]) as for tim_correct.
 * -------------------------------------------------------------------------- */
typedef struct {
  double clip_lo;         /* 1 - eps  (paper eq:ppo_loss) */
  double clip_hi;         /* 1 + eps                      */
  double hist_lo;         /* C(r) histogram: lower edge   */
  double hist_inv_width;  /* hist_bins / (hi - lo)        */
  int32_t hist_bins;      /* 1 .. 1024                    */
  int32_t reserved;
} tim_ppo_cfg;

typedef struct {
  int64_t n_tok, n_contrib, n_clipped, n_zero_adv, n_saturated;
  int64_t sum_loss[2], sum_k1[2], sum_k3[2];
  int64_t reserved[5];
} tim_ppo_partial_header;  /* 128 B; block = header + hist [2][bins + 2] int64 + n_seq tim_seq_partial */

typedef struct {
  int64_t n_tok, n_contrib, n_clipped, n_zero_adv, n_saturated, n_seq, n_seq_contrib;
  int64_t sum_loss_fx[2], sum_k1_fx[2], sum_k3_fx[2];   /* int128 {lo, hi}, scale 2^-52 */
  double batch_loss, clip_frac, mean_k1, mean_k3;       /* host: tim_ppo_stats_finalize */
} tim_ppo_stats;

size_t tim_ppo_partial_bytes(int64_t n_seq, int32_t hist_bins);
size_t tim_ppo_workspace_bytes(int64_t n_seq, int32_t hist_bins, int32_t nranks);
tim_status tim_ppo_loss(const float* logp_cur, const float* logp_old, const float* advantages,
                        const float* coeff_or_null, const uint8_t* resp_mask_or_null,
                        const int64_t* cu_seqlens_global, int64_t n_seq, int64_t tok_begin,
                        int64_t n_tok_local, const tim_ppo_cfg* cfg_host, tim_comm* comm_or_null,
                        float* loss_tok, float* grad_logp, uint8_t* clipped,
                        double* seq_loss_or_null, int64_t* hist_or_null, tim_ppo_stats* stats_dev_or_null,
                        void* workspace, size_t workspace_bytes, tim_device_status* dstatus, void* stream);
tim_status tim_ppo_local(const float* logp_cur, const float* logp_old, const float* advantages,
                         const float* coeff_or_null, const uint8_t* resp_mask_or_null,
                         const int64_t* cu_seqlens_global, int64_t n_seq, int64_t tok_begin,
                         int64_t n_tok_local, const tim_ppo_cfg* cfg_host,
                         float* loss_tok, float* grad_logp, uint8_t* clipped, void* partial_out,
                         tim_device_status* dstatus, void* stream);
tim_status tim_ppo_finish(const void* gathered_partials, int32_t nranks, int64_t n_seq,
                          const tim_ppo_cfg* cfg_host, double* seq_loss_or_null, int64_t* hist_or_null,
                          tim_ppo_stats* stats_dev_or_null, void* stream);
tim_status tim_ppo_stats_finalize(tim_ppo_stats* host_copy);

/* ----------------------------------------------------------------------------
 * Device L2 configuration (an application-level setting, never changed by any other call).
 * tim_l2_persisting: set the current device's persisting-L2 set-aside (cudaLimitPersistingL2CacheSize)
 * to min(bytes, the device maximum) and return the size the driver granted (it rounds up; 79 MB max
 * on B200).  The log-prob kernels load their live H tiles with the evict_last L2 policy; on boxes
 * whose C2 launches fall into the slow mode (W re-fetched) a ~48 MB set-aside kept every
 * launch in the fast mode, and it measured neutral elsewhere (profiles/r02_c2_bimodal.txt).  The
 * limit is context-wide: it also shrinks the L2 left to normal accesses of every other kernel in the
 * process -- with 48 MB the streaming correction / PPO passes ran 27% slower (0.565 -> 0.723 ms and
 * 0.623 -> 0.794 ms at 2^27 tokens), so bench.py leaves the driver default.  bytes < 0: TIM_ERR_VALUE; a CUDA failure: TIM_ERR_CUDA.  granted_bytes may be NULL.
 * -------------------------------------------------------------------------- */
tim_status tim_l2_persisting(int64_t bytes, int64_t* granted_bytes);

/* ----------------------------------------------------------------------------
 * NCCL communicator (NVLink / NVSwitch).  libnccl.so.2 is loaded at run time.
 * unique_id: 128 bytes from tim_comm_unique_id on rank 0, broadcast by the caller.
 * -------------------------------------------------------------------------- */
tim_status tim_comm_unique_id(void* unique_id_128B_out);
tim_status tim_comm_init(const void* unique_id_128B, int32_t nranks, int32_t rank, tim_comm** out);
tim_status tim_comm_destroy(tim_comm* comm);

#ifdef __cplusplus
}
#endif
#endif /* TIM_H_ */
