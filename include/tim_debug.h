/*
 * tim_debug.h -- TEST-ONLY entry points of libtim.so (GEMM bring-up and invariance tests).
 * Not part of the product ABI; never called on the hot path.
 */
#ifndef TIM_DEBUG_H_
#define TIM_DEBUG_H_

#include "tim.h"

#ifdef __cplusplus
extern "C" {
#endif

/* Same as tim_logprob (T = 1) but additionally writes the raw fp32 tcgen05 accumulators
 * z[t, v] = sum_k H[t,k] W[v,k] to logits_out[t * ld_logits + v] (device, ld_logits >= vocab),
 * so the TMA / UMMA-descriptor / TMEM layout can be checked against an fp64 matmul. */
tim_status tim_debug_logprob_logits(const void* hidden_bf16, int64_t ld_hidden, const void* weight_bf16,
                                    int32_t hidden, int32_t vocab, const int64_t* token_ids, int64_t n_tok,
                                    float* logits_out, int64_t ld_logits, float* logp_out, float* entropy_out,
                                    void* workspace, size_t workspace_bytes, void* stream);

/* Process-global knobs: use_pair = 1 (default) selects the cta_group::2 kernel (the numerics
 * contract), 0 the single-CTA cta_group::1 bring-up variant; max_ctas_or_clusters > 0 caps the
 * persistent grid (emulates a GPU with fewer SMs for batch-invariance tests), 0 = all SMs. */
tim_status tim_debug_set_kernel(int32_t use_pair, int32_t max_ctas_or_clusters);

/* Small-batch H staging (n_tok < 256, not a multiple of 128): 1 = copy the rows into zero-padded
 * whole 128-row boxes in the workspace before the kernel (default), 0 = let TMA zero-fill the
 * partial box on every load.  Never changes a result bit (rows are independent). */
tim_status tim_debug_set_pad_small(int32_t enable);

/* Performance knobs (never change results): L2 eviction policy of the hidden-state (H) and
 * weight (W) TMA tile loads, 0 = no hint, 1 = evict_normal, 2 = evict_first, 3 = evict_last;
 * sleep_waits (bits: 1 TMA producer, 2 epilogue, 4 MMA issuer; 0..7) makes those mbarrier waits sleep in hardware;
 * sync_slack > 0 bounds how many vocab tiles a CTA pair may run ahead of the slowest pair.
 * Defaults: h = 3, w = 2, sleep_waits = 0, sync_slack = 4. */
tim_status tim_debug_set_tuning(int32_t h_policy, int32_t w_policy, int32_t sleep_waits, int32_t sync_slack);

/* Schedule knobs (never change results): number of CTA pairs sharing one 256-token M-tile
 * (each sweeps S_v/group slices of it), 0 = automatic (smallest group whose live hidden-state
 * tiles fit in ~75% of L2); demote = 1 lowers finished hidden-state tiles to evict_normal in L2. */
tim_status tim_debug_set_schedule(int32_t group, int32_t demote);

/* Cluster shape knob (never changes results): 1 = clusters of one CTA pair; 2 = clusters of two
 * pairs that own different M-tiles and share every W tile through TMA multicast (used only when
 * the live hidden-state tiles of all pairs fit in L2). */
tim_status tim_debug_set_cluster(int32_t pairs_per_cluster);

/* Head-backward GEMM knob (never changes results): a CTA pair may run at most k_blocks 64-wide
 * K blocks ahead of the slowest pair (0 = no gate).  Default 128. */
tim_status tim_debug_set_gemm_slack(int32_t k_blocks);
/* L2 eviction policy of the backward GEMMs' operand loads (1 evict_normal, 2 evict_first, 3
 * evict_last) for dH's A (= G) / B (= W) and dW's A (= G^T) / B (= H).  Default 1, 1, 1, 3. */
tim_status tim_debug_set_gemm_policy(int32_t dh_a, int32_t dh_b, int32_t dw_a, int32_t dw_b);

/* Correction form at P = 1 (never changes results): 1 (default) = the split launches (local,
 * finish, zero) that P > 1 uses; 0 = pass 1, the sequence decisions and the coefficient zeroing in
 * ONE cooperative launch behind two grid barriers (SURVEY a7 "fused into pass 1 when P = 1";
 * measured 2.5% slower at 2^27 tokens, profiles/r02_correction_fused_ab.txt). */
tim_status tim_debug_set_correct_split(int32_t split);

/* Die-aware M-tile groups (never changes results): 1 (default) = when several CTA pairs share an
 * M-tile (G > 1, d = 4096 batches), pairs on the same die of the B200 form a group, from a one-time
 * per-device SM -> die latency probe; 0 = groups of consecutive cluster ids. */
tim_status tim_debug_set_die_groups(int32_t enable);
/* The probed SM -> die map of the current device (probing it now if needed): state 1 = valid,
 * -1 = unavailable (then the grouping falls back to cluster-id order); mask_out4[s / 64] bit s % 64
 * = die of SM s. */
tim_status tim_debug_die_map(int32_t* state_out, uint64_t* mask_out4);

#ifdef __cplusplus
}
#endif
#endif
