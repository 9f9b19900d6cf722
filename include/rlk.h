/*
 * rlk.h -- C ABI of the B200-native rolloutlab hot path (fusion + GRPO token objective).
 *
 * Plain pointers, sizes and a cudaStream_t (passed as void*); no torch types.  Every entry point
 * returns 0 on success or a negative RLK_ERR_* code; the message for the last failure on the calling
 * thread is available from rlk_last_error().  All device buffers are owned by the caller; the library
 * performs no allocations.  Entry points are reentrant and may be called concurrently on different
 * streams / devices.
 *
 * Reference interfaces replaced (paths relative to the reference tree pkg/src/rolloutlab/):
 *   rlk_fusion_sumsq        TaskVector.__post_init__ norm            fusion.py:37-44
 *                           ParamTable finite check                  toy_env.py:67-72
 *   rlk_fusion_finalize     normalize_magnitudes target/scale        fusion.py:86-102
 *   rlk_fusion_mask_bitmap  dropout_prune draw loop                  fusion.py:105-115, core.py:69-75, 95-103
 *   rlk_fusion_mask_bitmap_range  (the same, one index slice)       fusion.py:105-115
 *   rlk_fusion_merge        dropout_prune rescale, erase_minority,   fusion.py:114, 118-142
 *                           fuse weighted sum + FusionStats counts   fusion.py:154-188
 *   rlk_fusion_merge_ws     (the same, with a fix-up workspace)      fusion.py:114-188
 *   rlk_grpo_fwd            log_token_dist + objective_value         toy_env.py:157-175, objective.py:230-250
 *                           (tis_weight, _triplet_value_slope)       objective.py:133-165
 *   rlk_segment_sum_f64     per-group token-term sums                objective.py:238-250
 *   rlk_grpo_bwd            objective_gradient                       objective.py:253-283
 *   rlk_grpo_fused_bf16     objective_value + objective_gradient     objective.py:230-283 (one pass)
 *   rlk_grpo_fused          the same for bf16 or f32 logits          objective.py:230-283 (one pass)
 *   rlk_logsoftmax_rows     log_token_dist (full row)                toy_env.py:157-175
 *   rlk_nonfinite_count     ParamTable finite check                  toy_env.py:71-72
 *   rlk_scaled_add          ascent_step (params + lr * grad)         objective.py:286-293
 */
#ifndef RLK_H_
#define RLK_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RLK_OK 0
#define RLK_ERR_INVALID (-1)     /* bad argument (maps to the reference's ValueError) */
#define RLK_ERR_CUDA (-2)        /* CUDA runtime error */
#define RLK_ERR_UNSUPPORTED (-3) /* dtype / expert count not compiled */

#define RLK_BF16 0
#define RLK_F32 1
#define RLK_F64 2

#define RLK_MAX_EXPERTS 8
/* Norm-partial granularity: every piece is cut into items of this many elements, counted from the
 * start of its tensor, and one f64 partial per (item, expert) is produced.  Pieces handed to
 * different ranks must start on an item boundary, which makes the norms bit-identical at any world
 * size ("deterministic norms"). */
#define RLK_FUSION_ITEM 65536

/* One contiguous piece of one tensor: the base slice, the N expert slices (or N task-vector deltas
 * when delta_mode=1, base then unused), and the output slice. Element i of the piece is flat index
 * j0 + i of its tensor (the reference's ravel() index, which keys the dropout draw). */
typedef struct rlk_fusion_segment {
  const void* base;
  const void* expert[RLK_MAX_EXPERTS];
  void* out;
  uint64_t numel;
  uint64_t j0;    /* multiple of RLK_FUSION_ITEM */
  uint32_t tensor; /* row in the per-tensor scale / counter tables */
  uint32_t item0;  /* global item index of this piece's first item (row of the partials table) */
} rlk_fusion_segment;

/* A launch plan: device arrays built once per layout by the host.
 *   segs[n_segs]; seg_item_prefix[n_segs + 1] = exclusive prefix of ceil(numel / ITEM). */
typedef struct rlk_fusion_plan {
  const rlk_fusion_segment* segs; /* device */
  const uint32_t* seg_item_prefix; /* device */
  uint32_t n_segs;
  uint32_t n_items; /* = seg_item_prefix[n_segs] */
} rlk_fusion_plan;

const char* rlk_last_error(void);
int rlk_abi_version(void);
int rlk_device_sm_count(int device);

/* K1: partials[(item0 + k) * n_experts + i] = sum over item k of (expert_i - base)^2 in f64 (or
 * delta_i^2).  Non-finite inputs propagate into the partial (detected by rlk_fusion_finalize).
 * With nz_counters (device [n_tensors * 2N] u64, accumulated) it also counts, per (tensor, expert),
 * the entries that are non-zero after dropout (FusionStats.dropout_kept_fraction numerator,
 * fusion.py:172-174); the keep bits come from the K2 bitmap (dropout_mode 2), inline SplitMix64
 * (1, child_seeds a HOST array) or none (0), so K2 runs before K1. */
int rlk_fusion_sumsq(const rlk_fusion_plan* plan, int n_experts, int dtype, int delta_mode,
                     double* partials, unsigned long long* nz_counters, int dropout_mode,
                     const uint64_t* child_seeds, uint64_t thresh, const uint32_t* bitmap,
                     uint64_t words_per_row, void* stream);

/* Per tensor t: sumsq[t*N+i] = sum of its item partials in a fixed order (items
 * tensor_items[t] .. tensor_items[t+1]-1); norm = sqrt(sumsq); target per target_mode
 * (0 = none -> scale 1, 1 = mean of non-zero norms, 2 = target_value); scale = target / norm, or 1 for a
 * zero vector.  status[t]: 0 ok, 1 = all-zero task vectors under mean mode, 2 = non-finite input. */
int rlk_fusion_finalize(const double* partials, const uint32_t* tensor_items, uint32_t n_tensors,
                        int n_experts, int target_mode, double target_value, double* sumsq,
                        double* scale, int32_t* status, void* stream);

/* K2: bitmap[i * words_per_row + w] bit b = keep decision for draw j = 32*w + b of child stream i:
 * (mix64(child_seeds[i] + (j+1)*0x9E3779B97F4A7C15) >> 11) >= thresh.  child_seeds is a HOST array. */
int rlk_fusion_mask_bitmap(const uint64_t* child_seeds, int n_experts, uint64_t thresh, uint64_t n_bits,
                           uint32_t* bitmap, uint64_t words_per_row, void* stream);
/* The same bits for indices [bit_lo, bit_hi) only (bit_lo % 32 == 0): a sharded job draws its slice of
 * the rows and all-gathers them (FusionCall under a process group) instead of every rank drawing
 * every row. */
int rlk_fusion_mask_bitmap_range(const uint64_t* child_seeds, int n_experts, uint64_t thresh, uint64_t bit_lo,
                                 uint64_t bit_hi, uint32_t* bitmap, uint64_t words_per_row, void* stream);

/* K3 merge.  delta_mode: 0 = experts are expert tables (delta = expert - base); bit 0 set = experts are
 * task-vector deltas, and then bit 1 says whether the base stream is present (fused = base + sum) or
 * absent (fused = 0 + sum, used to materialise transformed task vectors).
 * scale: device [n_tensors * N] f64 (from finalize).  weights / child_seeds: HOST arrays.
 * dropout_mode: 0 none, 1 inline SplitMix64, 2 bitmap (bitmap/words_per_row from K2).
 * keep_prob = 1 - p (f64, as the reference computes it).  erase_mode: 0 off, 1 sum, 2 squared.
 * counters: device [n_tensors * 2N] u64, accumulated (caller zeroes): K3 adds the entries erased at
 * [t*2N + N + i] (the non-zero-after-dropout counts at [t*2N + i] come from K1).
 * bf16 -> bf16 with N <= 4 and dropout_mode 0/2 runs the f32x2 fast kernel with certified guards
 * (bit-identical to the f64 path); exact_path = 1 forces the reference-order f64 kernel instead (the
 * results are the same either way; the parity tests compare the two). */
int rlk_fusion_merge(const rlk_fusion_plan* plan, int n_experts, int dtype_in, int dtype_out,
                     int delta_mode, const double* scale, const double* weights, int dropout_mode,
                     const uint64_t* child_seeds, uint64_t thresh, double keep_prob,
                     const uint32_t* bitmap, uint64_t words_per_row, int erase_mode,
                     unsigned long long* counters, int exact_path, void* stream);

/* rlk_fusion_merge with a caller workspace for the bf16 fast path: elements whose certified f32
 * evaluation is inconclusive (~0.05% with normalisation) are queued per CTA and finished by a fix-up
 * kernel on the same stream (reference-order float64, one element per thread) instead of by one lane
 * of a warp inside the merge.  workspace: 16-byte aligned device memory, RLK_MERGE_WS_HEADER bytes of
 * queue lengths + 8 bytes per queued element (a full queue falls back to the in-kernel path); NULL or 0
 * = rlk_fusion_merge.  Results are identical either way. */
#define RLK_MERGE_WS_HEADER 4096
int rlk_fusion_merge_ws(const rlk_fusion_plan* plan, int n_experts, int dtype_in, int dtype_out, int delta_mode,
                        const double* scale, const double* weights, int dropout_mode, const uint64_t* child_seeds,
                        uint64_t thresh, double keep_prob, const uint32_t* bitmap, uint64_t words_per_row,
                        int erase_mode, unsigned long long* counters, int exact_path, void* workspace,
                        uint64_t workspace_bytes, void* stream);

/* GRPO token objective over packed rows (K4).  Token r reads logits row row_index[r] (or r when
 * row_index is NULL), row_stride elements between rows, vocab V.  Per token: token id, behaviour
 * log-probs on the train and inference engines (f64), and its sample id s into the per-sample arrays
 * adv[s], use[s] (1 = Mask.USE), temperature[s] and norm[s] = 1 / (G * T_max * n_groups).
 * Rows of masked samples are not read (objective.py:240-241).
 * Outputs per token (device, f64): logp (z_tok/T - lse), lse (natural log-sum-exp of z/T), term
 * (w * value, 0 if masked) and coef (norm * w * slope * r / T, the dJ/dlogit scale; 0 if masked).
 * flags[0] |= 1 when a row's logp is non-finite, |= 2 when a token id is out of [0, V).  Caller zeroes.
 * workspace (device f32, >= n_rows * 32 floats, nullable): with it, bf16/f32 logits run as two kernels
 * (K4a streams rows and writes per-(row, warp) log-sum-exp partials without block synchronisation;
 * K4b combines them and runs the epilogue); without it, one kernel reduces each row in-block. */
typedef struct rlk_clip {
  double eps_neg_low, eps_pos_high, eps_neg_high, tis_cap;
  int32_t guard_positive;
} rlk_clip;

int rlk_grpo_fwd(const void* logits, int dtype, uint64_t n_rows, uint64_t vocab, uint64_t row_stride,
                 const int64_t* row_index, const int32_t* tokens, const double* logp_train,
                 const double* logp_infer, const int32_t* sample_of_row, const double* adv,
                 const uint8_t* use, const double* temperature, const double* norm,
                 const rlk_clip* clip, double* logp_out, double* lse_out, double* term,
                 double* coef, int32_t* flags, float* workspace, uint64_t workspace_floats, void* stream);

/* Fused single-pass forward + backward for bf16 logits, one row per token (the LM layout): the same
 * per-token outputs as rlk_grpo_fwd plus grad[row, v] = grad_scale * coef * (onehot - softmax) written
 * as bf16 (grad_row_stride elements apart), reading every logit once.  2-CTA clusters split each row;
 * vocab % 16 == 0 and vocab <= 204800.  Replaces objective_value + objective_gradient
 * (objective.py:230-283) for that layout. */
int rlk_grpo_fused_bf16(const void* logits, uint64_t n_rows, uint64_t vocab, uint64_t row_stride,
                        const int64_t* row_index, const int32_t* tokens, const double* logp_train,
                        const double* logp_infer, const int32_t* sample_of_row, const double* adv,
                        const uint8_t* use, const double* temperature, const double* norm,
                        const rlk_clip* clip, double grad_scale, double* logp_out, double* lse_out,
                        double* term, double* coef, int32_t* flags, void* grad, uint64_t grad_row_stride,
                        void* stream);

/* The same for bf16 (2-CTA clusters, gradient bf16) or f32 logits (4-CTA clusters -- each CTA owns a
 * quarter row of 128 KiB -- gradient f32): 8 B of HBM traffic per f32 logit instead of 12 for
 * rlk_grpo_fwd + rlk_grpo_bwd.  vocab % (8 * cluster) == 0 and vocab <= 204800 (bf16) / 204800 (f32). */
int rlk_grpo_fused(const void* logits, int dtype, uint64_t n_rows, uint64_t vocab, uint64_t row_stride,
                   const int64_t* row_index, const int32_t* tokens, const double* logp_train,
                   const double* logp_infer, const int32_t* sample_of_row, const double* adv,
                   const uint8_t* use, const double* temperature, const double* norm,
                   const rlk_clip* clip, double grad_scale, double* logp_out, double* lse_out,
                   double* term, double* coef, int32_t* flags, void* grad, uint64_t grad_row_stride,
                   void* stream);

/* out[g] = sum of x[seg_ptr[g] .. seg_ptr[g+1]) in a fixed order (one block per segment). */
int rlk_segment_sum_f64(const double* x, const int64_t* seg_ptr, uint64_t n_segs, double* out, void* stream);

/* GRPO backward (K5).  Output row o of grad (grad_row_stride elements apart) is
 *   grad[o, v] = sum over tokens k listed for o (CSR row_tok_ptr[o] .. row_tok_ptr[o+1]-1 into row_tok, in
 *   order) of coef_k * (onehot(tokens_k)[v] - exp(z_v / T_k - lse_k)),
 * evaluated in the reference order (row -= coef * p; row[token] += coef; objective.py:278-282).  With
 * row_tok_ptr == NULL output row o is token o.  z is logits row logits_row[o] (NULL = o).  Rows with no
 * non-zero coef are written as zeros without reading logits.  T_k = temperature_tok[k]. */
int rlk_grpo_bwd(const void* logits, int dtype, uint64_t n_out_rows, uint64_t vocab, uint64_t row_stride,
                 const int64_t* logits_row, const int64_t* row_tok_ptr, const int64_t* row_tok,
                 const int32_t* tokens, const double* temperature_tok, const double* lse, const double* coef,
                 void* grad, int grad_dtype, uint64_t grad_row_stride, void* stream);

/* log_token_dist over rows: out[r, v] = z / T_r - lse_r for logits row row_index[r] (NULL = r). */
int rlk_logsoftmax_rows(const void* logits, int dtype, uint64_t n_rows, uint64_t vocab, uint64_t row_stride,
                        const int64_t* row_index, const double* temperature_row, void* out, int out_dtype,
                        void* stream);

/* Count of non-finite elements (ParamTable finite check). count: device u64, accumulated. */
int rlk_nonfinite_count(const void* x, int dtype, uint64_t n, unsigned long long* count, void* stream);

/* out = a + alpha * b elementwise in f64 semantics (ascent_step), dtype shared. */
int rlk_scaled_add(const void* a, const void* b, double alpha, void* out, int dtype, uint64_t n,
                   void* stream);

/* Benchmark / test data: out[i] = RN(base[i] + std * N(0,1)) with a counter-hash normal keyed by
 * (seed, j0 + i); base may be NULL (then 0) and has out's dtype. */
int rlk_synth_normal(void* out, int dtype, uint64_t n, uint64_t j0, uint64_t seed, double std_dev,
                     const void* base, void* stream);

/* Checkpoint checksum ("flat LE f64 + checksum"): *out += sum_i mix64(w_i ^ ((word_offset + i + 1)
 * * 0x9E3779B97F4A7C15)) mod 2^64 over n_words 64-bit words (8-byte aligned).  Chunks may be summed in
 * any order.  out is a device u64 (caller zeroes). */
int rlk_checksum64(const void* data, uint64_t n_words, uint64_t word_offset, unsigned long long* out,
                   void* stream);

/* ---- K7 host streaming loader (checkpoints larger than HBM) -------------------------------------
 * A ring of n_slots pinned host slots of slot_bytes each and n_threads host workers (0 = all cores).
 * h2d / d2h pipeline pageable<->pinned memcpy against cudaMemcpyAsync on `stream`; the device side of
 * a copy is complete when `stream` reaches the point of the call.  Host ranges that are already
 * page-locked (cudaHostAlloc / cudaHostRegister, e.g. torch pin_memory) skip the slots: one
 * cudaMemcpyAsync on `stream`, asynchronous to the host, so such a buffer must stay valid (and, for
 * d2h, unread) until `stream` reaches the call.  Loader state is not thread-safe:
 * one loader per host thread.  Replaces: no reference counterpart (the reference holds everything in
 * RAM as float64); the on-disk format it feeds is SPEC.md:588/727 (see loader.py). */
void* rlk_loader_create(uint64_t slot_bytes, int n_slots, int n_threads);
void rlk_loader_destroy(void* loader);
const char* rlk_loader_last_error(void);
int rlk_loader_h2d(void* loader, void* dst_dev, const void* src_host, uint64_t bytes, void* stream);
int rlk_loader_d2h(void* loader, void* dst_host, const void* src_dev, uint64_t bytes, void* stream);
/* Synthesise random-init parameters [j0, j0+n) into pinned slots on the host workers and DMA them:
 * value(j) = RN(base(j) + noise_std * N(noise_seed, j)), base(j) = RN(base_std * N(base_seed, j)),
 * noise_seed 0 = the base itself.  dtype RLK_BF16 or RLK_F32. */
int rlk_loader_synth_h2d(void* loader, void* dst_dev, int dtype, uint64_t n, uint64_t j0, uint64_t base_seed,
                         double base_std, uint64_t noise_seed, double noise_std, void* stream);
/* D2H through the slots, folding the data into *checksum (sum of 64-bit words mod 2^64); bytes % 8 == 0. */
int rlk_loader_d2h_checksum(void* loader, const void* src_dev, uint64_t bytes, uint64_t* checksum, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* RLK_H_ */
