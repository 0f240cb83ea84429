/*
 * hx_api.h -- C-ABI of the B200 (sm_100a) asymmetric TP/PP decoder data path.
 *
 * The reference (heteroplan, pure Python) has no FFI: its runtime boundary is
 * the plan document (reference pkg/src/heteroplan/cli.py:75-115) plus the
 * per-(replica, task) service-time table (pkg/src/heteroplan/simulate.py:135-142),
 * and the paper's per-layer math is what these entry points
 * execute. Each function below replaces one term of the reference's closed-form
 * stand-in for the path (pkg/src/heteroplan/costs.py:106-176):
 *
 *   hx_linear                 weight-scan + FLOP terms   costs.py:114-119
 *   hx_rope_kv_append,
 *   hx_attn_decode_paged,
 *   hx_attn_decode_rope_append,
 *   hx_attn_prefill           attention / KV concat
 *   hx_residual_add_rmsnorm   "+ x" residual after each all-reduce
 *   hx_argmax_*               greedy token selection (not modelled by the reference)
 *   hx_kv_bytes               KV part of mem_footprint   costs.py:168-176
 *
 * Conventions (no torch types cross this boundary):
 *   - every pointer is a device pointer owned by the caller; the library never
 *     allocates or frees; scratch is passed in as (workspace, bytes);
 *   - every call is asynchronous on `stream` (a cudaStream_t) and returns 0 on
 *     success or a positive hx error code / cudaError_t value (hx_error_string);
 *   - dtype codes: HX_F32 (fp32 mode) or HX_BF16 (bf16 mode); accumulation and
 *     softmax are always fp32; the residual stream `x` is always fp32;
 *   - matrices are row-major; weights are [out, in] (nn.Linear layout), so
 *     Y[t, n] = sum_k X[t, k] * W[n, k];
 *   - paged KV layout: cache[block][kv_head][page_size][head_dim] (K and V in
 *     separate arrays), block_table[seq][max_blocks] (int32 block ids),
 *     seq_lens[seq] = tokens already cached before this call (int32).
 */
#ifndef HX_API_H
#define HX_API_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef void *hx_stream_t; /* cudaStream_t */

enum hx_dtype { HX_F32 = 0, HX_BF16 = 1 };

enum hx_status {
  HX_OK = 0,
  HX_ERR_ARG = 1001,        /* bad shape / pointer / dtype combination */
  HX_ERR_UNSUPPORTED = 1002, /* shape the kernels do not implement */
  HX_ERR_WORKSPACE = 1003,   /* workspace too small */
  HX_ERR_DRIVER = 1004       /* cuTensorMapEncodeTiled unavailable / failed */
};

/* library identity, error text, and a count of kernels launched so far */
int hx_version(void);
const char *hx_error_string(int code);
uint64_t hx_launch_count(void);

/* x[t, :] = float(table[ids[t], :]);  table [vocab, hidden] (dtype) */
int hx_embed(const int32_t *ids, const void *table, int table_dtype, float *x,
             int n_tok, int hidden, int vocab, hx_stream_t stream);

/* out[t, :] = x[t * ldx, :] / sqrt(mean(x^2) + eps) * gain  (out in out_dtype,
 * rows contiguous). ldx = row pitch of x in elements (>= hidden), which lets
 * the last stage normalise only each sequence's last prompt token. */
int hx_rmsnorm(const float *x, int ldx, const float *gain, void *out, int out_dtype,
               int n_tok, int hidden, float eps, hx_stream_t stream);

/* x += delta (fp32, the all-reduced row-parallel output); out = rmsnorm(x)*gain.
 * out may be NULL (residual add only). */
int hx_residual_add_rmsnorm(float *x, const float *delta, const float *gain,
                            void *out, int out_dtype, int n_tok, int hidden,
                            float eps, hx_stream_t stream);

/* Y[t, n] (+)= sum_k X[t, k] W[n, k], t < n_tok, n < n_out, k < k_dim.
 * bf16 weights+activations: tcgen05/TMEM tensor-core kernel fed by TMA
 * (split-K for decode-sized n_tok, fp32 accumulate); fp32: CUDA-core kernel.
 * y_dtype HX_F32 or HX_BF16; ldy = row pitch of Y in elements; flags:
 * HX_LINEAR_ACCUMULATE (Y += .., fp32 Y only), HX_LINEAR_PACKED (w is in the
 * hx_pack_weight tile layout). workspace >= hx_linear_workspace(...), its
 * first 16 KB (ticket counters) zeroed once before first use.
 * Under PDL the kernel streams its first weight tiles before waiting on the
 * previous kernel: W must not be written by the kernel launched just before
 * it on the stream (weights are static; hx_pack_weight never triggers early). */
enum hx_linear_flags { HX_LINEAR_ACCUMULATE = 1, HX_LINEAR_PACKED = 2, HX_LINEAR_DEFER_REDUCE = 4,
                       HX_LINEAR_L2_PREFETCH = 8 };
/* HX_LINEAR_L2_PREFETCH (decode shapes): before its PDL wait each CTA also
 * prefetches its next weight tiles (HX_GEMM_L2PF, default 16) into L2 -- for a
 * GEMM that follows a latency-bound kernel (the TP all-reduce). */
/* HX_LINEAR_DEFER_REDUCE (decode shapes, fp32 Y): tiles split across CTAs are
 * left as fp32 partial slots in the workspace instead of being reduced by a
 * ticketed last CTA; the next kernel on the stream must be
 * hx_splitk_residual_rmsnorm with the same shape and workspace, which sums
 * them in the same order (bitwise identical to the in-kernel reduction). */
int hx_splitk_residual_rmsnorm(float *x, const float *y, int ldy, const void *workspace,
                               int n_tok, int n_out, int k_dim, const float *gain,
                               void *out, int out_dtype, float eps, hx_stream_t stream);
int hx_linear(const void *w, const void *x, void *y, int dtype, int y_dtype,
              int n_tok, int n_out, int k_dim, int ldy, int flags,
              void *workspace, size_t workspace_bytes, hx_stream_t stream);
size_t hx_linear_workspace(int dtype, int n_tok, int n_out, int k_dim);

/* Repack a bf16 weight [n_out, k_dim] into [ceil(n/128)][ceil(k/64)][128][64]
 * tiles (zero padded) so each 16 KB tile the decode GEMM streams is one
 * contiguous HBM range; packed holds hx_packed_weight_elems(n_out, k_dim). */
int hx_pack_weight(const void *w, void *packed, int n_out, int k_dim, hx_stream_t stream);
size_t hx_packed_weight_elems(int n_out, int k_dim);

/* Programmatic dependent launch on/off for subsequent launches (default on). */
void hx_set_pdl(int enabled);

/* Profiling aid: subsequent decode-GEMM launches record, per CTA, 8 u64
 * (globaltimer at start, after the dependency wait, at exit; SM id; first
 * accumulator ready, first epilogue done, last accumulator ready; segments) into buf
 * (device memory, `records` CTA slots). Returns the slots used since the
 * previous call; buf = NULL disables. */
size_t hx_debug_trace(void *buf, size_t records);

/* ---- TP all-reduce over NVLink peer memory (decode), fused with residual+RMSNorm.
 * Replaces NCCL all-reduce + hx_residual_add_rmsnorm after each row-parallel
 * projection of a TP>1 stage (reference tp_comm_cost, costs.py:123-147).
 * Buffers come from hx_ipc_alloc (zeroed cudaMalloc), are exported with
 * hx_ipc_handle (64-byte cudaIpcMemHandle) and mapped on peers with hx_ipc_open.
 * parts[r] = rank r's fp32 partial slot [n_tok][hidden] (peer-mapped; own local),
 * flags[r] = rank r's int flag array [sites][max_tok][8]; site_state = this
 * rank's int [sites][2] (zeroed). Every rank calls with the same site sequence;
 * x[t] += sum_r parts[r][t] (rank order: bitwise identical on all ranks);
 * out = rmsnorm(x) * gain (out may be NULL). Waits are bounded (trap, not hang). */
int hx_ipc_alloc(void **ptr, size_t bytes);
int hx_ipc_free(void *ptr);
int hx_ipc_handle(void *ptr, void *handle64);
int hx_ipc_open(const void *handle64, void **peer_ptr);
int hx_ipc_close(void *peer_ptr);
int hx_tp_allreduce_residual_rmsnorm(float *x, const float *const *parts, int *const *flags, int rank,
                                     int tp, int site, int max_tok, int *site_state,
                                     const float *gain, void *out, int out_dtype, int n_tok,
                                     int hidden, float eps, hx_stream_t stream);

/* Push (one-shot, flag-free) variant of the same all-reduce: each rank stores
 * its partial row into every peer's inbox over NVLink and polls its own inbox
 * for the peers' rows (sentinel -0.0f until the data lands). inboxes[r] = rank
 * r's inbox of hx_tp_inbox_bytes(tp, max_tok, hidden) bytes (peer-mapped; own
 * local), armed once with hx_tp_inbox_init; own_part = this rank's partial
 * [n_tok][hidden]; state = this rank's per-CTA call counters, int[4 * max_tok]
 * (zeroed once). Same result bits as hx_tp_allreduce_residual_rmsnorm. */
size_t hx_tp_inbox_bytes(int tp, int max_tok, int hidden);
int hx_tp_inbox_init(void *inbox, int tp, int max_tok, int hidden, hx_stream_t stream);
int hx_tp_allreduce_push_residual_rmsnorm(float *x, const float *own_part, float *const *inboxes,
                                          int rank, int tp, int max_tok, int *state,
                                          const float *gain, void *out, int out_dtype, int n_tok,
                                          int hidden, float eps, hx_stream_t stream);
/* _ex variants: payload_dtype HX_F32 (the calls above) or HX_BF16 -- each
 * partial row is rounded to bf16 once (on every rank, its own included) and
 * summed in fp32 in rank order: half the NVLink bytes, all ranks bitwise
 * identical; inbox halfwords armed with the bf16 sentinel 0x8000. hidden must be
 * a multiple of 32 for bf16 (16 for fp32). */
size_t hx_tp_inbox_bytes_ex(int tp, int max_tok, int hidden, int payload_dtype);
int hx_tp_inbox_init_ex(void *inbox, int tp, int max_tok, int hidden, int payload_dtype, hx_stream_t stream);
int hx_tp_allreduce_push_residual_rmsnorm_ex(float *x, const float *own_part, void *const *inboxes, int rank,
                                             int tp, int max_tok, int *state, const float *gain, void *out,
                                             int out_dtype, int n_tok, int hidden, float eps, int payload_dtype,
                                             hx_stream_t stream);
/* The same after a deferred row-parallel GEMM (hx_linear with
 * HX_LINEAR_DEFER_REDUCE into own_part, workspace gemm_workspace, reduction
 * dim k_dim): the GEMM's split tiles are summed from its partial slots in CTA
 * order while the row is read (bitwise the fix-up's result), so the O / down
 * GEMM ends without its split-K fix-up tail. push mode only. */
int hx_tp_allreduce_push_residual_rmsnorm_sk(float *x, const float *own_part, const void *gemm_workspace, int k_dim,
                                             void *const *inboxes, int rank, int tp, int max_tok, int *state,
                                             const float *gain, void *out, int out_dtype, int n_tok, int hidden,
                                             float eps, int payload_dtype, hx_stream_t stream);

/* ---- Inter-stage reshard over NVLink P2P (decode hand-off and token return).
 * Replaces the leader send + broadcast of PAPER.md:197 (modelled by
 * pp_comm_cost, costs.py:150-165): receiver r' of stage j+1 owns an inbox that
 * sender r' mod TP_j stores into directly (hx_handoff_push), and it polls the
 * inbox in place (hx_handoff_pull) -- 32-bit words armed with the sentinel
 * 0x80000000 by hx_handoff_inbox_init; pushed words equal to it travel as 0.
 * inbox = hx_handoff_inbox_bytes(max_words) bytes from hx_ipc_alloc, mapped on
 * the sender with hx_ipc_open; max_words % 4 == 0; words <= max_words; each
 * side's state = its own zeroed int[2] call counter. Both are graph-capturable
 * and need no host synchronisation; waits are bounded (trap, not hang). */
size_t hx_handoff_inbox_bytes(size_t max_words);
int hx_handoff_inbox_init(void *inbox, size_t max_words, hx_stream_t stream);
int hx_handoff_push(const void *src, void *const *dst_inboxes, int n_dst, size_t words,
                    size_t max_words, int *state, hx_stream_t stream);
int hx_handoff_pull(void *dst, void *inbox, size_t words, size_t max_words, int *state,
                    hx_stream_t stream);
/* Flow-controlled variant for streams of hand-offs the sender may run ahead on
 * (the pipelined prefill's micro-batches): the receiver drains hand-off k from
 * buffer k % 3, re-arms it in place and publishes credit k + 1 in the inbox's
 * credit word; the sender's hand-off k waits (over NVLink) for credit >= k - 2
 * before storing. One destination per call; state as above (int[2], zeroed),
 * separate from the decode links'. */
int hx_handoff_push_credit(const void *src, void *dst_inbox, size_t words, size_t max_words, int *state,
                           hx_stream_t stream);
int hx_handoff_pull_credit(void *dst, void *inbox, size_t words, size_t max_words, int *state, hx_stream_t stream);

/* ---- Prefill attention on tcgen05 (whole prompt, no earlier context).
 * hx_prefill_vt writes the prompt's V transposed per (sequence, kv head):
 * vt[((b * hkv + h) * 128 + d) * s + i] (bf16) from the packed qkv rows.
 * hx_attn_prefill_tc: o[b, i, h, :] = causal softmax(q k^T / sqrt(128)) v with q
 * [b*s][hq*128] (roped), K from the paged cache (page 64), V from vt; needs hd
 * 128, s % 128 == 0 (HX_ERR_UNSUPPORTED otherwise: use hx_attn_prefill). */
int hx_prefill_vt(const void *qkv, void *vt, int batch, int s_len, int hq, int hkv, int hd,
                  hx_stream_t stream);
int hx_attn_prefill_tc(const void *q, const void *k_cache, const void *vt, const int32_t *block_table,
                       void *o, int batch, int s_len, int hq, int hkv, int hd, int page_size,
                       int max_blocks, hx_stream_t stream);

/* Consumer of a deferred gate/up GEMM (hx_linear with HX_LINEAR_DEFER_REDUCE
 * into fp32 y [n_tok][ldy >= 2 inter], k_dim = its K): out (bf16) = silu(gate)
 * * up with gate/up reduced from the split-K slots and rounded to bf16 --
 * bit-identical to hx_linear (bf16 out) + hx_swiglu. */
int hx_splitk_swiglu(const float *y, int ldy, const void *workspace, int n_tok, int inter,
                     int k_dim, void *out, int ld_out, hx_stream_t stream);

/* out[t, j] = silu(gu[t, j]) * gu[t, inter + j], j < inter */
int hx_swiglu(const void *gu, void *out, int dtype, int n_tok, int inter,
              hx_stream_t stream);

/* RoPE (rotate-half, theta) on q and k of the packed qkv rows
 * [n_tok, (hq + 2 hkv) * hd], write roped q to q_out [n_tok, hq, hd] and k, v
 * into the paged cache. Decode (prefill_len == 0): token t is seq t at
 * position seq_lens[t]. Prefill (prefill_len = s): token t is seq t / s at
 * position seq_lens[t / s] + t % s. */
int hx_rope_kv_append(const void *qkv, void *q_out, void *k_cache, void *v_cache,
                      const int32_t *block_table, const int32_t *seq_lens,
                      int dtype, int n_tok, int prefill_len, int hq, int hkv,
                      int hd, int page_size, int max_blocks, float theta,
                      hx_stream_t stream);

/* Decode attention over the paged cache for one new token per sequence:
 * o[b, h, :] = softmax(q[b, h] . K[b, h/g]^T / sqrt(hd)) V, context length
 * seq_lens[b] + 1 (the token appended by hx_rope_kv_append). Split-KV with an
 * in-kernel combine; workspace >= hx_attn_decode_workspace(...). */
int hx_attn_decode_paged(const void *q, const void *k_cache, const void *v_cache,
                         const int32_t *block_table, const int32_t *seq_lens,
                         void *o, int dtype, int batch, int hq, int hkv, int hd,
                         int page_size, int max_blocks, int max_ctx,
                         void *workspace, size_t workspace_bytes,
                         hx_stream_t stream);
size_t hx_attn_decode_workspace(int batch, int hq, int hkv, int hd, int max_ctx);

/* hx_rope_kv_append + hx_attn_decode_paged of one decode step in one kernel:
 * q comes un-rotated from the packed qkv rows ([batch][(hq + 2 hkv) * hd]);
 * each CTA rotates its q heads, the CTA whose KV range holds position
 * seq_lens[b] rotates that token's k and appends k, v to the page, and pages
 * below the new token's page are prefetched before the kernel waits on the
 * QKV producer. Results are bit-identical to the two separate calls. bf16,
 * hd 128, page 64 only (else HX_ERR_UNSUPPORTED: use the separate calls);
 * workspace as hx_attn_decode_workspace. */
int hx_attn_decode_rope_append(const void *qkv, void *k_cache, void *v_cache,
                               const int32_t *block_table, const int32_t *seq_lens,
                               void *o, int dtype, int batch, int hq, int hkv, int hd,
                               int page_size, int max_blocks, int max_ctx, float theta,
                               void *workspace, size_t workspace_bytes,
                               hx_stream_t stream);
/* hx_attn_decode_rope_append for a QKV projection run as a deferred decode GEMM
 * (hx_linear(..., HX_LINEAR_DEFER_REDUCE) into fp32 qkv32 [batch][ld_qkv], its
 * workspace gemm_workspace, inner dimension k_dim): the kernel sums the split
 * tiles' partials in CTA order and rounds to bf16 (the bits the GEMM's fix-up
 * would have stored), so the GEMM has no fix-up tail. Same outputs as
 * hx_linear (bf16 qkv) + hx_attn_decode_rope_append, bit for bit. */
int hx_attn_decode_rope_append_sk(const float *qkv32, int ld_qkv, const void *gemm_workspace, int k_dim,
                                  void *k_cache, void *v_cache, const int32_t *block_table,
                                  const int32_t *seq_lens, void *o, int batch, int hq, int hkv, int hd,
                                  int page_size, int max_blocks, int max_ctx, float theta, void *workspace,
                                  size_t workspace_bytes, hx_stream_t stream);

/* Causal prefill attention: q [batch*s, hq, hd] (roped), keys/values are the
 * s prompt tokens already appended to the paged cache (positions
 * seq_lens[b] .. seq_lens[b]+s-1, with seq_lens the values BEFORE append). */
int hx_attn_prefill(const void *q, const void *k_cache, const void *v_cache,
                    const int32_t *block_table, const int32_t *seq_lens,
                    void *o, int dtype, int batch, int s, int hq, int hkv,
                    int hd, int page_size, int max_blocks, hx_stream_t stream);

/* seq_lens[b] += n for b < batch (end of a stage step). */
int hx_advance(int32_t *seq_lens, int batch, int n, hx_stream_t stream);

/* Greedy selection, vocab-parallel: key[t] = pack(max_j logits[t, j],
 * smallest argmax j + vocab_offset) as an int64 whose signed order is
 * (value, -index); MAX-reducing keys across TP ranks gives the global argmax
 * with torch.argmax tie-breaking (first index). */
int hx_argmax_partial(const float *logits, int64_t *keys, int n_tok, int n_cols,
                      int ld, int vocab_offset, hx_stream_t stream);

/* ids[t] = unpack(key[t]); if history != NULL also history[t * s_out + *step]
 * = ids[t] and, when bump_step != 0, ++*step (one thread, after all writes). */
int hx_argmax_finalize(const int64_t *keys, int32_t *ids, int32_t *history,
                       int32_t *step, int s_out, int n_tok, int bump_step,
                       hx_stream_t stream);

/* KV bytes one rank holds for `layers` layers (part of mem_footprint). */
size_t hx_kv_bytes(int dtype, int layers, int num_blocks, int hkv_rank, int page_size, int hd);

#ifdef __cplusplus
}
#endif
#endif /* HX_API_H */
