/*
 * sart.h -- C-ABI of the B200-native SART multi-branch decode engine.
 *
 * SART (arXiv 2505.13326): "redundant sampling with early stopping" (PAPER.md
 * P:141-143) plus "two-phase dynamic pruning" scheduled by
 * Algorithm 1 with prefix-KV sharing and immediate KV release
 * (P:306).  This library runs the data-parallel hot path of that method on one
 * GPU: cascade paged decode attention, the decoder GEMMs, a counter-based
 * sampler with EOS detection, and the on-device branch control (early stop,
 * pruning, KV-block reclamation, block-table compaction, vote).  Every reading
 * of the paper the implementation depends on is numbered "R<n>" in DESIGN.md.
 *
 * Conventions (all entry points):
 *   - Every call returns int: SART_OK (0) or a negative SART_E* code.
 *     sart_strerror(code) names the code; sart_last_error() returns a
 *     thread-local message for the most recent failure.
 *   - Input pointers are HOST pointers unless stated otherwise; they are
 *     borrowed only for the duration of the call (deep-copied when needed).
 *   - The ctx owns all device memory it allocates.  Outputs go to caller buffers.
 *   - One sart_ctx per GPU (or per tensor-parallel rank); a ctx is NOT thread-safe, but
 *     different ctx may be driven from different host threads concurrently.
 *   - After SART_ECUDA the ctx is poisoned: every later call except
 *     sart_destroy returns SART_ESTATE.
 *   - Validation is all-or-nothing: an error never leaves partial state.
 */
#ifndef SART_H_
#define SART_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct sart_ctx sart_ctx;

enum {
  SART_OK = 0,
  SART_EINVAL = -1, /* a parameter is outside its documented range            */
  SART_ENOMEM = -2, /* device memory, or a request that can never fit the pool */
  SART_ECUDA = -3,  /* CUDA runtime error; the ctx is poisoned                  */
  SART_EFULL = -4,  /* output buffers too small (partial fill, rest kept)      */
  SART_ESTATE = -5, /* call on a poisoned ctx                                  */
  SART_EDUP = -6    /* request_id reused                                       */
};
enum { SART_BF16 = 0, SART_FP32 = 1 };
enum { SART_SELECT_VOTE = 0, SART_SELECT_MAX_REWARD = 1 };
enum { SART_ATTN_CASCADE = 0, SART_ATTN_FLAT = 1 };

/* Branch states reported in sart_result.branch_state (Alg. 1 L28-40, R7, R17). */
enum {
  SART_BR_QUEUED = 0,
  SART_BR_RUNNING = 1,
  SART_BR_COMPLETED_EOS = 2,
  SART_BR_COMPLETED_CAP = 3, /* reached max_new_tokens; counts as completed (R17) */
  SART_BR_PRUNED = 4,
  SART_BR_EARLY_STOPPED = 5,
  SART_BR_DISCARDED = 6 /* still queued when its request finalized (R7)       */
};

/*
 * Engine configuration (init-time; copied).
 *
 * Model: a pre-norm GQA decoder (RMSNorm, QKV with bias, rotate-half RoPE,
 * SwiGLU MLP, untied LM head) plus a 2-way PRM head on the final-norm hidden
 * state (readings R14, R15, R29).  head_dim must be 64 or 128;
 * n_heads % n_kv_heads == 0 and n_heads / n_kv_heads <= 16.
 *
 * host_weights: optional HOST blob; tensors concatenated row-major in this
 * order and dtype (bf16 bit patterns for SART_BF16, fp32 for SART_FP32),
 * weight matrices in nn.Linear layout [out][in]:
 *   embed[V][d]
 *   per layer l: attn_norm[d], wqkv[(qh+2kvh)*hd][d], bqkv[(qh+2kvh)*hd],
 *                wo[d][qh*hd], mlp_norm[d], wgate[F][d], wup[F][d], wdown[d][F]
 *   final_norm[d], lm_head[V][d], prm_w1[d][d], prm_b1[d], prm_w2[2][d], prm_b2[2]
 * (q rows first, then k, then v inside wqkv).  NULL -> weights are generated
 * on the device from weight_seed: N(0, weight_std^2), norms 1 + N(0, 0.1^2).
 */
typedef struct {
  int32_t n_layers, d_model, n_heads, n_kv_heads, head_dim, d_ff, vocab;
  float rope_theta; /* RoPE base (Qwen2.5: 1e6)                                    */
  float rms_eps;    /* RMSNorm epsilon (1e-6)                                      */
  int32_t dtype;    /* SART_BF16 (bf16 storage, fp32 accumulate) or SART_FP32        */
  uint64_t weight_seed;
  float weight_std;           /* device init std (0 -> 0.02)                        */
  const void* host_weights;   /* optional host blob, see above                        */
  int32_t block_size;         /* tokens per KV block: 16, 32 or 64 (0 -> 64)          */
  int64_t num_blocks;         /* KV pool blocks NB; 0 -> size from free HBM           */
  int32_t max_rows;           /* B: max live branches; 0 -> 1024              */
  int32_t max_requests;       /* live request slots (prefilled, not finalized); 0->256*/
  int32_t max_prompt;         /* longest prompt accepted (tokens); 0 -> 8193         */
  int32_t ctl_interval;       /* T (default 400)                        */
  int32_t max_new_tokens;     /* cap: suffix length limit per branch (>= 1)           */
  int32_t eos_id;             /* end-of-sequence token                                */
  float temperature;          /* tau > 0: Gumbel-max sampling; 0: argmax (R24)       */
  uint64_t sampler_seed;      /* Philox key (R25)                                     */
  int32_t select_mode;        /* which branch's tokens sart_collect returns          */
  int32_t attn_mode;          /* SART_ATTN_CASCADE (default) or SART_ATTN_FLAT        */
  int32_t device;             /* CUDA device ordinal                                  */
  void* stream;               /* cudaStream_t to run on (NULL -> ctx-owned stream)    */
  int32_t enable_forced_tokens; /* allocate teacher-forcing buffers (tests)          */
  int32_t debug_capture;      /* keep per-layer attention outputs of the last step   */
  int32_t profile;            /* time the attention kernels with CUDA events         */
  /* NEXT row f2: a separate PRM decoder instead of the
   * 2-way head on the policy's hidden state.  prm_n_layers == 0: the head (row a8).
   * prm_n_layers > 0: a second pre-norm GQA decoder of these dims (vocab, rope_theta,
   * rms_eps and dtype are the policy's; head_dim 64 or 128; bf16 needs prm_d_ff % 128 == 0)
   * with its own 2-way head.  At every boundary it reads each branch's tokens decoded in
   * the window through its own paged KV cache -- the SAME block ids as the policy's pool
   * (so reclamation and compaction cover both), the prompt prefix prefilled once per
   * request -- and scores the last of them (reading R42: the PRM has read prompt + y_1 ..
   * y_{l-1} after l generated tokens).  prm_host_weights: optional HOST blob in the
   * host_weights layout with the PRM dims (its lm_head is unused); NULL -> generated on the
   * device from prm_weight_seed.  num_blocks == 0 sizes the pool for both caches. */
  int32_t prm_n_layers, prm_d_model, prm_n_heads, prm_n_kv_heads, prm_head_dim, prm_d_ff;
  uint64_t prm_weight_seed;
  const void* prm_host_weights;
  /* SURVEY §8(b) additions.
   * kv_pool / kv_pool_bytes: optional caller-owned DEVICE buffer (e.g. torch-allocated on
   *   `device`) that holds the policy's paged KV pool [L][NB][2][kvh][bs][hd]; the caller keeps
   *   it alive until sart_destroy, the ctx never frees it and zeroes it at init.  NB =
   *   num_blocks if > 0 (must fit: else ENOMEM), otherwise kv_pool_bytes / block bytes.  NULL:
   *   the ctx allocates the pool.  (The f2 PRM model's pool is always ctx-allocated.)
   * es_every_step: 0 = paper semantics (early stop is decided at T boundaries, P:300-305,
   *   reading R8); 1 = variant: once a request has M completed branches, its other running
   *   branches stop decoding at that step (reading R43); they are EarlyStopped at the boundary.
   * record_trace: 1 = record, at every boundary, each window row's generated tokens and the
   *   score the boundary used, plus a 64-bit FNV-1a hash of the control state after the
   *   boundary (sart_trace_fetch) -- the streams the oracle replays bit-exactly (PP2). */
  void* kv_pool;
  size_t kv_pool_bytes;
  int32_t es_every_step;
  int32_t record_trace;
  /* NEXT row f4 (the paper's 70B model): tensor parallelism over
   * tp_size GPUs (one ctx per GPU, tp_rank = its position).  The model dims above are the
   * FULL model's; this ctx holds q heads [rank*qh/tp, ...), kv heads [rank*kvh/tp, ...), FFN
   * rows [rank*F/tp, ...) (Megatron split: QKV / gate-up by output rows, O / down by input
   * columns; embedding, norms, LM head and PRM head replicated) and its share of the KV pool.
   * host_weights is the FULL blob (each rank extracts its shard); device-generated weights
   * equal the TP = 1 model's.  The O-projection and down-projection outputs are partial sums
   * over ranks: their GEMM epilogues store every partial tile straight into each peer's
   * receive buffer over NVLink (sart_tp_buffer / sart_tp_connect), then signal the peers;
   * the consuming RMSNorm waits for all ranks' tiles and sums them in (rank, split) order,
   * so every rank holds the same residual stream, the same logits and the same tokens, and
   * the (replicated) branch control stays identical across ranks.  Every rank must receive
   * the same sart_admit / sart_step calls.  Requires dtype SART_BF16, no PRM model,
   * n_heads and n_kv_heads divisible by tp_size, (d_ff / tp_size) % 128 == 0.
   * tp_size 0 or 1: no tensor parallelism. */
  int32_t tp_size, tp_rank;
  /* NEXT row f1: chunked prefill interleaved with decode (reading
   * R44).  0: each fill's prompts are prefilled before the window's first decode step (Alg. 1
   * L7 inline).  C in [1, 2048]: they are prefilled in C-token chunks, chunk c right before
   * window step min(c + 1, T), so resident rows keep decoding while long prompts are
   * prefilled; the rows of a request prefilled in this window start decoding at the step
   * whose chunk completes its prefix (ST_WAIT until then), every other row at step 1. */
  int32_t prefill_chunk;
} sart_config;

/* Create an engine.  Errors: EINVAL (shape/range), ENOMEM (allocation failure, or
 * a pool smaller than one branch: NB < ceil(cap/bs)), ECUDA. */
int sart_init(const sart_config* cfg, sart_ctx** out);

/*
 * Optional workload script (synthetic inputs).
 *   forced_len[N]   1 <= len <= cap: the step at which EOS is emitted; EOS is
 *                   masked at every other step (R36).  NULL: model EOS.
 *   scores[N][n_bnd] reward used at the k-th boundary the branch is running at
 *                   (k clamped to n_bnd-1) (R35); final_score[N] at completion.
 *                   Both NULL -> the PRM head scores; exactly one NULL -> EINVAL.
 *   answer[N]       labels for the vote; NULL -> last non-EOS token (R16).
 *   forced_tokens[N][cap] teacher forcing: y_s := forced_tokens[b][s-1]
 *                   (requires enable_forced_tokens); NULL -> sampled.
 */
typedef struct {
  const int32_t* forced_len;
  const float* scores;
  const float* final_score;
  const int32_t* answer;
  int32_t n_bnd;
  const int32_t* forced_tokens;
} sart_script;

/*
 * One request.  Admission deep-copies prompt and script and pushes
 * the request onto the FCFS request_queue.
 *   1 <= M <= N <= 32; 0 <= beta <= N-1 or -1 (-> N/2);
 *   prune_threshold alpha <= 1; alpha < 0 disables pruning in BOTH phases (R20);
 *   1 <= prompt_len <= max_prompt.
 * Errors: EINVAL, EDUP (request_id seen before), ENOMEM (the request could never
 * be admitted even into an empty pool: ceil((P-1)/bs) + ceil(cap/bs) > NB).
 */
typedef struct {
  int64_t request_id;
  const int32_t* prompt;
  int32_t prompt_len;
  int32_t N, M;
  float prune_threshold;
  int32_t beta;
  const sart_script* script; /* may be NULL */
  int64_t arrival_ns;        /* for queuing latency; 0 -> time of admission */
} sart_request;
int sart_admit(sart_ctx* ctx, const sart_request* req);

typedef struct {
  int32_t windows;          /* boundaries processed since init            */
  int32_t steps;            /* decode steps executed since init           */
  int32_t live_rows;        /* rows in current_batch after the last boundary */
  int32_t queued_branches;  /* len(branch_queue)                          */
  int32_t queued_requests;  /* len(request_queue)                         */
  int32_t finalized_total;  /* requests finalized since init              */
  int32_t free_blocks;      /* free-stack size                            */
  int32_t committed_blocks; /* commitment (R34)                           */
  int64_t branch_tokens;    /* tokens produced by live rows since init    */
} sart_stats;

/*
 * Run up to max_windows windows.  A window is: admission (Alg. 1 L3-11 with
 * commitment, R34) -> up to T decode steps (L22; ends early when no row is
 * live, R31) -> boundary on the device (PRM, L23-40, block reclamation,
 * compaction, reservation, vote).  Returns early when nothing is live and both
 * queues are empty.  Blocks only on the per-window counter read.
 */
int sart_step(sart_ctx* ctx, int32_t max_windows, sart_stats* out);

/* Write the 16-int32 admission-counter record (live_rows, queued_branches,
 * queued_requests, free_blocks, committed_blocks, finalized_total, windows,
 * steps, branch_tokens lo/hi, 0...) into DEVICE memory dev_int32x16 (16 int32 on
 * this ctx's device, caller-owned), for the multi-GPU all-gather of SURVEY §8(e)
 * (torch.distributed).  The copy is issued on the ctx stream and completed before
 * the call returns, so a collective on any stream may read the record.
 * Errors: EINVAL (null), ESTATE (poisoned ctx), ECUDA. */
int sart_export_counters(sart_ctx* ctx, void* dev_int32x16);

/* One finalized request (O9 / P:279). */
typedef struct {
  int64_t request_id;
  int32_t answer_vote, vote_count;             /* plurality, ties -> lowest branch (R16) */
  int32_t chosen_max_reward, answer_max_reward; /* argmax final reward, ties -> lowest    */
  int32_t num_completed, num_pruned, num_early_stopped, num_discarded_queued;
  int32_t finalize_reason; /* 0: num_completed >= M; 1: completed + pruned == N         */
  int32_t phase_at_end;    /* 0 explore, 1 exploit                                     */
  float threshold_at_end;
  int32_t branch_len[32];
  uint8_t branch_state[32];
  float branch_score[32];
  int64_t t_arrival_ns, t_prefill_ns, t_final_ns;
  int32_t window_final, selected_branch;
  int64_t tokens_offset; /* into tokens_out: the selected branch's generated tokens */
  int32_t tokens_len;
} sart_result;

/* Copy finalized records (finalization order: window, ascending request_id) and
 * the selected branches' tokens into caller HOST buffers.  EFULL: what fits is
 * written and the rest is kept for the next call. */
int sart_collect(sart_ctx* ctx, sart_result* out, int32_t cap, int32_t* n_out,
                 int32_t* tokens_out, int64_t tokens_cap);

/*
 * PP2 trace (record_trace = 1).  One record per row of every window's batch, in window order
 * then batch-row order:
 *   window      boundary index (0-based)
 *   ell_start   tokens the branch had generated before the window
 *   n_tokens    tokens it generated in the window; they are tokens_out[tokens_offset ..)
 *   running     1: incomplete at the boundary -- still running, or stopped by es_every_step --
 *               (score = its k-th running score, k counting the boundaries it was incomplete
 *               at); 0: completed in the window (score = final)
 *   score       the reward the boundary used (PRM head / PRM model / script), fp32
 * hashes[w]: FNV-1a 64 of the control state after boundary w, over the little-endian bytes of
 *   for each row in batch order: int64 request_id, int32 branch, int32 ell, int32 nblk,
 *                                 int32 table[0..nblk)
 *   int32 n_free, int32 free_stack[0..n_free) (bottom -> top), int64 committed,
 *   int32 n_live, then per live request in ascending id: int64 id, int32 phase, uint32
 *   threshold bits, int32 max_num_pruned, int32 num_completed, int32 num_pruned, int32 npre,
 *   int32 prefix[0..npre).
 * sart_trace_fetch moves everything recorded so far into the caller's HOST buffers and clears
 * it.  *n_rows / *n_tokens / *n_hashes always receive the recorded counts; if any buffer is
 * too small nothing is moved (EFULL).  EINVAL if record_trace is off or a pointer is null.
 */
typedef struct {
  int64_t request_id;
  int32_t branch, window, ell_start, n_tokens, running;
  float score;
  int64_t tokens_offset;
} sart_trace_row;
int sart_trace_fetch(sart_ctx* ctx, sart_trace_row* rows, int64_t rows_cap, int64_t* n_rows, int32_t* tokens_out,
                     int64_t tokens_cap, int64_t* n_tokens, uint64_t* hashes, int64_t hashes_cap, int64_t* n_hashes);

/*
 * Tensor parallelism (tp_size > 1): the symmetric receive buffer of this ctx -- device
 * memory on its GPU that every rank's O / down GEMMs write their partial tiles into, with
 * the arrival counters.  *dev_ptr gets its address (valid in this process); ipc_handle, if
 * not NULL, receives a 64-byte cudaIpcMemHandle_t for it (for peers in other processes).
 * Errors: EINVAL (tp_size <= 1, null dev_ptr).
 */
int sart_tp_buffer(sart_ctx* ctx, void** dev_ptr, void* ipc_handle);
/*
 * Connect the tp_size ranks.  Exactly one of peer_ptrs / ipc_handles is non-NULL:
 *   peer_ptrs[r]    the sart_tp_buffer address of rank r, valid in THIS process (ranks of one
 *                   process, e.g. on one GPU or GPUs with peer access enabled);
 *   ipc_handles     tp_size x 64 bytes: rank r's handle at offset 64 r (entry tp_rank is
 *                   ignored); opened with cudaIpcOpenMemHandle (one process per GPU).
 * Must be called once, after every rank's sart_init and before the first sart_step.
 * Errors: EINVAL, ESTATE (already connected), ECUDA (handle open failed).
 */
int sart_tp_connect(sart_ctx* ctx, void* const* peer_ptrs, const void* ipc_handles);
/* Host-only test hook (no GPU): where rank cfg->tp_rank's copy of tensor `tensor` (host_weights
 * order, FULL dims in cfg) comes from.  out receives *n_out records of 6 int64
 * {local offset, count, cl, cf, c0, global offset}: local element loff + i is full-tensor element
 * goff + (i / cl) * cf + c0 + i % cl.  EFULL if cap records do not suffice (count written). */
int sart_debug_tp_segments(const sart_config* cfg, int32_t tensor, int64_t* out, int32_t cap, int32_t* n_out);

int sart_destroy(sart_ctx* ctx);
const char* sart_strerror(int code);
const char* sart_last_error(void);

/* ------------------------------------------------------------------------
 * Test / measurement hooks.  Not needed by a serving user.
 * ---------------------------------------------------------------------- */

/* Control state after the last boundary (compared bit-exactly with the oracle).
 * All pointers are HOST buffers the caller sizes from the *_cap fields. */
typedef struct {
  int32_t n_rows;
  int64_t* row_request_id; /* [rows_cap] */
  int32_t* row_branch;     /* [rows_cap] */
  int32_t* row_ell;        /* [rows_cap] */
  int32_t* row_nbnd;       /* [rows_cap] */
  int32_t* row_table;      /* [rows_cap][table_cap]: first ceil(min(l+T,cap)/bs) valid */
  int32_t rows_cap, table_cap;
  int32_t n_free;
  int32_t* free_stack;     /* [free_cap] bottom -> top */
  int32_t free_cap;
  int32_t committed;
  int32_t n_live;          /* live (prefilled, unfinalized) requests, ascending id */
  int64_t* live_request_id;/* [live_cap] */
  int32_t* live_phase;
  float* live_threshold;
  int32_t* live_max_pruned;
  int32_t* live_completed;
  int32_t* live_pruned;
  int32_t* live_prefix;    /* [live_cap][prefix_cap] */
  int32_t* live_prefix_n;
  int32_t live_cap, prefix_cap;
} sart_state;
int sart_get_state(sart_ctx* ctx, sart_state* st);

enum {
  SART_DBG_LOGITS = 0, /* fp32 [n][V]  logits of the last decode step            */
  SART_DBG_TOKENS = 1, /* int32 [n]    tokens sampled at the last step            */
  SART_DBG_ROWIDS = 2, /* int64 [n]    request_id << 8 | branch of the step's rows */
  SART_DBG_SCORES = 3, /* fp32 [n]     PRM-head scores of the last boundary        */
  SART_DBG_ATTN = 4,   /* fp32 [n][qh*hd] attention output of `layer`, last step (debug_capture) */
  SART_DBG_Z = 5,      /* fp32 [n][d]  final-norm hidden state of the last step     */
  SART_DBG_PRM_SCORES = 6 /* fp32 [n]  PRM-head score of each row at the last boundary */
};
/* Copy a debug tensor of the most recent step into a HOST buffer; *n_rows gets
 * the number of rows of that step (batch order at the start of the window). */
int sart_debug_fetch(sart_ctx* ctx, int32_t what, int32_t layer, void* host_out,
                     size_t bytes, int32_t* n_rows);

/* Stand-alone run of the tcgen05 GEMM on the current device (unit tests):
 * C[M][N] (+)= A[M][K] . B[N][K]^T (+ bias[N]); A, B bf16 bit patterns, row-major HOST
 * buffers.  mode 0: store, 1: accumulate into C (C is read), 2: SwiGLU on gate/up rows
 * interleaved in 256-row tiles; C receives M x N/2 values (bf16 rounded).
 * splits (1..8): split-K, C receives splits x M x N partial products (caller sums);
 * bn: output tile width 64, 128 or 256 (SwiGLU needs 256 and splits = 1; 64: store only);
 * bm: output tile height 128 or 256 (256: two 128-row tensor-core tiles share each weight
 * stage; store with bn 128/256, SwiGLU with bn 256).  Unsupported combinations: SART_EINVAL. */
int sart_debug_gemm(int32_t M, int32_t N, int32_t K, const uint16_t* A, const uint16_t* B, const float* bias,
                    float* C, int32_t mode, int32_t splits, int32_t bn, int32_t bm);

/* Host-only test hook (no GPU needed): the packing plan of one f2 PRM pass.  Row r (n rows)
 * has ell[r] - ell_ws[r] >= 0 new suffix entries starting at entry ell_ws[r]; they are laid
 * back to back in chunks of <= chunk tokens, rows straddling chunk boundaries in order.
 * out receives int32x4 records [segments | query blocks | gathers] (cap records):
 *   segment {first token in chunk, count, row, first entry};
 *   query block {first token, count <= qp, row, first entry} (inside one segment);
 *   gather {row, token of the row's last entry, 0, 0} (in the chunk where the row ends);
 * chunks receives (tokens, segments, query blocks, gathers) per chunk (chunk_cap chunks).
 * Counts are always written; EFULL when a buffer is too small (nothing else written). */
int sart_debug_prm_plan(const int32_t* ell_ws, const int32_t* ell, int32_t n, int32_t chunk, int32_t qp,
                        int32_t* out, int32_t cap, int32_t* n_seg, int32_t* n_qb, int32_t* n_gat, int32_t* chunks,
                        int32_t chunk_cap, int32_t* n_chunks);

typedef struct {
  double attn_ms;          /* sum of attention-kernel durations (CUDA events)    */
  int64_t attn_launches;
  double attn_bytes;       /* algorithmic KV bytes those launches had to move    */
  int64_t kernel_launches; /* kernels this library launched                      */
  double prefill_ms;       /* host-observed prefill time                         */
  double prm_ms;           /* GPU time of the f2 PRM passes (CUDA events)         */
  int64_t prm_tokens;      /* suffix entries the PRM model read in those passes   */
  int64_t prm_passes;      /* boundaries with a PRM pass                          */
  int64_t h2d_bytes;       /* host->device bytes the serving path copied (prompts, scripts,
                              admission events, prefill token lists, counter exports) */
  int64_t d2h_bytes;       /* device->host bytes it copied (per-window counter records, live
                              polls, finalized records, selected branches' tokens)  */
  double first_step_ms_max; /* profile mode: longest time from a window's start to its first
                              decode step's completion (includes an inline prefill)  */
  double step_ms_max;       /* profile mode: longest single decode step (incl. an interleaved
                              prefill chunk), both over the windows since the last reset */
  int64_t prefix_tc_windows; /* windows whose decode steps ran the tensor-core prefix pass of the
                              cascade attention (a request with >= 64 query rows: N x g) */
  double attn_stream_ms;    /* profile mode 2: the part of attn_ms spent in the streaming kernel(s)
                              (k_attn_cascade, + k_attn_prefix_tc when on), merge excluded */
} sart_profile;
int sart_get_profile(sart_ctx* ctx, sart_profile* out);
/* Turn per-launch attention timing on or off.  While on, decode steps are launched eagerly
 * with CUDA events around each attention launch (enable = 1: around the whole operator, the
 * streaming kernel + merge -> attn_ms; enable = 2: also an event between the streaming kernel
 * and the merge -> attn_stream_ms, which delays the merge's launch); while off, each window's
 * decode step is captured once as a CUDA graph and replayed (the default serving mode). */
int sart_set_profile(sart_ctx* ctx, int32_t enable);
int sart_reset_profile(sart_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif /* SART_H_ */
