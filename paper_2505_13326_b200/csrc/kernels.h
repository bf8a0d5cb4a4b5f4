// Host-callable launchers of the SART device kernels (all on the given stream).
#pragma once
#include "common.cuh"

struct RopeArgs {
  // decode mode (pf_slot == sf_row == nullptr): per-row positions from Rows/Reqs.  Prefill
  // mode: row i of the batch is prompt position pf_pos[i] of request slot pf_slot[i]
  // (batched prefill).  Suffix mode (sf_row != nullptr, the f2 PRM pass): row i of the
  // batch is suffix entry pf_pos[i] of batch row sf_row[i] (-1: padding, no KV written),
  // at position P-1+entry, appended through that row's block table.
  const int* pf_slot;
  const int* pf_pos;
  const int* sf_row = nullptr;
};

// Packed f2 PRM pass: a chunk's tokens are the new suffix entries of its rows back to back.
// Descriptors (int4) built on the host from the rows' entry counts:
//   segment  {first token, count, batch row, first entry}   (k_prm_tokens, one CTA each)
//   qblock   {first token, count <= QP, batch row, first entry}   (suffix attention CTAs)
//   gather   {batch row, token of its last entry, 0, 0}      (k_prm_gather)

// ---- model (k_model.cu)
template <typename T> void launch_init_tensor(T* p, long long n, int tensor_id, int is_norm, float std,
                                              unsigned long long seed, cudaStream_t s);
template <typename T> void launch_embed(const int* tok, const T* emb, float* h, int n, int d, cudaStream_t s);
// h[r] += sum_{s<np} parts[s][r] (fixed order; np may be 0), then out = RMSNorm(h) * g
// tp_cnt / tp_expect (tensor parallelism, may be null): wait until the local arrival counter
// reaches the expected count before reading the partials (they include other ranks' tiles)
template <typename T> void launch_rmsnorm(float* h, const float* parts, int np, const T* g, T* out, float* out32,
                                          const int* status, int n, int d, float eps, cudaStream_t s,
                                          const unsigned long long* tp_cnt = nullptr,
                                          const unsigned long long* tp_expect = nullptr);
// device weight init of a (sliced) tensor: local element i is global element
// goff + (i / cl) * cf + c0 + i % cl of tensor tensor_id (row / column shards of TP ranks)
template <typename T> void launch_init_slice(T* p, long long n, int tensor_id, int is_norm, float std,
                                             unsigned long long seed, long long cl, long long cf, long long c0,
                                             long long goff, cudaStream_t s);
// qkv = sum_{s<np} parts[s] + bias (fixed order), then RoPE + paged KV append
template <typename T> void launch_rope_append(const float* parts, int np, const float* bias, T* qout, T* pool,
                                              const float* rope_cs, Dims D, int layer, Rows rows, Reqs reqs,
                                              RopeArgs a, int n, cudaStream_t s);
template <typename T> void launch_swiglu(const float* gu, T* act, int n, int F, cudaStream_t s);
void launch_prm_head2(const float* hid, const float* w2, const float* b2, float* score, int n, int d,
                      cudaStream_t s);
template <typename T> void launch_convert(const float* in, T* out, long long n, cudaStream_t s);
template <typename T> void launch_to_f32(const T* in, float* out, long long n, cudaStream_t s);

// ---- GEMM (k_gemm.cu): C[m][n] (+)= A[m][k] . B[n][k]^T (+ bias[n]); fp32 accumulate.
enum { GEMM_STORE = 0, GEMM_ACCUM = 1, GEMM_SWIGLU = 2, GEMM_QKV = 3,
       // QKV epilogue on half-head tiles (hd = 128, BN = 64): tile (head, p) holds head dims
       // [32p, 32p + 32) and [64 + 32p, 64 + 32p + 32) -- the rotate-half pairs stay in one tile,
       // so a head is split over 2 CTAs (2x the CTAs of the one-head tiling at small M)
       GEMM_QKV_HALF = 4,
       GEMM_SAMPLE = 5 };   // LM head with the sampler's per-(row, tile) Gumbel argmax in the epilogue
// QKV epilogue: bias, rotate-half RoPE, q -> qout (bf16), k/v -> paged pool (decode: running
// rows only; prefill: prefix positions p0 + row)
struct QkvEpi {
  const float* bias;
  bf16* qout;
  bf16* pool;
  const float* rope_cs;
  Dims D;
  int layer;
  Rows rows;
  Reqs reqs;
  RopeArgs a;
  float* parts;   // split-K partials [S][M][N] (S > 1)
  int* cnt;       // per (head, m-tile, lane quarter) arrival counters, zero between launches
  int cnt_cap;    // entries in cnt (split-K is used only when heads x m-tiles x 4 fits)
  int evict_b;    // weights (B) loaded with an L2 evict-first policy (SART_GEMM_EVICT)
  float* skey;    // GEMM_SAMPLE: best key per (row, slot), nsl slots per row
  int* sv;        //              and its vocab id
  int nsl;
};
// LM head + sampler phase 1 (GEMM_SAMPLE): every running row's best Gumbel key over each
// 128-column half of every 256-wide vocab tile -> skey / sv[row][2 * tile + half]; C (debug
// capture only, else null) also receives the fp32 logits.  Then launch_sample_final(nsl).
bool launch_gemm_sample(const bf16* A, const bf16* B, float* C, int M, int N, int K, const QkvEpi& epi,
                        cudaStream_t s);
int gemm_sample_slots(int V);
void launch_sample_final(Dims D, Rows rows, Reqs reqs, Ctr* ctr, int n, int* dbg_tok, const float* pkey, const int* pv,
                         int nchunk, cudaStream_t s);
// Tensor parallelism (row f4): the split-K partials of an O / down projection are partial sums
// over the tp ranks.  The GEMM epilogue stores partial tile (rank, split) into EVERY rank's
// receive buffer (dst[p] + (rank * S + split) * M * N, remote stores over NVLink), then each CTA
// adds 1 to counter k of every rank (system scope).  The consumer (k_rmsnorm) waits until its
// counter k reaches expect[k], which CTA 0 of the local producer raised by gridDim.x * tp.
constexpr int SART_MAX_TP = 8;
struct TpOut {
  float* dst[SART_MAX_TP];
  unsigned long long* cnt[SART_MAX_TP];   // counter arrays of every rank (index k)
  unsigned long long* expect;             // this rank's expected arrivals (index k)
  int tp, rank, k;
};
template <typename T> void launch_gemm_simt(const T* A, const T* B, const float* bias, float* C, int M, int N,
                                            int K, int mode, cudaStream_t s);

// tcgen05 GEMM (k_gemm_tc.cu), bf16 operands.  GEMM_SWIGLU: B rows interleaved in 256-row
// tiles as [gate 128 | up 128]; writes act[m][N/2] = SiLU(gate) * up as bf16.
// Returns false when the shape is unsupported (caller falls back to nothing: it is an error).
void gemm_ts_reset();
void gemm_ts_fetch(unsigned long long* h);
void gemm_trace_fetch(unsigned long long* h);
bool launch_gemm_tc(const bf16* A, const bf16* B, const float* bias, float* C, bf16* act, int M, int N, int K,
                    int mode, cudaStream_t s, const bf16* Bt = nullptr);
void launch_interleave_gate_up(bf16* w, bf16* tmp, int F, int d, cudaStream_t s);
// split-K variant: S partial products written to C + s*M*N (summed by the consumer kernel)
bool launch_gemm_tc_split(const bf16* A, const bf16* B, const float* bias, float* C, bf16* act, int M, int N, int K,
                          int mode, int S, int BN, int MSUB, cudaStream_t s, const bf16* Bt = nullptr,
                          const TpOut* tp = nullptr);
// CTA-pair (cta_group::2) variant: pair tiles 256 x NP (NP 256 / 512), GEMM_STORE (split-K S) or
// GEMM_SWIGLU (S = 1); returns false for unsupported shapes.  gemm_2sm_mask(): which call sites use it.
bool launch_gemm_2sm(const bf16* A, const bf16* B, const float* bias, float* C, bf16* act, int M, int N, int K,
                     int mode, int S, int NP, cudaStream_t s);
int gemm_2sm_mask();
// pre-tiled weight layout for the tcgen05 GEMM (k_gemm_tc.cu)
size_t tiled_b_elems(int N, int K, int BN);
void launch_tile_b(const bf16* W, bf16* Wt, int N, int K, int BN, cudaStream_t s);
void choose_split(int M, int N, int K, int& S, int& BN, int& MSUB);
// QKV projection with the bias + RoPE + paged KV append fused into the epilogue (tile = 1 head)
bool launch_gemm_qkv(const bf16* A, const bf16* B, int M, int N, int K, const QkvEpi& epi, cudaStream_t s, const bf16* Bt = nullptr);

// ---- attention (k_attn.cu)
template <typename T> void launch_attn_decode_simple(const T* q, const T* pool, T* out, float* dbg, Dims D,
                                                     int layer, Rows rows, Reqs reqs, int n, cudaStream_t s);
// causal attention of a batch of prompt tokens (row i: slot pf_slot[i], position pf_pos[i])
// over their requests' prefix blocks
template <typename T> void launch_attn_prefill(const T* q, const T* pool, T* out, Dims D, int layer, Reqs reqs,
                                               const int* pf_slot, const int* pf_pos, int n, cudaStream_t s);
// f2 PRM pass: causal attention of suffix-entry queries (row i: batch row sf_row[i], entry
// pf_pos[i]) over [prefix ; that row's suffix entries 0..entry]
template <typename T> void launch_attn_suffix(const T* q, const T* pool, T* out, Dims D, int layer, Rows rows,
                                              Reqs reqs, const int* sf_row, const int* sf_ent, int n, cudaStream_t s);

// cascade attention (k_attn_cascade.cu).  Per-window plan of work units.
struct AttnPlan {
  int4* units;      // tasks {type (1 prefix / 0 suffix), group or row, chunk, m-tile}
  int* n_units;
  int* work;        // [L] dynamic work counters (reset by the merge kernel)
  int* grp_slot;    // [R]
  int* grp_n;       // [R]
  int* grp_rows;    // [R][qr_max]
  int* row_pos;     // [R] position of the row inside its prefix group
  int* row_rank;    // [R] scratch of k_attn_plan: rank of the row among its request's rows
  int* row_nreq;    // [R] scratch of k_attn_plan: rows of the row's request
  int* done;        // [L] finished CTAs per layer launch
  int4* items;      // [2 * max tasks] per-step packed items {t0, t1, table base, slot} {type, row|group, mtile, nq}
  int* n_items;     // valid items this step
  // tensor-core prefix pass (k_attn_prefix_tc.cu): groups with >= tcq query rows (<= 128)
  // get type-2 units {2, group, chunk, 0}: one item covers all the group's query rows
  int4* tc_items;   // [2 * max tasks] per-step items of the tensor-core prefix pass (same packing)
  int* n_tc;        // valid tensor-core items this step
  int tcq;          // 0: off
  int* tc_done;     // [L] finished CTAs of the prefix pass per layer launch
  int tc_grid;      // CTAs of this window's prefix pass (0: no pass): the pass runs on tc_grid SMs
                    // CONCURRENTLY with k_attn_cascade (which skips its PDL wait and, in its last
                    // CTA, waits for tc_done == tc_grid, so the merge sees both kernels' partials)
  int qr_grp;       // branch rows per group of the mma.sync prefix tasks (16-row m-tiles)
  int qr_max, CH, npc_max, nslot;   // qr_max: row stride of grp_rows (>= every group size)
  int evict;        // 1: suffix KV streamed with an L2 evict-first policy (SART_ATTN_EVICT)
  int PC;           // suffix piece length (0: off): a row's whole CH-chunks stay items, its last
                    // partial chunk is cut into PC-token pieces so the queue ends with short items
};
void launch_attn_plan(Dims D, Rows rows, Reqs reqs, AttnPlan pl, int n, int flat, cudaStream_t s);
// tensor-core prefix pass of the cascade attention (k_attn_prefix_tc.cu): writes the prefix
// partials of the plan's type-2 items; kv_map from make_kv_map (bf16 pool, hd = 128)
void launch_attn_prefix_tc(const bf16* q, const void* kv_map, float* part_o, float* part_lse, Dims D, int layer,
                           Rows rows, Reqs reqs, AttnPlan pl, cudaStream_t s);
// 3-D tensor map over the paged pool for the prefix pass: {64 elements, HD/64 halves, token
// rows}; map_out must hold 128 bytes.  False if the driver cannot encode it.
bool make_kv_map(void* map_out, const bf16* pool, long long token_rows, int hd, int bs);
// tensor-core (tcgen05) causal prefill, hd = 128 (k_attn_prefix_tc.cu, CAUSAL): blocks[i] =
// {first batch row, rows (<= 128), request slot, first position}; out[row][qh][hd] bf16
void launch_attn_prefill_umma(const bf16* q, const void* kv_map, bf16* out, Dims D, int layer, Reqs reqs,
                              const int4* blocks, int nblocks, cudaStream_t s);
// the same for one f2 PRM chunk: qblocks[i] = {first token, entries (<= 128), row, first entry}
void launch_attn_suffix_umma(const bf16* q, const void* kv_map, bf16* out, Dims D, int layer, Rows rows, Reqs reqs,
                             const int4* qblocks, int nqb, cudaStream_t s);
void launch_attn_items(Dims D, Rows rows, Reqs reqs, AttnPlan pl, cudaStream_t s);
// tensor-core causal prefill: blocks[i] = {first batch row, rows (<= prefill_query_block(D)),
// slot, first position}
void launch_attn_prefill_tc(const bf16* q, const bf16* pool, bf16* out, Dims D, int layer, Reqs reqs,
                            const int4* blocks, int nblocks, cudaStream_t s);
int prefill_query_block(const Dims& D);   // query positions per prefill CTA (16, 32 or 64)
// tensor-core variant for one f2 PRM chunk: 64-entry query blocks of each row's new suffix
// entries over [prefix ; suffix entries 0..entry] (causal)
void launch_attn_suffix_tc(const bf16* q, const bf16* pool, bf16* out, Dims D, int layer, Rows rows, Reqs reqs,
                           const int4* qblocks, int nqb, cudaStream_t s);
extern thread_local cudaEvent_t g_attn_mid_event;   // profile mode: recorded between the streaming kernel and the merge
extern thread_local bool g_attn_skip_merge;   // measurement only (SART_ABLATE): launch the cascade kernel without its merge
void launch_attn_account(Dims D, Rows rows, Reqs reqs, AttnPlan pl, int n, double* acc, cudaStream_t s);
void launch_attn_cascade(const bf16* q, const bf16* pool, bf16* out, float* dbg, float* part_o, float* part_lse,
                         Dims D, int layer, Rows rows, Reqs reqs, AttnPlan pl, int n, cudaStream_t s);

// ---- sampler (k_sample.cu)
void launch_sample(const float* logits, Dims D, Rows rows, Reqs reqs, Ctr* ctr, int n, int* dbg_tok, float* pkey,
                   int* pv, cudaStream_t s);
int sample_chunks(int V);
void launch_step_begin(Ctr* ctr, int es, int wake, Dims D, Rows rows, Reqs reqs, int n, cudaStream_t s);

// ---- control (k_ctl.cu)
// type 0 = prefill (pop the prefix blocks, init meta[i], Alg. 1 L16), 1 = new row (L5)
struct AdmitEvent {
  int type, slot, b, pop_off, row, first_tok;
  int N, M, P, beta, prune, npre, has_script, has_answer, has_forced, nbnd;
  int start;   // new row: window step of its first decode (R44; 1 = immediately)
  float alpha;
  long long id;
};
void launch_admit(const AdmitEvent* ev, int n_ev, int total_pop, int new_rows, int commit_delta, Dims D,
                  Rows rows, Reqs reqs, int* free_stack, Ctr* ctr, cudaStream_t s);
// record_trace (PP2): per window row, the score the boundary used, its status at the end of
// the window (RUNNING, EOS, CAP) and its step count -- before compaction.  All null: off.
struct BoundaryTrace {
  float* score;
  int* state;
  int* ell;
};
void launch_boundary(Dims D, Rows rows, Rows tmp, Reqs reqs, const float* prm_score, int* free_stack,
                     Ctr* ctr, DevResult* res, int* slot_row, int n, BoundaryTrace tr, cudaStream_t s);
void launch_window_begin(Ctr* ctr, int n, cudaStream_t s);
// f2 PRM pass: token list of one chunk from its segments (tok: input token of the entry,
// row: batch row, ent: suffix entry), and the gather of each row's last-entry state
void launch_prm_tokens(Dims D, Rows rows, Reqs reqs, const int4* seg, int nseg, int* tok, int* row, int* ent,
                       cudaStream_t s);
template <typename T> void launch_prm_gather(const T* z, T* zrow, const int4* gat, int ng, int d, cudaStream_t s);
