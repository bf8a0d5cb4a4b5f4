// C-ABI (include/sart.h) and host orchestrator of the SART decode engine.
//
// Host side (this file): the FCFS request_queue and branch_queue of Algorithm 1
// (P:218-219), the fill loop L3-11 with commitment admission (R34), prefill launches
// (L14-20), the window loop (L12, L21-22) and result collection.  Everything
// that touches per-branch state -- sampling, EOS, pruning, early stop, reclamation,
// compaction, voting -- runs in device kernels; the host reads one counter record per
// window.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <map>
#include <set>
#include <string>
#include <type_traits>
#include <vector>

#include "../../include/sart.h"
#include "kernels.h"
#include <cuda_profiler_api.h>

namespace {
thread_local std::string g_last_error;

int set_err(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

int64_t now_ns() {
  return std::chrono::duration_cast<std::chrono::nanoseconds>(
             std::chrono::steady_clock::now().time_since_epoch())
      .count();
}

int cdiv(long long a, long long b) { return (int)((a + b - 1) / b); }

struct HostScript {
  std::vector<int32_t> forced_len, answer, forced_tokens;
  std::vector<float> scores, final_score;
  int n_bnd = 0;
};
struct HostReq {
  int64_t id;
  std::vector<int32_t> prompt;
  int N, M, beta;
  float alpha;
  bool has_script = false;
  HostScript sc;
  int64_t arrival_ns, admit_ns;
};
struct SlotInfo {
  int64_t id = -1;
  int N = 0;
  int64_t arrival_ns = 0, prefill_ns = 0;
  int first_tok = 0;
  bool live = false;
};
struct HostResult {
  sart_result r;
  std::vector<int32_t> tokens;
};
}  // namespace

struct sart_ctx {
  sart_config cfg{};
  Dims D{};
  bool bf16 = true;
  cudaStream_t st = nullptr;
  bool own_stream = false;
  bool poisoned = false;
  alignas(64) unsigned char kv_map[128] = {};   // CUtensorMap of the pool (tensor-core prefix pass)
  bool tc_prefix_window = false;
  bool kv_map_ok = false;   // kv_map describes this ctx's pool (bf16, hd 128)
  bool fused_sample = false;   // GEMM_SAMPLE: LM head + sampler phase 1 (SART_FUSED_SAMPLE)
  bool pf_umma = false;     // causal prefill on tcgen05 (k_attn_prefix_tc<CAUSAL>); SART_PF_UMMA=0: mma.sync
  long long prefix_tc_windows = 0;
  bool gemm_failed = false;
  int W = 0;   // workspace rows
  int ablate = 0;   // SART_ABLATE bit mask (measurement only: skip decode-step kernels, results invalid)
  int PC = 0;  // prefill chunk

  // device memory
  std::vector<void*> allocs;
  void* wblob = nullptr;   // all weight tensors (model dtype)
  std::vector<size_t> woff;  // element offset of each tensor in weight_names order
  float* fparams = nullptr;  // fp32 copies: bqkv per layer, prm_b1, prm_w2, prm_b2
  size_t f_bqkv = 0, f_prm_b1 = 0, f_prm_w2 = 0, f_prm_b2 = 0;
  void* pool = nullptr;
  Rows rows{}, tmp{};
  Reqs reqs{};
  Ctr* ctr = nullptr;
  int* free_stack = nullptr;
  DevResult* res = nullptr;
  int* slot_row = nullptr;
  float *h = nullptr, *parts = nullptr, *gu = nullptr, *z32 = nullptr, *logits = nullptr, *prm_hid = nullptr,
        *prm_score = nullptr, *rope_cs = nullptr, *dbg_attn = nullptr;
  void *a = nullptr, *q = nullptr, *o = nullptr, *act = nullptr, *zT = nullptr;
  int* dbg_tok = nullptr;
  int *dbg_slot = nullptr, *dbg_b = nullptr;
  int* d_prompt = nullptr;     // batched prefill: tokens, request slots, positions
  int *d_pf_slot = nullptr, *d_pf_pos = nullptr;
  int pf_cap = 0;
  int* qkv_cnt = nullptr;   // split-K QKV arrival counters
  int qkv_cnt_cap = 0;
  std::vector<int> pf_tok, pf_slot, pf_pos;
  std::vector<int> pf_slot_h, pf_pos_h;   // host copies used to build the query blocks
  int4* d_pf_blocks = nullptr;
  cudaEvent_t pf_ev[2] = {nullptr, nullptr};
  bool pf_pending = false;
  // R44 (row f1): chunked prefill interleaved with the window's decode steps
  int pf_chunk = 0;            // tokens per interleaved chunk (0: inline prefill)
  int pf_ntok = 0, pf_done = 0;   // this fill's prefill tokens, tokens already processed
  std::vector<int> fill_ready;    // per slot: start step of the rows of a request prefilled in this fill
  std::vector<cudaEvent_t> step_ev;   // profile mode: per-step completion events of a window
  double first_step_ms_max = 0, step_ms_max = 0;
  AdmitEvent* d_events = nullptr;
  int ev_cap = 0;
  AttnPlan plan{};
  float *part_o = nullptr, *part_lse = nullptr;
  float* skey = nullptr;   // sampler per-chunk partial argmax
  int* sv = nullptr;

  // host state
  std::deque<HostReq> request_queue;
  std::deque<std::pair<int, int>> branch_queue;  // (slot, branch)
  std::vector<SlotInfo> slots;
  std::vector<int> free_slots;
  std::set<int64_t> seen_ids;
  std::deque<HostResult> results;
  int n_rows = 0;
  long long free_top = 0, committed = 0;
  int windows = 0, steps = 0, finalized_total = 0;
  long long branch_tokens = 0;
  int last_n = 0;
  Ctr* h_ctr = nullptr;  // pinned
  int* h_live = nullptr; // pinned [2]
  cudaEvent_t poll_ev[2] = {nullptr, nullptr};
  cudaGraphExec_t step_exec = nullptr;
  bool use_graphs = true;
  std::vector<int64_t> last_slot_id;

  // profiling
  std::vector<cudaEvent_t> ev_pool;
  int ev_used = 0;
  double attn_ms = 0, attn_bytes = 0, attn_bytes_base = 0, prefill_ms = 0;
  double attn_stream_ms = 0;   // profile mode: the streaming kernel(s) alone (merge excluded)
  long long attn_launches = 0, launches = 0;
  long long h2d_bytes = 0, d2h_bytes = 0;   // host<->device bytes of the serving path (sart_profile)
  // record_trace (PP2): per-window streams and per-boundary state hashes for oracle replay
  std::vector<sart_trace_row> trace_rows;
  std::vector<int32_t> trace_tokens;
  std::vector<uint64_t> trace_hashes;
  std::vector<int> trace_ell0;   // rows.ell at window start
  BoundaryTrace dtr{nullptr, nullptr, nullptr};
  bool own_pool = true;          // false: caller-owned kv_pool (never freed here)
  // tensor parallelism (row f4): symmetric receive buffer [counters | partials] and the peers'
  int tp = 1, tp_rank = 0;
  void* tp_buf = nullptr;                  // this rank's receive buffer (cudaMalloc base)
  float* tp_parts = nullptr;               // its partial regions: 2 x [tp][S <= 8][W][max(d, qkv)] fp32
  size_t tp_region = 0;                    // floats per region (exchange k uses region k & 1)
  unsigned long long* tp_cnt = nullptr;    // its arrival counters [2 L]
  unsigned long long* tp_expect = nullptr; // expected arrivals [2 L] (local)
  std::vector<void*> tp_peer;              // every rank's buffer base as seen from here
  std::vector<void*> tp_opened;            // IPC mappings to close at destroy
  bool tp_connected = false;
  size_t tp_parts_off = 0;

  // row f2: the separate PRM decoder is a sub-context holding its own dims, weights, KV pool
  // and workspaces; it shares rows / reqs / stream with the policy ctx.
  sart_ctx* prm = nullptr;
  bool is_prm = false;
  int *h_ell_ws = nullptr, *h_ell = nullptr;   // pinned [R]: rows.ell at window start / at the boundary
  int *prm_tok = nullptr, *prm_row = nullptr, *prm_ent = nullptr;   // one PRM chunk's tokens
  int4 *prm_desc = nullptr, *h_prm_desc = nullptr;   // packed-pass descriptors (device / pinned host)
  size_t prm_desc_cap = 0;
  int prm_chunk = 0;                      // tokens per PRM-pass chunk (<= W)
  void* zrow = nullptr;                   // [R][d] final-norm state of each row's last entry
  cudaEvent_t prm_ev[2] = {nullptr, nullptr};
  double prm_ms = 0;
  long long prm_tokens = 0, prm_passes = 0;

  template <typename T> T* W_(int idx) const { return (T*)wblob + woff[idx]; }
};

namespace {
// tensor indices in weight_names order
int t_embed() { return 0; }
int t_layer(int l, int k) { return 1 + 8 * l + k; }  // k: 0 attn_norm 1 wqkv 2 bqkv 3 wo 4 mlp_norm 5 wgate 6 wup 7 wdown
int t_final(const Dims& D) { return 1 + 8 * D.L; }
int t_lm(const Dims& D) { return 2 + 8 * D.L; }
int t_prm_w1(const Dims& D) { return 3 + 8 * D.L; }
int t_prm_b1(const Dims& D) { return 4 + 8 * D.L; }
int t_prm_w2(const Dims& D) { return 5 + 8 * D.L; }
int t_prm_b2(const Dims& D) { return 6 + 8 * D.L; }

std::vector<size_t> tensor_sizes(const Dims& D) {
  std::vector<size_t> s;
  s.push_back((size_t)D.V * D.d);
  for (int l = 0; l < D.L; ++l) {
    s.push_back(D.d);
    s.push_back((size_t)D.qkv * D.d);
    s.push_back(D.qkv);
    s.push_back((size_t)D.d * D.qh * D.hd);
    s.push_back(D.d);
    s.push_back((size_t)D.F * D.d);
    s.push_back((size_t)D.F * D.d);
    s.push_back((size_t)D.d * D.F);
  }
  s.push_back(D.d);
  s.push_back((size_t)D.V * D.d);
  s.push_back((size_t)D.d * D.d);
  s.push_back(D.d);
  s.push_back((size_t)2 * D.d);
  s.push_back(2);
  return s;
}
bool is_norm_tensor(const Dims& D, int idx) {
  if (idx == t_final(D)) return true;
  if (idx >= 1 && idx < 1 + 8 * D.L) {
    int k = (idx - 1) % 8;
    return k == 0 || k == 4;
  }
  return false;
}

#define CK(x)                                                                              \
  do {                                                                                     \
    cudaError_t e_ = (x);                                                                  \
    if (e_ != cudaSuccess) {                                                               \
      ctx->poisoned = true;                                                                \
      return set_err(SART_ECUDA, std::string(#x) + ": " + cudaGetErrorString(e_));        \
    }                                                                                      \
  } while (0)
#define CK_VOID(x)                                                                         \
  do {                                                                                     \
    cudaError_t e_ = (x);                                                                  \
    if (e_ != cudaSuccess) {                                                               \
      ctx->poisoned = true;                                                                \
      set_err(SART_ECUDA, std::string(#x) + ": " + cudaGetErrorString(e_));               \
      return;                                                                              \
    }                                                                                      \
  } while (0)

// Every host<->device copy of the serving path goes through here so that sart_get_profile can
// report the bytes actually moved (bench.py's e2e h2d / d2h per step).
cudaError_t xfer(sart_ctx* ctx, void* dst, const void* src, size_t bytes, cudaMemcpyKind k, cudaStream_t s) {
  if (k == cudaMemcpyHostToDevice) ctx->h2d_bytes += (long long)bytes;
  else if (k == cudaMemcpyDeviceToHost) ctx->d2h_bytes += (long long)bytes;
  return cudaMemcpyAsync(dst, src, bytes, k, s);
}

// Host <-> device operations on the legacy default stream (initialisation uploads) complete
// before anything on the ctx's non-blocking stream may touch the same memory.
inline cudaError_t dsync(cudaError_t e) { return e == cudaSuccess ? cudaDeviceSynchronize() : e; }

template <typename P>
cudaError_t dalloc(sart_ctx* ctx, P** p, size_t bytes, bool zero = true) {
  void* v = nullptr;
  cudaError_t e = cudaMalloc(&v, bytes ? bytes : 16);
  if (e != cudaSuccess) return e;
  ctx->allocs.push_back(v);
  // zeroed on the ctx's own stream and completed before returning: a plain cudaMemset runs on
  // the legacy default stream, which a non-blocking ctx stream does not wait for -- executed
  // late (seen with two processes time-sharing one GPU) it wiped state the ctx's kernels had
  // already written (work counters, TP arrival counters / receive buffers): tests/test_gpu_tp.py
  // two-process IPC, profiles/r2_tp_ipc_flake.txt
  if (zero) {
    if (ctx->st) {
      e = cudaMemsetAsync(v, 0, bytes ? bytes : 16, ctx->st);
      if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->st);
    } else {
      e = cudaMemset(v, 0, bytes ? bytes : 16);
      if (e == cudaSuccess) e = cudaDeviceSynchronize();
    }
  }
  *p = (P*)v;
  return e;
}

cudaError_t alloc_rows(sart_ctx* ctx, Rows& r) {
  const Dims& D = ctx->D;
  cudaError_t e;
  int** ints[] = {&r.slot, &r.b, &r.ell, &r.status, &r.done_step, &r.done_wstep, &r.nbnd, &r.tok, &r.term, &r.nblk,
                  &r.start};
  for (auto p : ints)
    if ((e = dalloc(ctx, p, sizeof(int) * D.R)) != cudaSuccess) return e;
  if ((e = dalloc(ctx, &r.score, sizeof(float) * D.R)) != cudaSuccess) return e;
  return dalloc(ctx, &r.table, sizeof(int) * (size_t)D.R * D.MBR);
}

cudaError_t alloc_reqs(sart_ctx* ctx) {
  const Dims& D = ctx->D;
  Reqs& q = ctx->reqs;
  cudaError_t e;
  size_t S = D.S, S32 = (size_t)D.S * SART_MAXN;
  if ((e = dalloc(ctx, &q.id, sizeof(long long) * S)) != cudaSuccess) return e;
  int** ints[] = {&q.N, &q.M, &q.P, &q.beta, &q.prune, &q.phase, &q.maxp, &q.nc, &q.ncw, &q.np, &q.nes, &q.npre,
                  &q.first_tok, &q.has_script, &q.has_answer, &q.has_forced, &q.nbnd, &q.final_flag};
  for (auto p : ints)
    if ((e = dalloc(ctx, p, sizeof(int) * S)) != cudaSuccess) return e;
  if ((e = dalloc(ctx, &q.alpha, sizeof(float) * S)) != cudaSuccess) return e;
  if ((e = dalloc(ctx, &q.thr, sizeof(float) * S)) != cudaSuccess) return e;
  if ((e = dalloc(ctx, &q.prefix, sizeof(int) * S * D.MPB)) != cudaSuccess) return e;
  int** i32[] = {&q.br_state, &q.br_len, &q.br_label, &q.sc_len, &q.sc_answer};
  for (auto p : i32)
    if ((e = dalloc(ctx, p, sizeof(int) * S32)) != cudaSuccess) return e;
  if ((e = dalloc(ctx, &q.br_score, sizeof(float) * S32)) != cudaSuccess) return e;
  if ((e = dalloc(ctx, &q.sc_final, sizeof(float) * S32)) != cudaSuccess) return e;
  if ((e = dalloc(ctx, &q.sc_scores, sizeof(float) * S32 * D.nbnd_max)) != cudaSuccess) return e;
  if ((e = dalloc(ctx, &q.hist, sizeof(int) * S32 * D.cap)) != cudaSuccess) return e;
  q.forced = nullptr;
  if (ctx->cfg.enable_forced_tokens)
    if ((e = dalloc(ctx, &q.forced, sizeof(int) * S32 * D.cap)) != cudaSuccess) return e;
  return cudaSuccess;
}

// ------------------------------------------------------------------ model step
// bf16: tcgen05 GEMM; fp32 parity mode: SIMT FFMA GEMM (tf32 tensor cores would not hold 1e-5).
template <typename T>
void gemm(sart_ctx* ctx, const T* A, const T* B, const float* bias, float* C, int M, int N, int K, int mode) {
  if constexpr (std::is_same<T, bf16>::value) {
    if (!launch_gemm_tc(A, B, bias, C, nullptr, M, N, K, mode, ctx->st)) ctx->gemm_failed = true;
  } else {
    launch_gemm_simt<T>(A, B, bias, C, M, N, K, mode, ctx->st);
  }
  ctx->launches++;
}

// Projection whose consumer is a reduction kernel (RMSNorm residual add or RoPE): the bf16
// path uses split-K so that small-N projections still cover all SMs; the S partials land in
// ctx->parts and the consumer sums them in split order.  Returns S.
template <typename T>
int proj(sart_ctx* ctx, const T* A, const T* B, int M, int N, int K) {
  int S = 1;
  if constexpr (std::is_same<T, bf16>::value) {
    int BN = 256, MS = 1;
    choose_split(M, N, K, S, BN, MS);
    if ((gemm_2sm_mask() & 2) && K >= 4096 && M > 256 && N % 256 == 0 && BN == 256) {
      // CTA pairs (256 x 256 pair tiles) with the SAME split count, so every split covers the same
      // K-blocks and the partials are bit-identical to the one-SM kernel's.  Only above 256 rows:
      // C2 (M ~ 470) gains 0.2-0.8%, C3 (M ~ 200, one pair-row) loses 1.6% (profiles/r2_gemm_2sm_ab.txt)
      if (!launch_gemm_2sm(A, B, nullptr, ctx->parts, nullptr, M, N, K, GEMM_STORE, S, 256, ctx->st))
        ctx->gemm_failed = true;
    } else if (!launch_gemm_tc_split(A, B, nullptr, ctx->parts, nullptr, M, N, K, GEMM_STORE, S, BN, MS, ctx->st))
      ctx->gemm_failed = true;
  } else {
    launch_gemm_simt<T>(A, B, nullptr, ctx->parts, M, N, K, GEMM_STORE, ctx->st);
  }
  ctx->launches++;
  return S;
}

// Residual partials of an O / down projection as the consuming RMSNorm reads them: this
// rank's split-K partials, or (tensor parallelism) every rank's, with the arrival wait.
struct ResParts {
  const float* parts;
  int np;
  const unsigned long long* cnt;
  const unsigned long long* expect;
};
// proj() for the residual projections; k = the TP exchange index (2 l: O-proj, 2 l + 1: down)
template <typename T>
ResParts proj_res(sart_ctx* ctx, const T* A, const T* B, int M, int N, int K, int k) {
  if constexpr (std::is_same<T, bf16>::value) {
    if (ctx->tp > 1) {
      int S = 1, BN = 256, MS = 1;
      choose_split(M, N, K, S, BN, MS);
      TpOut t{};
      t.tp = ctx->tp;
      t.rank = ctx->tp_rank;
      t.k = k;
      t.expect = ctx->tp_expect;
      // two receive regions, alternating by exchange: a rank runs at most one exchange ahead of
      // a peer, so it never overwrites tiles the peer's consumer may still be reading
      const size_t roff = (size_t)(k & 1) * ctx->tp_region;
      for (int p = 0; p < ctx->tp; ++p) {
        t.dst[p] = (float*)((char*)ctx->tp_peer[p] + ctx->tp_parts_off) + roff;
        t.cnt[p] = (unsigned long long*)ctx->tp_peer[p];
      }
      if (!launch_gemm_tc_split(A, B, nullptr, ctx->tp_parts + roff, nullptr, M, N, K, GEMM_STORE, S, BN, MS,
                                ctx->st, nullptr, &t))
        ctx->gemm_failed = true;
      ctx->launches++;
      return ResParts{ctx->tp_parts + roff, S * ctx->tp, ctx->tp_cnt + k, ctx->tp_expect + k};
    }
  }
  return ResParts{ctx->parts, proj<T>(ctx, A, B, M, N, K), nullptr, nullptr};
}
template <typename T>
void norm(sart_ctx* ctx, const ResParts& rp, const T* g, T* out, float* out32, const int* status, int n) {
  launch_rmsnorm<T>(ctx->h, rp.parts, rp.np, g, out, out32, status, n, ctx->D.d, ctx->D.eps, ctx->st, rp.cnt,
                    rp.expect);
}

// QKV projection + bias + RoPE + paged KV append: one fused tcgen05 launch in bf16 (tile =
// one head); fp32 mode: SIMT GEMM into the partial buffer + the RoPE/append kernel.
template <typename T>
void qkv_rope(sart_ctx* ctx, int l, int n, RopeArgs ra) {
  const Dims& D = ctx->D;
  const float* bias = ctx->fparams + ctx->f_bqkv + (size_t)l * D.qkv;
  // long-K QKV (14B / 70B, K >= 4096) at small M: the fused kernel has one CTA per (head,
  // m-tile) -- 80 CTAs on 148 SMs for 70B at M <= 128 -- and streams the weights at half the
  // HBM rate, so it runs as a wave-split GEMM + the RoPE / append kernel instead
  bool fused = true;
  if constexpr (std::is_same<T, bf16>::value) {
    const int nsm = device_sms();
    fused = !(D.d >= 4096 && (D.qkv / D.hd) * ((n + 127) / 128) < nsm * 3 / 4);
  }
  if (!fused) {
    int np = proj<T>(ctx, (T*)ctx->a, ctx->W_<T>(t_layer(l, 1)), n, D.qkv, D.d);
    launch_rope_append<T>(ctx->parts, np, bias, (T*)ctx->q, (T*)ctx->pool, ctx->rope_cs, D, l, ctx->rows, ctx->reqs,
                          ra, n, ctx->st);
    ctx->launches++;
    return;
  }
  if constexpr (std::is_same<T, bf16>::value) {
    QkvEpi e{bias,       (bf16*)ctx->q, (bf16*)ctx->pool, ctx->rope_cs, D,           l,
             ctx->rows, ctx->reqs,    ra,               ctx->parts,    ctx->qkv_cnt, ctx->qkv_cnt_cap};
    if (!launch_gemm_qkv((bf16*)ctx->a, ctx->W_<bf16>(t_layer(l, 1)), n, D.qkv, D.d, e, ctx->st))
      ctx->gemm_failed = true;
    ctx->launches++;
  } else {
    int np = proj<T>(ctx, (T*)ctx->a, ctx->W_<T>(t_layer(l, 1)), n, D.qkv, D.d);
    launch_rope_append<T>(ctx->parts, np, bias, (T*)ctx->q, (T*)ctx->pool, ctx->rope_cs, D, l, ctx->rows, ctx->reqs,
                          ra, n, ctx->st);
    ctx->launches++;
  }
}

// MLP up-projection + SwiGLU: fused tcgen05 epilogue on gate/up-interleaved weights (bf16),
// or GEMM + elementwise kernel (fp32 mode).
template <typename T>
void mlp_up(sart_ctx* ctx, int l, int n) {
  const Dims& D = ctx->D;
  if constexpr (std::is_same<T, bf16>::value) {
    if (!launch_gemm_tc((bf16*)ctx->a, ctx->W_<bf16>(t_layer(l, 5)), nullptr, nullptr, (bf16*)ctx->act, n, 2 * D.F,
                        D.d, GEMM_SWIGLU, ctx->st))
      ctx->gemm_failed = true;
    ctx->launches++;
  } else {
    gemm<T>(ctx, (T*)ctx->a, ctx->W_<T>(t_layer(l, 5)), nullptr, ctx->gu, n, 2 * D.F, D.d, GEMM_STORE);
    launch_swiglu<T>(ctx->gu, (T*)ctx->act, n, D.F, ctx->st);
    ctx->launches++;
  }
}

template <typename T>
void layer_attention(sart_ctx* ctx, int l, int n) {
  const Dims& D = ctx->D;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  // profile mode: events before the attention, between the streaming kernel and the merge
  // (g_attn_mid_event, recorded by launch_attn_cascade) and after the merge
  if (ctx->cfg.profile && ctx->ev_used + 3 <= (int)ctx->ev_pool.size()) {
    e0 = ctx->ev_pool[ctx->ev_used++];
    cudaEvent_t em = ctx->ev_pool[ctx->ev_used++];
    if (ctx->cfg.profile == 2) g_attn_mid_event = em;   // (the mid event delays the merge's launch)
    e1 = ctx->ev_pool[ctx->ev_used++];
    cudaEventRecord(e0, ctx->st);
  }
  float* dbg = ctx->dbg_attn ? ctx->dbg_attn + (size_t)l * D.R * D.qh * D.hd : nullptr;
  if constexpr (std::is_same<T, bf16>::value) {
    if (ctx->tc_prefix_window) {   // tensor-core prefix pass: partials of the type-2 items
      launch_attn_prefix_tc((bf16*)ctx->q, ctx->kv_map, ctx->part_o, ctx->part_lse, D, l, ctx->rows, ctx->reqs,
                            ctx->plan, ctx->st);
      ctx->launches++;
    }
    launch_attn_cascade((bf16*)ctx->q, (bf16*)ctx->pool, (bf16*)ctx->o, dbg, ctx->part_o, ctx->part_lse, D, l,
                        ctx->rows, ctx->reqs, ctx->plan, n, ctx->st);
    ctx->launches += 2;
  } else {
    launch_attn_decode_simple<T>((T*)ctx->q, (T*)ctx->pool, (T*)ctx->o, dbg, D, l, ctx->rows, ctx->reqs, n, ctx->st);
    ctx->launches++;
  }
  ctx->attn_launches++;
  if (e1) cudaEventRecord(e1, ctx->st);
  g_attn_mid_event = nullptr;
}

// SART_ABLATE bits (measurement only, tools/ablate_c2.py): the in-graph marginal cost of a
// kernel class is the step time with it minus without it.  Results are meaningless when set.
enum { AB_RMSNORM = 1, AB_QKV = 2, AB_ATTN = 4, AB_MERGE = 8, AB_OPROJ = 16, AB_GATEUP = 32, AB_DOWN = 64,
       AB_HEAD = 128, AB_SAMPLE = 256 };

template <typename T>
void decode_step(sart_ctx* ctx, int n) {
  const Dims& D = ctx->D;
  cudaStream_t s = ctx->st;
  const int ab = ctx->ablate;
  launch_step_begin(ctx->ctr, ctx->cfg.es_every_step, ctx->pf_chunk > 0, D, ctx->rows, ctx->reqs, n, s);
  launch_embed<T>(ctx->rows.tok, ctx->W_<T>(t_embed()), ctx->h, n, D.d, s);
  ctx->launches += 2;
  if (ctx->cfg.profile) {
    launch_attn_account(D, ctx->rows, ctx->reqs, ctx->plan, n, &ctx->ctr->attn_bytes, s);
    ctx->launches++;
  }
  if constexpr (std::is_same<T, bf16>::value) {   // this step's attention items (all layers)
    launch_attn_items(D, ctx->rows, ctx->reqs, ctx->plan, s);
    ctx->launches++;
  }
  g_attn_skip_merge = (ab & AB_MERGE) != 0;
  ResParts res{ctx->parts, 0, nullptr, nullptr};   // pending residual partials (previous layer's down)
  for (int l = 0; l < D.L; ++l) {
    if (!(ab & AB_RMSNORM)) norm<T>(ctx, res, ctx->W_<T>(t_layer(l, 0)), (T*)ctx->a, nullptr, nullptr, n);
    if (!(ab & AB_QKV)) qkv_rope<T>(ctx, l, n, RopeArgs{nullptr, nullptr});
    if (!(ab & AB_ATTN)) layer_attention<T>(ctx, l, n);
    ResParts ro{ctx->parts, 0, nullptr, nullptr};
    if (!(ab & AB_OPROJ)) ro = proj_res<T>(ctx, (T*)ctx->o, ctx->W_<T>(t_layer(l, 3)), n, D.d, D.qh * D.hd, 2 * l);
    if (!(ab & AB_RMSNORM)) norm<T>(ctx, ro, ctx->W_<T>(t_layer(l, 4)), (T*)ctx->a, nullptr, nullptr, n);
    if (!(ab & AB_GATEUP)) mlp_up<T>(ctx, l, n);
    res = ResParts{ctx->parts, 0, nullptr, nullptr};
    if (!(ab & AB_DOWN)) res = proj_res<T>(ctx, (T*)ctx->act, ctx->W_<T>(t_layer(l, 7)), n, D.d, D.F, 2 * l + 1);
    ctx->launches += 1;
  }
  norm<T>(ctx, res, ctx->W_<T>(t_final(D)), (T*)ctx->zT, ctx->z32, ctx->rows.status, n);
  if constexpr (std::is_same<T, bf16>::value) {
    if (ctx->fused_sample && !(ab & (AB_HEAD | AB_SAMPLE))) {   // LM head + sampler phase 1 in one kernel
      QkvEpi e{};
      e.D = D;
      e.rows = ctx->rows;
      e.reqs = ctx->reqs;
      e.skey = ctx->skey;
      e.sv = ctx->sv;
      e.nsl = gemm_sample_slots(D.V);
      if (!launch_gemm_sample((bf16*)ctx->zT, ctx->W_<bf16>(t_lm(D)), ctx->cfg.debug_capture ? ctx->logits : nullptr, n,
                              D.V, D.d, e, s))
        ctx->gemm_failed = true;
      launch_sample_final(D, ctx->rows, ctx->reqs, ctx->ctr, n, ctx->dbg_tok, ctx->skey, ctx->sv, e.nsl, s);
      ctx->launches += 2;
      g_attn_skip_merge = false;
      return;
    }
  }
  if (!(ab & AB_HEAD)) gemm<T>(ctx, (T*)ctx->zT, ctx->W_<T>(t_lm(D)), nullptr, ctx->logits, n, D.V, D.d, GEMM_STORE);
  if (!(ab & AB_SAMPLE))
    launch_sample(ctx->logits, D, ctx->rows, ctx->reqs, ctx->ctr, n, ctx->dbg_tok, ctx->skey, ctx->sv, s);
  ctx->launches += 2;
  g_attn_skip_merge = false;
}

// Batched prefill (Alg. 1 L15): the prompts of every request admitted in this fill
// loop are processed together, token i being position pf_pos[i] of request slot pf_slot[i];
// chunks of up to PC tokens run all layers (a later chunk's tokens attend to the KV that
// earlier chunks wrote).  The last layer only needs its K/V (the prefix has no output).
//
// ctx is the decoder being prefilled (the policy, or the f2 PRM model into its own pool);
// src holds the batch's token lists (always the policy ctx).
template <typename T>
void prefill_batch(sart_ctx* ctx, sart_ctx* src, int t_begin, int t_end) {
  const Dims& D = ctx->D;
  cudaStream_t s = ctx->st;
  for (int t0 = t_begin; t0 < t_end; t0 += ctx->PC) {
    const int c = std::min(ctx->PC, t_end - t0);
    const RopeArgs ra{src->d_pf_slot + t0, src->d_pf_pos + t0};
    // query blocks of each request segment of this chunk (tensor-core prefill): 128 positions
    // (tcgen05, one TMEM lane each; largest key range first for the static CTA assignment) or
    // 16-64 (mma.sync)
    int nqb = 0;
    if constexpr (std::is_same<T, bf16>::value) {
      std::vector<int4> qb;
      const int QP = ctx->pf_umma ? 128 : prefill_query_block(D);
      for (int i = 0; i < c;) {
        const int slot = src->pf_slot_h[t0 + i];
        int j = i;
        while (j < c && src->pf_slot_h[t0 + j] == slot && j - i < QP) ++j;
        qb.push_back(make_int4(i, j - i, slot, src->pf_pos_h[t0 + i]));
        i = j;
      }
      if (ctx->pf_umma)
        std::stable_sort(qb.begin(), qb.end(), [](const int4& a, const int4& b) { return a.w + a.y > b.w + b.y; });
      nqb = (int)qb.size();
      xfer(src, src->d_pf_blocks, qb.data(), sizeof(int4) * qb.size(), cudaMemcpyHostToDevice, s);
    }
    launch_embed<T>(src->d_prompt + t0, ctx->W_<T>(t_embed()), ctx->h, c, D.d, s);
    ctx->launches++;
    ResParts res{ctx->parts, 0, nullptr, nullptr};
    for (int l = 0; l < D.L; ++l) {
      norm<T>(ctx, res, ctx->W_<T>(t_layer(l, 0)), (T*)ctx->a, nullptr, nullptr, c);
      qkv_rope<T>(ctx, l, c, ra);
      if (l == D.L - 1) break;
      if constexpr (std::is_same<T, bf16>::value) {
        if (ctx->pf_umma)
          launch_attn_prefill_umma((bf16*)ctx->q, ctx->kv_map, (bf16*)ctx->o, D, l, ctx->reqs, src->d_pf_blocks, nqb, s);
        else
          launch_attn_prefill_tc((bf16*)ctx->q, (bf16*)ctx->pool, (bf16*)ctx->o, D, l, ctx->reqs, src->d_pf_blocks,
                                 nqb, s);
      }
      else
        launch_attn_prefill<T>((T*)ctx->q, (T*)ctx->pool, (T*)ctx->o, D, l, ctx->reqs, ra.pf_slot, ra.pf_pos, c, s);
      const ResParts ro = proj_res<T>(ctx, (T*)ctx->o, ctx->W_<T>(t_layer(l, 3)), c, D.d, D.qh * D.hd, 2 * l);
      norm<T>(ctx, ro, ctx->W_<T>(t_layer(l, 4)), (T*)ctx->a, nullptr, nullptr, c);
      mlp_up<T>(ctx, l, c);
      res = proj_res<T>(ctx, (T*)ctx->act, ctx->W_<T>(t_layer(l, 7)), c, D.d, D.F, 2 * l + 1);
      ctx->launches += 3;
    }
  }
}

// Packing plan of one f2 PRM pass (host only; also exported as sart_debug_prm_plan): row r
// has ell[r] - ell_ws[r] new suffix entries starting at entry ell_ws[r]; they are laid back
// to back in chunks of <= Wc tokens (a row that does not fit continues in the next chunk).
// Per chunk: segments {first token, count, row, first entry}, query blocks of <= QP entries
// inside a segment {first token, count, row, first entry}, and gathers {row, token of its
// last entry} for the rows that end in the chunk.
struct PrmPlan {
  struct Chunk { int ntok, seg, nseg, qb, nqb, gat, ngat; };
  std::vector<Chunk> chunks;
  std::vector<int4> seg, qb, gat;
  long long entries = 0;
};
PrmPlan plan_prm_pass(const int* ell_ws, const int* ell, int n, int Wc, int QP) {
  PrmPlan P;
  int fill = 0;
  PrmPlan::Chunk cur{0, 0, 0, 0, 0, 0, 0};
  auto close_chunk = [&]() {
    if (cur.ntok == 0) return;
    P.chunks.push_back(cur);
    cur = PrmPlan::Chunk{0, (int)P.seg.size(), 0, (int)P.qb.size(), 0, (int)P.gat.size(), 0};
    fill = 0;
  };
  for (int r = 0; r < n; ++r) {
    const int cnt = ell[r] - ell_ws[r];
    P.entries += std::max(0, cnt);
    for (int j = 0; j < cnt;) {
      const int take = std::min(cnt - j, Wc - fill);
      const int e0 = ell_ws[r] + j;
      P.seg.push_back(make_int4(fill, take, r, e0));
      cur.nseg++;
      for (int k = 0; k < take; k += QP) {
        P.qb.push_back(make_int4(fill + k, std::min(QP, take - k), r, e0 + k));
        cur.nqb++;
      }
      if (j + take == cnt) {
        P.gat.push_back(make_int4(r, fill + take - 1, 0, 0));
        cur.ngat++;
      }
      fill += take;
      cur.ntok = fill;
      j += take;
      if (fill == Wc) close_chunk();
    }
  }
  close_chunk();
  return P;
}

// Row f2: the separate PRM decoder reads every row's suffix entries decoded in this window
// (entries ell_ws .. ell-1, reading R42) through its own paged KV -- the prefix was
// prefilled at admission -- and its head scores the last entry's final-norm state.  The
// host reads the rows' entry counts and packs the entries back to back into chunks of at
// most prm_chunk tokens (a row longer than the room left continues in the next chunk,
// processed in order, so its later entries attend to the KV its earlier ones appended):
// no padding, exact GEMM sizes.  Descriptors for every chunk go up in one copy.
template <typename T>
void prm_model_scores(sart_ctx* ctx, int n) {
  sart_ctx* m = ctx->prm;
  const Dims& D = m->D;
  cudaStream_t s = ctx->st;
  // SART_NCU_PRM_PASS=k: bracket the k-th pass (1-based) with cudaProfilerStart/Stop so
  // that `ncu --profile-from-start off` captures exactly one PRM pass
  static const int ncu_pass = getenv("SART_NCU_PRM_PASS") ? atoi(getenv("SART_NCU_PRM_PASS")) : 0;
  const bool ncu_range = ncu_pass > 0 && ctx->prm_passes + 1 == ncu_pass;
  CK_VOID(xfer(ctx, m->h_ell, ctx->rows.ell, sizeof(int) * n, cudaMemcpyDeviceToHost, s));
  CK_VOID(cudaStreamSynchronize(s));
  if (ncu_range) cudaProfilerStart();
  CK_VOID(cudaEventRecord(m->prm_ev[0], s));
  const PrmPlan pl = plan_prm_pass(m->h_ell_ws, m->h_ell, n, m->prm_chunk, m->pf_umma ? 128 : prefill_query_block(D));
  const std::vector<int4>&seg = pl.seg, &qb = pl.qb, &gat = pl.gat;
  const std::vector<PrmPlan::Chunk>& chunks = pl.chunks;
  const long long entries = pl.entries;
  // one upload: [all segments | all q-blocks | all gathers]
  const size_t nd = seg.size() + qb.size() + gat.size();
  if (nd > m->prm_desc_cap) {
    ctx->poisoned = true;
    set_err(SART_ECUDA, "PRM-pass descriptor buffer too small");
    return;
  }
  std::copy(seg.begin(), seg.end(), m->h_prm_desc);
  std::copy(qb.begin(), qb.end(), m->h_prm_desc + seg.size());
  std::copy(gat.begin(), gat.end(), m->h_prm_desc + seg.size() + qb.size());
  if (nd) CK_VOID(xfer(ctx, m->prm_desc, m->h_prm_desc, sizeof(int4) * nd, cudaMemcpyHostToDevice, s));
  const int4* dseg = m->prm_desc;
  const int4* dqb = m->prm_desc + seg.size();
  const int4* dgat = m->prm_desc + seg.size() + qb.size();
  for (const PrmPlan::Chunk& c : chunks) {
    const int nt = c.ntok;
    const RopeArgs ra{nullptr, m->prm_ent, m->prm_row};
    launch_prm_tokens(D, m->rows, m->reqs, dseg + c.seg, c.nseg, m->prm_tok, m->prm_row, m->prm_ent, s);
    launch_embed<T>(m->prm_tok, m->W_<T>(t_embed()), m->h, nt, D.d, s);
    m->launches += 2;
    int np_res = 0;
    for (int l = 0; l < D.L; ++l) {
      launch_rmsnorm<T>(m->h, m->parts, np_res, m->W_<T>(t_layer(l, 0)), (T*)m->a, nullptr, nullptr, nt, D.d, D.eps,
                        s);
      qkv_rope<T>(m, l, nt, ra);
      if constexpr (std::is_same<T, bf16>::value) {
        if (m->pf_umma)
          launch_attn_suffix_umma((bf16*)m->q, m->kv_map, (bf16*)m->o, D, l, m->rows, m->reqs, dqb + c.qb, c.nqb, s);
        else
          launch_attn_suffix_tc((bf16*)m->q, (bf16*)m->pool, (bf16*)m->o, D, l, m->rows, m->reqs, dqb + c.qb, c.nqb,
                                s);
      }
      else
        launch_attn_suffix<T>((T*)m->q, (T*)m->pool, (T*)m->o, D, l, m->rows, m->reqs, m->prm_row, m->prm_ent, nt, s);
      int np = proj<T>(m, (T*)m->o, m->W_<T>(t_layer(l, 3)), nt, D.d, D.qh * D.hd);
      launch_rmsnorm<T>(m->h, m->parts, np, m->W_<T>(t_layer(l, 4)), (T*)m->a, nullptr, nullptr, nt, D.d, D.eps, s);
      mlp_up<T>(m, l, nt);
      np_res = proj<T>(m, (T*)m->act, m->W_<T>(t_layer(l, 7)), nt, D.d, D.F);
      m->launches += 3;
    }
    launch_rmsnorm<T>(m->h, m->parts, np_res, m->W_<T>(t_final(D)), (T*)m->a, nullptr, nullptr, nt, D.d, D.eps, s);
    launch_prm_gather<T>((T*)m->a, (T*)m->zrow, dgat + c.gat, c.ngat, D.d, s);
    m->launches += 2;
  }
  gemm<T>(m, (T*)m->zrow, m->W_<T>(t_prm_w1(D)), m->fparams + m->f_prm_b1, m->prm_hid, n, D.d, D.d, GEMM_STORE);
  launch_prm_head2(m->prm_hid, m->fparams + m->f_prm_w2, m->fparams + m->f_prm_b2, m->prm_score, n, D.d, s);
  m->launches++;
  CK_VOID(cudaEventRecord(m->prm_ev[1], s));
  if (ncu_range) cudaProfilerStop();
  ctx->launches += m->launches;
  m->launches = 0;
  ctx->prm_tokens += entries;
  if (m->gemm_failed) ctx->gemm_failed = true;
}

template <typename T>
void prm_scores(sart_ctx* ctx, int n) {
  const Dims& D = ctx->D;
  gemm<T>(ctx, (T*)ctx->zT, ctx->W_<T>(t_prm_w1(D)), ctx->fparams + ctx->f_prm_b1, ctx->prm_hid, n, D.d, D.d,
          GEMM_STORE);
  launch_prm_head2(ctx->prm_hid, ctx->fparams + ctx->f_prm_w2, ctx->fparams + ctx->f_prm_b2, ctx->prm_score, n,
                   D.d, ctx->st);
  ctx->launches++;
}

// ------------------------------------------------------------------ admission (fill loop)
int flush_events(sart_ctx* ctx, std::vector<AdmitEvent>& ev, int& pop_off, int& new_rows, int& commit_delta) {
  if (ev.empty()) return SART_OK;
  if ((int)ev.size() > ctx->ev_cap) return set_err(SART_EINVAL, "too many admission events");
  CK(xfer(ctx, ctx->d_events, ev.data(), sizeof(AdmitEvent) * ev.size(), cudaMemcpyHostToDevice, ctx->st));
  launch_admit(ctx->d_events, (int)ev.size(), pop_off, new_rows, commit_delta, ctx->D, ctx->rows, ctx->reqs,
               ctx->free_stack, ctx->ctr, ctx->st);
  ctx->launches++;
  CK(cudaGetLastError());
  ctx->free_top -= pop_off;
  ctx->n_rows += new_rows;
  ev.clear();
  pop_off = new_rows = commit_delta = 0;
  return SART_OK;
}

int upload_request(sart_ctx* ctx, const HostReq& q, int slot) {
  const Dims& D = ctx->D;
  cudaStream_t s = ctx->st;
  size_t sb = (size_t)slot * SART_MAXN;
  if (!q.sc.forced_len.empty()) {
    CK(xfer(ctx, ctx->reqs.sc_len + sb, q.sc.forced_len.data(), sizeof(int) * q.N, cudaMemcpyHostToDevice, s));
  } else {
    std::vector<int> z(q.N, 0);
    CK(xfer(ctx, ctx->reqs.sc_len + sb, z.data(), sizeof(int) * q.N, cudaMemcpyHostToDevice, s));
  }
  if (q.has_script) {
    CK(xfer(ctx, ctx->reqs.sc_final + sb, q.sc.final_score.data(), sizeof(float) * q.N,
                       cudaMemcpyHostToDevice, s));
    int nb = std::min(q.sc.n_bnd, D.nbnd_max);
    ctx->h2d_bytes += (long long)sizeof(float) * nb * q.N;
    CK(cudaMemcpy2DAsync(ctx->reqs.sc_scores + sb * D.nbnd_max, sizeof(float) * D.nbnd_max, q.sc.scores.data(),
                         sizeof(float) * q.sc.n_bnd, sizeof(float) * nb, q.N, cudaMemcpyHostToDevice, s));
  }
  if (!q.sc.answer.empty())
    CK(xfer(ctx, ctx->reqs.sc_answer + sb, q.sc.answer.data(), sizeof(int) * q.N, cudaMemcpyHostToDevice, s));
  if (!q.sc.forced_tokens.empty())
    CK(xfer(ctx, ctx->reqs.forced + sb * D.cap, q.sc.forced_tokens.data(), sizeof(int) * (size_t)q.N * D.cap,
                       cudaMemcpyHostToDevice, s));
  return SART_OK;
}

// Prefill tokens [pf_done, upto) of this fill's batch (policy, then the f2 PRM model's cache).
int run_prefill(sart_ctx* ctx, int upto) {
  upto = std::min(upto, ctx->pf_ntok);
  if (upto <= ctx->pf_done) return SART_OK;
  if (ctx->bf16) prefill_batch<bf16>(ctx, ctx, ctx->pf_done, upto);
  else prefill_batch<float>(ctx, ctx, ctx->pf_done, upto);
  if (ctx->prm) {   // f2: the PRM model's own prefix KV (same block ids)
    if (ctx->bf16) prefill_batch<bf16>(ctx->prm, ctx, ctx->pf_done, upto);
    else prefill_batch<float>(ctx->prm, ctx, ctx->pf_done, upto);
    ctx->launches += ctx->prm->launches;
    ctx->prm->launches = 0;
    if (ctx->prm->gemm_failed) return set_err(SART_EINVAL, "GEMM shape unsupported by the tcgen05 kernel (PRM model)");
  }
  ctx->pf_done = upto;
  CK(cudaGetLastError());
  return SART_OK;
}

int fill(sart_ctx* ctx) {
  const Dims& D = ctx->D;
  const int RC = cdiv(D.cap, D.bs);
  const int nfirst = cdiv(std::min(D.T, D.cap), D.bs);
  std::vector<AdmitEvent> ev;
  int pop_off = 0, new_rows = 0, commit_delta = 0;
  std::fill(ctx->fill_ready.begin(), ctx->fill_ready.end(), 1);
  while (ctx->n_rows + new_rows < ctx->cfg.max_rows) {  // L3
    if (!ctx->branch_queue.empty()) {                   // L4-5
      auto [slot, b] = ctx->branch_queue.front();
      if (ctx->committed + RC > D.NB) break;            // R34: no skipping
      ctx->branch_queue.pop_front();
      ctx->committed += RC;
      commit_delta += RC;
      AdmitEvent e{};
      e.type = 1;
      e.slot = slot;
      e.b = b;
      e.pop_off = pop_off;
      e.row = ctx->n_rows + new_rows;
      e.first_tok = ctx->slots[slot].first_tok;   // prompt[P-1] (R22)
      e.start = ctx->fill_ready[slot];            // R44: 1 unless its prefix is prefilled in this window
      ev.push_back(e);
      pop_off += nfirst;
      new_rows++;
    } else if (!ctx->request_queue.empty()) {           // L6-7
      HostReq& q = ctx->request_queue.front();
      const int P = (int)q.prompt.size();
      const int npre = cdiv(P - 1, D.bs);
      if (ctx->committed + npre + RC > D.NB) break;
      if (ctx->free_slots.empty()) break;               // slot table full (max_requests)
      const int slot = ctx->free_slots.back();
      ctx->free_slots.pop_back();
      ctx->committed += npre;
      commit_delta += npre;
      AdmitEvent e{};
      e.type = 0;
      e.slot = slot;
      e.pop_off = pop_off;
      e.first_tok = q.prompt[P - 1];
      e.N = q.N;
      e.M = q.M;
      e.P = P;
      e.beta = q.beta;
      e.prune = q.alpha >= 0.f ? 1 : 0;
      e.npre = npre;
      e.has_script = q.has_script ? 1 : 0;
      e.has_answer = q.sc.answer.empty() ? 0 : 1;
      e.has_forced = q.sc.forced_tokens.empty() ? 0 : 1;
      e.nbnd = q.has_script ? std::min(q.sc.n_bnd, D.nbnd_max) : 0;
      e.alpha = q.alpha;
      e.id = q.id;
      ev.push_back(e);
      pop_off += npre;
      int rc = upload_request(ctx, q, slot);
      if (rc) return rc;
      // L15: the prompt joins this fill's prefill batch (prefix = prompt[0:P-1], R22)
      for (int p = 0; p + 1 < P; ++p) {
        ctx->pf_tok.push_back(q.prompt[p]);
        ctx->pf_slot.push_back(slot);
        ctx->pf_pos.push_back(p);
      }
      if (ctx->pf_chunk > 0 && P > 1)   // R44: its rows start at the step whose chunk completes the prefix
        ctx->fill_ready[slot] = std::min(((int)ctx->pf_tok.size() - 1) / ctx->pf_chunk + 1, D.T);
      SlotInfo& si = ctx->slots[slot];
      si.id = q.id;
      si.N = q.N;
      si.arrival_ns = q.arrival_ns;
      si.prefill_ns = now_ns();
      si.first_tok = q.prompt[P - 1];
      si.live = true;
      ctx->last_slot_id[slot] = q.id;
      for (int j = 0; j < q.N; ++j) ctx->branch_queue.emplace_back(slot, j);  // L17-19
      ctx->request_queue.pop_front();
    } else {
      break;  // L8-9
    }
  }
  int rc = flush_events(ctx, ev, pop_off, new_rows, commit_delta);   // all pops, in event order
  if (rc) return rc;
  const int ntok = (int)ctx->pf_tok.size();
  if (ntok > 0) {
    if (ntok > ctx->pf_cap) return set_err(SART_EINVAL, "prefill batch exceeds its buffer");
    CK(xfer(ctx, ctx->d_prompt, ctx->pf_tok.data(), 4 * (size_t)ntok, cudaMemcpyHostToDevice, ctx->st));
    CK(xfer(ctx, ctx->d_pf_slot, ctx->pf_slot.data(), 4 * (size_t)ntok, cudaMemcpyHostToDevice, ctx->st));
    CK(xfer(ctx, ctx->d_pf_pos, ctx->pf_pos.data(), 4 * (size_t)ntok, cudaMemcpyHostToDevice, ctx->st));
    ctx->pf_slot_h.swap(ctx->pf_slot);
    ctx->pf_pos_h.swap(ctx->pf_pos);
    ctx->pf_tok.clear();
    ctx->pf_slot.clear();
    ctx->pf_pos.clear();
    ctx->pf_ntok = ntok;
    ctx->pf_done = 0;
    if (ctx->pf_chunk == 0) {   // Alg. 1 L7: the whole batch before the window's first decode step
      CK(cudaEventRecord(ctx->pf_ev[0], ctx->st));
      int rc = run_prefill(ctx, ntok);
      if (rc) return rc;
      CK(cudaEventRecord(ctx->pf_ev[1], ctx->st));
      ctx->pf_pending = true;
    }
  }
  return SART_OK;
}

// ------------------------------------------------------------------ boundary read-back
int read_boundary(sart_ctx* ctx) {
  const Dims& D = ctx->D;
  CK(xfer(ctx, ctx->h_ctr, ctx->ctr, sizeof(Ctr) + sizeof(int) * D.S, cudaMemcpyDeviceToHost, ctx->st));
  CK(cudaStreamSynchronize(ctx->st));
  Ctr& c = *ctx->h_ctr;
  if (ctx->pf_pending) {   // GPU time of this window's batched prefill
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, ctx->pf_ev[0], ctx->pf_ev[1]) == cudaSuccess) ctx->prefill_ms += ms;
    ctx->pf_pending = false;
  }
  // the device applied the releases; the host mirror adopts its counters
  ctx->n_rows = c.n_rows;
  ctx->free_top = c.free_top;
  ctx->committed = c.committed;
  ctx->windows = c.windows;
  ctx->steps = c.steps;
  ctx->branch_tokens = c.branch_tokens;
  ctx->attn_bytes = c.attn_bytes - ctx->attn_bytes_base;
  const int nf = c.n_final;
  if (nf == 0) return SART_OK;
  std::vector<int> fslots(c.final_slots, c.final_slots + nf);
  std::sort(fslots.begin(), fslots.end(),
            [&](int a, int b) { return ctx->slots[a].id < ctx->slots[b].id; });
  std::vector<DevResult> dr(nf);
  for (int i = 0; i < nf; ++i)
    CK(xfer(ctx, &dr[i], ctx->res + fslots[i], sizeof(DevResult), cudaMemcpyDeviceToHost, ctx->st));
  CK(cudaStreamSynchronize(ctx->st));
  const int64_t tnow = now_ns();
  for (int i = 0; i < nf; ++i) {
    const int slot = fslots[i];
    SlotInfo& si = ctx->slots[slot];
    HostResult hr;
    sart_result& r = hr.r;
    memset(&r, 0, sizeof(r));
    const DevResult& d = dr[i];
    r.request_id = d.request_id;
    r.answer_vote = d.answer_vote;
    r.vote_count = d.vote_count;
    r.chosen_max_reward = d.chosen_max_reward;
    r.answer_max_reward = d.answer_max_reward;
    r.num_completed = d.num_completed;
    r.num_pruned = d.num_pruned;
    r.num_early_stopped = d.num_early_stopped;
    r.finalize_reason = d.finalize_reason;
    r.phase_at_end = d.phase_at_end;
    r.threshold_at_end = d.threshold_at_end;
    r.selected_branch = d.selected_branch;
    for (int b = 0; b < si.N; ++b) {
      r.branch_len[b] = d.branch_len[b];
      r.branch_state[b] = (uint8_t)d.branch_state[b];
      r.branch_score[b] = d.branch_score[b];
    }
    // R7: queued branches of a finalized request are discarded at no cost
    int disc = 0;
    std::deque<std::pair<int, int>> keep;
    for (auto& p : ctx->branch_queue) {
      if (p.first == slot) {
        r.branch_state[p.second] = SART_BR_DISCARDED;
        ++disc;
      } else {
        keep.push_back(p);
      }
    }
    ctx->branch_queue.swap(keep);
    r.num_discarded_queued = disc;
    r.t_arrival_ns = si.arrival_ns;
    r.t_prefill_ns = si.prefill_ns;
    r.t_final_ns = tnow;
    r.window_final = ctx->windows - 1;
    const int sel = d.selected_branch;
    r.tokens_len = d.branch_len[sel];
    hr.tokens.resize(r.tokens_len);
    if (r.tokens_len > 0)
      CK(xfer(ctx, hr.tokens.data(), ctx->reqs.hist + ((size_t)slot * SART_MAXN + sel) * D.cap,
                         sizeof(int) * r.tokens_len, cudaMemcpyDeviceToHost, ctx->st));
    ctx->results.push_back(std::move(hr));
    si.live = false;
    ctx->free_slots.push_back(slot);
    ctx->finalized_total++;
  }
  CK(cudaStreamSynchronize(ctx->st));
  return SART_OK;
}

// ------------------------------------------------------------------ PP2 trace (record_trace)
struct Fnv {
  uint64_t h = 1469598103934665603ull;
  void bytes(const void* p, size_t n) {
    const unsigned char* c = (const unsigned char*)p;
    for (size_t i = 0; i < n; ++i) { h ^= c[i]; h *= 1099511628211ull; }
  }
  void i32(int32_t v) { bytes(&v, 4); }
  void i64(int64_t v) { bytes(&v, 8); }
};

// FNV-1a 64 of the control state after a boundary (layout: include/sart.h, sart_trace_fetch)
int state_hash(sart_ctx* ctx, uint64_t* out) {
  const Dims& D = ctx->D;
  const int n = ctx->n_rows;
  std::vector<int> slot(n), b(n), ell(n), nblk(n), tab((size_t)n * D.MBR);
  if (n) {
    CK(cudaMemcpy(slot.data(), ctx->rows.slot, 4 * (size_t)n, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(b.data(), ctx->rows.b, 4 * (size_t)n, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(ell.data(), ctx->rows.ell, 4 * (size_t)n, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(nblk.data(), ctx->rows.nblk, 4 * (size_t)n, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(tab.data(), ctx->rows.table, 4 * tab.size(), cudaMemcpyDeviceToHost));
  }
  Fnv f;
  for (int r = 0; r < n; ++r) {
    f.i64(ctx->slots[slot[r]].id);
    f.i32(b[r]);
    f.i32(ell[r]);
    f.i32(nblk[r]);
    for (int j = 0; j < nblk[r]; ++j) f.i32(tab[(size_t)r * D.MBR + j]);
  }
  std::vector<int> fs((size_t)ctx->free_top);
  if (!fs.empty()) CK(cudaMemcpy(fs.data(), ctx->free_stack, 4 * fs.size(), cudaMemcpyDeviceToHost));
  f.i32((int32_t)fs.size());
  for (int x : fs) f.i32(x);
  f.i64(ctx->committed);
  std::vector<std::pair<int64_t, int>> live;
  for (int s = 0; s < D.S; ++s)
    if (ctx->slots[s].live) live.emplace_back(ctx->slots[s].id, s);
  std::sort(live.begin(), live.end());
  f.i32((int32_t)live.size());
  for (auto& [id, s] : live) {
    int v[5];
    float thr;
    CK(cudaMemcpy(&v[0], ctx->reqs.phase + s, 4, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(&thr, ctx->reqs.thr + s, 4, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(&v[1], ctx->reqs.maxp + s, 4, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(&v[2], ctx->reqs.nc + s, 4, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(&v[3], ctx->reqs.np + s, 4, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(&v[4], ctx->reqs.npre + s, 4, cudaMemcpyDeviceToHost));
    uint32_t tb;
    memcpy(&tb, &thr, 4);
    f.i64(id);
    f.i32(v[0]);
    f.i32((int32_t)tb);
    f.i32(v[1]);
    f.i32(v[2]);
    f.i32(v[3]);
    f.i32(v[4]);
    std::vector<int> pre(v[4]);
    if (v[4]) CK(cudaMemcpy(pre.data(), ctx->reqs.prefix + (size_t)s * D.MPB, 4 * (size_t)v[4], cudaMemcpyDeviceToHost));
    for (int x : pre) f.i32(x);
  }
  *out = f.h;
  return SART_OK;
}

// After the boundary of a window of n rows: each row's new tokens (reqs.hist [ell_start, ell))
// and the score the boundary used, then the state hash.  The finalized requests' slots were
// released by read_boundary, but nothing has overwritten their history yet (the next fill
// runs after this).
int record_trace_window(sart_ctx* ctx, int n) {
  const Dims& D = ctx->D;
  std::vector<int> slot(n), b(n), st(n), ell(n);
  std::vector<float> sc(n);
  if (n) {
    CK(cudaMemcpy(slot.data(), ctx->dbg_slot, 4 * (size_t)n, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(b.data(), ctx->dbg_b, 4 * (size_t)n, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(st.data(), ctx->dtr.state, 4 * (size_t)n, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(ell.data(), ctx->dtr.ell, 4 * (size_t)n, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(sc.data(), ctx->dtr.score, 4 * (size_t)n, cudaMemcpyDeviceToHost));
  }
  for (int r = 0; r < n; ++r) {
    sart_trace_row t{};
    t.request_id = ctx->last_slot_id[slot[r]];
    t.branch = b[r];
    t.window = ctx->windows - 1;
    t.ell_start = ctx->trace_ell0[r];
    t.n_tokens = ell[r] - t.ell_start;
    t.running = (st[r] == RUNNING_ST || st[r] == ST_STOP) ? 1 : 0;   // incomplete: a running score (R43)
    t.score = sc[r];
    t.tokens_offset = (int64_t)ctx->trace_tokens.size();
    ctx->trace_tokens.resize(ctx->trace_tokens.size() + t.n_tokens);
    if (t.n_tokens > 0)
      CK(cudaMemcpy(ctx->trace_tokens.data() + t.tokens_offset,
                    ctx->reqs.hist + ((size_t)slot[r] * SART_MAXN + b[r]) * D.cap + t.ell_start,
                    4 * (size_t)t.n_tokens, cudaMemcpyDeviceToHost));
    ctx->trace_rows.push_back(t);
  }
  uint64_t h = 0;
  const int rc = state_hash(ctx, &h);
  if (rc) return rc;
  ctx->trace_hashes.push_back(h);
  return SART_OK;
}

template <typename T>
int run_window(sart_ctx* ctx) {
  const Dims& D = ctx->D;
  const int n = ctx->n_rows;
  ctx->last_n = n;
  ctx->ev_used = 0;
  launch_window_begin(ctx->ctr, n, ctx->st);
  ctx->launches++;
  if (ctx->cfg.record_trace) {   // PP2: steps each row had before this window
    ctx->trace_ell0.resize(n);
    if (n) CK(cudaMemcpyAsync(ctx->trace_ell0.data(), ctx->rows.ell, sizeof(int) * n, cudaMemcpyDeviceToHost, ctx->st));
    CK(cudaStreamSynchronize(ctx->st));
  }
  if (ctx->prm)   // entries decoded this window = ell(boundary) - ell(now), per row (f2 pass)
    CK(xfer(ctx, ctx->prm->h_ell_ws, ctx->rows.ell, sizeof(int) * n, cudaMemcpyDeviceToHost, ctx->st));
  if (ctx->bf16) {   // work units of the cascade attention for this window's batch
    // the tensor-core prefix pass runs this window if a live request can form a group of
    // >= tcq query rows (its launch finds no items otherwise)
    ctx->tc_prefix_window = false;
    if (ctx->plan.tcq > 0 && ctx->cfg.attn_mode != SART_ATTN_FLAT)
      for (const SlotInfo& si : ctx->slots)
        if (si.live && si.N * D.g >= ctx->plan.tcq) ctx->tc_prefix_window = true;
    ctx->prefix_tc_windows += ctx->tc_prefix_window;
    // the pass's SMs (SART_TC_SMS); the cascade kernel streams the suffixes on the others
    static const int tc_sms = getenv("SART_TC_SMS") ? atoi(getenv("SART_TC_SMS")) : 64;
    ctx->plan.tc_grid = ctx->tc_prefix_window ? std::max(1, std::min(tc_sms, device_sms())) : 0;
    launch_attn_plan(D, ctx->rows, ctx->reqs, ctx->plan, n, ctx->cfg.attn_mode == SART_ATTN_FLAT, ctx->st);
    ctx->launches++;
  }
  // Decode steps.  Without profiling, the step (~260 kernels) is captured once per window as
  // a CUDA graph and replayed T times (row count and pointers are fixed within a window; all
  // per-step state is read from device memory).  A window ends early when no row is live
  // (R31): the live count is copied back asynchronously every POLL steps and the host stops
  // enqueuing once a completed copy shows 0; steps enqueued after that are no-ops.
  const bool graph = !ctx->cfg.profile && ctx->use_graphs;
  long long per_step = 0;
  if (graph) {
    const long long before = ctx->launches;
    cudaGraph_t g = nullptr;
    CK(cudaStreamBeginCapture(ctx->st, cudaStreamCaptureModeThreadLocal));
    decode_step<T>(ctx, n);
    CK(cudaStreamEndCapture(ctx->st, &g));
    per_step = ctx->launches - before;
    ctx->launches = before;
    bool updated = false;
    if (ctx->step_exec) {
      cudaGraphExecUpdateResultInfo info;
      updated = cudaGraphExecUpdate(ctx->step_exec, g, &info) == cudaSuccess;
      if (!updated) {
        cudaGetLastError();
        cudaGraphExecDestroy(ctx->step_exec);
        ctx->step_exec = nullptr;
      }
    }
    if (!updated) CK(cudaGraphInstantiate(&ctx->step_exec, g, 0));
    CK(cudaGraphDestroy(g));
  }
  constexpr int POLL = 16;
  int polls = 0;
  // profile mode: per-step completion times; step_ev[0] was recorded by sart_step before the
  // fill, so an inline prefill counts toward the first step (R44 stall measurement)
  const bool step_times = ctx->cfg.profile != 0 && (int)ctx->step_ev.size() > D.T;
  int steps_launched = 0;
  for (int k = 1; k <= D.T; ++k) {
    if (k > 1 && (k % POLL) == 1) {
      if (polls >= 2) {   // bound the run-ahead: wait for the poll two periods back
        CK(cudaEventSynchronize(ctx->poll_ev[polls & 1]));
        if (ctx->h_live[polls & 1] == 0) break;
      }
      CK(xfer(ctx, &ctx->h_live[polls & 1], &ctx->ctr->live, sizeof(int), cudaMemcpyDeviceToHost, ctx->st));
      CK(cudaEventRecord(ctx->poll_ev[polls & 1], ctx->st));
      ++polls;
      if (polls >= 2 && cudaEventQuery(ctx->poll_ev[(polls - 2) & 1]) == cudaSuccess &&
          ctx->h_live[(polls - 2) & 1] == 0)
        break;
    }
    if (ctx->pf_done < ctx->pf_ntok) {   // R44: chunk k-1 before step k (all the rest before step T)
      const int upto = k < D.T ? k * ctx->pf_chunk : ctx->pf_ntok;
      const int rc = run_prefill(ctx, upto);
      if (rc) return rc;
    }
    if (graph) {
      CK(cudaGraphLaunch(ctx->step_exec, ctx->st));
      ctx->launches += per_step;
    } else {
      decode_step<T>(ctx, n);
    }
    if (step_times) CK(cudaEventRecord(ctx->step_ev[k], ctx->st));
    steps_launched = k;
  }
  if (ctx->pf_done < ctx->pf_ntok) {   // a window that ended early (R31) still completes this fill's prefixes
    const int rc = run_prefill(ctx, ctx->pf_ntok);
    if (rc) return rc;
  }
  CK(cudaGetLastError());
  if (ctx->gemm_failed) return set_err(SART_EINVAL, "GEMM shape unsupported by the tcgen05 kernel");
  // rows of this window (debug), then the boundary: PRM head -> control kernel
  CK(cudaMemcpyAsync(ctx->dbg_slot, ctx->rows.slot, sizeof(int) * n, cudaMemcpyDeviceToDevice, ctx->st));
  CK(cudaMemcpyAsync(ctx->dbg_b, ctx->rows.b, sizeof(int) * n, cudaMemcpyDeviceToDevice, ctx->st));
  if (ctx->prm) {
    prm_model_scores<T>(ctx, n);
    if (ctx->poisoned) return SART_ECUDA;
    if (ctx->gemm_failed) return set_err(SART_EINVAL, "GEMM shape unsupported by the tcgen05 kernel (PRM model)");
  } else {
    prm_scores<T>(ctx, n);
  }
  launch_boundary(D, ctx->rows, ctx->tmp, ctx->reqs, ctx->prm ? ctx->prm->prm_score : ctx->prm_score, ctx->free_stack, ctx->ctr, ctx->res,
                  ctx->slot_row, n, ctx->dtr, ctx->st);
  ctx->launches++;
  CK(cudaGetLastError());
  int rc = read_boundary(ctx);
  if (rc) return rc;
  if (ctx->cfg.record_trace && (rc = record_trace_window(ctx, n)) != SART_OK) return rc;
  if (ctx->prm) {
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, ctx->prm->prm_ev[0], ctx->prm->prm_ev[1]) == cudaSuccess) ctx->prm_ms += ms;
    ctx->prm_passes++;
  }
  if (getenv("SART_GEMM_TS_PRINT")) {   // phase timestamps of the last 4 recorded GEMM launches
    unsigned long long hts[4][10];        // (CTA 0; build with -DSART_GEMM_TS [-DSART_GEMM_TS_MODE=m])
    CK(cudaStreamSynchronize(ctx->st));
    gemm_ts_fetch(&hts[0][0]);
    for (int i = 0; i < 4; ++i) {
      fprintf(stderr, "GEMMTS window %d launch %d (ns from CTA start): setup %lld wait %lld mma0 %lld mma_last %lld "
              "epi_start %lld epi_end %lld end %lld dealloc %lld\n", ctx->windows, i,
              (long long)(hts[i][1] - hts[i][0]), (long long)(hts[i][2] - hts[i][0]), (long long)(hts[i][3] - hts[i][0]),
              (long long)(hts[i][4] - hts[i][0]), (long long)(hts[i][5] - hts[i][0]), (long long)(hts[i][6] - hts[i][0]),
              (long long)(hts[i][7] - hts[i][0]), (long long)(hts[i][8] - hts[i][0]));
    }
  }
  if (step_times && steps_launched > 0) {   // window start -> first decode step done; longest step
    float first = 0.f, mx = 0.f;
    cudaEventElapsedTime(&first, ctx->step_ev[0], ctx->step_ev[1]);
    mx = first;
    for (int k = 2; k <= steps_launched; ++k) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, ctx->step_ev[k - 1], ctx->step_ev[k]);
      mx = std::max(mx, ms);
    }
    ctx->first_step_ms_max = std::max(ctx->first_step_ms_max, (double)first);
    ctx->step_ms_max = std::max(ctx->step_ms_max, (double)mx);
  }
  if (ctx->cfg.profile) {
    for (int i = 0; i + 2 < ctx->ev_used; i += 3) {
      float ms = 0.f, ms_s = 0.f;
      cudaEventElapsedTime(&ms, ctx->ev_pool[i], ctx->ev_pool[i + 2]);
      ctx->attn_ms += ms;
      if (ctx->cfg.profile == 2 && cudaEventElapsedTime(&ms_s, ctx->ev_pool[i], ctx->ev_pool[i + 1]) == cudaSuccess)
        ctx->attn_stream_ms += ms_s;
    }
  }
  return SART_OK;
}
}  // namespace

// Weights (host blob or device-generated), fp32 epilogue vectors, RoPE table and the
// per-token workspaces of one decoder: the policy, or the f2 PRM model (sub-context).
// Tensor parallelism: where a rank's tensor t comes from in the FULL model's tensor t --
// segments {local element offset, count, cl, cf, c0, global offset} in the k_init_tensor
// slice mapping (local i -> global goff + (i / cl) * cf + c0 + i % cl).
struct Seg { long long loff, n, cl, cf, c0, goff; };
std::vector<Seg> shard_segments(const Dims& F, int tp, int rank, int idx) {
  const long long d = F.d, hd = F.hd, qr = F.qh / tp, kr = F.kvh / tp, fr = F.F / tp;
  std::vector<size_t> sz = tensor_sizes(F);
  const long long n = (long long)sz[idx];
  if (idx >= 1 && idx < 1 + 8 * F.L) {
    const int k = (idx - 1) % 8;
    const long long rows_q = F.qh * hd, rows_k = F.kvh * hd;
    if (k == 1 || k == 2) {   // wqkv rows / bqkv: q heads, k heads, v heads of this rank
      const long long w = k == 1 ? d : 1;
      const long long q0 = rank * qr * hd, k0 = rows_q + rank * kr * hd, v0 = rows_q + rows_k + rank * kr * hd;
      const long long nq = qr * hd * w, nk = kr * hd * w;
      return {Seg{0, nq, nq, nq, 0, q0 * w}, Seg{nq, nk, nk, nk, 0, k0 * w}, Seg{nq + nk, nk, nk, nk, 0, v0 * w}};
    }
    if (k == 3)               // wo [d][qh hd]: this rank's input columns
      return {Seg{0, d * qr * hd, qr * hd, F.qh * hd, rank * qr * hd, 0}};
    if (k == 5 || k == 6)     // wgate / wup [F][d]: this rank's rows
      return {Seg{0, fr * d, fr * d, fr * d, 0, rank * fr * d}};
    if (k == 7)               // wdown [d][F]: this rank's input columns
      return {Seg{0, d * fr, fr, F.F, rank * fr, 0}};
  }
  return {Seg{0, n, n, n, 0, 0}};   // replicated
}

int init_model(sart_ctx* ctx, const void* host_w, uint64_t seed, float wstd) {
  const Dims& D = ctx->D;
  const size_t es = ctx->bf16 ? 2 : 4;
  const size_t W = ctx->W;
  cudaError_t e;
#define MC(x)                                                                   \
  do {                                                                          \
    e = (x);                                                                    \
    if (e != cudaSuccess)                                                       \
      return set_err(e == cudaErrorMemoryAllocation ? SART_ENOMEM : SART_ECUDA, \
                     std::string(#x) + ": " + cudaGetErrorString(e));           \
  } while (0)
  // ---- weights
  std::vector<size_t> sizes = tensor_sizes(D);
  size_t total = 0;
  for (size_t s : sizes) { ctx->woff.push_back(total); total += s; }
  MC(cudaMalloc(&ctx->wblob, total * es));
  if (ctx->tp > 1) {   // row f4: this rank's shard of the full model (host blob or generated)
    Dims Fd = D;
    Fd.qh *= ctx->tp; Fd.kvh *= ctx->tp; Fd.F *= ctx->tp; Fd.qkv = (Fd.qh + 2 * Fd.kvh) * Fd.hd;
    std::vector<size_t> fsz = tensor_sizes(Fd), foff;
    size_t ft = 0;
    for (size_t x : fsz) { foff.push_back(ft); ft += x; }
    for (size_t i = 0; i < sizes.size(); ++i) {
      const bool nrm = is_norm_tensor(D, (int)i);
      for (const Seg& g : shard_segments(Fd, ctx->tp, ctx->tp_rank, (int)i)) {
        char* dst = (char*)ctx->wblob + (ctx->woff[i] + g.loff) * es;
        if (host_w) {
          const char* src = (const char*)host_w + foff[i] * es;
          const long long rows = g.n / g.cl;
          if (rows == 1)
            MC(dsync(cudaMemcpy(dst, src + (g.goff + g.c0) * es, g.n * es, cudaMemcpyHostToDevice)));
          else
            MC(dsync(cudaMemcpy2D(dst, g.cl * es, src + (g.goff + g.c0) * es, g.cf * es, g.cl * es, rows,
                            cudaMemcpyHostToDevice)));
        } else if (ctx->bf16) {
          launch_init_slice<bf16>((bf16*)dst, g.n, (int)i, nrm, wstd, seed, g.cl, g.cf, g.c0, g.goff, ctx->st);
        } else {
          launch_init_slice<float>((float*)dst, g.n, (int)i, nrm, wstd, seed, g.cl, g.cf, g.c0, g.goff, ctx->st);
        }
      }
    }
    MC(cudaGetLastError());
  } else if (host_w) {
    MC(dsync(cudaMemcpy(ctx->wblob, host_w, total * es, cudaMemcpyHostToDevice)));
  } else {
    for (size_t i = 0; i < sizes.size(); ++i) {
      bool norm = is_norm_tensor(D, (int)i);
      if (ctx->bf16)
        launch_init_tensor<bf16>((bf16*)ctx->wblob + ctx->woff[i], (long long)sizes[i], (int)i, norm, wstd,
                                 seed, ctx->st);
      else
        launch_init_tensor<float>((float*)ctx->wblob + ctx->woff[i], (long long)sizes[i], (int)i, norm,
                                  wstd, seed, ctx->st);
    }
    MC(cudaGetLastError());
  }
  if (ctx->bf16) {
    if (D.F % 128 != 0) {
      return set_err(SART_EINVAL, "bf16 mode needs d_ff % 128 == 0 (fused SwiGLU tiles)");
    }
    bf16* tmpw = nullptr;
    MC(cudaMalloc(&tmpw, sizeof(bf16) * 2 * (size_t)D.F * D.d));
    for (int l = 0; l < D.L; ++l) launch_interleave_gate_up(ctx->W_<bf16>(t_layer(l, 5)), tmpw, D.F, D.d, ctx->st);
    MC(cudaStreamSynchronize(ctx->st));
    cudaFree(tmpw);
  }
  // fp32 copies of the small vectors used in epilogues
  size_t nf = (size_t)D.L * D.qkv + D.d + 2 * (size_t)D.d + 2;
  MC(dalloc(ctx, &ctx->fparams, nf * sizeof(float)));
  ctx->f_bqkv = 0;
  ctx->f_prm_b1 = (size_t)D.L * D.qkv;
  ctx->f_prm_w2 = ctx->f_prm_b1 + D.d;
  ctx->f_prm_b2 = ctx->f_prm_w2 + 2 * (size_t)D.d;
  auto tof = [&](int idx, size_t off, size_t n) {
    if (ctx->bf16) launch_to_f32<bf16>(ctx->W_<bf16>(idx), ctx->fparams + off, (long long)n, ctx->st);
    else launch_to_f32<float>(ctx->W_<float>(idx), ctx->fparams + off, (long long)n, ctx->st);
  };
  for (int l = 0; l < D.L; ++l) tof(t_layer(l, 2), (size_t)l * D.qkv, D.qkv);
  tof(t_prm_b1(D), ctx->f_prm_b1, D.d);
  tof(t_prm_w2(D), ctx->f_prm_w2, 2 * (size_t)D.d);
  tof(t_prm_b2(D), ctx->f_prm_b2, 2);
  MC(cudaGetLastError());
  // ---- RoPE table (fp64 on the host, stored fp32): [pos][cos(hd/2) | sin(hd/2)]
  {
    std::vector<float> cs((size_t)D.max_pos * D.hd);
    const int half = D.hd / 2;
    for (int p = 0; p < D.max_pos; ++p)
      for (int i = 0; i < half; ++i) {
        double inv = std::pow((double)D.theta, -2.0 * i / D.hd);
        double ang = p * inv;
        cs[(size_t)p * D.hd + i] = (float)std::cos(ang);
        cs[(size_t)p * D.hd + half + i] = (float)std::sin(ang);
      }
    MC(dalloc(ctx, &ctx->rope_cs, cs.size() * sizeof(float), false));
    MC(dsync(cudaMemcpy(ctx->rope_cs, cs.data(), cs.size() * sizeof(float), cudaMemcpyHostToDevice)));
  }
  MC(dalloc(ctx, &ctx->h, W * D.d * 4));
  MC(dalloc(ctx, &ctx->parts, W * std::max(D.qkv, D.d) * 8 * 4, false));   // split-K partials (S <= 8)
  ctx->qkv_cnt_cap = (D.qkv / D.hd) * ((int)((W + 127) / 128)) * 8;
  MC(dalloc(ctx, &ctx->qkv_cnt, sizeof(int) * (size_t)ctx->qkv_cnt_cap));   // QKV split-K arrivals (zeroed)
  if (!ctx->bf16) MC(dalloc(ctx, &ctx->gu, W * 2 * D.F * 4));   // bf16: fused SwiGLU epilogue
  MC(dalloc(ctx, &ctx->z32, (size_t)D.R * D.d * 4));
  MC(dalloc(ctx, &ctx->prm_hid, (size_t)D.R * D.d * 4));
  MC(dalloc(ctx, &ctx->prm_score, (size_t)D.R * 4));
  MC(dalloc(ctx, &ctx->a, W * D.d * es));
  MC(dalloc(ctx, &ctx->q, W * D.qh * D.hd * es));
  MC(dalloc(ctx, &ctx->o, W * D.qh * D.hd * es));
  MC(dalloc(ctx, &ctx->act, W * D.F * es));
  MC(dalloc(ctx, &ctx->zT, (size_t)D.R * D.d * es));
#undef MC
  return SART_OK;
}

// ====================================================================== C-ABI
extern "C" {

const char* sart_strerror(int code) {
  switch (code) {
    case SART_OK: return "SART_OK";
    case SART_EINVAL: return "SART_EINVAL";
    case SART_ENOMEM: return "SART_ENOMEM";
    case SART_ECUDA: return "SART_ECUDA";
    case SART_EFULL: return "SART_EFULL";
    case SART_ESTATE: return "SART_ESTATE";
    case SART_EDUP: return "SART_EDUP";
    default: return "SART_UNKNOWN";
  }
}
const char* sart_last_error(void) { return g_last_error.c_str(); }

int sart_destroy(sart_ctx* ctx) {
  if (!ctx) return SART_OK;
  cudaSetDevice(ctx->cfg.device);
  if (ctx->st) cudaStreamSynchronize(ctx->st);
  if (ctx->prm) {
    sart_destroy(ctx->prm);   // shares the stream; frees its own weights, pool, workspaces
    ctx->prm = nullptr;
  }
  for (auto e : ctx->prm_ev)
    if (e) cudaEventDestroy(e);
  for (auto e : ctx->ev_pool) cudaEventDestroy(e);
  for (auto e : ctx->step_ev) cudaEventDestroy(e);
  for (auto e : ctx->poll_ev)
    if (e) cudaEventDestroy(e);
  for (auto e : ctx->pf_ev)
    if (e) cudaEventDestroy(e);
  if (ctx->step_exec) cudaGraphExecDestroy(ctx->step_exec);
  for (void* p : ctx->tp_opened) cudaIpcCloseMemHandle(p);
  for (void* p : ctx->allocs) cudaFree(p);
  if (ctx->wblob) cudaFree(ctx->wblob);
  if (ctx->h_ctr) cudaFreeHost(ctx->h_ctr);
  if (ctx->h_ell_ws) cudaFreeHost(ctx->h_ell_ws);
  if (ctx->h_ell) cudaFreeHost(ctx->h_ell);
  if (ctx->h_prm_desc) cudaFreeHost(ctx->h_prm_desc);
  if (ctx->h_live) cudaFreeHost(ctx->h_live);
  if (ctx->own_stream && ctx->st) cudaStreamDestroy(ctx->st);
  delete ctx;
  return SART_OK;
}

int sart_init(const sart_config* cfg_in, sart_ctx** out) {
  if (!cfg_in || !out) return set_err(SART_EINVAL, "null argument");
  *out = nullptr;
  sart_config cfg = *cfg_in;
  if (cfg.block_size == 0) cfg.block_size = 64;
  if (cfg.max_rows == 0) cfg.max_rows = 1024;
  if (cfg.max_requests == 0) cfg.max_requests = 256;
  if (cfg.max_prompt == 0) cfg.max_prompt = 8193;
  if (cfg.ctl_interval == 0) cfg.ctl_interval = 400;
  if (cfg.weight_std == 0.f) cfg.weight_std = 0.02f;
  if (cfg.n_layers < 1 || cfg.d_model < 1 || cfg.n_heads < 1 || cfg.n_kv_heads < 1 || cfg.d_ff < 1 ||
      cfg.vocab < 2)
    return set_err(SART_EINVAL, "model dims must be positive");
  if (cfg.head_dim != 64 && cfg.head_dim != 128) return set_err(SART_EINVAL, "head_dim must be 64 or 128");
  if (cfg.n_heads % cfg.n_kv_heads || cfg.n_heads / cfg.n_kv_heads > 16)
    return set_err(SART_EINVAL, "n_heads must be a multiple of n_kv_heads with ratio <= 16");
  if (cfg.d_model % 8 || cfg.d_ff % 8) return set_err(SART_EINVAL, "d_model and d_ff must be multiples of 8");
  if (cfg.dtype != SART_BF16 && cfg.dtype != SART_FP32) return set_err(SART_EINVAL, "dtype");
  if (cfg.block_size != 16 && cfg.block_size != 32 && cfg.block_size != 64)
    return set_err(SART_EINVAL, "block_size must be 16, 32 or 64");
  if (cfg.max_new_tokens < 1 || cfg.ctl_interval < 1 || cfg.max_rows < 1 || cfg.max_requests < 1 ||
      cfg.max_requests > 1024 || cfg.max_prompt < 1)
    return set_err(SART_EINVAL, "cap, T, max_rows >= 1; 1 <= max_requests <= 1024");
  if (cfg.eos_id < 0 || cfg.eos_id >= cfg.vocab) return set_err(SART_EINVAL, "eos_id out of range");
  if (!(cfg.temperature >= 0.f)) return set_err(SART_EINVAL, "temperature must be >= 0");
  if (cfg.select_mode != 0 && cfg.select_mode != 1) return set_err(SART_EINVAL, "select_mode");
  if (cfg.attn_mode != 0 && cfg.attn_mode != 1) return set_err(SART_EINVAL, "attn_mode");
  if (cfg.prm_n_layers < 0) return set_err(SART_EINVAL, "prm_n_layers < 0");
  if (cfg.es_every_step != 0 && cfg.es_every_step != 1) return set_err(SART_EINVAL, "es_every_step must be 0 or 1");
  if (cfg.record_trace != 0 && cfg.record_trace != 1) return set_err(SART_EINVAL, "record_trace must be 0 or 1");
  if (cfg.kv_pool && cfg.kv_pool_bytes == 0) return set_err(SART_EINVAL, "kv_pool given with kv_pool_bytes == 0");
  if (cfg.prefill_chunk < 0 || cfg.prefill_chunk > 2048) return set_err(SART_EINVAL, "prefill_chunk must be in [0, 2048]");
  if (cfg.tp_size == 0) cfg.tp_size = 1;
  if (cfg.tp_size < 1 || cfg.tp_size > SART_MAX_TP || cfg.tp_rank < 0 || cfg.tp_rank >= cfg.tp_size)
    return set_err(SART_EINVAL, "need 1 <= tp_size <= 8 and 0 <= tp_rank < tp_size");
  if (cfg.tp_size > 1) {   // row f4
    if (cfg.dtype != SART_BF16) return set_err(SART_EINVAL, "tensor parallelism needs dtype SART_BF16");
    if (cfg.prm_n_layers > 0) return set_err(SART_EINVAL, "tensor parallelism with a separate PRM model is not supported");
    if (cfg.n_heads % cfg.tp_size || cfg.n_kv_heads % cfg.tp_size || (cfg.d_ff / cfg.tp_size) % 128 ||
        cfg.d_ff % cfg.tp_size)
      return set_err(SART_EINVAL, "tp_size must divide n_heads and n_kv_heads, and d_ff / tp_size % 128 == 0");
  }
  if (cfg.prm_n_layers > 0) {   // row f2: separate PRM decoder
    if (cfg.prm_d_model < 1 || cfg.prm_n_heads < 1 || cfg.prm_n_kv_heads < 1 || cfg.prm_d_ff < 1)
      return set_err(SART_EINVAL, "PRM model dims must be positive");
    if (cfg.prm_head_dim != 64 && cfg.prm_head_dim != 128) return set_err(SART_EINVAL, "prm_head_dim must be 64 or 128");
    if (cfg.prm_n_heads % cfg.prm_n_kv_heads || cfg.prm_n_heads / cfg.prm_n_kv_heads > 16)
      return set_err(SART_EINVAL, "prm_n_heads must be a multiple of prm_n_kv_heads with ratio <= 16");
    if (cfg.prm_d_model % 8 || cfg.prm_d_ff % 8) return set_err(SART_EINVAL, "prm_d_model and prm_d_ff: multiples of 8");
  }

  sart_ctx* ctx = new sart_ctx();
  ctx->cfg = cfg;
  ctx->bf16 = cfg.dtype == SART_BF16;
  Dims& D = ctx->D;
  D.L = cfg.n_layers; D.d = cfg.d_model; D.qh = cfg.n_heads; D.kvh = cfg.n_kv_heads; D.hd = cfg.head_dim;
  D.F = cfg.d_ff; D.V = cfg.vocab;
  ctx->tp = cfg.tp_size;
  ctx->tp_rank = cfg.tp_rank;
  D.qh /= ctx->tp; D.kvh /= ctx->tp; D.F /= ctx->tp;   // this rank's heads and FFN rows (row f4)
  D.qkv = (D.qh + 2 * D.kvh) * D.hd; D.g = D.qh / D.kvh;
  D.bs = cfg.block_size; D.R = cfg.max_rows; D.S = cfg.max_requests;
  D.cap = cfg.max_new_tokens; D.T = cfg.ctl_interval; D.eos = cfg.eos_id;
  D.MBR = cdiv(D.cap, D.bs);
  D.MPB = std::max(1, cdiv(cfg.max_prompt - 1, D.bs));
  D.nbnd_max = cdiv(D.cap, D.T) + 1;
  D.max_pos = cfg.max_prompt + D.cap;
  D.theta = cfg.rope_theta; D.eps = cfg.rms_eps; D.tau = cfg.temperature; D.seed = cfg.sampler_seed;
  D.select_mode = cfg.select_mode;
  ctx->PC = 2048;   // prefill chunk (tokens)
  ctx->pf_chunk = cfg.prefill_chunk;
  ctx->W = std::max(D.R, ctx->PC);
  const size_t es = ctx->bf16 ? 2 : 4;

  cudaError_t e;
#define IC(x)                                                                   \
  do {                                                                          \
    e = (x);                                                                    \
    if (e != cudaSuccess) {                                                     \
      int code = e == cudaErrorMemoryAllocation ? SART_ENOMEM : SART_ECUDA;     \
      set_err(code, std::string(#x) + ": " + cudaGetErrorString(e));            \
      sart_destroy(ctx);                                                        \
      return code;                                                              \
    }                                                                           \
  } while (0)
  IC(cudaSetDevice(cfg.device));
  if (cfg.stream) {
    ctx->st = (cudaStream_t)cfg.stream;
  } else {
    IC(cudaStreamCreateWithFlags(&ctx->st, cudaStreamNonBlocking));
    ctx->own_stream = true;
  }
  {
    const int rc = init_model(ctx, cfg.host_weights, cfg.weight_seed, cfg.weight_std);
    if (rc) {
      sart_destroy(ctx);
      return rc;
    }
  }
  // ---- state
  IC(alloc_rows(ctx, ctx->rows));
  IC(alloc_rows(ctx, ctx->tmp));
  IC(alloc_reqs(ctx));
  if (cfg.prm_n_layers > 0) {   // row f2: the PRM decoder as a sub-context sharing rows / reqs / stream
    sart_ctx* m = new sart_ctx();
    ctx->prm = m;
    m->is_prm = true;
    m->cfg = cfg;
    m->bf16 = ctx->bf16;
    m->st = ctx->st;
    m->D = D;
    Dims& P = m->D;
    P.L = cfg.prm_n_layers; P.d = cfg.prm_d_model; P.qh = cfg.prm_n_heads; P.kvh = cfg.prm_n_kv_heads;
    P.hd = cfg.prm_head_dim; P.F = cfg.prm_d_ff; P.qkv = (P.qh + 2 * P.kvh) * P.hd; P.g = P.qh / P.kvh;
    m->PC = ctx->PC;
    // chunk of the boundary pass: all rows x T entries when that is small, else 8192 tokens
    m->W = std::max(m->PC, (int)std::min<long long>(8192, (long long)((D.R + 63) / 64 * 64) * D.T));
    m->prm_chunk = m->W;
    if (const char* ev = getenv("SART_PRM_CHUNK"))   // tests: exercise the multi-chunk paths
      m->prm_chunk = std::max(64, std::min(m->W, atoi(ev)));
    m->rows = ctx->rows;
    m->reqs = ctx->reqs;
    {
      const int rc = init_model(m, cfg.prm_host_weights, cfg.prm_weight_seed, cfg.weight_std);
      if (rc) {
        sart_destroy(ctx);
        return rc;
      }
    }
    IC(dalloc(m, &m->prm_tok, sizeof(int) * (size_t)m->W));
    IC(dalloc(m, &m->prm_row, sizeof(int) * (size_t)m->W));
    IC(dalloc(m, &m->prm_ent, sizeof(int) * (size_t)m->W));
    IC(dalloc(m, &m->zrow, (size_t)D.R * P.d * es));
    IC(cudaEventCreate(&m->prm_ev[0]));
    IC(cudaEventCreate(&m->prm_ev[1]));
    IC(cudaMallocHost(&m->h_ell_ws, sizeof(int) * (size_t)D.R));
    IC(cudaMallocHost(&m->h_ell, sizeof(int) * (size_t)D.R));
    // descriptors: segments <= rows + chunks, q-blocks <= rows + tokens / 16, gathers <= rows
    const size_t max_tok = (size_t)D.R * D.T;
    m->prm_desc_cap = 3 * (size_t)D.R + 2 * (max_tok / m->prm_chunk + 1) + max_tok / 16 + 16;
    IC(dalloc(m, &m->prm_desc, sizeof(int4) * m->prm_desc_cap, false));
    IC(cudaMallocHost(&m->h_prm_desc, sizeof(int4) * m->prm_desc_cap));
  }
  if (ctx->tp > 1) {   // row f4: [arrival counters 2L (4 KB-aligned) | partials [tp][8][W][max(d, qkv)]]
    ctx->tp_parts_off = ((size_t)2 * D.L * sizeof(unsigned long long) + 4095) / 4096 * 4096;
    ctx->tp_region = (size_t)ctx->tp * 8 * ctx->W * std::max(D.d, D.qkv);
    const size_t bytes = ctx->tp_parts_off + sizeof(float) * 2 * ctx->tp_region;
    IC(dalloc(ctx, &ctx->tp_buf, bytes));
    ctx->tp_cnt = (unsigned long long*)ctx->tp_buf;
    ctx->tp_parts = (float*)((char*)ctx->tp_buf + ctx->tp_parts_off);
    IC(dalloc(ctx, &ctx->tp_expect, sizeof(unsigned long long) * 2 * D.L));
  }
  IC(dalloc(ctx, &ctx->ctr, sizeof(Ctr) + sizeof(int) * D.S));
  IC(dalloc(ctx, &ctx->res, sizeof(DevResult) * D.S));
  IC(dalloc(ctx, &ctx->slot_row, sizeof(int) * (size_t)D.S * SART_MAXN));
  IC(dsync(cudaMemset(ctx->slot_row, 0xff, sizeof(int) * (size_t)D.S * SART_MAXN)));
  // ---- workspaces
  IC(dalloc(ctx, &ctx->logits, (size_t)D.R * D.V * 4));
  IC(dalloc(ctx, &ctx->dbg_tok, (size_t)D.R * 4));
  // LM head with the sampler's first phase in its epilogue (SART_FUSED_SAMPLE=1; bf16)
  ctx->fused_sample = ctx->bf16 && getenv("SART_FUSED_SAMPLE") && atoi(getenv("SART_FUSED_SAMPLE")) != 0;
  {
    const int nsl = std::max(sample_chunks(D.V), ctx->bf16 ? gemm_sample_slots(D.V) : 0);
    IC(dalloc(ctx, &ctx->skey, (size_t)D.R * nsl * 4));
    IC(dalloc(ctx, &ctx->sv, (size_t)D.R * nsl * 4));
  }
  IC(dalloc(ctx, &ctx->dbg_slot, (size_t)D.R * 4));
  IC(dalloc(ctx, &ctx->dbg_b, (size_t)D.R * 4));
  ctx->pf_cap = (int)std::min<long long>((long long)D.S * cfg.max_prompt, 1LL << 24);
  IC(dalloc(ctx, &ctx->d_prompt, (size_t)ctx->pf_cap * 4));
  IC(dalloc(ctx, &ctx->d_pf_slot, (size_t)ctx->pf_cap * 4));
  IC(dalloc(ctx, &ctx->d_pf_pos, (size_t)ctx->pf_cap * 4));
  IC(dalloc(ctx, &ctx->d_pf_blocks, sizeof(int4) * (size_t)(ctx->PC / 16 + D.S + 8)));   // >= 16-position blocks
  IC(cudaEventCreate(&ctx->pf_ev[0]));
  IC(cudaEventCreate(&ctx->pf_ev[1]));
  ctx->ev_cap = D.R + D.S + 64;
  IC(dalloc(ctx, &ctx->d_events, sizeof(AdmitEvent) * ctx->ev_cap));
  if (cfg.debug_capture) IC(dalloc(ctx, &ctx->dbg_attn, (size_t)D.L * D.R * D.qh * D.hd * 4));
  if (cfg.record_trace) {
    IC(dalloc(ctx, &ctx->dtr.score, sizeof(float) * D.R));
    IC(dalloc(ctx, &ctx->dtr.state, sizeof(int) * D.R));
    IC(dalloc(ctx, &ctx->dtr.ell, sizeof(int) * D.R));
  }
  {  // cascade attention plan and partial outputs
    AttnPlan& pl = ctx->plan;
    pl.CH = 512;   // tokens per attention chunk (SART_ATTN_CH overrides; multiple of 64)
    if (const char* e = getenv("SART_ATTN_CH")) pl.CH = std::max(64, atoi(e) / 64 * 64);
    pl.qr_grp = std::max(1, std::min(SART_MAXN, 64 / D.g));
    if (const char* e = getenv("SART_ATTN_QR")) pl.qr_grp = std::max(1, std::min(SART_MAXN, atoi(e)));   // A/B
    // tensor-core prefix pass (hd 128, bf16 pool): groups of >= tcq query rows; SART_ATTN_TCQ
    // sets the threshold (0 = off).  Enabled after the pool's tensor map is encoded.
    // default 64 query rows (C3: N 16 x g 7, C5: 32 x 5; not C2: 8 x 6), running concurrently with
    // the cascade kernel on SART_TC_SMS = 64 SMs: C5 step -5.8%, C3 +1.6% throughput
    // (profiles/r2_prefix_tc_concurrent_ab.txt; serialised before the cascade it was a loss,
    // profiles/r2_prefix_tc_ab.txt)
    pl.tcq = D.hd == 128 ? 64 : 0;
    if (const char* e = getenv("SART_ATTN_TCQ")) pl.tcq = D.hd == 128 ? std::max(0, atoi(e)) : 0;
    pl.qr_max = std::max(pl.qr_grp, pl.tcq ? std::min(SART_MAXN, 128 / D.g) : 1);
    // suffix KV with an L2 evict-first policy: C2 step -1.7%, C3 +1.0% (profiles/r2_attn_evict_ab.txt)
    pl.evict = getenv("SART_ATTN_EVICT") ? atoi(getenv("SART_ATTN_EVICT")) : 1;
    // SART_ATTN_PIECE: suffix piece length (0 = off; a divisor of CH, multiple of 16)
    pl.PC = 0;
    if (const char* e = getenv("SART_ATTN_PIECE")) {
      const int pc = atoi(e) / 16 * 16;
      if (pc >= 16 && pc < pl.CH && pl.CH % pc == 0) pl.PC = pc;
    }
    pl.npc_max = std::max(1, cdiv(cfg.max_prompt - 1, pl.CH));
    const int nsc_max = cdiv(D.cap, pl.CH) + (pl.PC ? pl.CH / pl.PC : 0);   // chunks (+ pieces of the last)
    pl.nslot = pl.npc_max + nsc_max;
    const int nsu_max = pl.PC ? cdiv(D.cap, pl.PC) : nsc_max;             // suffix units per row
    const size_t max_units = (size_t)D.R * (4 * pl.npc_max + nsu_max);
    IC(dalloc(ctx, &pl.units, sizeof(int4) * max_units));
    IC(dalloc(ctx, &pl.n_units, sizeof(int)));
    IC(dalloc(ctx, &pl.work, sizeof(int) * D.L));
    IC(dalloc(ctx, &pl.done, sizeof(int) * D.L));
    IC(dalloc(ctx, &pl.tc_done, sizeof(int) * D.L));
    pl.tc_grid = 0;
    IC(dalloc(ctx, &pl.items, sizeof(int4) * 2 * max_units));
    IC(dalloc(ctx, &pl.n_items, sizeof(int)));
    IC(dalloc(ctx, &pl.tc_items, sizeof(int4) * 2 * max_units));
    IC(dalloc(ctx, &pl.n_tc, sizeof(int)));
    IC(dalloc(ctx, &pl.row_pos, sizeof(int) * D.R));
    IC(dalloc(ctx, &pl.row_rank, sizeof(int) * D.R));
    IC(dalloc(ctx, &pl.row_nreq, sizeof(int) * D.R));

    IC(dalloc(ctx, &pl.grp_slot, sizeof(int) * D.R));
    IC(dalloc(ctx, &pl.grp_n, sizeof(int) * D.R));
    IC(dalloc(ctx, &pl.grp_rows, sizeof(int) * (size_t)D.R * pl.qr_max));
    if (ctx->bf16) {
      IC(dalloc(ctx, &ctx->part_o, sizeof(float) * (size_t)D.R * D.qh * pl.nslot * D.hd, false));
      IC(dalloc(ctx, &ctx->part_lse, sizeof(float) * (size_t)D.R * D.qh * pl.nslot, false));
    }
  }
  IC(cudaMallocHost(&ctx->h_ctr, sizeof(Ctr) + sizeof(int) * D.S));
  IC(cudaMallocHost(&ctx->h_live, 2 * sizeof(int)));
  IC(cudaEventCreateWithFlags(&ctx->poll_ev[0], cudaEventDisableTiming));
  IC(cudaEventCreateWithFlags(&ctx->poll_ev[1], cudaEventDisableTiming));
  if (getenv("SART_NO_GRAPHS")) ctx->use_graphs = false;
  if (const char* ev = getenv("SART_ABLATE")) ctx->ablate = atoi(ev);
  // ---- KV pool
  const size_t blk_bytes = (size_t)D.L * 2 * D.kvh * D.bs * D.hd * es;
  // f2: the PRM cache uses the same block ids, so one block costs both decoders' pages
  const size_t prm_blk_bytes =
      ctx->prm ? (size_t)ctx->prm->D.L * 2 * ctx->prm->D.kvh * D.bs * ctx->prm->D.hd * es : 0;
  long long NB = cfg.num_blocks;
  if (cfg.kv_pool) {   // caller-owned pool: it bounds NB
    const long long fit = (long long)(cfg.kv_pool_bytes / blk_bytes);
    if (NB <= 0) NB = fit;
    if (NB > fit) {
      set_err(SART_ENOMEM, "kv_pool_bytes smaller than num_blocks x block bytes");
      sart_destroy(ctx);
      return SART_ENOMEM;
    }
  } else if (NB <= 0) {
    size_t fr = 0, tot = 0;
    IC(cudaMemGetInfo(&fr, &tot));
    const size_t reserve = (size_t)3 << 30;
    NB = fr > reserve ? (long long)((fr - reserve) / (blk_bytes + prm_blk_bytes)) : 0;
  }
  if (NB < cdiv(D.cap, D.bs)) {
    set_err(SART_ENOMEM, "KV pool cannot hold one branch of max_new_tokens");
    sart_destroy(ctx);
    return SART_ENOMEM;
  }
  D.NB = NB;
  if (cfg.kv_pool) {
    // never-written slots of a partially filled stage are multiplied by p = 0 in the attention
    // kernels: they must be finite, so the borrowed pool is zeroed like an allocated one
    ctx->pool = cfg.kv_pool;
    ctx->own_pool = false;
    IC(cudaMemsetAsync(ctx->pool, 0, (size_t)NB * blk_bytes, ctx->st));
  } else {
    IC(dalloc(ctx, &ctx->pool, (size_t)NB * blk_bytes));
  }
  // TMA map of the pool for the tensor-core attention kernels (prefix pass, causal prefill)
  static const bool pf_umma_env = !(getenv("SART_PF_UMMA") && atoi(getenv("SART_PF_UMMA")) == 0);
  ctx->kv_map_ok = ctx->bf16 && D.hd == 128 &&
                   make_kv_map(ctx->kv_map, (const bf16*)ctx->pool, (long long)D.L * NB * 2 * D.kvh * D.bs, D.hd, D.bs);
  if (!ctx->kv_map_ok) ctx->plan.tcq = 0;   // no tensor map: the mma.sync prefix tasks cover every group
  ctx->pf_umma = ctx->kv_map_ok && pf_umma_env;
  if (ctx->prm) {
    ctx->prm->D.NB = NB;
    IC(dalloc(ctx->prm, &ctx->prm->pool, (size_t)NB * prm_blk_bytes));
    const Dims& PD = ctx->prm->D;
    ctx->prm->kv_map_ok = ctx->prm->bf16 && PD.hd == 128 &&
                          make_kv_map(ctx->prm->kv_map, (const bf16*)ctx->prm->pool,
                                      (long long)PD.L * NB * 2 * PD.kvh * PD.bs, PD.hd, PD.bs);
    ctx->prm->pf_umma = ctx->prm->kv_map_ok && pf_umma_env;
  }
  IC(dalloc(ctx, &ctx->free_stack, sizeof(int) * (size_t)NB, false));
  {
    std::vector<int> fs(NB);
    for (long long i = 0; i < NB; ++i) fs[i] = (int)(NB - 1 - i);   // bottom -> top: NB-1 ... 0
    IC(dsync(cudaMemcpy(ctx->free_stack, fs.data(), sizeof(int) * NB, cudaMemcpyHostToDevice)));
    Ctr c0{};
    c0.free_top = NB;
    IC(dsync(cudaMemcpy(ctx->ctr, &c0, sizeof(Ctr), cudaMemcpyHostToDevice)));
  }
  ctx->free_top = NB;
  ctx->slots.resize(D.S);
  ctx->fill_ready.assign(D.S, 1);
  ctx->last_slot_id.assign(D.S, -1);
  for (int s = D.S - 1; s >= 0; --s) ctx->free_slots.push_back(s);
  if (cfg.profile) {
    ctx->ev_pool.resize(3 * D.L * D.T + 3);
    for (auto& ev : ctx->ev_pool) IC(cudaEventCreate(&ev));
  }
  IC(cudaStreamSynchronize(ctx->st));
  *out = ctx;
  return SART_OK;
}

int sart_admit(sart_ctx* ctx, const sart_request* r) {
  if (!ctx || !r) return set_err(SART_EINVAL, "null argument");
  if (ctx->poisoned) return set_err(SART_ESTATE, "ctx poisoned by an earlier CUDA error");
  const Dims& D = ctx->D;
  if (!(1 <= r->M && r->M <= r->N && r->N <= SART_MAXN)) return set_err(SART_EINVAL, "need 1 <= M <= N <= 32");
  int beta = r->beta == -1 ? r->N / 2 : r->beta;
  if (beta < 0 || beta > r->N - 1) return set_err(SART_EINVAL, "need 0 <= beta <= N-1");
  if (std::isnan(r->prune_threshold) || r->prune_threshold > 1.f) return set_err(SART_EINVAL, "alpha > 1 or NaN");
  if (!r->prompt || r->prompt_len < 1 || r->prompt_len > ctx->cfg.max_prompt)
    return set_err(SART_EINVAL, "prompt_len out of range");
  for (int i = 0; i < r->prompt_len; ++i)
    if (r->prompt[i] < 0 || r->prompt[i] >= D.V) return set_err(SART_EINVAL, "prompt token out of range");
  HostReq q;
  q.id = r->request_id;
  q.N = r->N;
  q.M = r->M;
  q.beta = beta;
  q.alpha = r->prune_threshold;
  if (r->script) {
    const sart_script* s = r->script;
    if ((s->scores == nullptr) != (s->final_score == nullptr))
      return set_err(SART_EINVAL, "scores and final_score must both be given or both NULL");
    if (s->scores) {
      if (s->n_bnd < 1) return set_err(SART_EINVAL, "n_bnd >= 1 required with scores");
      q.has_script = true;
      q.sc.n_bnd = s->n_bnd;
      q.sc.scores.assign(s->scores, s->scores + (size_t)r->N * s->n_bnd);
      q.sc.final_score.assign(s->final_score, s->final_score + r->N);
    }
    if (s->forced_len) {
      for (int b = 0; b < r->N; ++b)
        if (s->forced_len[b] < 1 || s->forced_len[b] > D.cap) return set_err(SART_EINVAL, "forced_len out of range");
      q.sc.forced_len.assign(s->forced_len, s->forced_len + r->N);
    }
    if (s->answer) q.sc.answer.assign(s->answer, s->answer + r->N);
    if (s->forced_tokens) {
      if (!ctx->cfg.enable_forced_tokens) return set_err(SART_EINVAL, "forced_tokens needs enable_forced_tokens");
      for (size_t i = 0; i < (size_t)r->N * D.cap; ++i)   // they become embedding indices and history
        if (s->forced_tokens[i] < 0 || s->forced_tokens[i] >= D.V) return set_err(SART_EINVAL, "forced token out of range");
      q.sc.forced_tokens.assign(s->forced_tokens, s->forced_tokens + (size_t)r->N * D.cap);
    }
  }
  const long long need = cdiv(r->prompt_len - 1, D.bs) + cdiv(D.cap, D.bs);
  if (need > D.NB) return set_err(SART_ENOMEM, "request can never fit the KV pool");
  if (ctx->seen_ids.count(r->request_id)) return set_err(SART_EDUP, "request_id reused");
  ctx->seen_ids.insert(r->request_id);
  q.prompt.assign(r->prompt, r->prompt + r->prompt_len);
  q.admit_ns = now_ns();
  q.arrival_ns = r->arrival_ns ? r->arrival_ns : q.admit_ns;
  ctx->request_queue.push_back(std::move(q));
  return SART_OK;
}

static void fill_stats(sart_ctx* ctx, sart_stats* o) {
  if (!o) return;
  o->windows = ctx->windows;
  o->steps = ctx->steps;
  o->live_rows = ctx->n_rows;
  o->queued_branches = (int)ctx->branch_queue.size();
  o->queued_requests = (int)ctx->request_queue.size();
  o->finalized_total = ctx->finalized_total;
  o->free_blocks = (int)ctx->free_top;
  o->committed_blocks = (int)ctx->committed;
  o->branch_tokens = ctx->branch_tokens;
}

int sart_step(sart_ctx* ctx, int32_t max_windows, sart_stats* out) {
  if (!ctx) return set_err(SART_EINVAL, "null ctx");
  if (ctx->poisoned) return set_err(SART_ESTATE, "ctx poisoned by an earlier CUDA error");
  if (max_windows < 0) return set_err(SART_EINVAL, "max_windows < 0");
  if (ctx->tp > 1 && !ctx->tp_connected) return set_err(SART_ESTATE, "tensor-parallel ctx not connected (sart_tp_connect)");
  cudaSetDevice(ctx->cfg.device);
  for (int w = 0; w < max_windows; ++w) {
    if (ctx->cfg.profile) {   // window start, before the fill (and an inline prefill)
      while ((int)ctx->step_ev.size() < ctx->D.T + 1) {
        cudaEvent_t e;
        if (cudaEventCreate(&e) != cudaSuccess) return set_err(SART_ECUDA, "event create");
        ctx->step_ev.push_back(e);
      }
      if (cudaEventRecord(ctx->step_ev[0], ctx->st) != cudaSuccess) return set_err(SART_ECUDA, "event record");
    }
    int rc = fill(ctx);
    if (rc) return rc;
    if (ctx->n_rows == 0) break;   // idle
    rc = ctx->bf16 ? run_window<bf16>(ctx) : run_window<float>(ctx);
    if (rc) return rc;
  }
  fill_stats(ctx, out);
  return SART_OK;
}

int sart_export_counters(sart_ctx* ctx, void* dev) {
  if (!ctx || !dev) return set_err(SART_EINVAL, "null argument");
  if (ctx->poisoned) return set_err(SART_ESTATE, "ctx poisoned");
  int32_t c[16] = {ctx->n_rows, (int32_t)ctx->branch_queue.size(), (int32_t)ctx->request_queue.size(),
                   (int32_t)ctx->free_top, (int32_t)ctx->committed, ctx->finalized_total, ctx->windows, ctx->steps,
                   (int32_t)(ctx->branch_tokens & 0xffffffff), (int32_t)(ctx->branch_tokens >> 32), 0, 0, 0, 0, 0, 0};
  CK(xfer(ctx, dev, c, sizeof(c), cudaMemcpyHostToDevice, ctx->st));
  CK(cudaStreamSynchronize(ctx->st));   // the record is in device memory on return (any stream may read it)
  return SART_OK;
}

int sart_collect(sart_ctx* ctx, sart_result* out, int32_t cap, int32_t* n_out, int32_t* tokens_out,
                 int64_t tokens_cap) {
  if (!ctx || !n_out || (cap > 0 && !out)) return set_err(SART_EINVAL, "null argument");
  if (ctx->poisoned) return set_err(SART_ESTATE, "ctx poisoned");
  int n = 0;
  int64_t used = 0;
  while (!ctx->results.empty() && n < cap) {
    HostResult& hr = ctx->results.front();
    if (used + hr.r.tokens_len > tokens_cap || (hr.r.tokens_len > 0 && !tokens_out)) break;
    out[n] = hr.r;
    out[n].tokens_offset = used;
    if (hr.r.tokens_len > 0) memcpy(tokens_out + used, hr.tokens.data(), sizeof(int32_t) * hr.r.tokens_len);
    used += hr.r.tokens_len;
    ++n;
    ctx->results.pop_front();
  }
  *n_out = n;
  if (!ctx->results.empty()) return set_err(SART_EFULL, "output buffers full; remaining results kept");
  return SART_OK;
}

int sart_get_state(sart_ctx* ctx, sart_state* st) {
  if (!ctx || !st) return set_err(SART_EINVAL, "null argument");
  if (ctx->poisoned) return set_err(SART_ESTATE, "ctx poisoned");
  const Dims& D = ctx->D;
  CK(cudaStreamSynchronize(ctx->st));
  const int n = ctx->n_rows;
  st->n_rows = n;
  st->n_free = (int)ctx->free_top;
  st->committed = (int)ctx->committed;
  if (n > st->rows_cap || st->n_free > st->free_cap) return set_err(SART_EFULL, "state buffers too small");
  std::vector<int> slot(n), b(n), ell(n), nbnd(n), nblk(n), tab((size_t)n * D.MBR);
  if (n) {
    CK(cudaMemcpy(slot.data(), ctx->rows.slot, 4 * n, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(b.data(), ctx->rows.b, 4 * n, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(ell.data(), ctx->rows.ell, 4 * n, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(nbnd.data(), ctx->rows.nbnd, 4 * n, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(nblk.data(), ctx->rows.nblk, 4 * n, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(tab.data(), ctx->rows.table, 4 * tab.size(), cudaMemcpyDeviceToHost));
  }
  for (int r = 0; r < n; ++r) {
    if (st->row_request_id) st->row_request_id[r] = ctx->slots[slot[r]].id;
    if (st->row_branch) st->row_branch[r] = b[r];
    if (st->row_ell) st->row_ell[r] = ell[r];
    if (st->row_nbnd) st->row_nbnd[r] = nbnd[r];
    if (st->row_table)
      for (int j = 0; j < st->table_cap; ++j)
        st->row_table[(size_t)r * st->table_cap + j] = j < nblk[r] && j < D.MBR ? tab[(size_t)r * D.MBR + j] : -1;
  }
  if (st->free_stack && st->n_free)
    CK(cudaMemcpy(st->free_stack, ctx->free_stack, 4 * (size_t)st->n_free, cudaMemcpyDeviceToHost));
  // live requests ascending by id
  std::vector<std::pair<int64_t, int>> live;
  for (int s = 0; s < D.S; ++s)
    if (ctx->slots[s].live) live.emplace_back(ctx->slots[s].id, s);
  std::sort(live.begin(), live.end());
  st->n_live = (int)live.size();
  if ((int)live.size() > st->live_cap) return set_err(SART_EFULL, "live_cap too small");
  for (size_t i = 0; i < live.size(); ++i) {
    const int s = live[i].second;
    int v[6];
    float thr;
    CK(cudaMemcpy(&v[0], ctx->reqs.phase + s, 4, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(&thr, ctx->reqs.thr + s, 4, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(&v[1], ctx->reqs.maxp + s, 4, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(&v[2], ctx->reqs.nc + s, 4, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(&v[3], ctx->reqs.np + s, 4, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(&v[4], ctx->reqs.npre + s, 4, cudaMemcpyDeviceToHost));
    if (st->live_request_id) st->live_request_id[i] = live[i].first;
    if (st->live_phase) st->live_phase[i] = v[0];
    if (st->live_threshold) st->live_threshold[i] = thr;
    if (st->live_max_pruned) st->live_max_pruned[i] = v[1];
    if (st->live_completed) st->live_completed[i] = v[2];
    if (st->live_pruned) st->live_pruned[i] = v[3];
    if (st->live_prefix_n) st->live_prefix_n[i] = v[4];
    if (st->live_prefix && v[4] > 0) {
      std::vector<int> pre(v[4]);
      CK(cudaMemcpy(pre.data(), ctx->reqs.prefix + (size_t)s * D.MPB, 4 * v[4], cudaMemcpyDeviceToHost));
      for (int j = 0; j < st->prefix_cap; ++j)
        st->live_prefix[i * st->prefix_cap + j] = j < v[4] ? pre[j] : -1;
    }
  }
  return SART_OK;
}

int sart_debug_fetch(sart_ctx* ctx, int32_t what, int32_t layer, void* host_out, size_t bytes, int32_t* n_rows) {
  if (!ctx || !host_out) return set_err(SART_EINVAL, "null argument");
  if (ctx->poisoned) return set_err(SART_ESTATE, "ctx poisoned");
  const Dims& D = ctx->D;
  const int n = ctx->last_n;
  if (n_rows) *n_rows = n;
  CK(cudaStreamSynchronize(ctx->st));
  size_t need = 0;
  const void* src = nullptr;
  switch (what) {
    case SART_DBG_LOGITS: need = (size_t)n * D.V * 4; src = ctx->logits; break;
    case SART_DBG_TOKENS: need = (size_t)n * 4; src = ctx->dbg_tok; break;
    case SART_DBG_SCORES:
    case SART_DBG_PRM_SCORES: need = (size_t)n * 4; src = ctx->prm ? ctx->prm->prm_score : ctx->prm_score; break;
    case SART_DBG_Z: need = (size_t)n * D.d * 4; src = ctx->z32; break;
    case SART_DBG_ATTN:
      if (!ctx->dbg_attn || layer < 0 || layer >= D.L) return set_err(SART_EINVAL, "needs debug_capture and a layer");
      need = (size_t)n * D.qh * D.hd * 4;
      src = ctx->dbg_attn + (size_t)layer * D.R * D.qh * D.hd;
      break;
    case SART_DBG_ROWIDS: {
      need = (size_t)n * 8;
      if (bytes < need) return set_err(SART_EFULL, "buffer too small");
      std::vector<int> slot(n), b(n);
      if (n) {
        CK(cudaMemcpy(slot.data(), ctx->dbg_slot, 4 * n, cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(b.data(), ctx->dbg_b, 4 * n, cudaMemcpyDeviceToHost));
      }
      int64_t* o = (int64_t*)host_out;
      for (int r = 0; r < n; ++r) o[r] = (ctx->last_slot_id[slot[r]] << 8) | b[r];
      return SART_OK;
    }
    default: return set_err(SART_EINVAL, "unknown debug tensor");
  }
  if (bytes < need) return set_err(SART_EFULL, "buffer too small");
  if (need) CK(cudaMemcpy(host_out, src, need, cudaMemcpyDeviceToHost));
  return SART_OK;
}

int sart_debug_gemm(int32_t M, int32_t N, int32_t K, const uint16_t* A, const uint16_t* B, const float* bias,
                    float* C, int32_t mode, int32_t splits, int32_t bn, int32_t bm) {
  if (M < 1 || N < 1 || K < 1 || !A || !B || !C || mode < 0 || mode > 2 || splits < 1 || splits > 8 ||
      (bn != 64 && bn != 128 && bn != 256 && !(bn == 512 && getenv("SART_DEBUG_2SM"))) || (bm != 128 && bm != 256))
    return set_err(SART_EINVAL, "bad args");
  bf16 *dA = nullptr, *dB = nullptr, *dact = nullptr, *dBt = nullptr;
  float *dC = nullptr, *dbias = nullptr;
  const size_t outn = mode == GEMM_SWIGLU ? (size_t)M * (N / 2) : (size_t)M * N;
  cudaError_t e = cudaSuccess;
  auto chk = [&](cudaError_t x) { if (x != cudaSuccess && e == cudaSuccess) e = x; };
  chk(cudaMalloc(&dA, 2 * (size_t)M * K));
  chk(cudaMalloc(&dB, 2 * (size_t)N * K));
  chk(cudaMalloc(&dC, 4 * (size_t)M * N * splits));
  chk(cudaMalloc(&dact, 2 * outn));
  if (bias) chk(cudaMalloc(&dbias, 4 * (size_t)N));
  if (e == cudaSuccess) {
    chk(cudaMemcpy(dA, A, 2 * (size_t)M * K, cudaMemcpyHostToDevice));
    chk(cudaMemcpy(dB, B, 2 * (size_t)N * K, cudaMemcpyHostToDevice));
    if (bias) chk(cudaMemcpy(dbias, bias, 4 * (size_t)N, cudaMemcpyHostToDevice));
    if (mode == GEMM_ACCUM) chk(cudaMemcpy(dC, C, 4 * (size_t)M * N, cudaMemcpyHostToDevice));
    // SART_GEMM_BTILED=1: run from the pre-tiled weight layout (what the engine uses)
    const bool tiled = getenv("SART_GEMM_BTILED") && atoi(getenv("SART_GEMM_BTILED"));
    if (tiled) {
      chk(cudaMalloc(&dBt, 2 * tiled_b_elems(N, K, bn)));
      if (e == cudaSuccess) launch_tile_b(dB, dBt, N, K, bn, 0);
    }
    chk(cudaDeviceSynchronize());   // the kernel prefetches B before its PDL wait: B must be resident
    if (getenv("SART_DEBUG_2SM")) {   // the CTA-pair kernel on the same problem (pair tile 256 x bn)
      if (!launch_gemm_2sm(dA, dB, dbias, dC, dact, M, N, K, mode, splits, bn, 0)) e = cudaErrorInvalidValue;
    } else if (!launch_gemm_tc_split(dA, dB, dbias, dC, dact, M, N, K, mode, splits, bn, bm / 128, 0, dBt))
      e = cudaErrorInvalidValue;
    chk(cudaGetLastError());
    chk(cudaDeviceSynchronize());
    if (const char* reps_s = getenv("SART_GEMM_BENCH_REPS")) {   // micro-benchmark (tools/gemm_sweep.py)
      const int reps = atoi(reps_s);
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      // SART_GEMM_BENCH_COPIES=n: cycle over n copies of B so that the weights stream from HBM
      // (n x |B| > L2) as they do in a decode step, instead of staying L2-resident
      const int ncp = getenv("SART_GEMM_BENCH_COPIES") ? std::max(1, atoi(getenv("SART_GEMM_BENCH_COPIES"))) : 1;
      std::vector<bf16*> Bs(1, tiled ? dBt : dB);
      const size_t bel = tiled ? tiled_b_elems(N, K, bn) : (size_t)N * K;
      for (int i = 1; i < ncp; ++i) {
        bf16* p = nullptr;
        if (cudaMalloc(&p, 2 * bel) != cudaSuccess) break;
        cudaMemcpy(p, Bs[0], 2 * bel, cudaMemcpyDeviceToDevice);
        Bs.push_back(p);
      }
      auto run = [&](bf16* p) {
        if (tiled) launch_gemm_tc_split(dA, dB, dbias, dC, dact, M, N, K, mode, splits, bn, bm / 128, 0, p);
        else launch_gemm_tc_split(dA, p, dbias, dC, dact, M, N, K, mode, splits, bn, bm / 128, 0);
      };
      for (auto p : Bs) run(p);
      cudaDeviceSynchronize();
      cudaEventRecord(a, 0);
      for (int i = 0; i < reps; ++i) run(Bs[i % Bs.size()]);
      cudaEventRecord(b, 0);
      cudaEventSynchronize(b);
      float ms = 0.f;
      cudaEventElapsedTime(&ms, a, b);
      fprintf(stderr, "GEMMBENCH M=%d N=%d K=%d mode=%d S=%d BM=%d BN=%d copies=%d tiled=%d us=%.2f TFLOPs=%.1f\n", M,
              N, K, mode, splits, bm, bn, (int)Bs.size(), (int)tiled,
              1e3 * ms / reps, 2.0 * M * N * K / (ms / reps * 1e-3) / 1e12);
      cudaEventDestroy(a);
      cudaEventDestroy(b);
      for (size_t i = 1; i < Bs.size(); ++i) cudaFree(Bs[i]);
    }
    if (getenv("SART_GEMM_TS")) {
      gemm_ts_reset();
      for (int i = 0; i < 4; ++i) launch_gemm_tc_split(dA, dB, dbias, dC, dact, M, N, K, mode, splits, bn, bm / 128, 0);
      cudaDeviceSynchronize();
      unsigned long long h[4][10];
      gemm_ts_fetch(&h[0][0]);
      for (int i = 0; i < 4; ++i) {
        fprintf(stderr, "GEMMTS M=%d N=%d K=%d S=%d BM=%d BN=%d launch %d:", M, N, K, splits, bm, bn, i);
        for (int j = 1; j < 9; ++j) fprintf(stderr, " %lld", (long long)(h[i][j] - h[i][0]));
        if (i) fprintf(stderr, " | start-after-prev-start %lld prev-end->start %lld", (long long)(h[i][0] - h[i - 1][0]),
                       (long long)(h[i][0] - h[i - 1][8]));
        fprintf(stderr, "\n");
      }
      unsigned long long tr[2][64];
      gemm_trace_fetch(&tr[0][0]);
      fprintf(stderr, "GEMMTRACE M=%d N=%d K=%d S=%d BN=%d (ns from first issue) issue/landed:", M, N, K, splits, bn);
      for (int k = 0; k < 64 && tr[1][k] >= tr[0][0] && tr[1][k] - tr[0][0] < 1000000; ++k)
        fprintf(stderr, " %lld/%lld", (long long)(tr[0][k] - tr[0][0]), (long long)(tr[1][k] - tr[0][0]));
      fprintf(stderr, "\n");
    }
    if (mode == GEMM_SWIGLU) {
      std::vector<uint16_t> h(outn);
      chk(cudaMemcpy(h.data(), dact, 2 * outn, cudaMemcpyDeviceToHost));
      for (size_t i = 0; i < outn; ++i) {
        uint32_t u = (uint32_t)h[i] << 16;
        memcpy(&C[i], &u, 4);
      }
    } else {
      chk(cudaMemcpy(C, dC, 4 * (size_t)M * N * splits, cudaMemcpyDeviceToHost));
    }
  }
  cudaFree(dA); cudaFree(dB); cudaFree(dC); cudaFree(dact); if (dbias) cudaFree(dbias); if (dBt) cudaFree(dBt);
  if (e != cudaSuccess) return set_err(SART_ECUDA, cudaGetErrorString(e));
  return SART_OK;
}

int sart_debug_prm_plan(const int32_t* ell_ws, const int32_t* ell, int32_t n, int32_t chunk, int32_t qp,
                        int32_t* out, int32_t cap, int32_t* n_seg, int32_t* n_qb, int32_t* n_gat, int32_t* chunks,
                        int32_t chunk_cap, int32_t* n_chunks) {
  if ((n > 0 && (!ell_ws || !ell)) || !out || !n_seg || !n_qb || !n_gat || !chunks || !n_chunks || n < 0 ||
      chunk < 1 || qp < 1)
    return set_err(SART_EINVAL, "bad args");
  for (int r = 0; r < n; ++r)
    if (ell[r] < ell_ws[r]) return set_err(SART_EINVAL, "ell < ell_ws");
  const PrmPlan P = plan_prm_pass(ell_ws, ell, n, chunk, qp);
  *n_seg = (int32_t)P.seg.size();
  *n_qb = (int32_t)P.qb.size();
  *n_gat = (int32_t)P.gat.size();
  *n_chunks = (int32_t)P.chunks.size();
  const size_t nd = P.seg.size() + P.qb.size() + P.gat.size();
  if (nd > (size_t)cap || P.chunks.size() > (size_t)chunk_cap) return set_err(SART_EFULL, "buffers too small");
  int32_t* o = out;
  for (const auto* v : {&P.seg, &P.qb, &P.gat})
    for (const int4& x : *v) { o[0] = x.x; o[1] = x.y; o[2] = x.z; o[3] = x.w; o += 4; }
  for (size_t c = 0; c < P.chunks.size(); ++c) {
    const PrmPlan::Chunk& k = P.chunks[c];
    chunks[4 * c] = k.ntok; chunks[4 * c + 1] = k.nseg; chunks[4 * c + 2] = k.nqb; chunks[4 * c + 3] = k.ngat;
  }
  return SART_OK;
}

int sart_debug_tp_segments(const sart_config* cfg, int32_t tensor, int64_t* out, int32_t cap, int32_t* n_out) {
  if (!cfg || !out || !n_out) return set_err(SART_EINVAL, "null argument");
  const int tp = cfg->tp_size < 1 ? 1 : cfg->tp_size;
  if (cfg->tp_rank < 0 || cfg->tp_rank >= tp || cfg->n_heads % tp || cfg->n_kv_heads % tp || cfg->d_ff % tp ||
      cfg->n_layers < 1 || cfg->head_dim < 1)
    return set_err(SART_EINVAL, "bad tp / dims");
  Dims F{};
  F.L = cfg->n_layers; F.d = cfg->d_model; F.qh = cfg->n_heads; F.kvh = cfg->n_kv_heads; F.hd = cfg->head_dim;
  F.F = cfg->d_ff; F.V = cfg->vocab; F.qkv = (F.qh + 2 * F.kvh) * F.hd;
  if (tensor < 0 || tensor >= (int)tensor_sizes(F).size()) return set_err(SART_EINVAL, "tensor index");
  const std::vector<Seg> g = shard_segments(F, tp, cfg->tp_rank, tensor);
  *n_out = (int32_t)g.size();
  if ((int)g.size() > cap) return set_err(SART_EFULL, "cap too small");
  for (size_t i = 0; i < g.size(); ++i) {
    const int64_t v[6] = {g[i].loff, g[i].n, g[i].cl, g[i].cf, g[i].c0, g[i].goff};
    memcpy(out + 6 * i, v, sizeof(v));
  }
  return SART_OK;
}

int sart_tp_buffer(sart_ctx* ctx, void** dev_ptr, void* ipc_handle) {
  if (!ctx || !dev_ptr) return set_err(SART_EINVAL, "null argument");
  if (ctx->tp <= 1) return set_err(SART_EINVAL, "tp_size <= 1");
  *dev_ptr = ctx->tp_buf;
  if (ipc_handle) {
    cudaSetDevice(ctx->cfg.device);
    cudaIpcMemHandle_t h;
    CK(cudaIpcGetMemHandle(&h, ctx->tp_buf));
    static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
    memcpy(ipc_handle, &h, 64);
  }
  return SART_OK;
}

int sart_tp_connect(sart_ctx* ctx, void* const* peer_ptrs, const void* ipc_handles) {
  if (!ctx) return set_err(SART_EINVAL, "null ctx");
  if (ctx->tp <= 1) return set_err(SART_EINVAL, "tp_size <= 1");
  if ((peer_ptrs == nullptr) == (ipc_handles == nullptr)) return set_err(SART_EINVAL, "give peer_ptrs or ipc_handles");
  if (ctx->tp_connected) return set_err(SART_ESTATE, "already connected");
  cudaSetDevice(ctx->cfg.device);
  std::vector<void*> peers(ctx->tp, nullptr);
  for (int r = 0; r < ctx->tp; ++r) {
    if (r == ctx->tp_rank) { peers[r] = ctx->tp_buf; continue; }
    if (peer_ptrs) {
      if (!peer_ptrs[r]) return set_err(SART_EINVAL, "null peer pointer");
      peers[r] = peer_ptrs[r];
    } else {
      cudaIpcMemHandle_t h;
      memcpy(&h, (const char*)ipc_handles + 64 * (size_t)r, 64);
      void* p = nullptr;
      const cudaError_t e = cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess);
      if (e != cudaSuccess) {
        for (void* q : ctx->tp_opened) cudaIpcCloseMemHandle(q);
        ctx->tp_opened.clear();
        return set_err(SART_ECUDA, std::string("cudaIpcOpenMemHandle: ") + cudaGetErrorString(e));
      }
      ctx->tp_opened.push_back(p);
      peers[r] = p;
    }
  }
  ctx->tp_peer = peers;
  ctx->tp_connected = true;
  return SART_OK;
}

int sart_trace_fetch(sart_ctx* ctx, sart_trace_row* rows, int64_t rows_cap, int64_t* n_rows, int32_t* tokens_out,
                     int64_t tokens_cap, int64_t* n_tokens, uint64_t* hashes, int64_t hashes_cap, int64_t* n_hashes) {
  if (!ctx || !n_rows || !n_tokens || !n_hashes) return set_err(SART_EINVAL, "null argument");
  if (!ctx->cfg.record_trace) return set_err(SART_EINVAL, "record_trace is off");
  *n_rows = (int64_t)ctx->trace_rows.size();
  *n_tokens = (int64_t)ctx->trace_tokens.size();
  *n_hashes = (int64_t)ctx->trace_hashes.size();
  if (*n_rows > rows_cap || *n_tokens > tokens_cap || *n_hashes > hashes_cap)
    return set_err(SART_EFULL, "trace buffers too small (counts written, nothing moved)");
  if ((*n_rows && !rows) || (*n_tokens && !tokens_out) || (*n_hashes && !hashes))
    return set_err(SART_EINVAL, "null buffer");
  if (*n_rows) memcpy(rows, ctx->trace_rows.data(), sizeof(sart_trace_row) * (size_t)*n_rows);
  if (*n_tokens) memcpy(tokens_out, ctx->trace_tokens.data(), sizeof(int32_t) * (size_t)*n_tokens);
  if (*n_hashes) memcpy(hashes, ctx->trace_hashes.data(), sizeof(uint64_t) * (size_t)*n_hashes);
  ctx->trace_rows.clear();
  ctx->trace_tokens.clear();
  ctx->trace_hashes.clear();
  return SART_OK;
}

int sart_get_profile(sart_ctx* ctx, sart_profile* o) {
  if (!ctx || !o) return set_err(SART_EINVAL, "null argument");
  o->attn_ms = ctx->attn_ms;
  o->attn_launches = ctx->attn_launches;
  o->attn_bytes = ctx->attn_bytes;
  o->kernel_launches = ctx->launches;
  o->prefill_ms = ctx->prefill_ms;
  o->prm_ms = ctx->prm_ms;
  o->prm_tokens = ctx->prm_tokens;
  o->prm_passes = ctx->prm_passes;
  o->h2d_bytes = ctx->h2d_bytes;
  o->d2h_bytes = ctx->d2h_bytes;
  o->first_step_ms_max = ctx->first_step_ms_max;
  o->step_ms_max = ctx->step_ms_max;
  o->prefix_tc_windows = ctx->prefix_tc_windows;
  o->attn_stream_ms = ctx->attn_stream_ms;
  return SART_OK;
}
int sart_set_profile(sart_ctx* ctx, int32_t enable) {
  if (!ctx) return set_err(SART_EINVAL, "null argument");
  if (enable && ctx->ev_pool.empty()) {
    ctx->ev_pool.resize(3 * ctx->D.L * ctx->D.T + 3);
    for (auto& ev : ctx->ev_pool)
      if (cudaEventCreate(&ev) != cudaSuccess) return set_err(SART_ECUDA, "event create");
  }
  ctx->cfg.profile = enable == 2 ? 2 : (enable ? 1 : 0);
  return SART_OK;
}

int sart_reset_profile(sart_ctx* ctx) {
  if (!ctx) return set_err(SART_EINVAL, "null argument");
  ctx->attn_bytes_base += ctx->attn_bytes;
  ctx->attn_ms = ctx->attn_bytes = ctx->prefill_ms = ctx->prm_ms = ctx->attn_stream_ms = 0;
  ctx->prm_tokens = ctx->prm_passes = 0;
  ctx->attn_launches = ctx->launches = 0;
  ctx->h2d_bytes = ctx->d2h_bytes = 0;
  ctx->first_step_ms_max = ctx->step_ms_max = 0;
  ctx->prefix_tc_windows = 0;
  return SART_OK;
}

}  // extern "C"
