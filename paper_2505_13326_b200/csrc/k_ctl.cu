// On-device branch control: admission append, and the window
// boundary -- PRM score selection, Algorithm 1 L23-40 (phase switch, completions, pruning,
// finalize / early stop), vote and max-reward selection, KV-block reclamation onto the
// free stack, stable compaction of current_batch and next-window reservation.
//
// Everything runs in ONE CTA of 1024 threads so every ordering rule of the allocator
// (R23: batch-row order, logical block order, ascending request_id for prefixes, LIFO)
// is a deterministic prefix sum.  Readings R2-R8, R16-R21, R31, R34, R35.
#include "kernels.h"

namespace {
constexpr int NT = 1024;

__device__ __forceinline__ int cdiv(int a, int b) { return (a + b - 1) / b; }

// Exclusive prefix sum over the CTA; *total gets the sum.  All threads must call.
__device__ int cta_excl_scan(int v, int* total) {
  __shared__ int ws[NT / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  __syncthreads();
  if (lane == 31) ws[warp] = x;
  __syncthreads();
  if (warp == 0) {
    int w = ws[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    ws[lane] = w;
  }
  __syncthreads();
  int before = warp > 0 ? ws[warp - 1] : 0;
  *total = ws[NT / 32 - 1];
  return before + x - v;
}

__device__ __forceinline__ void copy_row(const Dims& D, Rows dst, int di, Rows src, int si) {
  dst.slot[di] = src.slot[si];
  dst.b[di] = src.b[si];
  dst.ell[di] = src.ell[si];
  dst.status[di] = src.status[si];
  dst.done_step[di] = src.done_step[si];
  dst.done_wstep[di] = src.done_wstep[si];
  dst.nbnd[di] = src.nbnd[si];
  dst.tok[di] = src.tok[si];
  dst.term[di] = src.term[si];
  dst.nblk[di] = src.nblk[si];
  dst.start[di] = src.start[si];
  dst.score[di] = src.score[si];
  for (int j = 0; j < src.nblk[si]; ++j) dst.table[(long long)di * D.MBR + j] = src.table[(long long)si * D.MBR + j];
}
}  // namespace

// ------------------------------------------------------------------ window begin
__global__ void k_window_begin(Ctr* ctr, int n) {
  ctr->live = n;
  ctr->wstep = 0;
  ctr->n_final = 0;
}
void launch_window_begin(Ctr* ctr, int n, cudaStream_t s) { k_window_begin<<<1, 1, 0, s>>>(ctr, n); }

// ------------------------------------------------------------------ admission (Alg. 1 L3-19)
// Events come from the host fill loop in order; pops are taken from the top of the free
// stack in event order (R23 step 4: a prefill pops its prefix blocks, a new row pops its
// first-window blocks).  Offsets are precomputed by the host.
__global__ void __launch_bounds__(NT) k_admit(const AdmitEvent* __restrict__ ev, int n_ev, int total_pop,
                                               int new_rows, int commit_delta, Dims D, Rows rows, Reqs reqs,
                                               int* __restrict__ fs, Ctr* ctr) {
  const long long top = ctr->free_top;
  const int nfirst = cdiv(min(D.T, D.cap), D.bs);
  for (int e = threadIdx.x; e < n_ev; e += NT) {
    const AdmitEvent E = ev[e];
    const int slot = E.slot;
    if (E.type == 0) {
      for (int j = 0; j < E.npre; ++j) reqs.prefix[(long long)slot * D.MPB + j] = fs[top - 1 - (E.pop_off + j)];
      reqs.id[slot] = E.id;
      reqs.N[slot] = E.N;
      reqs.M[slot] = E.M;
      reqs.P[slot] = E.P;
      reqs.beta[slot] = E.beta;
      reqs.prune[slot] = E.prune;
      reqs.npre[slot] = E.npre;
      reqs.first_tok[slot] = E.first_tok;
      reqs.has_script[slot] = E.has_script;
      reqs.has_answer[slot] = E.has_answer;
      reqs.has_forced[slot] = E.has_forced;
      reqs.nbnd[slot] = E.nbnd;
      reqs.alpha[slot] = E.alpha;
      // Alg. 1 L16: meta[i] <- {phase = explore, threshold = alpha, max_num_pruned = beta, 0, 0}
      reqs.phase[slot] = 0;
      reqs.thr[slot] = E.alpha;
      reqs.maxp[slot] = E.beta;
      reqs.nc[slot] = 0;
      reqs.ncw[slot] = 0;
      reqs.np[slot] = 0;
      reqs.nes[slot] = 0;
      reqs.final_flag[slot] = 0;
      for (int b = 0; b < SART_MAXN; ++b) {
        long long sb = (long long)slot * SART_MAXN + b;
        reqs.br_state[sb] = 0;
        reqs.br_len[sb] = 0;
        reqs.br_label[sb] = -1;
        reqs.br_score[sb] = 0.f;
      }
    } else {
      const int r = E.row;
      for (int j = 0; j < nfirst; ++j) rows.table[(long long)r * D.MBR + j] = fs[top - 1 - (E.pop_off + j)];
      rows.slot[r] = slot;
      rows.b[r] = E.b;
      rows.ell[r] = 0;
      rows.start[r] = E.start;
      rows.status[r] = E.start > 1 ? ST_WAIT : RUNNING_ST;   // R44: waits for its interleaved prefill
      rows.done_step[r] = 0;
      rows.done_wstep[r] = 0;
      rows.nbnd[r] = 0;
      rows.tok[r] = E.first_tok;           // prompt[P-1] is every branch's first input (R22)
      rows.term[r] = RUNNING_ST;
      rows.nblk[r] = nfirst;
      rows.score[r] = 0.f;
    }
  }
  __syncthreads();
  // branch state RUNNING after the meta init above (a prefill and its rows can share a launch)
  for (int e = threadIdx.x; e < n_ev; e += NT) {
    const AdmitEvent E = ev[e];
    if (E.type == 1) reqs.br_state[(long long)E.slot * SART_MAXN + E.b] = RUNNING_ST;
  }
  if (threadIdx.x == 0) {
    ctr->free_top = top - total_pop;
    ctr->committed += commit_delta;
    ctr->n_rows += new_rows;
  }
}
void launch_admit(const AdmitEvent* ev, int n_ev, int total_pop, int new_rows, int commit_delta, Dims D,
                  Rows rows, Reqs reqs, int* free_stack, Ctr* ctr, cudaStream_t s) {
  k_admit<<<1, NT, 0, s>>>(ev, n_ev, total_pop, new_rows, commit_delta, D, rows, reqs, free_stack, ctr);
}

// ------------------------------------------------------------------ boundary
__global__ void __launch_bounds__(NT) k_boundary(Dims D, Rows rows, Rows tmp, Reqs reqs,
                                                  const float* __restrict__ prm, int* __restrict__ fs, Ctr* ctr,
                                                  DevResult* __restrict__ res, int* __restrict__ slot_row, int n,
                                                  BoundaryTrace tr) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  __shared__ int s_nlead;
  __shared__ int s_lead[NT];
  __shared__ int s_sorted[NT];
  __shared__ int s_preoff[NT + 1];
  __shared__ long long s_top;
  if (tid == 0) { s_nlead = 0; ctr->n_final = 0; }

  // ---- A. PRM / script scores for every row of the window's batch (L25, L33; O6, R35)
  for (int r = tid; r < n; r += NT) {
    const int slot = rows.slot[r], b = rows.b[r];
    const long long sb = (long long)slot * SART_MAXN + b;
    float score;
    if (rows.status[r] == RUNNING_ST || rows.status[r] == ST_STOP || rows.status[r] == ST_WAIT) {   // incomplete (R43, R44)
      const int k = rows.nbnd[r];
      score = reqs.has_script[slot] ? reqs.sc_scores[sb * D.nbnd_max + min(k, reqs.nbnd[slot] - 1)] : prm[r];
      rows.nbnd[r] = k + 1;
    } else {
      score = reqs.has_script[slot] ? reqs.sc_final[sb] : prm[r];
    }
    rows.score[r] = score;
    rows.term[r] = RUNNING_ST;
    slot_row[sb] = r;
    if (tr.score) {   // record_trace (PP2): the score used and the row's state, in window-row order
      tr.score[r] = score;
      tr.state[r] = rows.status[r];
      tr.ell[r] = rows.ell[r];
    }
  }
  __syncthreads();
  // involved requests (R19): one leader row per request (its lowest batch row)
  for (int r = tid; r < n; r += NT) {
    const int slot = rows.slot[r];
    bool lead = true;
    for (int b = 0; b < reqs.N[slot]; ++b) {
      int o = slot_row[(long long)slot * SART_MAXN + b];
      if (o >= 0 && o < r) { lead = false; break; }
    }
    if (lead) s_lead[atomicAdd(&s_nlead, 1)] = slot;
  }
  __syncthreads();

  // ---- B. Alg. 1 L24-40 for each involved request, one warp each (lane = branch index)
  for (int li = warp; li < s_nlead; li += NT / 32) {
    const int slot = s_lead[li];
    const long long sb = (long long)slot * SART_MAXN + lane;
    const int N = reqs.N[slot], M = reqs.M[slot];
    const int r = lane < N ? slot_row[sb] : -1;
    const bool has = r >= 0;
    const int st = has ? rows.status[r] : 0;
    // stopped (es_every_step, R43): incomplete, not prunable, EarlyStopped by the finalize below
    const bool stopped = has && st == ST_STOP;
    const bool running = has && (st == RUNNING_ST || stopped || st == ST_WAIT),
               done = has && (st == ST_EOS || st == ST_CAP);
    const float sc = has ? rows.score[r] : 0.f;
    int phase = reqs.phase[slot], maxp = reqs.maxp[slot], nc = reqs.nc[slot], np = reqs.np[slot];
    float thr = reqs.thr[slot];
    const unsigned dmask = __ballot_sync(0xffffffffu, done);
    // L24-27: first completion (smallest window step, ties lowest branch: R2) sets alpha' (R3, R6)
    if (phase == 0 && dmask) {
      int key = done ? rows.done_wstep[r] * SART_MAXN + lane : 0x7fffffff;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) key = min(key, __shfl_xor_sync(0xffffffffu, key, o));
      thr = __shfl_sync(0xffffffffu, sc, key % SART_MAXN);
      maxp = N - 1;
      phase = 1;
    }
    // L28-31: completed branches (EOS or cap, R17)
    int label = -1;
    if (done) {
      if (reqs.has_answer[slot]) {
        label = reqs.sc_answer[sb];
      } else {                                          // R16: last non-EOS token
        const int len = rows.done_step[r];
        const int idx = st == ST_EOS ? len - 2 : len - 1;
        label = idx >= 0 ? reqs.hist[sb * D.cap + idx] : -1;
      }
      rows.term[r] = st;
      reqs.br_state[sb] = st;
      reqs.br_len[sb] = rows.done_step[r];
      reqs.br_score[sb] = sc;
      reqs.br_label[sb] = label;
    }
    nc += __popc(dmask);
    // L32-37: prune running branches below the threshold in ascending branch index (R4, R5),
    // while num_pruned < max_num_pruned; alpha < 0 disables pruning (R20)
    bool pr = false;
    if (reqs.prune[slot]) {
      const bool cand = running && !stopped && sc < thr;
      const unsigned cm = __ballot_sync(0xffffffffu, cand);
      const int allow = maxp - np;
      const int rank = __popc(cm & ((1u << lane) - 1u));
      pr = cand && rank < allow;
      const unsigned pm = __ballot_sync(0xffffffffu, pr);
      np += __popc(pm);
      if (pr) {
        rows.term[r] = ST_PRUNED;
        reqs.br_state[sb] = ST_PRUNED;
        reqs.br_len[sb] = rows.ell[r];
        reqs.br_score[sb] = sc;
      }
    }
    // L38-40: output; remaining running branches are early-stopped (R7)
    const bool fin = nc >= M || nc + np == N;
    int nes = reqs.nes[slot];
    if (fin) {
      const bool es = running && !pr;
      if (es) {
        rows.term[r] = ST_ES;
        reqs.br_state[sb] = ST_ES;
        reqs.br_len[sb] = rows.ell[r];
        reqs.br_score[sb] = sc;
      }
      nes += __popc(__ballot_sync(0xffffffffu, es));
      __syncwarp();
      // O9 aggregation over all Completed branches of the request
      const int bst = lane < N ? reqs.br_state[sb] : 0;
      const bool comp = bst == ST_EOS || bst == ST_CAP;
      const int lab = comp ? reqs.br_label[sb] : 0;
      const float scr = comp ? reqs.br_score[sb] : 0.f;
      int count = 0;
      for (int j = 0; j < SART_MAXN; ++j) {
        int lj = __shfl_sync(0xffffffffu, lab, j);
        bool cj = __shfl_sync(0xffffffffu, comp, j);
        count += (cj && lj == lab) ? 1 : 0;
      }
      int best = comp ? count : 0;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) best = max(best, __shfl_xor_sync(0xffffffffu, best, o));
      const unsigned wm = __ballot_sync(0xffffffffu, comp && count == best);
      const int winner = __ffs(wm) - 1;
      const int vote = __shfl_sync(0xffffffffu, lab, winner);
      float ms = comp ? scr : -INFINITY;
      int ml = comp ? lane : SART_MAXN;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        float os = __shfl_xor_sync(0xffffffffu, ms, o);
        int ol = __shfl_xor_sync(0xffffffffu, ml, o);
        if (os > ms || (os == ms && ol < ml)) { ms = os; ml = ol; }
      }
      const int amr = __shfl_sync(0xffffffffu, lab, ml & 31);
      DevResult* R = res + slot;
      if (lane < N) {
        R->branch_len[lane] = reqs.br_len[sb];
        R->branch_state[lane] = bst;
        R->branch_score[lane] = reqs.br_score[sb];
      }
      if (lane == 0) {
        R->request_id = reqs.id[slot];
        R->answer_vote = vote;
        R->vote_count = best;
        R->chosen_max_reward = ml;
        R->answer_max_reward = amr;
        R->num_completed = nc;
        R->num_pruned = np;
        R->num_early_stopped = nes;
        R->finalize_reason = nc >= M ? 0 : 1;
        R->phase_at_end = phase;
        R->threshold_at_end = thr;
        R->selected_branch = D.select_mode == 0 ? winner : ml;
        reqs.final_flag[slot] = 1;
        ctr->final_slots[atomicAdd(&ctr->n_final, 1)] = slot;
      }
    }
    if (lane == 0) {
      reqs.phase[slot] = phase;
      reqs.thr[slot] = thr;
      reqs.maxp[slot] = maxp;
      reqs.nc[slot] = nc;
      reqs.ncw[slot] = nc;
      reqs.np[slot] = np;
      reqs.nes[slot] = nes;
    }
  }
  __syncthreads();

  // ---- C. free (R23 step 1): terminated rows in batch-row order, blocks in logical order
  if (tid == 0) s_top = ctr->free_top;
  __syncthreads();
  const long long top0 = s_top;
  int carry = 0, nterm = 0;
  for (int base = 0; base < n; base += NT) {
    const int r = base + tid;
    const bool term = r < n && rows.term[r] != RUNNING_ST;
    int tot, tcount;
    const int off = cta_excl_scan(term ? rows.nblk[r] : 0, &tot);
    const int dummy = cta_excl_scan(term ? 1 : 0, &tcount);
    (void)dummy;
    if (term)
      for (int j = 0; j < rows.nblk[r]; ++j) fs[top0 + carry + off + j] = rows.table[(long long)r * D.MBR + j];
    carry += tot;
    nterm += tcount;
    __syncthreads();
  }
  // then prefix blocks of requests finalized at this boundary, ascending request_id (R21)
  const int nf = ctr->n_final;
  for (int i = tid; i < nf; i += NT) {
    const int si = ctr->final_slots[i];
    const long long id = reqs.id[si];
    int rank = 0;
    for (int j = 0; j < nf; ++j) rank += reqs.id[ctr->final_slots[j]] < id ? 1 : 0;
    s_sorted[rank] = si;
  }
  __syncthreads();
  if (tid == 0) {
    int acc = 0;
    for (int i = 0; i < nf; ++i) { s_preoff[i] = acc; acc += reqs.npre[s_sorted[i]]; }
    s_preoff[nf] = acc;
  }
  __syncthreads();
  for (int i = tid; i < nf; i += NT) {
    const int si = s_sorted[i];
    for (int j = 0; j < reqs.npre[si]; ++j)
      fs[top0 + carry + s_preoff[i] + j] = reqs.prefix[(long long)si * D.MPB + j];
  }
  const int pre_total = s_preoff[nf];
  long long top = top0 + carry + pre_total;
  // reset the slot -> row map for the next boundary
  for (int r = tid; r < n; r += NT) slot_row[(long long)rows.slot[r] * SART_MAXN + rows.b[r]] = -1;
  __syncthreads();

  // ---- D. stable compaction of current_batch (R23 step 2)
  int nk = 0;
  for (int base = 0; base < n; base += NT) {
    const int r = base + tid;
    const bool keep = r < n && rows.term[r] == RUNNING_ST;
    int tot;
    const int off = cta_excl_scan(keep ? 1 : 0, &tot);
    if (keep) copy_row(D, tmp, nk + off, rows, r);
    nk += tot;
    __syncthreads();
  }
  for (int r = tid; r < nk; r += NT) copy_row(D, rows, r, tmp, r);
  __syncthreads();

  // ---- E. reserve next-window blocks: each row owns ceil(min(l + T, cap) / bs) (R23 step 3)
  int popped = 0;
  for (int base = 0; base < nk; base += NT) {
    const int r = base + tid;
    int need = 0;
    if (r < nk) need = cdiv(min(rows.ell[r] + D.T, D.cap), D.bs) - rows.nblk[r];
    int tot;
    const int off = cta_excl_scan(need, &tot);
    for (int j = 0; j < need; ++j)
      rows.table[(long long)r * D.MBR + rows.nblk[r] + j] = fs[top - 1 - (popped + off + j)];
    if (r < nk) rows.nblk[r] += need;
    popped += tot;
    __syncthreads();
  }
  top -= popped;
  if (tid == 0) {
    ctr->free_top = top;
    ctr->committed -= (long long)nterm * cdiv(D.cap, D.bs) + pre_total;
    ctr->n_rows = nk;
    ctr->windows += 1;
  }
}
void launch_boundary(Dims D, Rows rows, Rows tmp, Reqs reqs, const float* prm_score, int* free_stack, Ctr* ctr,
                     DevResult* res, int* slot_row, int n, BoundaryTrace tr, cudaStream_t s) {
  k_boundary<<<1, NT, 0, s>>>(D, rows, tmp, reqs, prm_score, free_stack, ctr, res, slot_row, n, tr);
}
