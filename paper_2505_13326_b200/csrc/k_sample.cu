// Seeded counter-based sampler with EOS / cap / forced-length detection.
//   y_s = argmax_v ( logit_v / tau + G_v ),  G_v = -ln(-ln u_v),
//   u_v = ((w >> 8) + 0.5) 2^-24,  w = Philox4x32-10((v>>2, s, rid, b), seed)[v & 3]
// (readings R24, R25).  Ties go to the lowest v.  fp32 arithmetic; -ln u is evaluated as
// log1p(-(2^24 - x - 0.5) 2^-24) in the upper half so u is represented exactly.
#include "kernels.h"
#include "sample_math.cuh"

// Phase 1: one CTA per (row, vocab chunk of SCHUNK entries) -> the chunk's best (key, v).
// (Fusing phase 1 into the LM-head GEMM epilogue was measured slower: 691 us vs 233 + 344 us
// per C2 step -- the epilogue's 8 warps per SM cannot hide the Philox/log latency that the
// stand-alone kernel hides with full occupancy.)
// Phase 2: one warp per row reduces the chunks (exact max with the lowest-v tie rule, so the
// reduction order does not matter) and updates the row: history, EOS / cap, counters.
constexpr int SCHUNK = 16384;   // 16 groups of 4 per thread: pruning bound warms up early

__global__ void __launch_bounds__(256) k_sample_part(const float* __restrict__ logits, Dims D, Rows rows, Reqs reqs,
                                                      float* __restrict__ pkey, int* __restrict__ pv, int nchunk) {
  pdl_wait();
  pdl_trigger();
  const int r = blockIdx.x, c = blockIdx.y;
  if (rows.status[r] != RUNNING_ST) return;
  const int slot = rows.slot[r], b = rows.b[r];
  const int s = rows.ell[r] + 1;
  const long long sb = (long long)slot * SART_MAXN + b;
  const int forced_len = reqs.sc_len[sb];   // 0 = no scripted EOS step
  if (forced_len > 0 && s == forced_len) return;
  const bool mask_eos = forced_len > 0;
  const float* lg = logits + (long long)r * D.V;
  const uint32_t rid = (uint32_t)reqs.id[slot];
  const uint32_t k0 = (uint32_t)D.seed, k1 = (uint32_t)(D.seed >> 32);
  float bk = -INFINITY;
  int bv = 0x7fffffff;
  const int g_lo = c * (SCHUNK / 4), g_hi = min((c + 1) * (SCHUNK / 4), (D.V + 3) >> 2);
  if (D.tau > 0.f && g_lo + (int)threadIdx.x < g_hi) {
    // pilot: the first entry of this thread's first group seeds the pruning bound (it is a
    // legitimate candidate; re-visiting it in the loop cannot change (bk, bv))
    const int v = 4 * (g_lo + threadIdx.x);
    if (!(mask_eos && v == D.eos)) {
      const u32x4 w = philox4x32_10(u32x4{(uint32_t)(v >> 2), (uint32_t)s, rid, (uint32_t)b}, k0, k1);
      better(bk, bv, (D.tau == 1.0f ? lg[v] : lg[v] / D.tau) + gumbel_from_word(w.x), v);
    }
  }
  float wb = -INFINITY;
  int it = 0;
  for (int base = g_lo; base < g_hi; base += blockDim.x, ++it) {   // uniform trip count (warp shuffles)
    // a key some entry already has is a valid pruning bound: the lane's own best every
    // iteration, the warp's best every 4th (a stale bound only prunes less)
    wb = fmaxf(wb, bk);
    if ((it & 3) == 0) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) wb = fmaxf(wb, __shfl_xor_sync(0xffffffffu, wb, o));
    }
    const int g4 = base + threadIdx.x;
    if (g4 >= g_hi) continue;
    const float4 l4 = (D.V % 4 == 0 && 4 * g4 + 3 < D.V) ? *reinterpret_cast<const float4*>(lg + 4 * g4)
                                         : make_float4(lg[4 * g4], 4 * g4 + 1 < D.V ? lg[4 * g4 + 1] : 0.f,
                                                       4 * g4 + 2 < D.V ? lg[4 * g4 + 2] : 0.f, 0.f);
    const float lv[4] = {l4.x, l4.y, l4.z, l4.w};
#ifdef SART_SAMPLE_NOPRUNE
    wb = -INFINITY;
#endif
    sample_group4(bk, bv, lv, 4 * g4, D.V, s, rid, (uint32_t)b, k0, k1, D.tau, mask_eos, D.eos, wb);
  }
  __shared__ float sk[8];
  __shared__ int sv[8];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    float ok = __shfl_xor_sync(0xffffffffu, bk, o);
    int ov = __shfl_xor_sync(0xffffffffu, bv, o);
    better(bk, bv, ok, ov);
  }
  if ((threadIdx.x & 31) == 0) { sk[threadIdx.x >> 5] = bk; sv[threadIdx.x >> 5] = bv; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w2 = 1; w2 < (int)(blockDim.x >> 5); ++w2) better(bk, bv, sk[w2], sv[w2]);
    pkey[(long long)r * nchunk + c] = bk;
    pv[(long long)r * nchunk + c] = bv;
  }
}

__global__ void __launch_bounds__(32) k_sample_final(Dims D, Rows rows, Reqs reqs, Ctr* ctr, const float* pkey,
                                                     const int* pv, int nchunk, int* dbg_tok) {
  pdl_wait();
  pdl_trigger();
  const int r = blockIdx.x, lane = threadIdx.x;
  if (rows.status[r] != RUNNING_ST) return;
  const int slot = rows.slot[r], b = rows.b[r];
  const int s = rows.ell[r] + 1;
  const long long sb = (long long)slot * SART_MAXN + b;
  const int forced_len = reqs.sc_len[sb];
  int y;
  if (forced_len > 0 && s == forced_len) {
    y = D.eos;
  } else {
    float bk = -INFINITY;
    int bv = 0x7fffffff;
    for (int c = lane; c < nchunk; c += 32) better(bk, bv, pkey[(long long)r * nchunk + c], pv[(long long)r * nchunk + c]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      float ok = __shfl_xor_sync(0xffffffffu, bk, o);
      int ov = __shfl_xor_sync(0xffffffffu, bv, o);
      better(bk, bv, ok, ov);
    }
    y = bv;
  }
  if (lane != 0) return;
  if (dbg_tok) dbg_tok[r] = y;
  if (reqs.has_forced[slot]) y = reqs.forced[sb * D.cap + (s - 1)];   // teacher forcing
  reqs.hist[sb * D.cap + (s - 1)] = y;
  rows.tok[r] = y;
  rows.ell[r] = s;
  atomicAdd((unsigned long long*)&ctr->branch_tokens, 1ull);
  int st = RUNNING_ST;
  if (y == D.eos) st = ST_EOS;                  // O5 / R17
  else if (s == D.cap) st = ST_CAP;
  if (st != RUNNING_ST) {
    atomicAdd(&reqs.ncw[slot], 1);              // completions so far (es_every_step, R43)
    rows.status[r] = st;
    rows.done_step[r] = s;
    rows.done_wstep[r] = ctr->wstep;
    atomicSub(&ctr->live, 1);
  }
}

void launch_sample(const float* logits, Dims D, Rows rows, Reqs reqs, Ctr* ctr, int n, int* dbg_tok,
                   float* pkey, int* pv, cudaStream_t s) {
  if (n <= 0) return;
  const int nchunk = (D.V + SCHUNK - 1) / SCHUNK;
  launch_pdl(k_sample_part, dim3(n, nchunk), dim3(256), 0, s, logits, D, rows, reqs, pkey, pv, nchunk);
  launch_pdl(k_sample_final, dim3(n), dim3(32), 0, s, D, rows, reqs, ctr, pkey, pv, nchunk, dbg_tok);
}
int sample_chunks(int V) { return (V + SCHUNK - 1) / SCHUNK; }
void launch_sample_final(Dims D, Rows rows, Reqs reqs, Ctr* ctr, int n, int* dbg_tok, const float* pkey, const int* pv,
                         int nchunk, cudaStream_t s) {
  if (n <= 0) return;
  launch_pdl(k_sample_final, dim3(n), dim3(32), 0, s, D, rows, reqs, ctr, pkey, pv, nchunk, dbg_tok);
}


// Start of a decode step.  es_every_step (reading R43): a running row whose request already
// has M completed branches -- counted at the end of the previous step -- stops here: it keeps
// the steps it has (done_step = l) and is EarlyStopped at the boundary.
__global__ void k_step_begin(Ctr* ctr, int es, int wake, Dims D, Rows rows, Reqs reqs, int n) {
  pdl_wait();
  pdl_trigger();
  if (wake) {   // R44: rows whose interleaved prefill has completed start decoding at this step
    for (int r = threadIdx.x; r < n; r += blockDim.x)
      if (rows.status[r] == ST_WAIT && rows.start[r] <= ctr->wstep + 1) rows.status[r] = RUNNING_ST;
    __syncthreads();
  }
  if (es) {
    int stopped = 0;
    for (int r = threadIdx.x; r < n; r += blockDim.x) {
      if (rows.status[r] != RUNNING_ST) continue;
      const int slot = rows.slot[r];
      if (reqs.ncw[slot] >= reqs.M[slot]) {
        rows.status[r] = ST_STOP;
        rows.done_step[r] = rows.ell[r];
        rows.done_wstep[r] = ctr->wstep;
        ++stopped;
      }
    }
    if (stopped) atomicSub(&ctr->live, stopped);
    __syncthreads();
  }
  if (threadIdx.x == 0 && ctr->live > 0) { ctr->wstep += 1; ctr->steps += 1; }
}
void launch_step_begin(Ctr* ctr, int es, int wake, Dims D, Rows rows, Reqs reqs, int n, cudaStream_t s) {
  launch_pdl(k_step_begin, dim3(1), dim3(es || wake ? 1024 : 1), 0, s, ctr, es, wake, D, rows, reqs, n);
}
