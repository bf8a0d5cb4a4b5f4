// tcgen05 GEMM for the decoder projections:
//   C[m][n] (+)= sum_k A[m][k] B[n][k]  (+ bias[n]),  A = activations [M][K] bf16,
//   B = weights [N][K] bf16 (nn.Linear layout; both operands K-major), fp32 accumulate.
//
// Blackwell structure (one CTA per SM, persistent over output tiles):
//   warp 0      TMA producer: 2-D tensor-map loads of A (128 x 64) and B (BN x 64) tiles
//               into a 4-stage shared-memory ring, 128-byte swizzle, mbarrier complete_tx.
//   warp 1      allocates TMEM (2 x BN fp32 columns: double-buffered accumulator) and one
//               elected lane issues tcgen05.mma.cta_group::1.kind::f16 (M=128, N=BN, K=16);
//               tcgen05.commit releases smem stages / publishes finished accumulators.
//   warps 2..5  epilogue: tcgen05.ld 32x32b (each warp owns its TMEM lane quarter = 32 rows),
//               bias / residual-accumulate / SwiGLU, vector stores to global memory.
// Tiles are ordered m-fastest so the CTAs that share a weight tile run together and the
// weight stream is read from HBM once (small-M decode GEMMs are weight-bandwidth-bound).
#include <cuda.h>

#include <cstdio>
#include <cstdlib>

#include <map>
#include <mutex>
#include <tuple>

#include "kernels.h"
#include "umma.cuh"
#include "sample_math.cuh"

namespace {
constexpr int BM = 128, BK = 64;
// pipeline depth: ~192 KB of A+B stages in flight per SM whatever the tile shape
template <int BN, int MS> struct Stages { static constexpr int value = (192 * 1024) / ((MS * BM + BN) * BK * 2); };
// TMEM accumulators: MS m-subtiles x BN columns, double-buffered when that fits in 512 columns
template <int BN, int MS> struct Tmem {
  static constexpr int NBUF = 2 * MS * BN <= 512 ? 2 : 1;
  static constexpr int COLS = NBUF * MS * BN;
};
// warp 0 TMA producer, warp 1 MMA issuer, then NEPI epilogue warps: NEPI / 4 per TMEM lane
// quarter (warp % 4), splitting the 32-column chunks between them
#ifndef SART_GEMM_NEPI
#define SART_GEMM_NEPI 4   // 8 (two warps per lane quarter) for every mode measured 1.3% slower per C2 step
#endif
#ifndef SART_GEMM_NEPI_SWIGLU
#define SART_GEMM_NEPI_SWIGLU 8   // the SwiGLU epilogue (2 MUFU ops per output, one tile per CTA) runs alone
#endif                            // after the mainloop: two warps per lane quarter halve it
template <int MODE> struct Epi {
  static constexpr int NEPI = MODE == GEMM_SWIGLU ? SART_GEMM_NEPI_SWIGLU : (MODE == GEMM_SAMPLE ? 8 : SART_GEMM_NEPI);
  static constexpr int NTHREADS = 64 + 32 * NEPI;
  static constexpr int CSTEP = 32 * (NEPI / 4);   // chunk stride of one epilogue warp
  static constexpr int SLAB = MODE == GEMM_SWIGLU ? 1 : NEPI;   // transpose slabs (store epilogues)
};

// fp32 output of one 32-row TMEM lane quarter (BN columns): each lane holds one row of a
// 32 x 32 chunk; transpose it through a 16-byte-swizzled shared slab (chunk k of row r at
// k ^ (r & 7): conflict-free both ways) so that each 16-byte store instruction writes 4 full
// 128-byte lines.  MODE == GEMM_ACCUM adds into C.
// ndst > 1 (tensor parallelism): the same values go to every destination tile in dsts[] (this
// rank's and each peer's receive buffer).
template <int BN, int MODE>
__device__ __forceinline__ void store_tile_f32(uint32_t tbase, float* Cs, int mrow0, int n0, int M, int N,
                                               const float* bias, uint32_t slab, int lane, int c_begin, int c_step,
                                               float* const* dsts = nullptr, int ndst = 0) {
  const int kk = lane & 7, r4 = lane >> 3;
  const bool vec = (N & 3) == 0;
#pragma unroll 1
  for (int c = c_begin; c < BN; c += c_step) {
    float v[32];
    tmem_ld32(tbase + c, v);
#pragma unroll
    for (int k = 0; k < 8; ++k)
      asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(slab + (uint32_t)(lane * 32 + ((k ^ (lane & 7)) << 2)) * 4),
                   "f"(v[4 * k]), "f"(v[4 * k + 1]), "f"(v[4 * k + 2]), "f"(v[4 * k + 3])
                   : "memory");
    __syncwarp();
    const int gn = n0 + c + kk * 4;
    float4 bv = make_float4(0.f, 0.f, 0.f, 0.f);
    if (bias) {
      if (vec && gn + 4 <= N) bv = *reinterpret_cast<const float4*>(bias + gn);
      else {
        if (gn < N) bv.x = bias[gn];
        if (gn + 1 < N) bv.y = bias[gn + 1];
        if (gn + 2 < N) bv.z = bias[gn + 2];
        if (gn + 3 < N) bv.w = bias[gn + 3];
      }
    }
    float4 x[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int rr = i * 4 + r4;
      asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                   : "=f"(x[i].x), "=f"(x[i].y), "=f"(x[i].z), "=f"(x[i].w)
                   : "r"(slab + (uint32_t)(rr * 32 + ((kk ^ (rr & 7)) << 2)) * 4)
                   : "memory");
      x[i].x += bv.x; x[i].y += bv.y; x[i].z += bv.z; x[i].w += bv.w;
    }
    __syncwarp();
    if (ndst > 0) {   // TP exchange: plain stores (no accumulate) into every rank's buffer
      for (int p = 0; p < ndst; ++p) {
        float* dst = dsts[p] + (size_t)(mrow0 + r4) * N + gn;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          if (mrow0 + i * 4 + r4 >= M) continue;
          float* d = dst + (size_t)i * 4 * N;
          if (vec && gn + 4 <= N) {
            *reinterpret_cast<float4*>(d) = x[i];
          } else {
            const float xs[4] = {x[i].x, x[i].y, x[i].z, x[i].w};
            for (int e = 0; e < 4; ++e)
              if (gn + e < N) d[e] = xs[e];
          }
        }
      }
      continue;
    }
    float* dst = Cs + (size_t)(mrow0 + r4) * N + gn;
    if (vec && gn + 4 <= N) {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        if (mrow0 + i * 4 + r4 < M) {
          float4* d4 = reinterpret_cast<float4*>(dst + (size_t)i * 4 * N);
          if (MODE == GEMM_ACCUM) {
            const float4 o = *d4;
            x[i].x += o.x; x[i].y += o.y; x[i].z += o.z; x[i].w += o.w;
          }
          *d4 = x[i];
        }
      }
    } else {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        if (mrow0 + i * 4 + r4 < M) {
          float* d = dst + (size_t)i * 4 * N;
          const float xs[4] = {x[i].x, x[i].y, x[i].z, x[i].w};
#pragma unroll
          for (int e = 0; e < 4; ++e)
            if (gn + e < N) d[e] = MODE == GEMM_ACCUM ? d[e] + xs[e] : xs[e];
        }
      }
    }
  }
}

template <int BN, int MS, int NSLAB>
struct Smem {
  static constexpr int STAGES = Stages<BN, MS>::value;
  alignas(1024) bf16 a[STAGES][MS * BM * BK];
  alignas(1024) bf16 b[STAGES][BN * BK];
  uint64_t full[STAGES], empty[STAGES], tfull[2], tempty[2];
  uint32_t tmem_base;
  alignas(16) float slab[NSLAB][32 * 32];   // epilogue transpose staging (explicit st/ld.shared)
};

// MS m-subtiles of 128 rows share each B stage (tile = MS*128 x BN): per-SM operand traffic
// per flop falls from (128 + BN) / (128 BN) to (MS 128 + BN) / (MS 128 BN) -- the decode GEMMs are
// bound by L2 -> SM operand delivery, not by the tensor pipe (profiles/r1_gemm_ncu.txt).
// MODE: GEMM_STORE (C = AB^T + bias), GEMM_ACCUM (C += AB^T), GEMM_SWIGLU (columns of each
// BN tile are [gate(BN/2) | up(BN/2)] of interleaved weights; writes bf16 act[m][F]).
// Split-K: work unit u -> (m-tile = u % mt, split, n-tile); split s covers k-blocks
// [s*kb/S, (s+1)*kb/S) and writes its fp32 partial tile to C + s*M*N.  The consumer kernel
// (RMSNorm / RoPE) sums the S partials in split order, so the result is deterministic.
}  // namespace
__device__ unsigned long long g_gemm_ts[4][10];
__device__ int g_gemm_ts_idx;
__device__ unsigned long long g_gemm_trace[2][64];   // CTA 0, first tile: [0] load issue, [1] stage landed
namespace {
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
// QKV epilogue: where row gm's k / v go and at which RoPE position (decode: the row's next
// suffix entry; prefill: a prompt position; f2 PRM pass: a suffix entry of a batch row)
struct RowMeta {
  int pos, sib;
  long long blk;
  bool kv_ok;
};
__device__ __forceinline__ RowMeta qkv_row_meta(const QkvEpi& epi, int gm, int M) {
  const Dims& D = epi.D;
  RowMeta r{0, 0, 0, false};
  if (gm >= M) return r;
  if (epi.a.sf_row) {
    const int row = epi.a.sf_row[gm];
    if (row >= 0) {
      const int l = epi.a.pf_pos[gm];
      r.pos = epi.reqs.P[epi.rows.slot[row]] - 1 + l;
      r.blk = epi.rows.table[(long long)row * D.MBR + l / D.bs];
      r.sib = l % D.bs;
      r.kv_ok = true;
    }
  } else if (epi.a.pf_slot) {
    r.pos = epi.a.pf_pos[gm];
    r.blk = epi.reqs.prefix[(long long)epi.a.pf_slot[gm] * D.MPB + r.pos / D.bs];
    r.sib = r.pos % D.bs;
    r.kv_ok = true;
  } else if (epi.rows.status[gm] == RUNNING_ST) {
    const int l = epi.rows.ell[gm];
    r.pos = epi.reqs.P[epi.rows.slot[gm]] - 1 + l;
    r.blk = epi.rows.table[(long long)gm * D.MBR + l / D.bs];
    r.sib = l % D.bs;
    r.kv_ok = true;
  }
  return r;
}

template <int BN, int MODE, int MS>
__global__ void __launch_bounds__(Epi<MODE>::NTHREADS, 1)
    k_gemm_tc(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, const bf16* __restrict__ Bt,
              float* C, const float* __restrict__ bias, bf16* act, int M, int N, int K, int S,
              const __grid_constant__ QkvEpi epi, const __grid_constant__ TpOut tp) {
  extern __shared__ __align__(16) uint8_t smem_raw[];   // 1024-aligned below (+1024 B slack)
  Smem<BN, MS, Epi<MODE>::SLAB>& sm =
      *reinterpret_cast<Smem<BN, MS, Epi<MODE>::SLAB>*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  constexpr int STAGES = Smem<BN, MS, Epi<MODE>::SLAB>::STAGES;
  constexpr int NEPI = Epi<MODE>::NEPI, CSTEP = Epi<MODE>::CSTEP;
  constexpr int NBUF = Tmem<BN, MS>::NBUF, TCOLS = Tmem<BN, MS>::COLS;
  constexpr uint32_t STAGE_TX = (MS * BM + BN) * BK * 2;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int mt = (M + MS * BM - 1) / (MS * BM), nt = (N + BN - 1) / BN, ntiles = mt * nt * S;
  const int kb_all = (K + BK - 1) / BK;
  auto unit_of = [&](int t, int& m0, int& n0, int& kb0, int& kb1, int& sp) {
    m0 = (t % mt) * (MS * BM);
    const int rest = t / mt;
    sp = rest % S;
    n0 = (rest / S) * BN;
    kb0 = sp * kb_all / S;
    kb1 = (sp + 1) * kb_all / S;
  };

#ifdef SART_GEMM_TS   // phase timestamps of CTA 0 (build with -DSART_GEMM_TS; SART_GEMM_TS=1 prints them)
  __shared__ int ts_slot;
#ifndef SART_GEMM_TS_MODE
#define SART_GEMM_TS_MODE -1   // record launches of this MODE only (-1: every launch)
#endif
  const bool tsb = blockIdx.x == 0 && (SART_GEMM_TS_MODE < 0 || MODE == SART_GEMM_TS_MODE);
  if (threadIdx.x == 0 && tsb) { ts_slot = atomicAdd(&g_gemm_ts_idx, 1) & 3; g_gemm_ts[ts_slot][0] = gtime(); }
#define TS(i) if (tsb) g_gemm_ts[ts_slot][i] = gtime()
#else
#define TS(i) do {} while (0)
#endif
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) { mbar_init(&sm.full[s], 1); mbar_init(&sm.empty[s], 1); }
    for (int s = 0; s < NBUF; ++s) { mbar_init(&sm.tfull[s], 1); mbar_init(&sm.tempty[s], NEPI); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&sm.tmem_base)),
                 "r"(TCOLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = sm.tmem_base;
  if (threadIdx.x == 0) { TS(1); }
  if (threadIdx.x == 0) pdl_trigger();

  if (warp == 0) {
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(&tmA) : "memory");
      if (!Bt) asm volatile("prefetch.tensormap [%0];" ::"l"(&tmB) : "memory");
      // weights: pre-tiled (Bt: [n-tile][k-block] images of the swizzled shared tile, one
      // contiguous bulk copy each) or row-major through the 2-D tensor map
      const uint64_t polb = l2_policy_evict_first();
      auto load_b = [&](int st, int kbi, int n0_) {
        if constexpr (MODE == GEMM_QKV_HALF) {
          // half-head tile: weight rows [32p, 32p + 32) and [64 + 32p, ...) of head n0_ / 128
          // as two 32-row boxes (four whole 8-row swizzle atoms each, so the 64-row smem tile
          // keeps the layout one 64-row box would have)
          const int hb = (n0_ / 128) * 128 + ((n0_ / 64) & 1) * 32;
          tma_load_2d(sm.b[st], &tmB, &sm.full[st], kbi * BK, hb);
          tma_load_2d(sm.b[st] + 32 * BK, &tmB, &sm.full[st], kbi * BK, hb + 64);
        } else if (Bt) {
          bulk_load(sm.b[st], Bt + ((size_t)(n0_ / BN) * kb_all + kbi) * (BN * BK), BN * BK * 2, &sm.full[st]);
        } else if (epi.evict_b) {
          tma_load_2d_hint(sm.b[st], &tmB, &sm.full[st], kbi * BK, n0_, polb);
        } else {
          tma_load_2d(sm.b[st], &tmB, &sm.full[st], kbi * BK, n0_);
        }
      };
      auto load_a = [&](int st, int j, int kbi, int m0_) {
        tma_load_2d(sm.a[st] + j * BM * BK, &tmA, &sm.full[st], kbi * BK, m0_ + j * BM);
      };
      int stage = 0;
      uint32_t phase = 0;
      bool first = true;
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
        int m0, n0, kb0, kb1, sp;
        unit_of(t, m0, n0, kb0, kb1, sp);
        int kb = kb0;
        if (first) {
          // PDL: the weight tiles of the first stages do not depend on the previous kernel;
          // start them before waiting for it, then load the activations.
          first = false;
          const int pre = min(STAGES, kb1 - kb0);
          for (int i = 0; i < pre; ++i) {
            mbar_expect_tx(&sm.full[i], STAGE_TX);
            load_b(i, kb0 + i, n0);
          }
          pdl_wait();
          TS(2);
          for (int i = 0; i < pre; ++i) {
#pragma unroll
            for (int j = 0; j < MS; ++j)
              load_a(i, j, kb0 + i, m0);
#ifdef SART_GEMM_TS
            if (blockIdx.x == 0 && i < 64) g_gemm_trace[0][i] = gtime();
#endif
          }
          kb += pre;
          stage = pre % STAGES;
          phase = pre == STAGES ? 1 : 0;
        }
        for (; kb < kb1; ++kb) {
          mbar_wait(&sm.empty[stage], phase ^ 1);
          mbar_expect_tx(&sm.full[stage], STAGE_TX);
#pragma unroll
          for (int j = 0; j < MS; ++j) load_a(stage, j, kb, m0);
          load_b(stage, kb, n0);
#ifdef SART_GEMM_TS
          if (blockIdx.x == 0 && t == blockIdx.x && kb - kb0 < 64) g_gemm_trace[0][kb - kb0] = gtime();
#endif
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
      if (first) pdl_wait();
    }
  } else if (warp == 1) {
    // instruction descriptor: D f32, A/B bf16, both K-major, N = BN, M = 128
    const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
    int stage = 0;
    uint32_t phase = 0;
    int it = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
      const int as = it % NBUF;
      const uint32_t aph = (it / NBUF) & 1;
      int m0, n0, kb0, kb1, sp;
      unit_of(t, m0, n0, kb0, kb1, sp);
      mbar_wait(&sm.tempty[as], aph ^ 1);
      asm volatile("tcgen05.fence::after_thread_sync;");
      const uint32_t d = tmem + as * MS * BN;
      for (int kb = kb0; kb < kb1; ++kb) {
        mbar_wait(&sm.full[stage], phase);
        asm volatile("tcgen05.fence::after_thread_sync;");
        if (lane == 0 && it == 0 && kb == kb0) { TS(3); }
#ifdef SART_GEMM_TS
        if (lane == 0 && blockIdx.x == 0 && it == 0 && kb - kb0 < 64) g_gemm_trace[1][kb - kb0] = gtime();
#endif
        if (lane == 0) {
          const uint32_t a0 = smem_u32(sm.a[stage]), b0 = smem_u32(sm.b[stage]);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k)
#pragma unroll
            for (int j = 0; j < MS; ++j)
              umma_bf16(d + j * BN, umma_desc(a0 + j * BM * BK * 2 + k * 32), umma_desc(b0 + k * 32), idesc,
                        (kb > kb0 || k) ? 1u : 0u);
          umma_commit(&sm.empty[stage]);
          if (kb == kb1 - 1) umma_commit(&sm.tfull[as]);
          if (kb == kb1 - 1 && it == 0) { TS(4); }
        }
        __syncwarp();
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
    }
  } else {
    // epilogue warps 2..5 -> TMEM lane quarter (warp % 4)
    pdl_wait();   // outputs may be read by the previous kernel; inputs (bias, rows) are visible
    // TP: this rank's consumer of projection k expects gridDim.x arrivals from each rank
    if (tp.tp > 1 && blockIdx.x == 0 && warp == 2 && lane == 0) {
      tp.expect[tp.k] += (unsigned long long)gridDim.x * tp.tp;
#ifdef SART_TP_DEBUG
      printf("tp gemm rank %d k %d grid %d expect %llu cnt0 %p cnt1 %p\n", tp.rank, tp.k, gridDim.x, tp.expect[tp.k],
             (void*)tp.cnt[0], (void*)tp.cnt[1]);
#endif
    }
    const int q = warp & 3;            // TMEM lane quarter this warp may access
    const int half = (warp - 2) >> 2;  // which 32-column chunks of the tile it handles
    const int row = q * 32 + lane;
    int it = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
      const int as = it % NBUF;
      const uint32_t aph = (it / NBUF) & 1;
      int m0_, n0, kb0, kb1, sp;
      unit_of(t, m0_, n0, kb0, kb1, sp);
      const int n0_ = n0;
      float* Cs = C + (size_t)sp * M * N;
      // QKV: this row's position and KV slot are dependent global loads (status, ell, request
      // prompt length, block table); resolve them -- and pull the row's RoPE cos / sin lines
      // toward L1 -- while the mainloop still runs, off the epilogue's critical path (MS == 1)
      RowMeta rm{};
      if constexpr (MODE == GEMM_QKV || MODE == GEMM_QKV_HALF) {
        rm = qkv_row_meta(epi, m0_ + row, M);
        constexpr int HD = MODE == GEMM_QKV_HALF ? 128 : BN;
        const float* cs = epi.rope_cs + (long long)rm.pos * HD + (MODE == GEMM_QKV_HALF ? ((n0_ / 64) & 1) * 32 : 0);
        asm volatile("prefetch.global.L1 [%0];" ::"l"(cs));
        asm volatile("prefetch.global.L1 [%0];" ::"l"(cs + HD / 2));
        if (HD == 128 && MODE == GEMM_QKV) {
          asm volatile("prefetch.global.L1 [%0];" ::"l"(cs + 32));
          asm volatile("prefetch.global.L1 [%0];" ::"l"(cs + HD / 2 + 32));
        }
      }
      mbar_wait(&sm.tfull[as], aph);
      asm volatile("tcgen05.fence::after_thread_sync;");
      if (warp == 2 && lane == 0 && it == 0) { TS(5); }
#pragma unroll 1
      for (int ms = 0; ms < MS; ++ms) {
      const int m0 = m0_ + ms * BM;
      const int gm = m0 + row;
      const uint32_t tbase = tmem + ((uint32_t)(q * 32) << 16) + (as * MS + ms) * BN;
      if (MODE == GEMM_QKV || MODE == GEMM_QKV_HALF) {
        // tile = one head (GEMM_QKV, BN == head_dim) or half a head (GEMM_QKV_HALF, hd = 128):
        // q / k heads are rotated (pairs i, i + hd/2), k and v are appended to the paged pool
        // at the row's slot (common.cuh layout and swizzle).  Tile column c < HALF is head dim
        // i0 + c and column HALF + c is dim hd/2 + i0 + c.
        // Split-K (S > 1, GEMM_QKV only): every unit publishes its fp32 partial tile (C + split
        // * M * N); the last of the S units of a (m-tile, head, lane quarter) -- an atomic
        // arrival count -- sums the S partials in split order (deterministic) and runs the
        // epilogue.
        const Dims& D = epi.D;
        constexpr int HD = MODE == GEMM_QKV_HALF ? 128 : BN;
        constexpr int HALF = BN / 2, HHD = HD / 2;
        const int head = n0 / HD;
        const int i0 = MODE == GEMM_QKV_HALF ? ((n0 / 64) & 1) * 32 : 0;
        if (MODE == GEMM_QKV && S > 1) {
          store_tile_f32<BN, GEMM_STORE>(tbase, Cs, m0 + q * 32, n0, M, N, nullptr, smem_u32(sm.slab[warp - 2]), lane, half * 32, CSTEP);
          __threadfence();
          __syncwarp();
          int old = 0;
          if (lane == 0) {
            int* cnt = epi.cnt + (((size_t)head * mt + m0_ / BM) * 4 + q) * 2 + half;
            old = atomicAdd(cnt, 1);
            if (old == S - 1) *cnt = 0;   // reset for the next launch (stream-ordered)
          }
          old = __shfl_sync(0xffffffffu, old, 0);
          if (old != S - 1) continue;
          __threadfence();
        }
        const int pos = rm.pos, sib = rm.sib;
        const bool kv_ok = rm.kv_ok;
        const long long blk = rm.blk;
        const bool rot = head < D.qh + D.kvh;
        const float* cs = epi.rope_cs + (long long)pos * HD;   // [cos(hd/2) | sin(hd/2)]
#pragma unroll 1
        for (int c = half * 32; c < HALF; c += CSTEP) {
          float x1[32], x2[32];
          if (S == 1) {
            tmem_ld32(tbase + c, x1);
            tmem_ld32(tbase + HALF + c, x2);
          } else if (gm < M) {
#pragma unroll
            for (int j = 0; j < 32; ++j) x1[j] = x2[j] = 0.f;
            for (int sp2 = 0; sp2 < S; ++sp2) {   // split order
              const float* p = C + (size_t)sp2 * M * N + (size_t)gm * N + n0 + c;
#pragma unroll
              for (int j4 = 0; j4 < 8; ++j4) {
                const float4 a = __ldcg(reinterpret_cast<const float4*>(p + 4 * j4));
                const float4 b = __ldcg(reinterpret_cast<const float4*>(p + HALF + 4 * j4));
                x1[4 * j4] += a.x; x1[4 * j4 + 1] += a.y; x1[4 * j4 + 2] += a.z; x1[4 * j4 + 3] += a.w;
                x2[4 * j4] += b.x; x2[4 * j4 + 1] += b.y; x2[4 * j4 + 2] += b.z; x2[4 * j4 + 3] += b.w;
              }
            }
          }
          if (gm < M) {
            const float* bh = epi.bias + head * HD + i0 + c;
#pragma unroll
            for (int j = 0; j < 32; ++j) { x1[j] += bh[j]; x2[j] += bh[HHD + j]; }
            if (rot) {
#pragma unroll
              for (int j4 = 0; j4 < 8; ++j4) {
                const float4 co = *reinterpret_cast<const float4*>(cs + i0 + c + 4 * j4);
                const float4 sn = *reinterpret_cast<const float4*>(cs + HHD + i0 + c + 4 * j4);
                const float cv[4] = {co.x, co.y, co.z, co.w}, sv[4] = {sn.x, sn.y, sn.z, sn.w};
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                  const int j = 4 * j4 + e;
                  const float a = x1[j], b = x2[j];
                  x1[j] = a * cv[e] - b * sv[e];
                  x2[j] = b * cv[e] + a * sv[e];
                }
              }
            }
            if (head < D.qh) {
              bf16* qd = epi.qout + ((long long)gm * D.qh + head) * HD + i0;
#pragma unroll
              for (int j = 0; j < 32; j += 8) {
                __align__(16) bf16 o1[8], o2[8];
#pragma unroll
                for (int e = 0; e < 8; ++e) { o1[e] = __float2bfloat16_rn(x1[j + e]); o2[e] = __float2bfloat16_rn(x2[j + e]); }
                *reinterpret_cast<uint4*>(qd + c + j) = *reinterpret_cast<uint4*>(o1);
                *reinterpret_cast<uint4*>(qd + HHD + c + j) = *reinterpret_cast<uint4*>(o2);
              }
            } else if (kv_ok) {
              const int kv = head < D.qh + D.kvh ? 0 : 1;
              const int hh = kv == 0 ? head - D.qh : head - D.qh - D.kvh;
              bf16* tile = epi.pool + kv_tile_off(D, epi.layer, blk, kv, hh);
#pragma unroll
              for (int j = 0; j < 32; j += 8) {
                __align__(16) bf16 o1[8], o2[8];
#pragma unroll
                for (int e = 0; e < 8; ++e) { o1[e] = __float2bfloat16_rn(x1[j + e]); o2[e] = __float2bfloat16_rn(x2[j + e]); }
                *reinterpret_cast<uint4*>(tile + kv_swz<bf16>(sib, i0 + c + j, HD)) = *reinterpret_cast<uint4*>(o1);
                *reinterpret_cast<uint4*>(tile + kv_swz<bf16>(sib, HHD + i0 + c + j, HD)) = *reinterpret_cast<uint4*>(o2);
              }
            }
          }
        }
      } else if (MODE == GEMM_SWIGLU) {
        const int F = N / 2;   // N = 2F interleaved in BN-wide tiles
        const int f0 = n0 / 2;
#pragma unroll 1
        for (int c = half * 32; c < BN / 2; c += CSTEP) {
          float g[32], u[32];
          tmem_ld32(tbase + c, g);
          tmem_ld32(tbase + BN / 2 + c, u);
          if (gm < M) {
            bf16* dst = act + (size_t)gm * F + f0 + c;
#pragma unroll
            for (int j = 0; j < 32; j += 8) {
              if (f0 + c + j + 8 <= F) {
                __align__(16) bf16 o[8];
#pragma unroll
                for (int e = 0; e < 8; ++e) {
                  float x = g[j + e];
                  o[e] = __float2bfloat16_rn(__fdividef(x, 1.0f + __expf(-x)) * u[j + e]);
                }
                *reinterpret_cast<uint4*>(dst + j) = *reinterpret_cast<uint4*>(o);
              }
            }
          }
        }
      } else if (MODE == GEMM_SAMPLE) {
        // phase 1 of the sampler on this tile: the thread owns row gm and, with its twin warp,
        // half of the tile's columns (32-column chunks half, half + 2, ...); its own best key
        // so far is the pruning bound (sample_math.cuh: skipped entries cannot win)
        if (Cs) store_tile_f32<BN, GEMM_STORE>(tbase, Cs, m0 + q * 32, n0, M, N, nullptr, smem_u32(sm.slab[warp - 2]),
                                                lane, half * 32, CSTEP);
        const Dims& D = epi.D;
        bool live = false, mask_eos = false;
        int s_ = 0, b_ = 0;
        uint32_t rid = 0;
        if (gm < M && epi.rows.status[gm] == RUNNING_ST) {
          const int slot = epi.rows.slot[gm];
          b_ = epi.rows.b[gm];
          s_ = epi.rows.ell[gm] + 1;
          const int fl = epi.reqs.sc_len[(long long)slot * SART_MAXN + b_];
          live = !(fl > 0 && s_ == fl);   // a scripted EOS step needs no sample (phase 2 sets it)
          mask_eos = fl > 0;
          rid = (uint32_t)epi.reqs.id[slot];
        }
        const uint32_t k0 = (uint32_t)D.seed, k1 = (uint32_t)(D.seed >> 32);
        float bk = -INFINITY;
        int bv = 0x7fffffff;
#pragma unroll 1
        for (int c = half * 32; c < BN; c += CSTEP) {
          float v[32];
          tmem_ld32(tbase + c, v);
          if (live)
#pragma unroll
            for (int g4 = 0; g4 < 8; ++g4)
              if (n0 + c + 4 * g4 < N)
                sample_group4(bk, bv, v + 4 * g4, n0 + c + 4 * g4, N, s_, rid, (uint32_t)b_, k0, k1, D.tau, mask_eos,
                              D.eos, bk);
        }
        if (live) {
          const long long si = (long long)gm * epi.nsl + (n0 / BN) * (NEPI / 4) + half;
          epi.skey[si] = bk;
          epi.sv[si] = bv;
        }
      } else if (tp.tp > 1) {
        float* dsts[SART_MAX_TP];
        for (int p = 0; p < tp.tp; ++p) dsts[p] = tp.dst[p] + ((size_t)tp.rank * S + sp) * M * N;
        store_tile_f32<BN, MODE>(tbase, Cs, m0 + q * 32, n0, M, N, bias, smem_u32(sm.slab[warp - 2]), lane, half * 32,
                                 CSTEP, dsts, tp.tp);
      } else {
        store_tile_f32<BN, MODE>(tbase, Cs, m0 + q * 32, n0, M, N, bias, smem_u32(sm.slab[warp - 2]), lane, half * 32, CSTEP);
      }
      }  // m-subtile
      asm volatile("tcgen05.fence::before_thread_sync;");
      __syncwarp();
      if (warp == 2 && lane == 0 && it == 0) { TS(6); }
      if (lane == 0) mbar_arrive(&sm.tempty[as]);
    }
  }
  if (tp.tp > 1) __threadfence_system();   // this thread's remote partial stores, before the signal
  __syncthreads();
  if (threadIdx.x == 0) { TS(7); }
  if (tp.tp > 1 && threadIdx.x == 0) {      // every rank: one more CTA of projection k has landed
    __threadfence_system();
    for (int p = 0; p < tp.tp; ++p)
      asm volatile("red.release.sys.global.add.u64 [%0], 1;" ::"l"(tp.cnt[p] + tp.k) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TCOLS));
    if (lane == 0) { TS(8); }
  }
}

// ------------------------------------------------------------------ CTA-pair variant
// cta_group::2 (two SMs of a TPC cooperate on one MMA): a pair tile is 256 rows x NP columns.
// CTA r of the pair loads its own 128 A rows and half of the pair's B rows (for each 256-column
// MMA chunk c: B rows [c 256 + r 128, +128)), so per SM the operand bytes per flop drop by a
// quarter (NP = 256) to a third (NP = 512) against the one-SM 256 x 256 tile -- the decode GEMMs
// are bound by per-SM operand delivery (profiles/r2_gemm_phase_ts.txt).  Only the leader (even
// CTA) issues tcgen05.mma.cta_group::2; both CTAs' TMA loads complete on the leader's stage
// barrier; the leader's commits multicast to both CTAs' stage-empty / accumulator-full barriers;
// both CTAs' epilogue warps release the accumulator on the leader's barrier.  Each CTA's TMEM
// holds its own 128 rows x NP columns, so the epilogue is the one-SM epilogue on 128 rows.
// Modes: GEMM_STORE (split-K partial or bias store) and GEMM_SWIGLU (NP / 256 interleaved
// [gate 128 | up 128] tiles).  Every output element accumulates the same K-blocks in the same
// order as the one-SM kernel.
template <int NP>
struct Smem2 {
  static constexpr int BH = NP / 2;                                      // B rows per CTA
  static constexpr int STAGES = (192 * 1024) / ((BM + BH) * BK * 2);
  alignas(1024) bf16 a[STAGES][BM * BK];
  alignas(1024) bf16 b[STAGES][BH * BK];
  uint64_t full[STAGES], empty[STAGES], tfull[2], tempty[2];
  uint32_t tmem_base;
  alignas(16) float slab[4][32 * 32];
};
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t mapa_shared(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
// TMA load whose bytes complete on the PAIR LEADER's barrier (CUTLASS SM100_TMA_2SM_LOAD_2D:
// clearing bit 24 of the shared::cluster barrier address selects the even CTA of the pair)
__device__ __forceinline__ void tma_load_2sm(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
      "%3}], [%4];" ::"r"(smem_u32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(smem_u32(bar) & 0xFEFFFFFFu)
      : "memory");
}
__device__ __forceinline__ void umma_bf16_2sm(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void umma_commit_2sm(uint64_t* bar) {   // arrive on bar in BOTH CTAs
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"((uint16_t)3)
      : "memory");
}

template <int NP, int MODE>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(Epi<MODE>::NTHREADS, 1)
    k_gemm_2sm(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, float* C,
               const float* __restrict__ bias, bf16* act, int M, int N, int K, int S) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  Smem2<NP>& sm = *reinterpret_cast<Smem2<NP>*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  constexpr int STAGES = Smem2<NP>::STAGES, BH = Smem2<NP>::BH;
  constexpr int NEPI = Epi<MODE>::NEPI, CSTEP = Epi<MODE>::CSTEP;
  constexpr int NBUF = 2 * NP <= 512 ? 2 : 1, TCOLS = NBUF * NP;
  constexpr uint32_t PAIR_TX = 2u * (BM + BH) * BK * 2;   // bytes of one stage over both CTAs
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;
  const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
  const int mt = (M + 2 * BM - 1) / (2 * BM), nt = (N + NP - 1) / NP, ntiles = mt * nt * S;
  const int kb_all = (K + BK - 1) / BK;
  auto unit_of = [&](int t, int& m0, int& n0, int& kb0, int& kb1, int& sp) {
    m0 = (t % mt) * (2 * BM) + (int)rank * BM;   // this CTA's 128 rows of the pair's 256
    const int rest = t / mt;
    sp = rest % S;
    n0 = (rest / S) * NP;
    kb0 = sp * kb_all / S;
    kb1 = (sp + 1) * kb_all / S;
  };
  if (threadIdx.x == 0) {
    for (int i = 0; i < STAGES; ++i) { mbar_init(&sm.full[i], 1); mbar_init(&sm.empty[i], 1); }
    for (int i = 0; i < NBUF; ++i) { mbar_init(&sm.tfull[i], 1); mbar_init(&sm.tempty[i], 2 * NEPI); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&sm.tmem_base)),
                 "r"(TCOLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  cluster_sync_all();   // both CTAs' barriers initialised and TMEM allocated before any cross-CTA signal
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = sm.tmem_base;
  if (threadIdx.x == 0) pdl_trigger();

  if (warp == 0) {
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(&tmA) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(&tmB) : "memory");
      auto load_b = [&](int st, int kbi, int n0_) {
#pragma unroll
        for (int c = 0; c < NP / 256; ++c)
          tma_load_2sm(sm.b[st] + c * 128 * BK, &tmB, &sm.full[st], kbi * BK, n0_ + c * 256 + (int)rank * 128);
      };
      int stage = 0;
      uint32_t phase = 0;
      bool first = true;
      for (int t = pair; t < ntiles; t += npairs) {
        int m0, n0, kb0, kb1, sp;
        unit_of(t, m0, n0, kb0, kb1, sp);
        int kb = kb0;
        if (first) {   // PDL: weight stages before waiting for the previous kernel
          first = false;
          const int pre = min(STAGES, kb1 - kb0);
          for (int i = 0; i < pre; ++i) {
            if (leader) mbar_expect_tx(&sm.full[i], PAIR_TX);
            load_b(i, kb0 + i, n0);
          }
          pdl_wait();
          for (int i = 0; i < pre; ++i) tma_load_2sm(sm.a[i], &tmA, &sm.full[i], (kb0 + i) * BK, m0);
          kb += pre;
          stage = pre % STAGES;
          phase = pre == STAGES ? 1 : 0;
        }
        for (; kb < kb1; ++kb) {
          mbar_wait(&sm.empty[stage], phase ^ 1);
          if (leader) mbar_expect_tx(&sm.full[stage], PAIR_TX);
          tma_load_2sm(sm.a[stage], &tmA, &sm.full[stage], kb * BK, m0);
          load_b(stage, kb, n0);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
      if (first) pdl_wait();
    }
  } else if (warp == 1) {
    if (leader) {
      // D f32, A/B bf16, K-major, N = 256 per instruction, M = 256 (the pair)
      const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(256 >> 3) << 17) | ((uint32_t)(256 >> 4) << 24);
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int t = pair; t < ntiles; t += npairs, ++it) {
        const int as = it % NBUF;
        const uint32_t aph = (it / NBUF) & 1;
        int m0, n0, kb0, kb1, sp;
        unit_of(t, m0, n0, kb0, kb1, sp);
        mbar_wait(&sm.tempty[as], aph ^ 1);
        asm volatile("tcgen05.fence::after_thread_sync;");
        const uint32_t d = tmem + as * NP;
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&sm.full[stage], phase);
          asm volatile("tcgen05.fence::after_thread_sync;");
          if (lane == 0) {
            const uint32_t a0 = smem_u32(sm.a[stage]), b0 = smem_u32(sm.b[stage]);
#pragma unroll
            for (int k = 0; k < BK / 16; ++k)
#pragma unroll
              for (int c = 0; c < NP / 256; ++c)
                umma_bf16_2sm(d + c * 256, umma_desc(a0 + k * 32), umma_desc(b0 + c * 128 * BK * 2 + k * 32), idesc,
                              (kb > kb0 || k) ? 1u : 0u);
            umma_commit_2sm(&sm.empty[stage]);
            if (kb == kb1 - 1) umma_commit_2sm(&sm.tfull[as]);
          }
          __syncwarp();
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else {
    pdl_wait();
    const int q = warp & 3;
    const int half = (warp - 2) >> 2;
    const int row = q * 32 + lane;
    const uint32_t tempty_leader0 = mapa_shared(smem_u32(&sm.tempty[0]), 0);
    int it = 0;
    for (int t = pair; t < ntiles; t += npairs, ++it) {
      const int as = it % NBUF;
      const uint32_t aph = (it / NBUF) & 1;
      int m0, n0, kb0, kb1, sp;
      unit_of(t, m0, n0, kb0, kb1, sp);
      mbar_wait(&sm.tfull[as], aph);
      asm volatile("tcgen05.fence::after_thread_sync;");
      const int gm = m0 + row;
      const uint32_t tbase = tmem + ((uint32_t)(q * 32) << 16) + as * NP;
      if constexpr (MODE == GEMM_SWIGLU) {
        const int F = N / 2;
#pragma unroll 1
        for (int g2 = 0; g2 < NP / 256; ++g2) {
          const int f0 = n0 / 2 + g2 * 128;
#pragma unroll 1
          for (int c = half * 32; c < 128; c += CSTEP) {
            float g[32], u[32];
            tmem_ld32(tbase + g2 * 256 + c, g);
            tmem_ld32(tbase + g2 * 256 + 128 + c, u);
            if (gm < M) {
              bf16* dst = act + (size_t)gm * F + f0 + c;
#pragma unroll
              for (int j = 0; j < 32; j += 8) {
                if (f0 + c + j + 8 <= F) {
                  __align__(16) bf16 o[8];
#pragma unroll
                  for (int e = 0; e < 8; ++e) {
                    float x = g[j + e];
                    o[e] = __float2bfloat16_rn(__fdividef(x, 1.0f + __expf(-x)) * u[j + e]);
                  }
                  *reinterpret_cast<uint4*>(dst + j) = *reinterpret_cast<uint4*>(o);
                }
              }
            }
          }
        }
      } else {
        float* Cs = C + (size_t)sp * M * N;
        store_tile_f32<NP, GEMM_STORE>(tbase, Cs, m0 + q * 32, n0, M, N, bias, smem_u32(sm.slab[(warp - 2) & 3]), lane,
                                       half * 32, CSTEP);
      }
      asm volatile("tcgen05.fence::before_thread_sync;");
      __syncwarp();
      if (lane == 0)   // release the accumulator on the LEADER's barrier (both CTAs' epilogues count)
        asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(tempty_leader0 + as * 8)
                     : "memory");
    }
  }
  __syncwarp();
  asm volatile("tcgen05.fence::before_thread_sync;");
  cluster_sync_all();   // the leader's MMAs into this CTA's TMEM / smem are done before either CTA exits
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TCOLS));
}

}  // namespace
void gemm_ts_reset() { int z = 0; cudaMemcpyToSymbol(g_gemm_ts_idx, &z, 4); }
void gemm_ts_fetch(unsigned long long* h) { cudaMemcpyFromSymbol(h, g_gemm_ts, sizeof(g_gemm_ts)); }
void gemm_trace_fetch(unsigned long long* h) { cudaMemcpyFromSymbol(h, g_gemm_trace, sizeof(g_gemm_trace)); }
// ------------------------------------------------------------------ host side
EncodeTiled get_encode() {
  static EncodeTiled fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (EncodeTiled)p;
  });
  return fn;
}
namespace {

bool make_map(CUtensorMap* m, const void* ptr, int rows, int K, int box_rows) {
  EncodeTiled enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)K * 2};
  cuuint32_t box[2] = {BK, (cuuint32_t)box_rows};
  cuuint32_t es[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Process-wide and used by every ctx: several ctx may launch from different host threads (one
// thread per rank of a tensor-parallel group), so lookups and inserts are serialised.  Entries
// are std::map nodes, so returned pointers stay valid across later inserts.
struct MapCache {
  std::map<std::tuple<const void*, int, int, int>, CUtensorMap> m;
  std::mutex mu;
  const CUtensorMap* get(const void* p, int rows, int K, int box) {
    std::lock_guard<std::mutex> lk(mu);
    auto key = std::make_tuple(p, rows, K, box);
    auto it = m.find(key);
    if (it != m.end()) return &it->second;
    CUtensorMap t;
    if (!make_map(&t, p, rows, K, box)) return nullptr;
    return &(m[key] = t);
  }
};
MapCache g_maps;

template <int BN, int MODE, int MS = 1>
bool launch_bn(const bf16* A, const bf16* B, const float* bias, float* C, bf16* act, int M, int N, int K, int S,
               cudaStream_t s, const QkvEpi* epi = nullptr, const bf16* Bt = nullptr, const TpOut* tpo = nullptr) {
  const CUtensorMap* ma = g_maps.get(A, M, K, BM);
  const CUtensorMap* mb = Bt ? ma : g_maps.get(B, N, K, MODE == GEMM_QKV_HALF ? 32 : BN);
  if (!ma || !mb) return false;
  const size_t smem = sizeof(Smem<BN, MS, Epi<MODE>::SLAB>) + 1024;
  ensure_dyn_smem(k_gemm_tc<BN, MODE, MS>, (int)smem);
  const int g_num_sms = device_sms();
  const int ntiles = ((M + MS * BM - 1) / (MS * BM)) * ((N + BN - 1) / BN) * S;
  const int grid = ntiles < g_num_sms ? ntiles : g_num_sms;
  QkvEpi e{};
  if (epi) e = *epi;
  static const int evict_b = getenv("SART_GEMM_EVICT") ? atoi(getenv("SART_GEMM_EVICT")) : 0;
  e.evict_b = evict_b;
  TpOut t{};
  if (tpo) t = *tpo;
  launch_pdl(k_gemm_tc<BN, MODE, MS>, dim3(grid), dim3(Epi<MODE>::NTHREADS), smem, s, *ma, *mb, Bt, C, bias, act, M, N, K, S, e,
             t);
  return true;
}
template <int NP, int MODE>
bool launch_2sm(const bf16* A, const bf16* B, const float* bias, float* C, bf16* act, int M, int N, int K, int S,
                cudaStream_t s) {
  const CUtensorMap* ma = g_maps.get(A, M, K, BM);
  const CUtensorMap* mb = g_maps.get(B, N, K, 128);
  if (!ma || !mb) return false;
  const size_t smem = sizeof(Smem2<NP>) + 1024;
  ensure_dyn_smem(k_gemm_2sm<NP, MODE>, (int)smem);
  const int npairs_max = device_sms() / 2;
  const int ntiles = ((M + 2 * BM - 1) / (2 * BM)) * ((N + NP - 1) / NP) * S;
  const int pairs = ntiles < npairs_max ? ntiles : npairs_max;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(2 * pairs);
  cfg.blockDim = dim3(Epi<MODE>::NTHREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k_gemm_2sm<NP, MODE>, *ma, *mb, C, bias, act, M, N, K, S) == cudaSuccess;
}
}  // namespace
// CTA-pair routing (bit mask; SART_GEMM_2SM overrides): 1 = fused gate/up SwiGLU, 2 = split-K
// long-K projections (down), 4 = LM head
int gemm_2sm_mask() {
  // default 2: measured on C2 in-graph -- down -0.8%, SwiGLU and LM head neutral (the SwiGLU
  // mainloop already runs at ~77% of the per-SM MMA rate; profiles/r2_gemm_2sm_ab.txt)
  static const int v = getenv("SART_GEMM_2SM") ? atoi(getenv("SART_GEMM_2SM")) : 2;
  return v;
}

bool launch_gemm_2sm(const bf16* A, const bf16* B, const float* bias, float* C, bf16* act, int M, int N, int K,
                     int mode, int S, int NP, cudaStream_t s) {
  if (M <= 0 || N <= 0) return true;
  if (K % 8 || N % 256) return false;
  if (mode == GEMM_SWIGLU && S == 1 && NP == 512) return launch_2sm<512, GEMM_SWIGLU>(A, B, bias, C, act, M, N, K, 1, s);
  if (mode == GEMM_SWIGLU && S == 1 && NP == 256) return launch_2sm<256, GEMM_SWIGLU>(A, B, bias, C, act, M, N, K, 1, s);
  if (mode == GEMM_STORE && NP == 256) return launch_2sm<256, GEMM_STORE>(A, B, bias, C, act, M, N, K, S, s);
  if (mode == GEMM_STORE && NP == 512) return launch_2sm<512, GEMM_STORE>(A, B, bias, C, act, M, N, K, S, s);
  return false;
}

bool launch_gemm_sample(const bf16* A, const bf16* B, float* C, int M, int N, int K, const QkvEpi& epi,
                        cudaStream_t s) {
  if (M <= 0) return true;
  if (K % 8) return false;
  return launch_bn<256, GEMM_SAMPLE, 1>(A, B, nullptr, C, nullptr, M, N, K, 1, s, &epi);
}
int gemm_sample_slots(int V) { return (V + 255) / 256 * (Epi<GEMM_SAMPLE>::NEPI / 4); }

bool launch_gemm_tc(const bf16* A, const bf16* B, const float* bias, float* C, bf16* act, int M, int N, int K,
                    int mode, cudaStream_t s, const bf16* Bt) {
  // 256-row tiles (two MMA tiles per weight stage) once they still fill ~3/4 of the SMs:
  // measured 7% faster on the C2 gate/up projection (profiles/r1_gemm_bm256_sweep.txt)
  const int g_num_sms = device_sms();
  if (!Bt && M > BM && N % 512 == 0 && (gemm_2sm_mask() & (mode == GEMM_SWIGLU ? 1 : 4)) &&
      (mode == GEMM_SWIGLU || mode == GEMM_STORE))
    return launch_gemm_2sm(A, B, bias, C, act, M, N, K, mode, 1, mode == GEMM_SWIGLU ? 512 : 256, s);
  const int ms = (mode == GEMM_SWIGLU && M > BM && ((M + 2 * BM - 1) / (2 * BM)) * ((N + 255) / 256) >= g_num_sms * 3 / 4)
                     ? 2 : 1;
  return launch_gemm_tc_split(A, B, bias, C, act, M, N, K, mode, 1, 256, ms, s, Bt);
}

bool launch_gemm_tc_split(const bf16* A, const bf16* B, const float* bias, float* C, bf16* act, int M, int N, int K,
                          int mode, int S, int BN, int MSUB, cudaStream_t s, const bf16* Bt, const TpOut* tp) {
  if (M <= 0 || N <= 0) return true;
  if (tp && tp->tp > 1) {   // TP exchange: plain partial stores only
    if (mode != GEMM_STORE || MSUB != 1) return false;
    if (BN == 128) return launch_bn<128, GEMM_STORE>(A, B, bias, C, act, M, N, K, S, s, nullptr, Bt, tp);
    if (BN == 256) return launch_bn<256, GEMM_STORE>(A, B, bias, C, act, M, N, K, S, s, nullptr, Bt, tp);
    return false;
  }
  if (K % 8) return false;   // TMA row stride must be a multiple of 16 bytes
  const int kb = (K + BK - 1) / BK;
  if (S < 1 || S > kb || (mode == GEMM_SWIGLU && S != 1)) return false;
  if (MSUB == 2) {
    if (BN == 128 && mode == GEMM_STORE) return launch_bn<128, GEMM_STORE, 2>(A, B, bias, C, act, M, N, K, S, s, nullptr, Bt);
    if (BN == 256 && mode == GEMM_STORE) return launch_bn<256, GEMM_STORE, 2>(A, B, bias, C, act, M, N, K, S, s, nullptr, Bt);
    if (BN == 256 && mode == GEMM_SWIGLU) return launch_bn<256, GEMM_SWIGLU, 2>(A, B, bias, C, act, M, N, K, S, s, nullptr, Bt);
    return false;
  }
  if (MSUB != 1) return false;
  if (BN == 64) {
    if (mode == GEMM_STORE) return launch_bn<64, GEMM_STORE>(A, B, bias, C, act, M, N, K, S, s, nullptr, Bt);
    return false;
  }
  if (BN == 128) {
    if (mode == GEMM_STORE) return launch_bn<128, GEMM_STORE>(A, B, bias, C, act, M, N, K, S, s, nullptr, Bt);
    if (mode == GEMM_ACCUM) return launch_bn<128, GEMM_ACCUM>(A, B, bias, C, act, M, N, K, S, s, nullptr, Bt);
    return false;
  }
  if (mode == GEMM_STORE) return launch_bn<256, GEMM_STORE>(A, B, bias, C, act, M, N, K, S, s, nullptr, Bt);
  if (mode == GEMM_ACCUM) return launch_bn<256, GEMM_ACCUM>(A, B, bias, C, act, M, N, K, S, s, nullptr, Bt);
  return launch_bn<256, GEMM_SWIGLU>(A, B, bias, C, act, M, N, K, S, s, nullptr, Bt);
}

// Split count that minimises the wave-quantised time of t output tiles x S splits on the SMs
// of a persistent launch: cost(S) = ceil(t S / SMs) / S (a unit does 1/S of a tile's K);
// ties go to fewer splits (less partial traffic).  E.g. t = 32 tiles: S = 4 (128 units, one
// wave) instead of 5 (160 units = two waves, the second 12 units long).
static int wave_split(int t, int smax) {
  const int g_num_sms = device_sms();
  int best = 1;
  double bc = 1e30;
  for (int S = 1; S <= smax; ++S) {
    const double c = (double)((t * S + g_num_sms - 1) / g_num_sms) / S;
    if (c < bc - 1e-9) { bc = c; best = S; }
  }
  return best;
}

bool launch_gemm_qkv(const bf16* A, const bf16* B, int M, int N, int K, const QkvEpi& epi, cudaStream_t s,
                     const bf16* Bt) {
  if (M <= 0) return true;
  if (K % 8) return false;
  // split-K so that (m-tiles x heads x splits) covers the SMs; the last split of each tile
  // runs the fused bias + RoPE + KV-append epilogue
  const int g_num_sms = device_sms();
  const int mt = (M + BM - 1) / BM, heads = N / epi.D.hd, kb = (K + BK - 1) / BK;
  int S = 1;
  if (epi.parts && epi.cnt && heads * mt * 8 <= epi.cnt_cap && epi.D.hd >= 128) {
    // measured on C2 (K = 1536): the fused single-pass kernel is 3% faster per step than S = 2
    // with the partial round trip; long-K projections (14B / 70B, K >= 4096) at small M leave
    // most SMs idle without splits.  SART_QKV_SPLIT = max splits overrides.
    static const int smax_env = getenv("SART_QKV_SPLIT") ? atoi(getenv("SART_QKV_SPLIT")) : 0;
    const int smax = smax_env ? smax_env : 1;
    S = wave_split(heads * mt, std::max(1, std::min(smax, std::min(8, kb / 2))));
  }
  // half-head tiles (2 CTAs per head) when the doubled tile count still fits one wave: C2's
  // 16 heads x 4 m-tiles = 64 one-head CTAs leave 84 SMs idle.  SART_QKV_HALF=0 disables.
  static const int half_env = getenv("SART_QKV_HALF") ? atoi(getenv("SART_QKV_HALF")) : 1;
  if (epi.D.hd == 128 && S == 1 && !Bt && half_env && 2 * heads * mt <= g_num_sms)
    return launch_bn<64, GEMM_QKV_HALF>(A, B, nullptr, epi.parts, nullptr, M, N, K, 1, s, &epi);
  if (epi.D.hd == 128) return launch_bn<128, GEMM_QKV>(A, B, nullptr, epi.parts, nullptr, M, N, K, S, s, &epi, Bt);
  if (epi.D.hd == 64) return launch_bn<64, GEMM_QKV>(A, B, nullptr, epi.parts, nullptr, M, N, K, S, s, &epi, Bt);
  return false;
}

// Split choice for the decode GEMMs: enough (tile x split) units to cover the SMs.
void choose_split(int M, int N, int K, int& S, int& BN, int& MSUB) {
  MSUB = 1;
  // measured on B200 at M = 512 (tools/gemm_sweep.py): long-K projections prefer 256-wide
  // tiles with more splits, short-K ones 128-wide tiles; aim for ~one unit per SM
  const int g_num_sms = device_sms();
  const int mt = (M + BM - 1) / BM;
  const int kb = (K + BK - 1) / BK;
  const int t256 = mt * ((N + 255) / 256);
  if (t256 >= g_num_sms * 3 / 4) { S = 1; BN = 256; return; }
  BN = K >= 4096 ? 256 : 128;
  const int t = mt * ((N + BN - 1) / BN);
  S = wave_split(t, std::max(1, std::min(8, kb / 2)));
}

// ------------------------------------------------------------------ pre-tiled weights
// Wt[n-tile][k-block] = the exact shared-memory image of the (BN x 64) K-major tile with the
// 128-byte swizzle (16-byte chunk c of row r stored at c ^ (r & 7)); rows >= N and columns >= K
// are zero.  One contiguous BN*128-byte bulk copy per stage replaces BN strided 128-byte rows.
__global__ void k_tile_b(const bf16* __restrict__ W, bf16* __restrict__ Wt, int N, int K, int BN, int KB,
                         long long chunks) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < chunks; i += (long long)gridDim.x * blockDim.x) {
    const int c = (int)(i & 7);                 // source 16-byte chunk within the row's 64 columns
    const long long rowid = i >> 3;             // (n-tile, k-block, r)
    const int r = (int)(rowid % BN);
    const long long tk = rowid / BN;
    const int kb = (int)(tk % KB);
    const int nt = (int)(tk / KB);
    const int n = nt * BN + r, k = kb * BK + c * 8;
    uint4 v = make_uint4(0, 0, 0, 0);
    if (n < N) {
      if (k + 8 <= K && (K & 7) == 0) v = *reinterpret_cast<const uint4*>(W + (size_t)n * K + k);
      else {
        __align__(16) bf16 t[8];
        for (int e = 0; e < 8; ++e) t[e] = (k + e < K) ? W[(size_t)n * K + k + e] : __float2bfloat16_rn(0.f);
        v = *reinterpret_cast<uint4*>(t);
      }
    }
    *reinterpret_cast<uint4*>(Wt + rowid * BK + ((c ^ (r & 7)) << 3)) = v;
  }
}

size_t tiled_b_elems(int N, int K, int BN) {
  return (size_t)((N + BN - 1) / BN) * BN * (size_t)((K + BK - 1) / BK) * BK;
}
void launch_tile_b(const bf16* W, bf16* Wt, int N, int K, int BN, cudaStream_t s) {
  const int KB = (K + BK - 1) / BK;
  const long long chunks = (long long)tiled_b_elems(N, K, BN) / 8;
  const int blocks = (int)std::min<long long>((chunks + 255) / 256, 148LL * 16);
  k_tile_b<<<blocks, 256, 0, s>>>(W, Wt, N, K, BN, KB, chunks);
}
