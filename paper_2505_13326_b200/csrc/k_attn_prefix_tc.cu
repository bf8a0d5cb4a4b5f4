// Tensor-core (tcgen05) prefix pass of the cascade decode attention (SURVEY §8(a) row a4,
// K1 "prefix pass"; PAPER P:306 shares the prompt's KV across a request's branches).
//
// For one item = (prefix group of one request, prefix chunk [t0, t1) of <= CH tokens, kv head
// h) it computes, for EVERY query row of the group at once (n_r branch rows x g q heads <= 128,
// one TMEM lane each), the chunk's normalised partial output and log-sum-exp
//
//   o_i = sum_{t in chunk} softmax_t(q_i . k_t / sqrt(hd)) v_t,   lse_i = log2 sum_t exp2(...)
//
// and writes them into the same partial slots (slot = chunk index) the mma.sync prefix tasks
// of k_attn_cascade would have written; k_attn_merge combines them with the suffix partials
// unchanged.  Each prefix KV byte is read from HBM once per (request, kv head) and multiplied
// by all 128 query rows on the tensor cores -- the mma.sync path re-reads it (from L2) once
// per 16-row m-tile and is bound by per-warp instruction latency (C5).
//
// Structure (one CTA per SM, persistent; items assigned round-robin, so which CTA computes an
// item never changes its result):
//   warp 0      TMA producer: 64-token K / V tiles of the paged pool through a 4-stage ring.
//               The pool's per-row XOR pre-swizzle (common.cuh kv_swz: 16-byte chunk c of
//               token row t at c ^ (t & 7)) IS the 128-byte-swizzle layout UMMA expects once
//               each 256-byte row is split into two 128-byte halves, so a 3-D tensor map
//               {64 elements, half, token row} with SWIZZLE_NONE lands every tile in
//               shared memory ready for the MMA (no re-layout pass).
//   warp 1      TMEM owner + MMA issuer (one lane):  S_j = Q K_j^T  (M 128, N 64, K hd; K-major
//               Q and K) into one of two S buffers, then O += P_{j-1} V_{j-1} (M 128, N hd, K 64;
//               K-major P, MN-major V straight from the tile).
//   warps 2..5  softmax, one query row per thread: tcgen05.ld of its S row, online softmax with
//               a lazy rescale (O in TMEM is rescaled only when the running max grows by more
//               than 2^8 -- exact, the stale max cancels in o / l), P (bf16) to shared memory,
//               and at the item's end O / l and the lse to the partial slot.
//
// MODE = PT_PREFILL is the tensor-core causal prefill of row f1 (Alg. 1 L15): an item is
// (a block of <= 128 prompt positions of one request, one q head); its rows see keys
// [0, position] of the request's prefix pages (written by this layer's QKV epilogue), and O / l
// is written in bf16 as the prefill's attention output.  MODE = PT_SUF is the same for the f2
// PRM pass: the rows are one batch row's new suffix entries, the keys its prefix pages
// (padding slots masked) followed by its suffix entries.
#include <algorithm>
#include <cstdlib>

#include "kernels.h"
#include "umma.cuh"

namespace {
constexpr int PT_KT = 64;    // key tokens per KV tile (one S buffer = 64 TMEM columns)
constexpr int PT_M = 128;    // query rows per item (TMEM lanes)
constexpr float PT_LAZY = 8.f;   // rescale O only when the max grows by more than 2^8 (log2 units)

// NS KV tile stages, NP P buffers (P(g) in buffer g % NP); (NS, NP) = (4, 2): one CTA per SM
// (~194 KB), (2, 1): two CTAs per SM (112 KB each, 256 TMEM columns each) whose softmax and
// MMA phases interleave.  Layout from a 1024-byte aligned base: q | k | v | p (all 1024-byte
// multiples, as the SW128 UMMA descriptors need) | mbarriers | TMEM base address.
template <int HD, int NS, int NP>
struct PtView {
  static constexpr int NH = HD / 64;                   // 128-byte column halves of a row
  static constexpr size_t QB = (size_t)NH * PT_M * 64 * 2, KB = (size_t)NS * NH * PT_KT * 64 * 2,
                          PB = (size_t)NP * PT_M * PT_KT * 2, NBAR = 2 * NS + 4 + 2 * NP + 1;
  static constexpr size_t BYTES = QB + 2 * KB + PB + 8 * NBAR + 16;
  static constexpr size_t XBYTES = 4 * 4 * PT_M;     // pair-exchange arrays (NSM = 8 only)
  bf16 (*q)[PT_M * 64];                                // Q, K-major SW128: [half][row][64]
  bf16 (*k)[NH][PT_KT * 64];                           // K tile: [half][token][64] (K-major B of S)
  bf16 (*v)[NH][PT_KT * 64];                           // V tile: same bytes, MN-major B of O
  bf16 (*p)[PT_M * PT_KT];                             // P, K-major SW128: [row][64 tokens]
  uint64_t *kv_full, *kv_empty, *s_full, *s_free, *p_full, *o_done;   // [NS] [NS] [2] [2] [NP] [NP]
  uint64_t& q_full;
  uint32_t& tmem_base;
  float* xch;     // [4][PT_M] two softmax warps per row (NSM = 8): max of each half, l after half 0, l
  __device__ explicit PtView(uint8_t* b)
      : q(reinterpret_cast<bf16 (*)[PT_M * 64]>(b)),
        k(reinterpret_cast<bf16 (*)[NH][PT_KT * 64]>(b + QB)),
        v(reinterpret_cast<bf16 (*)[NH][PT_KT * 64]>(b + QB + KB)),
        p(reinterpret_cast<bf16 (*)[PT_M * PT_KT]>(b + QB + 2 * KB)),
        kv_full(reinterpret_cast<uint64_t*>(b + QB + 2 * KB + PB)),
        kv_empty(kv_full + NS), s_full(kv_empty + NS), s_free(s_full + 2), p_full(s_free + 2), o_done(p_full + NP),
        q_full(o_done[NP]), tmem_base(*reinterpret_cast<uint32_t*>(o_done + NP + 1)),
        xch(reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(o_done + NP + 1) + 16)) {}
};

__device__ __forceinline__ uint32_t pack_bf16_pt(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}

struct PtItem {
  int t0, t1, tab, slot_idx, grp, nq, h;
  int head, r0, nr, p0;   // causal modes: q head, first batch row, rows, first key index of the block
  int rtab, npre, pbase;  // PT_SUF: row table offset; masked padding keys [npre, pbase) of the prefix pages
};
// modes: PT_PREFIX = the cascade's prefix pass (partials); PT_PREFILL = causal prefill of
// prompt positions; PT_SUF = the f2 PRM pass (a row's new suffix entries over the virtual key
// space [prefix pages (pbase slots, slots >= P - 1 masked) ; suffix entries])
enum { PT_PREFIX = 0, PT_PREFILL = 1, PT_SUF = 2 };
// item i: prefix pass = (tc task i / kvh, kv head i % kvh); causal modes = (query block i / qh
// of <= 128 rows, q head i % qh), keys [0, p0 + nr)
template <int MODE>
__device__ __forceinline__ PtItem pt_item(const AttnPlan& pl, const Dims& D, const Rows& rows, const Reqs& reqs,
                                          const int4* __restrict__ blocks, int i) {
  PtItem it;
  it.rtab = 0;
  it.npre = it.pbase = 0x7fffffff;
  if constexpr (MODE != PT_PREFIX) {
    const int4 b = __ldg(blocks + i / D.qh);
    it.head = i % D.qh;
    it.h = it.head / D.g;
    it.r0 = b.x;
    it.nr = b.y;
    it.t0 = 0;
    it.slot_idx = it.grp = it.nq = 0;
    if constexpr (MODE == PT_PREFILL) {                  // {first batch row, rows, slot, first position}
      it.p0 = b.w;
      it.tab = b.z * D.MPB;
    } else {                                             // {first token, entries, row, first entry}
      const int slot = rows.slot[b.z];
      it.npre = reqs.P[slot] - 1;
      it.pbase = (it.npre + D.bs - 1) / D.bs * D.bs;
      it.p0 = it.pbase + b.w;
      it.tab = slot * D.MPB;
      it.rtab = b.z * D.MBR;
    }
    it.t1 = it.p0 + it.nr;
  } else {
    const int task = i / D.kvh;
    it.h = i % D.kvh;
    const int4 a = __ldcg(pl.tc_items + 2 * task);
    const int4 b = __ldcg(pl.tc_items + 2 * task + 1);
    it.t0 = a.x;
    it.t1 = a.y;
    it.tab = a.z;
    it.slot_idx = a.w;
    it.grp = b.y;
    it.nq = b.w;
    it.head = it.r0 = it.nr = it.p0 = 0;
  }
  return it;
}

template <int HD, int MODE, int NS, int NP, int MINB, int NSM = 4>
__global__ void __launch_bounds__(64 + 32 * NSM, MINB)
    k_attn_prefix_tc(const __grid_constant__ CUtensorMap kvmap, const bf16* __restrict__ q, float* __restrict__ part_o,
                     float* __restrict__ part_lse, bf16* __restrict__ out, const int4* __restrict__ blocks, int nblocks,
                     Dims D, int layer, Rows rows, Reqs reqs, AttnPlan pl) {
  constexpr int NH = HD / 64;
  constexpr uint32_t TMEM_COLS = 256;                  // S0 | S1 | O (HD <= 128 columns)
  constexpr uint32_t O_COL = 128;
  extern __shared__ __align__(1024) uint8_t pt_raw[];
  // one CTA per SM: the launch adds 1024 bytes of slack to align the base here; two per SM
  // have no room for it, and rely on the dynamic window starting 1024-aligned (checked)
  uint8_t* base = pt_raw;
  if constexpr (MINB == 1) base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(pt_raw) + 1023) & ~uintptr_t(1023));
  else if (smem_u32(pt_raw) & 1023) __trap();
  PtView<HD, NS, NP> sm(base);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int i = 0; i < NS; ++i) {
      mbar_init(&sm.kv_full[i], 1);
      mbar_init(&sm.kv_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&sm.s_full[i], 1);
      mbar_init(&sm.s_free[i], NSM);
    }
    for (int i = 0; i < NP; ++i) {
      mbar_init(&sm.p_full[i], NSM);
      mbar_init(&sm.o_done[i], 1);
    }
    mbar_init(&sm.q_full, NSM);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&sm.tmem_base)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  // stale V rows of a partial last tile are multiplied by P = 0: keep them finite
  for (int e = threadIdx.x; e < NS * NH * PT_KT * 64 / 8; e += blockDim.x) {
    reinterpret_cast<uint4*>(&sm.k[0][0][0])[e] = make_uint4(0, 0, 0, 0);
    reinterpret_cast<uint4*>(&sm.v[0][0][0])[e] = make_uint4(0, 0, 0, 0);
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = sm.tmem_base;
  pdl_wait();        // q of this step (QKV GEMM) and the step's item list are visible
  pdl_trigger();
  constexpr bool CAUSAL = MODE != PT_PREFIX;
  const int n_items = CAUSAL ? nblocks * D.qh : *pl.n_tc * D.kvh;
  const float sl2 = 1.4426950408889634f * rsqrtf((float)HD);   // log2(e) / sqrt(hd)

  if (warp == 0) {
    // ---------------------------------------------------------------- TMA producer
    if (lane == 0) {
      const int tpb = D.bs < PT_KT ? D.bs : PT_KT;     // tokens per box (whole page pieces)
      uint32_t tile = 0;
      for (int i = blockIdx.x; i < n_items; i += gridDim.x) {
        const PtItem it = pt_item<MODE>(pl, D, rows, reqs, blocks, i);
        const int* tab = reqs.prefix + it.tab;
        const int* rtab = rows.table + it.rtab;            // PT_SUF: keys >= pbase are suffix entries
        for (int s0 = it.t0; s0 < it.t1; s0 += PT_KT, ++tile) {
          const int st = tile % NS;
          mbar_wait(&sm.kv_empty[st], ((tile / NS) & 1) ^ 1);
          const int ntok = min(PT_KT, it.t1 - s0);
          const int pieces = (ntok + tpb - 1) / tpb;
          mbar_expect_tx(&sm.kv_full[st], (uint32_t)(pieces * tpb * 2 * HD * 2));
          for (int pc = 0; pc < pieces; ++pc) {
            const int tok = s0 + pc * tpb;
            const long long blk = tok < it.pbase ? tab[tok / D.bs] : rtab[(tok - it.pbase) / D.bs];
            const long long base = ((((long long)layer * D.NB + blk) * 2) * D.kvh + it.h) * D.bs + tok % D.bs;
            const int rk = (int)base, rv = (int)(base + (long long)D.kvh * D.bs);
#pragma unroll
            for (int hh = 0; hh < NH; ++hh) {
              tma_load_3d(&sm.k[st][hh][pc * tpb * 64], &kvmap, &sm.kv_full[st], 0, hh, rk);
              tma_load_3d(&sm.v[st][hh][pc * tpb * 64], &kvmap, &sm.kv_full[st], 0, hh, rv);
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------------- MMA issuer
    // S = Q K^T: M 128, N 64, both K-major.  O += P V: M 128, N HD, P K-major, V MN-major.
    const uint32_t idesc_s = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(PT_KT >> 3) << 17) | ((uint32_t)(PT_M >> 4) << 24);
    const uint32_t idesc_o =
        (1u << 4) | (1u << 7) | (1u << 10) | (1u << 16) | ((uint32_t)(HD >> 3) << 17) | ((uint32_t)(PT_M >> 4) << 24);
    const uint32_t qa = smem_u32(&sm.q[0][0]);
    // PV of tile g reads P buffer g % NP and completes on o_done[g % NP] (phase g / NP)
    auto issue_pv = [&](uint32_t g, bool first) {
      const int st = g % NS;
      const uint32_t pa = smem_u32(&sm.p[g % NP][0]);
      mbar_wait(&sm.p_full[g % NP], (g / NP) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;");
      if (lane == 0) {
        const uint32_t va = smem_u32(&sm.v[st][0][0]);
#pragma unroll
        for (int kk = 0; kk < PT_KT / 16; ++kk)
          umma_bf16(tmem + O_COL, umma_desc_k(pa + kk * 32), umma_desc_mn(va + kk * 16 * 128, PT_KT * 128), idesc_o,
                    (first && kk == 0) ? 0u : 1u);
        umma_commit(&sm.kv_empty[st]);
        umma_commit(&sm.o_done[g % NP]);
      }
      __syncwarp();
    };
    uint32_t tile = 0, icnt = 0;
    for (int i = blockIdx.x; i < n_items; i += gridDim.x, ++icnt) {
      const PtItem it = pt_item<MODE>(pl, D, rows, reqs, blocks, i);
      const int nt = (it.t1 - it.t0 + PT_KT - 1) / PT_KT;
      mbar_wait(&sm.q_full, icnt & 1);
      for (int kt = 0; kt < nt; ++kt) {
        const uint32_t g = tile + kt;
        const int st = g % NS, b = g & 1;
        mbar_wait(&sm.kv_full[st], (g / NS) & 1);
        mbar_wait(&sm.s_free[b], ((g >> 1) & 1) ^ 1);
        asm volatile("tcgen05.fence::after_thread_sync;");
        if (lane == 0) {
          const uint32_t ka = smem_u32(&sm.k[st][0][0]);
#pragma unroll
          for (int kk = 0; kk < HD / 16; ++kk) {
            const uint32_t off = (kk / 4) * (PT_M * 128) + (kk % 4) * 32;
            const uint32_t koff = (kk / 4) * (PT_KT * 128) + (kk % 4) * 32;
            umma_bf16(tmem + b * PT_KT, umma_desc_k(qa + off), umma_desc_k(ka + koff), idesc_s, kk ? 1u : 0u);
          }
          umma_commit(&sm.s_full[b]);
        }
        __syncwarp();
        if (kt > 0) issue_pv(g - 1, kt == 1);
      }
      issue_pv(tile + nt - 1, nt == 1);
      tile += nt;
    }
  } else {
    // ---------------------------------------------------------------- softmax (one row / thread)
    // NSM = 8: two warps per TMEM lane quarter share each row, half of the 64 key columns each;
    // they exchange the half maxima and hand the row sum over in column order (half 0's chain
    // continues in half 1), so every value is the same as with one warp per row
    constexpr int HH = NSM / 4, KC = PT_KT / HH;
    const int quarter = warp & 3;
    const int hf = HH == 1 ? 0 : (warp - 2) >> 2;      // which key-column half this warp owns
    const int j = quarter * 32 + lane;                 // query row of the item = TMEM lane
    const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
    float* xmax = sm.xch;                              // [2][PT_M]
    float* xl0 = sm.xch + 2 * PT_M;                    // l after half 0's columns
    float* xlf = sm.xch + 3 * PT_M;                    // l after the whole tile
    auto pair_sync = [&]() {
      if constexpr (HH == 2) asm volatile("bar.sync %0, 64;" ::"r"(1 + quarter) : "memory");
    };
    uint32_t tile = 0, icnt = 0;
    for (int i = blockIdx.x; i < n_items; i += gridDim.x, ++icnt) {
      const PtItem it = pt_item<MODE>(pl, D, rows, reqs, blocks, i);
      const int nt = (it.t1 - it.t0 + PT_KT - 1) / PT_KT;
      int row = -1, head = 0;
      if constexpr (CAUSAL) {
        if (j < it.nr) { row = it.r0 + j; head = it.head; }
      } else if (j < it.nq) {
        row = pl.grp_rows[it.grp * pl.qr_max + j / D.g];
        head = it.h * D.g + j % D.g;
      }
      // Q row j -> shared memory, K-major SW128 (chunk c of row j at c ^ (j & 7)); the previous
      // item's MMAs that read Q are complete (its last o_done was waited on below)
      {
        const uint4* src = row >= 0 ? reinterpret_cast<const uint4*>(q + ((long long)row * D.qh + head) * HD) : nullptr;
#pragma unroll
        for (int hh = 0; hh < NH; ++hh) {
          if (HH == 2 && (hh & 1) != hf) continue;
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            const uint4 v = src ? __ldg(src + hh * 8 + c) : make_uint4(0, 0, 0, 0);
            *reinterpret_cast<uint4*>(reinterpret_cast<uint8_t*>(&sm.q[hh][0]) + j * 128 + ((c ^ (j & 7)) << 4)) = v;
          }
        }
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&sm.q_full);

      float m = -INFINITY, l = 0.f;
      for (int kt = 0; kt < nt; ++kt) {
        const uint32_t g = tile + kt;
        const int b = g & 1;
        mbar_wait(&sm.s_full[b], (g >> 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;");
        uint32_t sr[KC];
#pragma unroll
        for (int c = 0; c < KC; c += 32) tmem_ld32_nw(tmem + lane_off + b * PT_KT + hf * KC + c, sr + c);
        tmem_wait_ld();
        asm volatile("tcgen05.fence::before_thread_sync;");
        __syncwarp();
        if (lane == 0) mbar_arrive(&sm.s_free[b]);
        // keys of this tile the row may see: >= 1 in its first tile (key 0 precedes every
        // position); causal: key index <= the row's position p0 + j.  Column c of this
        // warp's half is key column hf * KC + c of the tile.
        int nvalid = it.t1 - (it.t0 + kt * PT_KT);
        if constexpr (CAUSAL) nvalid = min(nvalid, it.p0 + j - kt * PT_KT + 1);
        nvalid -= hf * KC;
        // PT_SUF: the prefix pages' padding slots [npre, pbase) of this tile are masked
        const int h0 = it.npre - (it.t0 + kt * PT_KT) - hf * KC, h1 = it.pbase - (it.t0 + kt * PT_KT) - hf * KC;
        // warp-uniform fast path: every key of the half is visible to every row of the warp
        // (all but the diagonal / ragged / padding tiles) -- no per-element predicates
        const bool wfull = __all_sync(0xffffffffu, nvalid >= KC && (MODE != PT_SUF || h1 <= 0 || h0 >= KC));
        auto vis = [&](int c) { return wfull || (c < nvalid && (MODE != PT_SUF || c < h0 || c >= h1)); };
        float mx8[8];   // 8 independent max chains (max is order-free)
#pragma unroll
        for (int e = 0; e < 8; ++e) mx8[e] = -INFINITY;
        if (wfull) {
#pragma unroll
          for (int c = 0; c < KC; ++c) mx8[c & 7] = fmaxf(mx8[c & 7], __uint_as_float(sr[c]));
        } else {
#pragma unroll
          for (int c = 0; c < KC; ++c)
            if (vis(c)) mx8[c & 7] = fmaxf(mx8[c & 7], __uint_as_float(sr[c]));
        }
        float mx = fmaxf(fmaxf(fmaxf(mx8[0], mx8[1]), fmaxf(mx8[2], mx8[3])),
                         fmaxf(fmaxf(mx8[4], mx8[5]), fmaxf(mx8[6], mx8[7])));
        if constexpr (HH == 2) {
          xmax[hf * PT_M + j] = mx;
          pair_sync();                                   // B1: both halves' maxima are written
          mx = fmaxf(mx, xmax[(1 - hf) * PT_M + j]);
          if (hf == 0 && kt > 0) l = xlf[j];             // the row sum through the previous tile
        }
        const float mn = fmaxf(m, mx);
        const bool grow = kt == 0 || (mn - m) * sl2 > PT_LAZY;
        // P buffer g % NP is free once PV(g - NP) has completed; O may be rescaled only after
        // PV(g - 1).  (No barrier can be two phases ahead of a wait: PV(t + NP) needs
        // P(t + NP), which is written only after PV(t) was waited for.)
        auto wait_pv = [&](uint32_t t) { mbar_wait(&sm.o_done[t % NP], (t / NP) & 1); };
        if (g >= NP) wait_pv(g - NP);
        asm volatile("tcgen05.fence::after_thread_sync;");
        if (kt > 0 && __any_sync(0xffffffffu, grow)) {
          wait_pv(g - 1);
          asm volatile("tcgen05.fence::after_thread_sync;");
          const float c = grow ? exp2f((m - mn) * sl2) : 1.f;
#pragma unroll 1
          for (int cb = hf * (HD / HH); cb < (hf + 1) * (HD / HH); cb += 32) {   // this warp's O columns
            uint32_t o[32];
            tmem_ld32_nw(tmem + lane_off + O_COL + cb, o);
            tmem_wait_ld();
#pragma unroll
            for (int e = 0; e < 32; ++e) o[e] = __float_as_uint(__uint_as_float(o[e]) * c);
            tmem_st32(tmem + lane_off + O_COL + cb, o);
          }
          tmem_wait_st();
          if (grow) l *= c;
        }
        if (grow) m = mn;
        const float mo = m * sl2;
        uint8_t* prow = reinterpret_cast<uint8_t*>(&sm.p[g % NP][0]) + j * 128;
        // l is one chain in column order and p = exp2f(.): the same arithmetic as the masked
        // form (a masked key adds an exact 0), so the fast path leaves every result unchanged
        // (a 4-chain sum moved a full-size C2 logits row from 0.0196 to 0.0200)
        if (!wfull)   // masked keys -> -inf: their p is exactly 0
#pragma unroll
          for (int c = 0; c < KC; ++c)
            if (!vis(c)) sr[c] = __float_as_uint(-INFINITY);
        float pk[KC];
#pragma unroll
        for (int c8 = 0; c8 < KC / 8; ++c8) {
#pragma unroll
          for (int e = 0; e < 8; ++e) pk[c8 * 8 + e] = exp2f(fmaf(__uint_as_float(sr[c8 * 8 + e]), sl2, -mo));
          uint4 w;
          w.x = pack_bf16_pt(pk[c8 * 8 + 0], pk[c8 * 8 + 1]);
          w.y = pack_bf16_pt(pk[c8 * 8 + 2], pk[c8 * 8 + 3]);
          w.z = pack_bf16_pt(pk[c8 * 8 + 4], pk[c8 * 8 + 5]);
          w.w = pack_bf16_pt(pk[c8 * 8 + 6], pk[c8 * 8 + 7]);
          const int cg = hf * (KC / 8) + c8;             // 16-byte chunk of the 64-key P row
          *reinterpret_cast<uint4*>(prow + ((cg ^ (j & 7)) << 4)) = w;
        }
        if constexpr (HH == 2) {                         // B2: half 0's running sum -> half 1
          if (hf == 0) {
#pragma unroll
            for (int c = 0; c < KC; ++c) l += pk[c];
            xl0[j] = l;
            pair_sync();
          } else {
            pair_sync();
            l = xl0[j];
#pragma unroll
            for (int c = 0; c < KC; ++c) l += pk[c];
            xlf[j] = l;
          }
        } else {
#pragma unroll
          for (int c = 0; c < KC; ++c) l += pk[c];
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("tcgen05.fence::before_thread_sync;");
        __syncwarp();
        if (lane == 0) mbar_arrive(&sm.p_full[g % NP]);
      }
      if constexpr (HH == 2) {                           // the whole row sum to both halves
        pair_sync();
        if (hf == 0) l = xlf[j];
      }
      // item done: O / l and the lse into the partial slot of (row, head)
      const uint32_t glast = tile + nt - 1;
      mbar_wait(&sm.o_done[glast % NP], (glast / NP) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;");
      const float inv = 1.f / l;
      if constexpr (CAUSAL) {   // the prefill's attention output, bf16 [row][qh][hd]
        bf16* dst = row >= 0 ? out + ((long long)row * D.qh + head) * HD : nullptr;
#pragma unroll 1
        for (int cb = hf * (HD / HH); cb < (hf + 1) * (HD / HH); cb += 32) {
          uint32_t o[32];
          tmem_ld32_nw(tmem + lane_off + O_COL + cb, o);
          tmem_wait_ld();
          if (dst)
#pragma unroll
            for (int e = 0; e < 32; e += 8) {
              uint4 w;
              w.x = pack_bf16_pt(__uint_as_float(o[e]) * inv, __uint_as_float(o[e + 1]) * inv);
              w.y = pack_bf16_pt(__uint_as_float(o[e + 2]) * inv, __uint_as_float(o[e + 3]) * inv);
              w.z = pack_bf16_pt(__uint_as_float(o[e + 4]) * inv, __uint_as_float(o[e + 5]) * inv);
              w.w = pack_bf16_pt(__uint_as_float(o[e + 6]) * inv, __uint_as_float(o[e + 7]) * inv);
              *reinterpret_cast<uint4*>(dst + cb + e) = w;
            }
        }
      } else {
        float* dst = row >= 0 ? part_o + (((long long)row * D.qh + head) * pl.nslot + it.slot_idx) * HD : nullptr;
#pragma unroll 1
        for (int cb = hf * (HD / HH); cb < (hf + 1) * (HD / HH); cb += 32) {
          uint32_t o[32];
          tmem_ld32_nw(tmem + lane_off + O_COL + cb, o);
          tmem_wait_ld();
          if (dst)
#pragma unroll
            for (int e = 0; e < 32; e += 4)
              *reinterpret_cast<float4*>(dst + cb + e) =
                  make_float4(__uint_as_float(o[e]) * inv, __uint_as_float(o[e + 1]) * inv,
                              __uint_as_float(o[e + 2]) * inv, __uint_as_float(o[e + 3]) * inv);
        }
        if (dst && hf == HH - 1) part_lse[((long long)row * D.qh + head) * pl.nslot + it.slot_idx] = m * sl2 + log2f(l);
      }
      asm volatile("tcgen05.fence::before_thread_sync;");
      tile += nt;
    }
  }
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS));
  }
  if constexpr (!CAUSAL) {   // the concurrent k_attn_cascade's last CTA waits for every CTA of the pass
    if (threadIdx.x == 0) {
      __threadfence();
      atomicAdd(pl.tc_done + layer, 1);
    }
  }
}
}  // namespace

bool make_kv_map(void* map_out, const bf16* pool, long long token_rows, int hd, int bs) {
  EncodeTiled enc = get_encode();
  if (!enc || hd % 64 != 0) return false;
  // {64 elements (128 B), hd / 64 halves of a token row, token rows}; SWIZZLE_NONE: the pool's
  // own XOR pre-swizzle already is the 128-byte-swizzle layout within each half
  cuuint64_t dims[3] = {64, (cuuint64_t)(hd / 64), (cuuint64_t)token_rows};
  cuuint64_t strides[2] = {128, (cuuint64_t)hd * 2};
  cuuint32_t box[3] = {64, 1, (cuuint32_t)(bs < PT_KT ? bs : PT_KT)};
  cuuint32_t es[3] = {1, 1, 1};
  return enc(reinterpret_cast<CUtensorMap*>(map_out), CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<bf16*>(pool), dims,
             strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

static bool tc_pair() {   // SART_TC_PAIR=1: two softmax warps per row (8 softmax warps per CTA)
  static const bool on = getenv("SART_TC_PAIR") && atoi(getenv("SART_TC_PAIR")) != 0;
  return on;
}
void launch_attn_prefix_tc(const bf16* q, const void* kv_map, float* part_o, float* part_lse, Dims D, int layer,
                           Rows rows, Reqs reqs, AttnPlan pl, cudaStream_t s) {
  const CUtensorMap& map = *reinterpret_cast<const CUtensorMap*>(kv_map);
  if (tc_pair()) {
    const size_t smem = PtView<128, 4, 2>::BYTES + PtView<128, 4, 2>::XBYTES + 1024;
    ensure_dyn_smem(k_attn_prefix_tc<128, PT_PREFIX, 4, 2, 1, 8>, (int)smem);
    launch_pdl(k_attn_prefix_tc<128, PT_PREFIX, 4, 2, 1, 8>, dim3(pl.tc_grid), dim3(64 + 32 * 8), smem, s, map, q, part_o,
               part_lse, (bf16*)nullptr, (const int4*)nullptr, 0, D, layer, rows, reqs, pl);
    return;
  }
  const size_t smem = PtView<128, 4, 2>::BYTES + 1024;
  ensure_dyn_smem(k_attn_prefix_tc<128, PT_PREFIX, 4, 2, 1>, (int)smem);
  launch_pdl(k_attn_prefix_tc<128, PT_PREFIX, 4, 2, 1>, dim3(pl.tc_grid), dim3(192), smem, s, map, q, part_o, part_lse,
             (bf16*)nullptr, (const int4*)nullptr, 0, D, layer, rows, reqs, pl);
}

// causal modes: one CTA per SM (4 KV stages, two P buffers); SART_PF_CTA2=1: two CTAs per SM
// (2 KV stages, one P buffer each) -- measured neutral (14B 8K prefill 252.3 vs 252.6 ms,
// profiles/r2_prefill_umma_ab.txt), kept as an option; SART_TC_PAIR=1: 8 softmax warps
template <int MODE>
static void launch_causal(const bf16* q, const void* kv_map, bf16* out, Dims D, int layer, Rows rows, Reqs reqs,
                          const int4* blocks, int nblocks, cudaStream_t s) {
  if (nblocks <= 0) return;
  static const bool two = getenv("SART_PF_CTA2") && atoi(getenv("SART_PF_CTA2")) != 0;
  const int items = nblocks * D.qh;
  const CUtensorMap& map = *reinterpret_cast<const CUtensorMap*>(kv_map);
  if (tc_pair()) {
    const size_t smem = PtView<128, 4, 2>::BYTES + PtView<128, 4, 2>::XBYTES + 1024;
    ensure_dyn_smem(k_attn_prefix_tc<128, MODE, 4, 2, 1, 8>, (int)smem);
    launch_pdl(k_attn_prefix_tc<128, MODE, 4, 2, 1, 8>, dim3(std::min(items, device_sms())), dim3(64 + 32 * 8), smem, s,
               map, q, (float*)nullptr, (float*)nullptr, out, blocks, nblocks, D, layer, rows, reqs, AttnPlan{});
  } else if (two) {
    const size_t smem = PtView<128, 2, 1>::BYTES;
    ensure_dyn_smem(k_attn_prefix_tc<128, MODE, 2, 1, 2>, (int)smem);
    static bool carve = false;   // the largest shared-memory carveout: room for two CTAs per SM
    if (!carve) carve = cudaFuncSetAttribute(k_attn_prefix_tc<128, MODE, 2, 1, 2>,
                                             cudaFuncAttributePreferredSharedMemoryCarveout, 100) == cudaSuccess;
    launch_pdl(k_attn_prefix_tc<128, MODE, 2, 1, 2>, dim3(std::min(items, 2 * device_sms())), dim3(192), smem, s, map,
               q, (float*)nullptr, (float*)nullptr, out, blocks, nblocks, D, layer, rows, reqs, AttnPlan{});
  } else {
    const size_t smem = PtView<128, 4, 2>::BYTES + 1024;
    ensure_dyn_smem(k_attn_prefix_tc<128, MODE, 4, 2, 1>, (int)smem);
    launch_pdl(k_attn_prefix_tc<128, MODE, 4, 2, 1>, dim3(std::min(items, device_sms())), dim3(192), smem, s, map,
               q, (float*)nullptr, (float*)nullptr, out, blocks, nblocks, D, layer, rows, reqs, AttnPlan{});
  }
}
void launch_attn_prefill_umma(const bf16* q, const void* kv_map, bf16* out, Dims D, int layer, Reqs reqs,
                              const int4* blocks, int nblocks, cudaStream_t s) {
  launch_causal<PT_PREFILL>(q, kv_map, out, D, layer, Rows{}, reqs, blocks, nblocks, s);
}
void launch_attn_suffix_umma(const bf16* q, const void* kv_map, bf16* out, Dims D, int layer, Rows rows, Reqs reqs,
                             const int4* qblocks, int nqb, cudaStream_t s) {
  launch_causal<PT_SUF>(q, kv_map, out, D, layer, rows, reqs, qblocks, nqb, s);
}
