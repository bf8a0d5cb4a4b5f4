// Cascade paged decode attention (the dominant HBM-bound kernel).
//
//   o_i = sum_t softmax_t(q_i . k_t / sqrt(hd)) v_t   over [prefix (P-1 tokens, shared) ;
//                                                           suffix (l+1 tokens, per branch)]
//
// PAPER P:306 shares the prompt's KV across a request's branches.  We read it ONCE per
// request and kv head: a "prefix task" multiplies a chunk of the shared prefix KV by up to
// 16 query rows (branches x g heads) of the request, a "suffix task" covers one branch's
// private KV.  Every task covers <= CH tokens and writes a normalised partial output and its
// log-sum-exp; a merge kernel combines the partials of each (row, kv head) in a fixed slot
// order, so the result does not depend on scheduling (deterministic, PP4).  (Merging inside
// the streaming kernel was measured slower: per-item fences and atomics stall the streams.)
//
// Kernel structure ("warp-autonomous" persistent kernel, one CTA per SM):
//   * every warp takes items (task, kv head) from a work counter (dynamic load balance; an
//     item's result does not depend on which warp computes it) and streams the item's KV
//     through its OWN 2-stage ring of 32-token stages with 1-D bulk copies
//     (cp.async.bulk ... mbarrier::complete_tx) of page-table tiles; the issue cursor runs
//     ahead across item boundaries, so a warp always has its next 2 stages in flight;
//   * mma.sync m16n8k16 bf16 computes S = Q K^T and O += P V with an fp32 online softmax;
//     the pool's XOR pre-swizzle (common.cuh kv_swz) keeps the ldmatrix reads conflict-free;
//   * no CTA-wide barriers and no cross-warp merges: warps never wait on each other.
// Tensor cores are used because QK^T / PV are dense contractions, but the kernel is
// HBM-bound (about g flop per byte): the design goal is bytes in flight per SM.
#include <cstdlib>

#include "kernels.h"

namespace {
// Partial outputs of the split items (normalised o of a chunk, per row / q head / slot): fp32.
// -DSART_PART_BF16 stores them in bf16 (half the partial round trip): +0.6% on the C2 step
// (profiles/r2_attn_partials_ab.txt), but the extra rounding moved one sampled row of the
// full-depth C2 logits parity to 2.09e-2 > north_star's 2e-2, so it is not the default.
#ifdef SART_PART_BF16
typedef bf16 PartT;
#else
typedef float PartT;
#endif
// launch configurations <warps per CTA, stages per warp ring, tokens per stage>; the
// default is chosen by measurement, SART_ATTN_CFG=<index> overrides it.

__device__ __forceinline__ uint32_t s_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mb_init(uint64_t* b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(s_u32(b)), "r"(c));
}
__device__ __forceinline__ void mb_expect(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mb_wait(uint64_t* b, uint32_t par) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tW_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra W_%=;\n\t}" ::"r"(s_u32(b)),
      "r"(par)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(s_u32(bar))
               : "memory");
}
// suffix KV is read exactly once per step: stream it with an L2 evict-first policy so it does
// not push the step's partials, q and the shared prefix (re-read by the prefix m-tiles) out of L2
__device__ __forceinline__ uint64_t l2_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void bulk_g2s_hint(uint32_t dst, const void* src, uint32_t bytes, uint64_t* bar,
                                              uint64_t pol) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
               ::"r"(dst), "l"(src), "r"(bytes), "r"(s_u32(bar)), "l"(pol)
               : "memory");
}
__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ void mma16816(float* c, const uint32_t* a, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}

// A decoded item: task (prefix/suffix chunk, m-tile) x kv head; token range for this step.
struct Item {
  int valid, task, h, t0, t1, nq, slot_idx, type, y, mt;
  const int* tab;
};

__device__ __forceinline__ Item decode_item(const AttnPlan& pl, const Dims& D, const Rows& rows, const Reqs& reqs,
                                            int item) {
  Item it;
  it.task = item / D.kvh;            // index into the per-step packed list
  it.h = item % D.kvh;
  const int4 a = __ldcg(pl.items + 2 * it.task);
  it.t0 = a.x;
  it.t1 = a.y;
  it.slot_idx = a.w;
  const int4 b = __ldcg(pl.items + 2 * it.task + 1);
  it.nq = b.w;
  it.tab = (b.x == 0 ? rows.table : reqs.prefix) + a.z;
  it.type = b.x;
  it.y = b.y;
  it.mt = b.z;
  it.valid = 1;
  return it;
}

// query row i (0..15) of an item -> (batch row, q head); false if beyond nq
__device__ __forceinline__ bool q_of(const AttnPlan& pl, const Dims& D, const Item& it, int i, int& row,
                                     int& head) {
  if (i >= it.nq) return false;
  if (it.type == 0) {
    row = it.y;
    head = it.h * D.g + i;
  } else {
    const int j = it.mt * 16 + i;
    row = pl.grp_rows[it.y * pl.qr_max + j / D.g];
    head = it.h * D.g + j % D.g;
  }
  return true;
}

// number of items that cover (row r, any kv head) this step
__device__ __forceinline__ int items_for_row(const AttnPlan& pl, const Dims& D, const Rows& rows, const Reqs& reqs,
                                             int r, int& npc, int& nsc) {
  npc = (reqs.P[rows.slot[r]] - 1 + pl.CH - 1) / pl.CH;
  const int len = rows.ell[r] + 1;
  if (pl.PC) {   // whole chunks, then the pieces of the partial last chunk
    const int nfull = len / pl.CH;
    nsc = nfull + (len - nfull * pl.CH + pl.PC - 1) / pl.PC;
  } else {
    nsc = (len + pl.CH - 1) / pl.CH;
  }
  const int j = pl.row_pos[r];
  const int tiles = (j * D.g + D.g - 1) / 16 - (j * D.g) / 16 + 1;   // prefix m-tiles holding this row
  return nsc + npc * tiles;
}

template <int HD, int NS, int SW>
struct WarpSmem {
  bf16 k[NS][SW * HD];
  bf16 v[NS][SW * HD];
  uint64_t full[NS];
  uint64_t pad[(NS & 1) ? 1 : 2];
};

template <int HD, int NW, int NS, int SW>
__global__ void __launch_bounds__(NW * 32, 1)
    k_attn_cascade(const bf16* __restrict__ q, const bf16* __restrict__ pool, float* __restrict__ part_o,
                   float* __restrict__ part_lse, bf16* __restrict__ out, float* __restrict__ dbg, Dims D, int layer,
                   Rows rows, Reqs reqs, AttnPlan pl) {
  extern __shared__ __align__(128) uint8_t sraw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  WarpSmem<HD, NS, SW>& sm = reinterpret_cast<WarpSmem<HD, NS, SW>*>(sraw)[warp];
  int* work = pl.work + layer;
  const float sl2 = 1.4426950408889634f * rsqrtf((float)HD);   // log2(e) / sqrt(hd)
  const uint64_t pol = l2_evict_first();

  // zero the ring once (masked tokens multiply V by 0, so stale smem must be finite)
  for (int e = lane; e < NS * SW * HD / 8; e += 32) {
    reinterpret_cast<uint4*>(sm.k)[e] = make_uint4(0, 0, 0, 0);
    reinterpret_cast<uint4*>(sm.v)[e] = make_uint4(0, 0, 0, 0);
  }
  if (lane == 0)
    for (int s = 0; s < NS; ++s) mb_init(&sm.full[s], 1);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  // predecessor's q / KV writes are visible from here on.  With a concurrent prefix pass
  // (pl.tc_grid > 0) the predecessor is that pass, whose CTAs release this grid only after
  // their own PDL wait on the QKV GEMM: q and the appended KV are complete before any CTA of
  // this grid starts, so it does not wait (q is read through L2, __ldcg)
  if (pl.tc_grid == 0) pdl_wait();
  pdl_trigger();
  const int n_items = *pl.n_items * D.kvh;

  // ---- issue side (warp-uniform state): ring of decoded items; the issue cursor runs up
  //      to NS stages ahead of the consume cursor, across item boundaries
  Item ring[NS + 1];
  int r_head = 0, r_cnt = 0;       // consume item = ring[r_head]
  int iss_idx = -1, iss_s0 = 0;    // ring index of the item being issued, next stage start
  uint32_t issued = 0, consumed = 0;
  bool exhausted = false;
  // the next work index is grabbed one item ahead, so the atomic's latency is hidden
  int next_grab = 0;
  if (lane == 0) next_grab = atomicAdd(work, 1);

  auto refill = [&]() {
    while (issued - consumed < (uint32_t)NS) {
      if (iss_idx < 0 || iss_s0 >= ring[iss_idx].t1) {
        if (exhausted || r_cnt == NS + 1) return;
        Item nx{};
        for (;;) {
          const int i = __shfl_sync(0xffffffffu, next_grab, 0);
          if (i >= n_items) { exhausted = true; return; }
          if (lane == 0) next_grab = atomicAdd(work, 1);
          nx = decode_item(pl, D, rows, reqs, i);
          break;
        }
        iss_idx = (r_head + r_cnt) % (NS + 1);
        ring[iss_idx] = nx;
        ++r_cnt;
        iss_s0 = nx.t0;
      }
      const Item& it = ring[iss_idx];
      const int slot = issued % NS;
      if (lane == 0) {
        // stage = tokens [iss_s0, iss_s0 + ntok): whole blocks (bs <= 32) or half a block (bs = 64)
        const int ntok = min(SW, it.t1 - iss_s0);
        const int tpb = min(D.bs, SW);
        const int pieces = (ntok + tpb - 1) / tpb;
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mb_expect(&sm.full[slot], 2u * pieces * tpb * HD * 2);
        for (int p = 0; p < pieces; ++p) {
          const int tok = iss_s0 + p * tpb;
          const long long blk = it.tab[tok / D.bs];
          const int inblk = tok % D.bs;
          const bf16* kt = pool + kv_tile_off(D, layer, blk, 0, it.h) + (long long)inblk * HD;
          const bf16* vt = pool + kv_tile_off(D, layer, blk, 1, it.h) + (long long)inblk * HD;
          if (it.type == 0 && pl.evict) {
            bulk_g2s_hint(s_u32(sm.k[slot] + p * tpb * HD), kt, tpb * HD * 2, &sm.full[slot], pol);
            bulk_g2s_hint(s_u32(sm.v[slot] + p * tpb * HD), vt, tpb * HD * 2, &sm.full[slot], pol);
          } else {
            bulk_g2s(s_u32(sm.k[slot] + p * tpb * HD), kt, tpb * HD * 2, &sm.full[slot]);
            bulk_g2s(s_u32(sm.v[slot] + p * tpb * HD), vt, tpb * HD * 2, &sm.full[slot]);
          }
        }
      }
      iss_s0 += SW;
      ++issued;
    }
  };

  refill();
  while (r_cnt > 0) {
    const Item it = ring[r_head];
    // Q fragments (16 rows x HD) of this item, zero beyond nq
    uint32_t qa[HD / 16][4];
    {
      const int r0 = lane >> 2, r1 = r0 + 8, cc = 2 * (lane & 3);
      int row, head;
      const bf16* q0 = q_of(pl, D, it, r0, row, head) ? q + ((long long)row * D.qh + head) * HD : nullptr;
      const bf16* q1 = q_of(pl, D, it, r1, row, head) ? q + ((long long)row * D.qh + head) * HD : nullptr;
#pragma unroll
      for (int kk = 0; kk < HD / 16; ++kk) {
        qa[kk][0] = q0 ? __ldcg(reinterpret_cast<const unsigned int*>(q0 + 16 * kk + cc)) : 0u;
        qa[kk][1] = q1 ? __ldcg(reinterpret_cast<const unsigned int*>(q1 + 16 * kk + cc)) : 0u;
        qa[kk][2] = q0 ? __ldcg(reinterpret_cast<const unsigned int*>(q0 + 16 * kk + 8 + cc)) : 0u;
        qa[kk][3] = q1 ? __ldcg(reinterpret_cast<const unsigned int*>(q1 + 16 * kk + 8 + cc)) : 0u;
      }
    }
    float o[HD / 8][4];
#pragma unroll
    for (int nt = 0; nt < HD / 8; ++nt) o[nt][0] = o[nt][1] = o[nt][2] = o[nt][3] = 0.f;
    float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;

    for (int s0 = it.t0; s0 < it.t1; s0 += SW) {
      const int slot = consumed % NS;
      mb_wait(&sm.full[slot], (consumed / NS) & 1);
      const int ntok = min(SW, it.t1 - s0);
      const uint32_t kb = s_u32(sm.k[slot]), vb = s_u32(sm.v[slot]);
#pragma unroll
      for (int sub = 0; sub < SW; sub += 16) {
        if (sub >= ntok) break;
        float s[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
        float s2[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};   // 2nd accumulator: shorter chains
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk) {
          const int mi = lane >> 3;
          const int tok = sub + (lane & 7) + 8 * (mi >> 1);
          const int ch = 2 * kk + (mi & 1);
          uint32_t b0, b1, b2, b3;
          ldsm_x4(kb + tok * (HD * 2) + ((ch ^ (tok & 7)) << 4), b0, b1, b2, b3);
          if (kk & 1) {
            mma16816(s2[0], qa[kk], b0, b1);
            mma16816(s2[1], qa[kk], b2, b3);
          } else {
            mma16816(s[0], qa[kk], b0, b1);
            mma16816(s[1], qa[kk], b2, b3);
          }
        }
#pragma unroll
        for (int nt = 0; nt < 2; ++nt)
#pragma unroll
          for (int e = 0; e < 4; ++e) s[nt][e] += s2[nt][e];
        const int cbase = sub + 2 * (lane & 3);
#pragma unroll
        for (int nt = 0; nt < 2; ++nt)
#pragma unroll
          for (int e = 0; e < 4; ++e)
            if (cbase + nt * 8 + (e & 1) >= ntok) s[nt][e] = -INFINITY;
        float mx0 = fmaxf(fmaxf(s[0][0], s[0][1]), fmaxf(s[1][0], s[1][1]));
        float mx1 = fmaxf(fmaxf(s[0][2], s[0][3]), fmaxf(s[1][2], s[1][3]));
        mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 1));
        mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 2));
        mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 1));
        mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 2));
        const float n0 = fmaxf(m0, mx0), n1 = fmaxf(m1, mx1);
        const float u0 = n0 == -INFINITY ? 0.f : n0, u1 = n1 == -INFINITY ? 0.f : n1;
        const float c0 = exp2f((m0 - u0) * sl2), c1 = exp2f((m1 - u1) * sl2);
        m0 = n0;
        m1 = n1;
        float p[2][4];
#pragma unroll
        for (int nt = 0; nt < 2; ++nt) {
          p[nt][0] = exp2f((s[nt][0] - u0) * sl2);
          p[nt][1] = exp2f((s[nt][1] - u0) * sl2);
          p[nt][2] = exp2f((s[nt][2] - u1) * sl2);
          p[nt][3] = exp2f((s[nt][3] - u1) * sl2);
        }
        l0 = l0 * c0 + p[0][0] + p[0][1] + p[1][0] + p[1][1];
        l1 = l1 * c1 + p[0][2] + p[0][3] + p[1][2] + p[1][3];
        // (skipping this rescale when c0 = c1 = 1 is bit-exact but measured neutral:
        // profiles/r2_attn_lazy_rescale_ab.txt -- the kernel waits on data, not on issue)
#pragma unroll
        for (int nt = 0; nt < HD / 8; ++nt) { o[nt][0] *= c0; o[nt][1] *= c0; o[nt][2] *= c1; o[nt][3] *= c1; }
        uint32_t pa[4];
        pa[0] = pack_bf16(p[0][0], p[0][1]);
        pa[1] = pack_bf16(p[0][2], p[0][3]);
        pa[2] = pack_bf16(p[1][0], p[1][1]);
        pa[3] = pack_bf16(p[1][2], p[1][3]);
#pragma unroll
        for (int dp = 0; dp < HD / 16; ++dp) {
          const int mi = lane >> 3;
          const int tok = sub + (lane & 7) + 8 * (mi & 1);
          const int ch = 2 * dp + (mi >> 1);
          uint32_t b0, b1, b2, b3;
          ldsm_x4_t(vb + tok * (HD * 2) + ((ch ^ (tok & 7)) << 4), b0, b1, b2, b3);
          mma16816(o[2 * dp], pa, b0, b1);
          mma16816(o[2 * dp + 1], pa, b2, b3);
        }
      }
      __syncwarp();
      ++consumed;
      refill();              // re-fill the slot just consumed (next stage of this or a later item)
    }
    // ---- item done: normalise and write the partial (rows r = lane/4 and r + 8)
    l0 += __shfl_xor_sync(0xffffffffu, l0, 1);
    l0 += __shfl_xor_sync(0xffffffffu, l0, 2);
    l1 += __shfl_xor_sync(0xffffffffu, l1, 1);
    l1 += __shfl_xor_sync(0xffffffffu, l1, 2);
    {
      const int r0 = lane >> 2, cc = 2 * (lane & 3);
#pragma unroll
      for (int half = 0; half < 2; ++half) {
        int row, head;
        if (!q_of(pl, D, it, r0 + 8 * half, row, head)) continue;
        const float m = half ? m1 : m0, l = half ? l1 : l0;
        const float inv = 1.0f / l;
        const long long pi = ((long long)row * D.qh + head) * pl.nslot + it.slot_idx;
        PartT* dst = reinterpret_cast<PartT*>(part_o) + pi * HD;
#pragma unroll
        for (int nt = 0; nt < HD / 8; ++nt) {
          if constexpr (sizeof(PartT) == 4)
            *reinterpret_cast<float2*>(dst + nt * 8 + cc) =
                make_float2(o[nt][2 * half] * inv, o[nt][2 * half + 1] * inv);
          else
            *reinterpret_cast<__nv_bfloat162*>(dst + nt * 8 + cc) =
                __floats2bfloat162_rn(o[nt][2 * half] * inv, o[nt][2 * half + 1] * inv);
        }
        if ((lane & 3) == 0) part_lse[pi] = (m == -INFINITY ? 0.f : m) * sl2 + log2f(l);
      }
    }
    r_head = (r_head + 1) % (NS + 1);
    --r_cnt;
    if (r_cnt == 0) iss_idx = -1;
    refill();
  }
  // the last CTA to finish resets this layer's counters for the next step
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(pl.done + layer, 1) == (int)gridDim.x - 1) {
      if (pl.tc_grid > 0) {   // this grid completes only after the concurrent prefix pass
        volatile int* td = pl.tc_done + layer;
        while (*td < pl.tc_grid) __nanosleep(256);
        __threadfence();
        pl.tc_done[layer] = 0;
      }
      pl.work[layer] = 0;
      pl.done[layer] = 0;
    }
  }
}

// merge kernel: one warp per (row, q head); each lane owns HD/32 contiguous columns (one
// vector load per slot), slots in fixed order (prefix chunks, then suffix chunks)
template <int HD>
__global__ void __launch_bounds__(256) k_attn_merge(const float* __restrict__ part_o,
                                                    const float* __restrict__ part_lse, bf16* __restrict__ out,
                                                    float* __restrict__ dbg, Dims D, Rows rows, Reqs reqs,
                                                    AttnPlan pl, int n) {
  pdl_wait();
  pdl_trigger();
  constexpr int C = HD / 32;
  const int wid = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (wid >= n * D.qh) return;
  const int r = wid / D.qh, head = wid % D.qh;
  if (rows.status[r] != RUNNING_ST) return;
  int npc, nsc;
  items_for_row(pl, D, rows, reqs, r, npc, nsc);
  const long long base = ((long long)r * D.qh + head) * pl.nslot;
  float M = -INFINITY;
  for (int k = 0; k < npc + nsc; ++k) M = fmaxf(M, part_lse[base + (k < npc ? k : pl.npc_max + k - npc)]);
  float acc[C] = {};
  float L = 0.f;
#pragma unroll 4
  for (int k = 0; k < npc + nsc; ++k) {
    const long long pi = base + (k < npc ? k : pl.npc_max + k - npc);
    const float w = exp2f(part_lse[pi] - M);
    L += w;
    const PartT* src = reinterpret_cast<const PartT*>(part_o) + pi * HD + lane * C;
    if constexpr (sizeof(PartT) == 4) {
      if constexpr (C == 4) {
        const float4 v = *reinterpret_cast<const float4*>(src);
        acc[0] += w * v.x; acc[1] += w * v.y; acc[2] += w * v.z; acc[3] += w * v.w;
      } else {
        const float2 v = *reinterpret_cast<const float2*>(src);
        acc[0] += w * v.x; acc[1] += w * v.y;
      }
    } else {
      if constexpr (C == 4) {
        const uint2 u = *reinterpret_cast<const uint2*>(src);
        const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.x));
        const float2 b = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.y));
        acc[0] += w * a.x; acc[1] += w * a.y; acc[2] += w * b.x; acc[3] += w * b.y;
      } else {
        const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(src));
        acc[0] += w * a.x; acc[1] += w * a.y;
      }
    }
  }
  const long long oi = ((long long)r * D.qh + head) * HD + lane * C;
  const float inv = 1.0f / L;
  if constexpr (C == 4) {
    __nv_bfloat162 a = __floats2bfloat162_rn(acc[0] * inv, acc[1] * inv), b = __floats2bfloat162_rn(acc[2] * inv, acc[3] * inv);
    uint2 u;
    u.x = *reinterpret_cast<uint32_t*>(&a);
    u.y = *reinterpret_cast<uint32_t*>(&b);
    *reinterpret_cast<uint2*>(out + oi) = u;
  } else {
    *reinterpret_cast<__nv_bfloat162*>(out + oi) = __floats2bfloat162_rn(acc[0] * inv, acc[1] * inv);
  }
  if (dbg)
    for (int c = 0; c < C; ++c) dbg[oi + c] = acc[c] * inv;
}

// ------------------------------------------------------------------ causal prefill (f1)
// Prompt positions of a batched prefill (Alg. 1 L15): CTA = (QP-position query block of one
// request, HG q heads of one kv head); warp w = 16 query rows (tile w % QT) of head w / QT,
// so each K/V stage -- key positions [64 kb, 64 kb + 64) through a 2-stage bulk-copy ring --
// serves every q head of the GQA group (read once per group, not once per q head); the last
// key block is masked causally.  QT, HG: pf_shape() (<= 8 warps).
//
// SUF (row f2, the PRM pass): the CTA is a block of <= QP of one batch row's new suffix
// entries (descriptor {first token, count, row, first entry}); keys live in a virtual index space [prefix blocks (pbase = ceil((P-1)/bs) * bs
// slots, slots >= P-1 masked) ; suffix entries], so every 64-key stage is whole pages of one
// table and the causal test stays "key index <= query index".
#ifndef SART_PF_MINB
#define SART_PF_MINB 1   // min CTAs per SM for the prefill kernel (2: <= 128 registers)
#endif
template <int HD, bool SUF, int NST>
__global__ void __launch_bounds__(256, SART_PF_MINB) k_attn_prefill_tc(const bf16* __restrict__ q, const bf16* __restrict__ pool,
                                                         bf16* __restrict__ out, Dims D, int layer, Reqs reqs,
                                                         const int4* __restrict__ blocks, Rows rows, int QT, int HG) {
  constexpr int KT = 64;                                   // key tokens per stage
  extern __shared__ __align__(128) uint8_t praw[];
  bf16 (*ks)[KT * HD] = reinterpret_cast<bf16 (*)[KT * HD]>(praw);
  bf16 (*vs)[KT * HD] = reinterpret_cast<bf16 (*)[KT * HD]>(praw + NST * KT * HD * sizeof(bf16));
  uint64_t* full = reinterpret_cast<uint64_t*>(praw + 2 * NST * KT * HD * sizeof(bf16));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int qt = warp % QT;                                // this warp's 16-row query tile
  const int head = blockIdx.y * HG + warp / QT, h = head / D.g;
  int r0, nr, slot, p0;                                    // first batch token, tokens, slot, first key index
  int npre = 0x7fffffff, pbase = 0x7fffffff;               // masked prefix padding [npre, pbase); suffix base
  const int* rtab = nullptr;
  if constexpr (SUF) {
    const int4 blk = blocks[blockIdx.x];                   // {first token, entries, row, first entry}
    const int row = blk.z;
    r0 = blk.x; nr = blk.y;
    slot = rows.slot[row];
    npre = reqs.P[slot] - 1;
    pbase = (npre + D.bs - 1) / D.bs * D.bs;
    p0 = pbase + blk.w;
    rtab = rows.table + (long long)row * D.MBR;
  } else {
    const int4 blk = blocks[blockIdx.x];                   // {first batch row, rows, slot, first position}
    r0 = blk.x; nr = blk.y; slot = blk.z; p0 = blk.w;
  }
  const int nkey = p0 + nr;                                // keys 0 .. p0 + nr - 1
  const int nkb = (nkey + KT - 1) / KT;
  const int* ptab = reqs.prefix + (long long)slot * D.MPB;
  const float sl2 = 1.4426950408889634f * rsqrtf((float)HD);
  if (threadIdx.x == 0) {
    for (int i = 0; i < NST; ++i) mb_init(&full[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto issue = [&](int kb) {
    const int st = kb % NST;
    const int t0 = kb * KT, ntok = min(KT, nkey - t0);
    const int tpb = min(D.bs, KT);
    const int pieces = (ntok + tpb - 1) / tpb;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    mb_expect(&full[st], 2u * pieces * tpb * HD * 2);
    for (int pc = 0; pc < pieces; ++pc) {
      const int tok = t0 + pc * tpb;
      const long long b = tok < pbase ? ptab[tok / D.bs] : rtab[(tok - pbase) / D.bs];
      const int inb = tok % D.bs;
      bulk_g2s(s_u32(ks[st] + pc * tpb * HD), pool + kv_tile_off(D, layer, b, 0, h) + (long long)inb * HD,
               tpb * HD * 2, &full[st]);
      bulk_g2s(s_u32(vs[st] + pc * tpb * HD), pool + kv_tile_off(D, layer, b, 1, h) + (long long)inb * HD,
               tpb * HD * 2, &full[st]);
    }
  };
  // stale smem of a partial stage is multiplied by P = 0: keep it finite
  for (int e = threadIdx.x; e < 2 * NST * KT * HD / 8; e += blockDim.x) reinterpret_cast<uint4*>(praw)[e] = make_uint4(0, 0, 0, 0);
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int i = 0; i < NST && i < nkb; ++i) issue(i);
  }
  // Q fragments of this warp's 16 rows (zero beyond nr)
  const int qr0 = qt * 16 + (lane >> 2), qr1 = qr0 + 8, cc = 2 * (lane & 3);
  const bf16* q0 = qr0 < nr ? q + ((long long)(r0 + qr0) * D.qh + head) * HD : nullptr;
  const bf16* q1 = qr1 < nr ? q + ((long long)(r0 + qr1) * D.qh + head) * HD : nullptr;
  uint32_t qa[HD / 16][4];
#pragma unroll
  for (int kk = 0; kk < HD / 16; ++kk) {
    qa[kk][0] = q0 ? *reinterpret_cast<const uint32_t*>(q0 + 16 * kk + cc) : 0u;
    qa[kk][1] = q1 ? *reinterpret_cast<const uint32_t*>(q1 + 16 * kk + cc) : 0u;
    qa[kk][2] = q0 ? *reinterpret_cast<const uint32_t*>(q0 + 16 * kk + 8 + cc) : 0u;
    qa[kk][3] = q1 ? *reinterpret_cast<const uint32_t*>(q1 + 16 * kk + 8 + cc) : 0u;
  }
  const int pos0 = p0 + qr0, pos1 = p0 + qr1;              // query positions (causal limits)
  float o[HD / 8][4];
#pragma unroll
  for (int nt = 0; nt < HD / 8; ++nt) o[nt][0] = o[nt][1] = o[nt][2] = o[nt][3] = 0.f;
  float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;
  for (int kb = 0; kb < nkb; ++kb) {
    const int st = kb % NST;
    mb_wait(&full[st], (kb / NST) & 1);
    const uint32_t kbase = s_u32(ks[st]), vbase = s_u32(vs[st]);
    const int t0 = kb * KT;
    if (t0 <= p0 + qt * 16 + 15) {                         // some key of this block is visible to the warp
#pragma unroll 1
      for (int sub = 0; sub < KT; sub += 16) {
        if (t0 + sub > p0 + qt * 16 + 15) break;
        float s[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk) {
          const int mi = lane >> 3;
          const int tok = sub + (lane & 7) + 8 * (mi >> 1);
          const int ch = 2 * kk + (mi & 1);
          uint32_t b0, b1, b2, b3;
          ldsm_x4(kbase + tok * (HD * 2) + ((ch ^ (tok & 7)) << 4), b0, b1, b2, b3);
          mma16816(s[0], qa[kk], b0, b1);
          mma16816(s[1], qa[kk], b2, b3);
        }
        const int kpos = t0 + sub + 2 * (lane & 3);
#pragma unroll
        for (int nt = 0; nt < 2; ++nt)
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int kp = kpos + nt * 8 + (e & 1);
            if (kp > (e < 2 ? pos0 : pos1) || (kp >= npre && kp < pbase)) s[nt][e] = -INFINITY;   // causal, padding
          }
        float mx0 = fmaxf(fmaxf(s[0][0], s[0][1]), fmaxf(s[1][0], s[1][1]));
        float mx1 = fmaxf(fmaxf(s[0][2], s[0][3]), fmaxf(s[1][2], s[1][3]));
        mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 1));
        mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 2));
        mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 1));
        mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 2));
        const float n0 = fmaxf(m0, mx0), n1 = fmaxf(m1, mx1);
        const float u0 = n0 == -INFINITY ? 0.f : n0, u1 = n1 == -INFINITY ? 0.f : n1;
        const float c0 = exp2f((m0 - u0) * sl2), c1 = exp2f((m1 - u1) * sl2);
        m0 = n0;
        m1 = n1;
        float pr[2][4];
#pragma unroll
        for (int nt = 0; nt < 2; ++nt) {
          pr[nt][0] = exp2f((s[nt][0] - u0) * sl2);
          pr[nt][1] = exp2f((s[nt][1] - u0) * sl2);
          pr[nt][2] = exp2f((s[nt][2] - u1) * sl2);
          pr[nt][3] = exp2f((s[nt][3] - u1) * sl2);
        }
        l0 = l0 * c0 + pr[0][0] + pr[0][1] + pr[1][0] + pr[1][1];
        l1 = l1 * c1 + pr[0][2] + pr[0][3] + pr[1][2] + pr[1][3];
#pragma unroll
        for (int nt = 0; nt < HD / 8; ++nt) { o[nt][0] *= c0; o[nt][1] *= c0; o[nt][2] *= c1; o[nt][3] *= c1; }
        uint32_t pa[4] = {pack_bf16(pr[0][0], pr[0][1]), pack_bf16(pr[0][2], pr[0][3]), pack_bf16(pr[1][0], pr[1][1]),
                          pack_bf16(pr[1][2], pr[1][3])};
#pragma unroll
        for (int dp = 0; dp < HD / 16; ++dp) {
          const int mi = lane >> 3;
          const int tok = sub + (lane & 7) + 8 * (mi & 1);
          const int ch = 2 * dp + (mi >> 1);
          uint32_t b0, b1, b2, b3;
          ldsm_x4_t(vbase + tok * (HD * 2) + ((ch ^ (tok & 7)) << 4), b0, b1, b2, b3);
          mma16816(o[2 * dp], pa, b0, b1);
          mma16816(o[2 * dp + 1], pa, b2, b3);
        }
      }
    }
    __syncthreads();                                       // every warp is done with this stage
    if (threadIdx.x == 0 && kb + NST < nkb) issue(kb + NST);
  }
  l0 += __shfl_xor_sync(0xffffffffu, l0, 1);
  l0 += __shfl_xor_sync(0xffffffffu, l0, 2);
  l1 += __shfl_xor_sync(0xffffffffu, l1, 1);
  l1 += __shfl_xor_sync(0xffffffffu, l1, 2);
#pragma unroll
  for (int half = 0; half < 2; ++half) {
    const int qr = half ? qr1 : qr0;
    if (qr >= nr) continue;
    const float inv = 1.0f / (half ? l1 : l0);
    bf16* dst = out + ((long long)(r0 + qr) * D.qh + head) * HD;
#pragma unroll
    for (int nt = 0; nt < HD / 8; ++nt)
      *reinterpret_cast<__nv_bfloat162*>(dst + nt * 8 + cc) =
          __floats2bfloat162_rn(o[nt][2 * half] * inv, o[nt][2 * half + 1] * inv);
  }
}

// ------------------------------------------------------------------ per-step item list
// Valid tasks of this step (rows finished mid-window are skipped) with their token ranges,
// ordered by size, largest first (counting sort on 16-token buckets), so that the dynamic
// work queue ends with small items.  One launch per step serves all layers.
__global__ void __launch_bounds__(1024) k_attn_items(Dims D, Rows rows, Reqs reqs, AttnPlan pl) {
  constexpr int NB = 64;                       // size buckets
  __shared__ int cnt[NB], base[NB];
  pdl_wait();
  pdl_trigger();
  const int tid = threadIdx.x;
  const int nu = *pl.n_units;
  const int bw = (pl.CH + NB - 1) / NB;        // tokens per bucket
  if (tid < NB) cnt[tid] = 0;
  if (tid == 0 && pl.n_tc) *pl.n_tc = 0;
  __syncthreads();
  for (int pass = 0; pass < 2; ++pass) {
    for (int t = tid; t < nu; t += 1024) {
      const int4 u = pl.units[t];
      int t0 = 0, t1 = 0, nq = 0, tabbase = 0, slot_idx = 0;
      bool ok;
      if (u.x == 2) {   // tensor-core prefix item: all query rows of the group (k_attn_prefix_tc)
        if (pass == 0) continue;
        const int gi = u.y;
        const int n = pl.grp_n[gi];
        ok = false;
        for (int j = 0; j < n; ++j) ok |= rows.status[pl.grp_rows[gi * pl.qr_max + j]] == RUNNING_ST;
        const int slot = pl.grp_slot[gi];
        t0 = u.z * pl.CH;
        t1 = min(t0 + pl.CH, reqs.P[slot] - 1);
        if (ok && t0 < t1) {
          const int pos = atomicAdd(pl.n_tc, 1);
          pl.tc_items[2 * pos] = make_int4(t0, t1, slot * D.MPB, u.z);
          pl.tc_items[2 * pos + 1] = make_int4(2, gi, 0, n * D.g);
        }
        continue;
      }
      if (u.x == 0) {
        const int r = u.y;
        ok = rows.status[r] == RUNNING_ST;
        const int len = rows.ell[r] + 1;
        if (pl.PC) {   // unit u.z = piece u.z: a whole chunk is emitted by its first piece
          const int q = pl.CH / pl.PC, nfull = len / pl.CH;
          t0 = u.z * pl.PC;
          if (u.z / q < nfull) {
            ok = ok && (u.z % q) == 0;
            t1 = t0 + pl.CH;
            slot_idx = pl.npc_max + u.z / q;
          } else {
            t1 = min(t0 + pl.PC, len);
            slot_idx = pl.npc_max + nfull + (u.z - nfull * q);
          }
        } else {
          t0 = u.z * pl.CH;
          t1 = min(t0 + pl.CH, len);
          slot_idx = pl.npc_max + u.z;
        }
        nq = D.g;
        tabbase = r * D.MBR;
      } else {
        const int gi = u.y;
        const int n = pl.grp_n[gi];
        const int q0 = u.w * 16, q1 = min(n * D.g, q0 + 16);
        ok = false;
        for (int j = q0 / D.g; j <= (q1 - 1) / D.g; ++j)
          ok |= rows.status[pl.grp_rows[gi * pl.qr_max + j]] == RUNNING_ST;
        const int slot = pl.grp_slot[gi];
        t0 = u.z * pl.CH;
        t1 = min(t0 + pl.CH, reqs.P[slot] - 1);
        nq = q1 - q0;
        tabbase = slot * D.MPB;
        slot_idx = u.z;
      }
      ok = ok && t0 < t1;
      if (!ok) continue;
      const int bkt = NB - 1 - min(NB - 1, (t1 - t0 - 1) / bw);   // larger first
      if (pass == 0) {
        atomicAdd(&cnt[bkt], 1);
      } else {
        const int pos = atomicAdd(&base[bkt], 1);
        pl.items[2 * pos] = make_int4(t0, t1, tabbase, slot_idx);
        pl.items[2 * pos + 1] = make_int4(u.x, u.y, u.w, nq);
      }
    }
    __syncthreads();
    if (pass == 0 && tid == 0) {
      int acc = 0;
      for (int b = 0; b < NB; ++b) { base[b] = acc; acc += cnt[b]; }
      *pl.n_items = acc;
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------------ per-window plan
// Tasks: prefix tasks first (type 1: group, chunk, m-tile), then suffix tasks (type 0: row,
// chunk).  Groups: the window's rows of one request in batch order, qr rows per group
// (cascade) or one row per group (flat mode).  Built once per window: the batch only
// changes at boundaries; tasks whose rows finished mid-window are skipped at run time.
__global__ void __launch_bounds__(1024) k_attn_plan(Dims D, Rows rows, Reqs reqs, AttnPlan pl, int n, int flat) {
  const int tid = threadIdx.x;
  // per-row rank inside its request and the request's row count: global scratch sized R, so
  // any max_rows works (a fixed shared array would overflow above 1024 rows)
  int* s_rank = pl.row_rank;
  int* s_nrows = pl.row_nreq;
  const int qr = flat ? 1 : pl.qr_grp;
  for (int r = tid; r < n; r += 1024) {
    const int slot = rows.slot[r];
    int rank = 0, tot = 0;
    for (int r2 = 0; r2 < n; ++r2)
      if (rows.slot[r2] == slot) { rank += r2 < r; ++tot; }
    s_rank[r] = rank;
    s_nrows[r] = tot;
  }
  __threadfence_block();
  __syncthreads();
  if (tid == 0) {
    int ng = 0, nu = 0;
    for (int r = 0; r < n; ++r) {
      if (s_rank[r] != 0) continue;
      const int slot = rows.slot[r];
      const int npc = (reqs.P[slot] - 1 + pl.CH - 1) / pl.CH;
      const int nr = s_nrows[r];
      // tensor-core prefix pass: the request's rows in ceil(nr g / 128) equal groups of <= 128
      // query rows, if a group has at least tcq of them
      int qg = qr;
      bool tc = false;
      if (!flat && pl.tcq > 0) {
        const int ngt = (nr * D.g + 127) / 128;
        const int qt = (nr + ngt - 1) / ngt;
        if (qt * D.g >= pl.tcq) { tc = true; qg = qt; }
      }
      const int ngr = (nr + qg - 1) / qg;
      for (int k = 0; k < ngr; ++k) {
        const int gi = ng + k;
        pl.grp_slot[gi] = slot;
        pl.grp_n[gi] = min(qg, nr - k * qg);
        const int mts = (pl.grp_n[gi] * D.g + 15) / 16;
        for (int c = 0; c < npc; ++c) {
          if (tc) pl.units[nu++] = make_int4(2, gi, c, 0);
          else
            for (int mt = 0; mt < mts; ++mt) pl.units[nu++] = make_int4(1, gi, c, mt);
        }
      }
      int k = 0;
      for (int r2 = r; r2 < n; ++r2)
        if (rows.slot[r2] == slot) {
          pl.grp_rows[(ng + k / qg) * pl.qr_max + k % qg] = r2;
          pl.row_pos[r2] = k % qg;
          ++k;
        }
      ng += ngr;
    }
    for (int r = 0; r < n; ++r) {
      const int maxlen = min(rows.ell[r] + D.T, D.cap);   // suffix length at the window's last step
      const int nsc = (maxlen + (pl.PC ? pl.PC : pl.CH) - 1) / (pl.PC ? pl.PC : pl.CH);
      for (int c = 0; c < nsc; ++c) pl.units[nu++] = make_int4(0, r, c, 0);
    }
    *pl.n_units = nu;
  }
}

// algorithmic KV bytes of one step's attention (all layers): prefix once per request with a
// running row, each running suffix once, plus q and o (profiling only)
__global__ void __launch_bounds__(1024) k_attn_account(Dims D, Rows rows, Reqs reqs, int n, double* acc) {
  __shared__ double red[32];
  pdl_wait();
  pdl_trigger();
  __shared__ unsigned char live[1024];     // request slots with a running row (S <= 1024)
  for (int i = threadIdx.x; i < D.S; i += 1024) live[i] = 0;
  __syncthreads();
  double b = 0.0;
  const double kvtok = 2.0 * D.kvh * D.hd * 2.0;   // K+V bytes per token per layer (bf16)
  for (int r = threadIdx.x; r < n; r += 1024) {
    if (rows.status[r] != RUNNING_ST) continue;
    b += (rows.ell[r] + 1) * kvtok + 2.0 * D.qh * D.hd * 2.0;
    live[rows.slot[r]] = 1;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < D.S; i += 1024)    // prefix once per request
    if (live[i]) b += (reqs.P[i] - 1) * kvtok;
  for (int o = 16; o > 0; o >>= 1) b += __shfl_xor_sync(0xffffffffu, b, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = b;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < 32; ++w) t += red[w];
    *acc += t * D.L;
  }
}
}  // namespace

void launch_attn_plan(Dims D, Rows rows, Reqs reqs, AttnPlan pl, int n, int flat, cudaStream_t s) {
  k_attn_plan<<<1, 1024, 0, s>>>(D, rows, reqs, pl, n, flat);
}
// GQA grouping of the prefill / PRM-pass attention: HG q heads (a divisor of g, <= 8) per
// CTA, QT 16-row query tiles per head, QT * HG <= 8 warps.
// SART_PF_GROUP=0: one q head per CTA (64 positions, 4 warps) -- the A/B baseline.
void pf_shape(const Dims& D, int& QT, int& HG) {
  static const int grp = getenv("SART_PF_GROUP") ? atoi(getenv("SART_PF_GROUP")) : 1;
  HG = 1;
  if (grp)
    for (int d = 1; d <= 8 && d <= D.g; ++d)
      if (D.g % d == 0) HG = d;
  QT = std::max(1, std::min(4, 8 / HG));
}
int prefill_query_block(const Dims& D) {
  int QT, HG;
  pf_shape(D, QT, HG);
  return 16 * QT;
}
template <int HD, bool SUF, int NST>
static void launch_pf_n(dim3 grid, int threads, const bf16* q, const bf16* pool, bf16* out, Dims D, int layer,
                        Reqs reqs, const int4* blocks, Rows rows, int QT, int HG, cudaStream_t s) {
  const size_t sm = 2 * NST * 64 * (size_t)HD * sizeof(bf16) + 8 * NST;
  ensure_dyn_smem(k_attn_prefill_tc<HD, SUF, NST>, (int)sm);
  k_attn_prefill_tc<HD, SUF, NST><<<grid, threads, sm, s>>>(q, pool, out, D, layer, reqs, blocks, rows, QT, HG);
}
// ring depth: 2 stages while two CTAs share an SM (<= 4 warps); 4 stages for the larger
// grouped CTAs, which the register file limits to one per SM (SART_PF_NST overrides)
template <int HD, bool SUF>
static void launch_pf(dim3 grid, const bf16* q, const bf16* pool, bf16* out, Dims D, int layer, Reqs reqs,
                      const int4* blocks, Rows rows, cudaStream_t s) {
  int QT, HG;
  pf_shape(D, QT, HG);
  grid.y = D.qh / HG;
  static const int nst_env = getenv("SART_PF_NST") ? atoi(getenv("SART_PF_NST")) : 0;
  const int nst = nst_env ? nst_env : (QT * HG > 4 ? 4 : 2);
  const int th = 32 * QT * HG;
  if (nst >= 4) launch_pf_n<HD, SUF, 4>(grid, th, q, pool, out, D, layer, reqs, blocks, rows, QT, HG, s);
  else launch_pf_n<HD, SUF, 2>(grid, th, q, pool, out, D, layer, reqs, blocks, rows, QT, HG, s);
}
void launch_attn_prefill_tc(const bf16* q, const bf16* pool, bf16* out, Dims D, int layer, Reqs reqs,
                            const int4* blocks, int nblocks, cudaStream_t s) {
  if (nblocks <= 0) return;
  dim3 grid(nblocks, D.qh);
  if (D.hd == 128) launch_pf<128, false>(grid, q, pool, out, D, layer, reqs, blocks, Rows{}, s);
  else launch_pf<64, false>(grid, q, pool, out, D, layer, reqs, blocks, Rows{}, s);
}
void launch_attn_suffix_tc(const bf16* q, const bf16* pool, bf16* out, Dims D, int layer, Rows rows, Reqs reqs,
                           const int4* qblocks, int nqb, cudaStream_t s) {
  if (nqb <= 0) return;
  dim3 grid(nqb, D.qh);
  if (D.hd == 128) launch_pf<128, true>(grid, q, pool, out, D, layer, reqs, qblocks, rows, s);
  else launch_pf<64, true>(grid, q, pool, out, D, layer, reqs, qblocks, rows, s);
}
void launch_attn_items(Dims D, Rows rows, Reqs reqs, AttnPlan pl, cudaStream_t s) {
  launch_pdl(k_attn_items, dim3(1), dim3(1024), 0, s, D, rows, reqs, pl);
}
void launch_attn_account(Dims D, Rows rows, Reqs reqs, AttnPlan pl, int n, double* acc, cudaStream_t s) {
  (void)pl;
  launch_pdl(k_attn_account, dim3(1), dim3(1024), 0, s, D, rows, reqs, n, acc);
}

template <int HD, int NW, int NS, int SW>
static void launch_cfg(const bf16* q, const bf16* pool, float* part_o, float* part_lse, bf16* out, float* dbg, Dims D,
                       int layer, Rows rows, Reqs reqs, AttnPlan pl, cudaStream_t s) {
  const size_t sm = sizeof(WarpSmem<HD, NS, SW>) * NW;
  ensure_dyn_smem(k_attn_cascade<HD, NW, NS, SW>, (int)sm);
  launch_pdl(k_attn_cascade<HD, NW, NS, SW>, dim3(device_sms()), dim3(NW * 32), sm, s, q, pool, part_o, part_lse, out, dbg,
             D, layer, rows, reqs, pl);
}
static int attn_cfg() {
  static int c = -1;
  if (c < 0) {
    const char* e = getenv("SART_ATTN_CFG");
    c = e ? atoi(e) : 0;
  }
  return c;
}
thread_local bool g_attn_skip_merge = false;   // per host thread (ctx of a TP group each drive one)
thread_local cudaEvent_t g_attn_mid_event = nullptr;
template <int HD>
static void launch_hd(const bf16* q, const bf16* pool, bf16* out, float* dbg, float* part_o, float* part_lse, Dims D,
                      int layer, Rows rows, Reqs reqs, AttnPlan pl, int n, cudaStream_t s) {
  switch (attn_cfg()) {
    case 0: launch_cfg<HD, 6, 2, 32>(q, pool, part_o, part_lse, out, dbg, D, layer, rows, reqs, pl, s); break;
    case 2: launch_cfg<HD, 6, 4, 16>(q, pool, part_o, part_lse, out, dbg, D, layer, rows, reqs, pl, s); break;
    case 3: launch_cfg<HD, 7, 3, 16>(q, pool, part_o, part_lse, out, dbg, D, layer, rows, reqs, pl, s); break;
    case 4: launch_cfg<HD, 7, 2, 32>(q, pool, part_o, part_lse, out, dbg, D, layer, rows, reqs, pl, s); break;   // 224 KB
    default: launch_cfg<HD, 8, 3, 16>(q, pool, part_o, part_lse, out, dbg, D, layer, rows, reqs, pl, s); break;
  }
  if (g_attn_mid_event) cudaEventRecord(g_attn_mid_event, s);
  if (g_attn_skip_merge) return;
  launch_pdl(k_attn_merge<HD>, dim3((n * D.qh * 32 + 255) / 256), dim3(256), 0, s, part_o, part_lse, out, dbg, D,
             rows, reqs, pl, n);
}
void launch_attn_cascade(const bf16* q, const bf16* pool, bf16* out, float* dbg, float* part_o, float* part_lse,
                         Dims D, int layer, Rows rows, Reqs reqs, AttnPlan pl, int n, cudaStream_t s) {
  if (n <= 0) return;
  if (D.hd == 128) launch_hd<128>(q, pool, out, dbg, part_o, part_lse, D, layer, rows, reqs, pl, n, s);
  else launch_hd<64>(q, pool, out, dbg, part_o, part_lse, D, layer, rows, reqs, pl, n, s);
}
